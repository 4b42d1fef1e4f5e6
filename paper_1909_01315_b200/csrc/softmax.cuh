// softmax.cuh - fused edge_softmax forward and backward.
//
// Forward replaces messaging.edge_softmax (messaging.py:105-126), which
// dispatches gspmm(copy_rhs(edge), max) -> gsddmm(sub(edge,dst)) -> exp ->
// gspmm(copy_rhs(edge), sum) -> gsddmm(div(edge,dst)) and keeps four (m,H) /
// (n,H) temporaries. Here two kernels do it:
//   stats : walk each destination's in-edges once (CSC row schedule of
//           spmm_rows.cuh: degree-sorted, CTA per heavy row, warp per light
//           row) computing the online (max, sum of exp) per head column;
//   apply : edge-parallel over the COO list in edge-id order - coalesced
//           reads of s and writes of alpha = exp(s - max[dst]) / sum[dst].
// Edge-keyed data is random in CSC order (one 32 B sector per edge, fetched
// at 64 B granularity), so reading it once in row order and once streaming
// beats two row-order passes, whose second pass misses L2 when many large
// rows are in flight (measured: 7.2 ms -> see profiles/).
// Backward (the composition of those four kernel backwards, autodiff.py:398-418)
// is the closed form  ds = alpha * (g - sum_{in-edges} alpha * g): the stats
// kernel computes the per-destination sums, the apply kernel the edges.
//
// Numerics: fp32 sums use the exact compensated pair of spmm_rows.cuh (no
// per-element fp32->fp64 conversions, which run on the XU pipe) and are
// folded to fp64 once per row; the backward's g - sum is formed with a
// two-float representation of the fp64 sum. The fp64 instantiation computes
// everything in double.
#pragma once

#include "gmp_common.cuh"
#include "spmm_rows.cuh"

namespace gmp {

struct SoftmaxArgs {
  const int64_t* indptr;
  const int32_t* indices;
  const int32_t* eids;
  const int32_t* order;
  int64_t n_rows;
  int64_t n_heavy;
  int64_t blocks_per_tile;
  int32_t H;
  int32_t tile_cols;
  int32_t g_log2;
  const void* s;   // scores (fwd) / alpha (bwd)
  int64_t lds;
  const void* g;   // upstream grad (bwd only)
  int64_t ldg;
  void* out;       // alpha (fwd) / ds (bwd)
  int64_t ldo;
  const int32_t* dst;  // COO destinations (apply kernel)
  int64_t m;
  void* stat;          // (n_rows, 2H) of T: [max | 1/sum] fwd, [sum_hi | sum_lo] bwd
  // fused u_add_v scores (forward only): s[e] = el[src e] + er[dst e], never
  // materialised (GAT attention logits, layers.py:110-113); null = read s
  const void* el;
  int64_t lde;
  const void* er;
  int64_t ldr;
  const int32_t* src;  // COO sources (apply kernel, fused mode)
};

__device__ __forceinline__ float exp_t(float x) { return expf(x); }
__device__ __forceinline__ double exp_t(double x) { return exp(x); }

// (m, l) online-softmax merge in fp64 for l; empty partials carry m = -inf.
template <typename T>
__device__ __forceinline__ void sm_merge(T& m, double& l, T om, double ol) {
  if (om == -INFINITY) return;
  if (m == -INFINITY) { m = om; l = ol; return; }
  if (om > m) { l = l * exp((double)m - (double)om) + ol; m = om; }
  else        { l += ol * exp((double)om - (double)m); }
}

// per-column running sum: compensated fp32 pair for float, plain fp64 for double
template <typename T> struct ColSum;
template <> struct ColSum<float> {
  float s = 0.f, c = 0.f;
  __device__ __forceinline__ void add(float x) { two_sum1(s, c, x); }
  __device__ __forceinline__ void add_prod(float x, float y) {
    const float p = __fmul_rn(x, y);
    two_sum1(s, c, p);
    c = __fadd_rn(c, __fmaf_rn(x, y, -p));
  }
  __device__ __forceinline__ void scale(float f) { s = __fmul_rn(s, f); c = __fmul_rn(c, f); }
  __device__ __forceinline__ double value() const { return (double)s + (double)c; }
};
template <> struct ColSum<double> {
  double s = 0.0;
  __device__ __forceinline__ void add(double x) { s += x; }
  __device__ __forceinline__ void add_prod(double x, double y) { s += x * y; }
  __device__ __forceinline__ void scale(double f) { s *= f; }
  __device__ __forceinline__ double value() const { return s; }
};

// Stats kernel: edges of a row are walked in chunks of kChunk whose edge ids
// are staged in shared memory (coalesced loads, one chunk ahead), so every
// lane keeps U independent score loads in flight even when 32 edges fit in
// one warp step.
constexpr int kChunk = 256;

template <typename T, int V, bool BWD, bool UV>
__global__ void __launch_bounds__(kWarpsPerCta * 32) edge_softmax_kernel(const SoftmaxArgs a) {
  constexpr int U = V == 4 ? 4 : 8;
  constexpr int B = kChunk / 32;
  __shared__ double s_l[kWarpsPerCta][32 * V];
  __shared__ T s_m[kWarpsPerCta][32 * V];
  __shared__ int32_t s_eid[kWarpsPerCta][kChunk];
  const int64_t bid = blockIdx.x;
  const int tile = (int)(bid / a.blocks_per_tile);
  const int64_t local = bid - (int64_t)tile * a.blocks_per_tile;
  const int c0 = tile * a.tile_cols, c1 = min(a.H, c0 + a.tile_cols);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = 1 << a.g_log2, E = 32 >> a.g_log2;
  const int slot = lane >> a.g_log2, gl = lane & (G - 1);
  const bool heavy = local < a.n_heavy;
  int64_t row;
  if (heavy) {
    row = a.order[local];
  } else {
    const int64_t r = a.n_heavy + (local - a.n_heavy) * kWarpsPerCta + warp;
    if (r >= a.n_rows) return;
    row = a.order ? (int64_t)a.order[r] : r;
  }
  const int64_t pb = a.indptr[row], pe = a.indptr[row + 1];
  if (pe == pb) return;  // no in-edges: nothing keyed to this row (heavy rows are never empty)
  const int col = c0 + gl * V;
  const bool valid = col < c1;
  const int ccol = valid ? col : 0;
  const T* S = static_cast<const T*>(a.s) + ccol;
  const T* Gd = static_cast<const T*>(a.g) + ccol;
  const T* EL = UV ? static_cast<const T*>(a.el) + ccol : nullptr;
  T er_row[V];
#pragma unroll
  for (int k = 0; k < V; ++k) er_row[k] = T(0);
  if (UV) load_vec<T, V>(static_cast<const T*>(a.er) + row * a.ldr + ccol, er_row);
  T* O = static_cast<T*>(a.out) + ccol;
  const int64_t first = heavy ? (int64_t)warp * kChunk : 0;
  const int64_t stride = heavy ? (int64_t)kChunk * kWarpsPerCta : kChunk;
  int32_t* buf = s_eid[warp];

  // stage chunk `cb` of edge ids into this warp's buffer (prefetched registers)
  int32_t pre[B];
  auto fetch = [&](int64_t cb) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const int64_t q = cb + i * 32 + lane;
      pre[i] = q < pe ? __ldg((UV ? a.indices : a.eids) + q) : 0;
    }
  };
  auto stage = [&]() {
    __syncwarp();
#pragma unroll
    for (int i = 0; i < B; ++i) buf[i * 32 + lane] = pre[i];
    __syncwarp();
  };

  // ---- pass 1: online max + sum (fwd) / sum of alpha * g (bwd) ----
  T m[V];
  ColSum<T> acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) m[k] = -INFINITY;
  fetch(pb + first);
  for (int64_t cb = pb + first; cb < pe; cb += stride) {
    const int cnt = (int)min((int64_t)kChunk, pe - cb);
    stage();
    fetch(cb + stride);
    for (int t = 0; t < cnt; t += E * U) {
      T x[U][V], gg[U][V];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = t + slot + E * u;
        ok[u] = j < cnt && valid;
        const int64_t e = buf[j & (kChunk - 1)];
#pragma unroll
        for (int k = 0; k < V; ++k) x[u][k] = gg[u][k] = T(0);
        if (UV && ok[u]) {  // e is the source node: score = el[u] + er[row]
          load_vec<T, V>(EL + e * a.lde, x[u]);
#pragma unroll
          for (int k = 0; k < V; ++k) x[u][k] = x[u][k] + er_row[k];
        } else if (ok[u]) {
          load_vec<T, V>(S + e * a.lds, x[u]);
          if constexpr (BWD) load_vec<T, V>(Gd + e * a.ldg, gg[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
#pragma unroll
        for (int k = 0; k < V; ++k) {
          if constexpr (BWD) {
            acc[k].add_prod(x[u][k], gg[u][k]);
          } else {
            if (x[u][k] > m[k]) {
              acc[k].scale(exp_t(T(m[k] - x[u][k])));
              m[k] = x[u][k];
            }
            acc[k].add(exp_t(T(x[u][k] - m[k])));
          }
        }
      }
    }
  }
  double l[V];
#pragma unroll
  for (int k = 0; k < V; ++k) l[k] = acc[k].value();
  for (int off = G; off < 32; off <<= 1) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const double ol = __shfl_xor_sync(kFull, l[k], off);
      if constexpr (BWD) {
        l[k] += ol;
      } else {
        const T om = __shfl_xor_sync(kFull, m[k], off);
        sm_merge<T>(m[k], l[k], om, ol);
      }
    }
  }
  if (heavy) {
    if (slot == 0) {
#pragma unroll
      for (int k = 0; k < V; ++k) { s_l[warp][gl * V + k] = l[k]; s_m[warp][gl * V + k] = m[k]; }
    }
    __syncthreads();
    if (warp == 0 && slot == 0) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        T mm = s_m[0][gl * V + k];
        double ll = s_l[0][gl * V + k];
        for (int w = 1; w < kWarpsPerCta; ++w) {
          if constexpr (BWD) ll += s_l[w][gl * V + k];
          else sm_merge<T>(mm, ll, s_m[w][gl * V + k], s_l[w][gl * V + k]);
        }
        s_m[0][gl * V + k] = mm;
        s_l[0][gl * V + k] = ll;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < V; ++k) { m[k] = s_m[0][gl * V + k]; l[k] = s_l[0][gl * V + k]; }
  }
  // every slot of the warp needs its lane-group's final (m, l)
#pragma unroll
  for (int k = 0; k < V; ++k) {
    l[k] = __shfl_sync(kFull, l[k], gl);
    m[k] = __shfl_sync(kFull, m[k], gl);
  }

  // ---- per-destination statistics: (max, 1/sum) fwd, (sum_hi, sum_lo) bwd ----
  if (slot == 0 && valid) {
    T* st = static_cast<T*>(a.stat) + row * 2 * (int64_t)a.H + col;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      if constexpr (BWD) {
        const T hi = (T)l[k];
        st[k] = hi;
        st[a.H + k] = (T)(l[k] - (double)hi);
      } else {
        st[k] = m[k];
        st[a.H + k] = (T)(1.0 / l[k]);
      }
    }
  }
}

// alpha[e] = exp(s[e] - max[dst e]) * inv_sum[dst e]   (fwd)
// ds[e]    = alpha[e] * (g[e] - sum[dst e])            (bwd)
// Edge-id order: s / g / alpha / ds stream coalesced; the per-destination
// statistics (T pairs, (n, H)) are L2-resident gathers. Each thread keeps
// kApplyU independent vectors in flight, and the destination ids of its next
// group are loaded while the current group computes, so the dependent
// statistics gather is not serialised behind a DRAM miss on dst[e].
constexpr int kApplyU = 4;

template <typename T, int V, bool BWD, bool UV>
__global__ void __launch_bounds__(256) edge_softmax_apply_kernel(const SoftmaxArgs a) {
  const int per_edge = a.H / V;  // vectors per edge row
  const int pe_log2 = (per_edge & (per_edge - 1)) == 0 ? __ffs(per_edge) - 1 : -1;
  const int64_t total = a.m * (int64_t)per_edge;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t step = nthreads * kApplyU;
  const T* st = static_cast<const T*>(a.stat);
  auto edge_of = [&](int64_t i) -> int64_t {
    return pe_log2 >= 0 ? (i >> pe_log2) : i / per_edge;
  };
  int32_t vn[kApplyU], un[kApplyU];
  auto fetch_ids = [&](int64_t ib) {
#pragma unroll
    for (int u = 0; u < kApplyU; ++u) {
      const int64_t i = ib + u * nthreads;
      const int64_t e = i < total ? edge_of(i) : 0;
      vn[u] = i < total ? __ldg(a.dst + e) : 0;
      if constexpr (UV) un[u] = i < total ? __ldg(a.src + e) : 0;
    }
  };
  int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  fetch_ids(i0);
  for (; i0 < total; i0 += step) {
    int32_t vc[kApplyU], uc[kApplyU];
#pragma unroll
    for (int u = 0; u < kApplyU; ++u) { vc[u] = vn[u]; uc[u] = UV ? un[u] : 0; }
    fetch_ids(i0 + step);
    T x[kApplyU][V], gg[kApplyU][V], p0[kApplyU][V], p1[kApplyU][V];
    int64_t ev[kApplyU];
    int cv[kApplyU];
    bool ok[kApplyU];
#pragma unroll
    for (int u = 0; u < kApplyU; ++u) {
      const int64_t i = i0 + u * nthreads;
      ok[u] = i < total;
      const int64_t e = ok[u] ? edge_of(i) : 0;
      const int c = ok[u] ? (int)(i - e * per_edge) * V : 0;
      ev[u] = e;
      cv[u] = c;
      const int64_t v = vc[u];
      if constexpr (UV) {
        T xr[V];
        load_vec<T, V>(static_cast<const T*>(a.el) + (int64_t)uc[u] * a.lde + c, x[u]);
        load_vec<T, V>(static_cast<const T*>(a.er) + v * a.ldr + c, xr);
#pragma unroll
        for (int k = 0; k < V; ++k) x[u][k] = x[u][k] + xr[k];
      } else {
        load_vec<T, V>(static_cast<const T*>(a.s) + e * a.lds + c, x[u]);
      }
      if constexpr (BWD) load_vec<T, V>(static_cast<const T*>(a.g) + e * a.ldg + c, gg[u]);
      // stats row v: [pair0 (H) | pair1 (H)] interleaved as 2*H per row
      load_vec<T, V>(st + v * 2 * a.H + c, p0[u]);
      load_vec<T, V>(st + v * 2 * a.H + a.H + c, p1[u]);
    }
#pragma unroll
    for (int u = 0; u < kApplyU; ++u) {
      if (!ok[u]) continue;
      T r[V];
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if constexpr (BWD) {
          if constexpr (sizeof(T) == 8) {
            r[k] = x[u][k] * (gg[u][k] - p0[u][k]);
          } else {
            // (g - l) to ~fp64 accuracy with l = lhi + llo (p0, p1)
            float dh = 0.f, dc = 0.f;
            two_sum1(dh, dc, (float)gg[u][k]);
            two_sum1(dh, dc, -(float)p0[u][k]);
            dc = __fsub_rn(dc, (float)p1[u][k]);
            r[k] = (T)__fmaf_rn((float)x[u][k], dh, __fmul_rn((float)x[u][k], dc));
          }
        } else {
          r[k] = exp_t(T(x[u][k] - p0[u][k])) * p1[u][k];
        }
      }
      store_vec<T, V>(static_cast<T*>(a.out) + ev[u] * a.ldo + cv[u], r);
    }
  }
}

cudaError_t launch_edge_softmax(int dtype_is_f64, int V, bool bwd, bool uv, const SoftmaxArgs& a,
                                int64_t grid, cudaStream_t s);
cudaError_t launch_edge_softmax_apply(int dtype_is_f64, int V, bool bwd, bool uv,
                                      const SoftmaxArgs& a, cudaStream_t s);

}  // namespace gmp
