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


// exp(x - m) of a softmax term: sm_exp / uv_score in spmm_rows.cuh (error
// relative to |x - m|, one formula for every fp32 softmax term).

// (m, l) online-softmax merge in fp64 for l; empty partials carry m = -inf.
template <typename T>
__device__ __forceinline__ void sm_merge(T& m, double& l, T om, double ol) {
  if (om == -INFINITY) return;
  if (m == -INFINITY) { m = om; l = ol; return; }
  // the rescale factor in the element precision: its error (~1 ulp of the
  // fp32 exponent difference) is weighted by the factor itself, < 3e-8 of l
  if (om > m) { l = l * (double)sm_exp(m, om) + ol; m = om; }
  else        { l += ol * (double)sm_exp(om, m); }
}

// per-column running sum: compensated fp32 pair for float, plain fp64 for double
template <typename T> struct ColSum;
template <> struct ColSum<float> {
  float s = 0.f, c = 0.f;
  __device__ __forceinline__ void add(float x) { two_sum1(s, c, x); }
  __device__ __forceinline__ void add_prod(float x, float y) { two_sum_prod1(s, c, x, y); }
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

// score rows in flight per lane: the forward's online max/exp work per
// element favours 4 for float4 rows, the backward's plain products 8
// (Reddit H=8, fwd / bwd ms: U=4 2.90 / 4.11, U=8 2.98 / 3.70, U=16 3.29 / 4.06)
template <int V, bool BWD>
struct StatsUnroll {
  static constexpr int value = (V == 4 && !BWD) ? 4 : 8;
};

// Pass 1 of the statistics for edges [pb, pe) of one row owned by this warp
// (chunks pb + first, + stride, ...): online (max, sum exp) per column (fwd)
// or sum alpha * g (bwd). ids: edge ids (UV: source node ids).
template <typename T, int V, bool BWD, bool UV>
__device__ __forceinline__ void stats_pass1(const SoftmaxArgs& a, const int32_t* __restrict__ ids,
                                            int64_t pb, int64_t pe, int64_t first,
                                            int64_t stride, int lane, int slot, int E, bool valid,
                                            int ccol, const T (&er_row)[V], int32_t* buf,
                                            T (&m)[V], ColSum<T> (&acc)[V]) {
  constexpr int U = StatsUnroll<V, BWD>::value;
  constexpr int B = kChunk / 32;
  const T* S = static_cast<const T*>(a.s) + ccol;
  const T* Gd = static_cast<const T*>(a.g) + ccol;
  const T* EL = UV ? static_cast<const T*>(a.el) + ccol : nullptr;
  int32_t pre[B];
  auto fetch = [&](int64_t cb) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const int64_t q = cb + i * 32 + lane;
      pre[i] = q < pe ? __ldg(ids + q) : 0;
    }
  };
  auto stage = [&]() {
    __syncwarp();
#pragma unroll
    for (int i = 0; i < B; ++i) buf[i * 32 + lane] = pre[i];
    __syncwarp();
  };
  fetch(pb + first);
  for (int64_t cb = pb + first; cb < pe; cb += stride) {
    const int cnt = (int)min((int64_t)kChunk, pe - cb);
    stage();
    fetch(cb + stride);
    for (int t = 0; t < cnt; t += E * U) {
      T x[U][V], gg[U][V];
      T xl[UV ? U : 1][V];  // UV: low part of the exact score el + er
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = t + slot + E * u;
        ok[u] = j < cnt && valid;
        const int64_t e = buf[j & (kChunk - 1)];
#pragma unroll
        for (int k = 0; k < V; ++k) x[u][k] = gg[u][k] = T(0);
        if constexpr (UV) {
#pragma unroll
          for (int k = 0; k < V; ++k) xl[u][k] = T(0);
        }
        if (UV && ok[u]) {  // e is the source node: score = el[u] + er[row]
          load_vec<T, V>(EL + e * a.lde, x[u]);
#pragma unroll
          for (int k = 0; k < V; ++k) {
            if constexpr (UV) uv_score(x[u][k], er_row[k], x[u][k], xl[u][k]);
          }
        } else if (ok[u]) {
          load_vec<T, V>(S + e * a.lds, x[u]);
          if constexpr (BWD) load_vec<T, V>(Gd + e * a.ldg, gg[u]);
        }
      }
      if constexpr (BWD) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!ok[u]) continue;
#pragma unroll
          for (int k = 0; k < V; ++k) acc[k].add_prod(x[u][k], gg[u][k]);
        }
      } else {
        // one rescale per group of U edges: the group max first, then one
        // exp per element relative to the (possibly raised) running max
#pragma unroll
        for (int k = 0; k < V; ++k) {
          T mx = m[k];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (ok[u] && x[u][k] > mx) mx = x[u][k];
          if (mx > m[k]) {
            if (m[k] != T(-INFINITY)) acc[k].scale(sm_exp(m[k], mx));
            m[k] = mx;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
            if constexpr (UV) acc[k].add(sm_exp(x[u][k], xl[u][k], m[k]));
            else acc[k].add(sm_exp(x[u][k], m[k]));
          }
        }
      }
    }
  }
}

// fold the slots of a warp: every lane group ends with its columns' (m, l)
template <typename T, int V, bool BWD>
__device__ __forceinline__ void stats_warp_combine(int G, T (&m)[V], double (&l)[V]) {
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
}

template <typename T, int V, bool BWD>
__device__ __forceinline__ void stats_write(const SoftmaxArgs& a, int64_t row, int col,
                                            const T (&m)[V], const double (&l)[V]) {
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

template <typename T, int V, bool BWD, bool UV>
__global__ void __launch_bounds__(kWarpsPerCta * 32) edge_softmax_kernel(const SoftmaxArgs a) {
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
  T er_row[V];
#pragma unroll
  for (int k = 0; k < V; ++k) er_row[k] = T(0);
  if (UV) load_vec<T, V>(static_cast<const T*>(a.er) + row * a.ldr + ccol, er_row);

  T m[V];
  ColSum<T> acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) m[k] = -INFINITY;
  stats_pass1<T, V, BWD, UV>(a, UV ? a.indices : a.eids, pb, pe,
                             heavy ? (int64_t)warp * kChunk : 0,
                             heavy ? (int64_t)kChunk * kWarpsPerCta : kChunk, lane, slot, E,
                             valid, ccol, er_row, s_eid[warp], m, acc);
  double l[V];
#pragma unroll
  for (int k = 0; k < V; ++k) l[k] = acc[k].value();
  stats_warp_combine<T, V, BWD>(G, m, l);
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
  if (slot == 0 && valid) stats_write<T, V, BWD>(a, row, col, m, l);
}

// Statistics of short rows (degree <= the schedule's light threshold; on
// Reddit 106k of the 135k non-empty rows have 1-16 in-edges): one row per
// lane group (E rows per warp), the row's edges walked U at a time with the
// same online update as stats_pass1 - no shared-memory staging, no warp
// combine.
template <typename T, int V, bool BWD, bool UV>
__global__ void __launch_bounds__(kWarpsPerCta * 32) edge_softmax_slot_kernel(const SoftmaxArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = 32 >> a.g_log2;
  const int slot = lane >> a.g_log2, gl = lane & ((1 << a.g_log2) - 1);
  const int64_t r = ((int64_t)blockIdx.x * kWarpsPerCta + warp) * E + slot;
  if (r >= a.n_rows) return;  // lanes are independent below
  const int64_t row = a.order ? (int64_t)a.order[r] : r;
  const int64_t pb = a.indptr[row], pe = a.indptr[row + 1];
  if (pe == pb) return;
  const int col = gl * V;
  const bool valid = col < a.H;
  const int ccol = valid ? col : 0;
  T er_row[V];
#pragma unroll
  for (int k = 0; k < V; ++k) er_row[k] = T(0);
  if (UV) load_vec<T, V>(static_cast<const T*>(a.er) + row * a.ldr + ccol, er_row);
  const T* S = static_cast<const T*>(a.s) + ccol;
  const T* Gd = static_cast<const T*>(a.g) + ccol;
  const T* EL = UV ? static_cast<const T*>(a.el) + ccol : nullptr;
  const int32_t* ids = UV ? a.indices : a.eids;
  T m[V];
  ColSum<T> acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) m[k] = -INFINITY;
  constexpr int U = 4;
  for (int64_t p0 = pb; p0 < pe; p0 += U) {
    T x[U][V], gg[U][V];
    T xl[UV ? U : 1][V];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ok[u] = p0 + u < pe && valid;
      const int64_t e = ok[u] ? (int64_t)__ldg(ids + p0 + u) : 0;
#pragma unroll
      for (int k = 0; k < V; ++k) x[u][k] = gg[u][k] = T(0);
      if constexpr (UV) {
#pragma unroll
        for (int k = 0; k < V; ++k) xl[u][k] = T(0);
        if (ok[u]) {
          load_vec<T, V>(EL + e * a.lde, x[u]);
#pragma unroll
          for (int k = 0; k < V; ++k) uv_score(x[u][k], er_row[k], x[u][k], xl[u][k]);
        }
      } else if (ok[u]) {
        load_vec<T, V>(S + e * a.lds, x[u]);
        if constexpr (BWD) load_vec<T, V>(Gd + e * a.ldg, gg[u]);
      }
    }
    if constexpr (BWD) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k].add_prod(x[u][k], gg[u][k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        T mx = m[k];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (ok[u] && x[u][k] > mx) mx = x[u][k];
        if (mx > m[k]) {
          if (m[k] != T(-INFINITY)) acc[k].scale(sm_exp(m[k], mx));
          m[k] = mx;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!ok[u]) continue;
          if constexpr (UV) acc[k].add(sm_exp(x[u][k], xl[u][k], m[k]));
          else acc[k].add(sm_exp(x[u][k], m[k]));
        }
      }
    }
  }
  if (!valid) return;
  double l[V];
#pragma unroll
  for (int k = 0; k < V; ++k) l[k] = acc[k].value();
  stats_write<T, V, BWD>(a, row, col, m, l);
}

// Windowed statistics for the heavy rows (edge-keyed scores only). A random
// 32 B score row costs a whole 128 B DRAM line (tools/micro/randread.cu), so
// walking heavy rows in CSC order moves ~4x the score bytes. Instead the edge
// ids are cut into windows of `win` consecutive ids whose score rows fit in L2
// together, and work items (window b, heavy row r) - the part of row r's
// edge list (ascending edge ids, `sorted_eids`) inside window b - are handed
// out in window-major order through an atomic counter, so the warps in flight
// share one or two windows and every score line is fetched from DRAM about
// once. Each item writes a partial (max, sum) per column; a merge kernel
// combines a row's partials in window order (deterministic).
struct WindowArgs {
  const int32_t* sorted_eids;  // in-adjacency edge ids, ascending inside each row
  int64_t win;                 // edge ids per window
  int64_t n_windows;
  unsigned long long* counter; // work-item counter (zeroed by the launcher)
  int64_t* bounds;             // (n_heavy, n_windows + 1): first position of each window in a row
  void* pm;                    // (n_windows, n_heavy, H) T: partial max (fwd)
  double* pl;                  // (n_windows, n_heavy, H): partial sum
};

template <typename T, int V, bool BWD>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    edge_softmax_window_kernel(const SoftmaxArgs a, const WindowArgs w) {
  __shared__ int32_t s_eid[kWarpsPerCta][kChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = 1 << a.g_log2, E = 32 >> a.g_log2;
  const int slot = lane >> a.g_log2, gl = lane & (G - 1);
  const int col = gl * V;  // one column tile (H <= 32 V)
  const bool valid = col < a.H;
  const int ccol = valid ? col : 0;
  const int64_t items = w.n_windows * a.n_heavy;
  T zero_row[V];
#pragma unroll
  for (int k = 0; k < V; ++k) zero_row[k] = T(0);
  // the next item's index is claimed one item ahead (hides the atomic's latency)
  unsigned long long nxt = 0;
  if (lane == 0) nxt = atomicAdd(w.counter, 1ull);
  for (;;) {
    const unsigned long long it = __shfl_sync(kFull, nxt, 0);
    if ((int64_t)it >= items) return;
    if (lane == 0) nxt = atomicAdd(w.counter, 1ull);
    const int64_t b = (int64_t)it / a.n_heavy, r = (int64_t)it - b * a.n_heavy;
    // [lo, hi): positions of row r's edge ids inside [b*win, (b+1)*win)
    const int64_t* bd = w.bounds + r * (w.n_windows + 1) + b;
    const int64_t lo = __ldg(bd), hi = __ldg(bd + 1);
    T m[V];
    ColSum<T> acc[V];
#pragma unroll
    for (int k = 0; k < V; ++k) m[k] = -INFINITY;
    if (hi > lo)
      stats_pass1<T, V, BWD, false>(a, w.sorted_eids, lo, hi, 0, kChunk, lane, slot, E, valid,
                                    ccol, zero_row, s_eid[warp], m, acc);
    double l[V];
#pragma unroll
    for (int k = 0; k < V; ++k) l[k] = acc[k].value();
    stats_warp_combine<T, V, BWD>(G, m, l);
    if (slot == 0 && valid) {
      const int64_t base = ((int64_t)b * a.n_heavy + r) * a.H + col;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if constexpr (!BWD) static_cast<T*>(w.pm)[base + k] = m[k];
        w.pl[base + k] = l[k];
      }
    }
  }
}

// bounds[r][b] = first position p in heavy row r with sorted_eids[p] >= b*win
// (b = 0..n_windows): one independent binary search per thread
static __global__ void edge_softmax_window_bounds(const SoftmaxArgs a, const WindowArgs w) {
  const int64_t per = w.n_windows + 1;
  const int64_t total = a.n_heavy * per;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per, b = i - r * per;
    const int64_t row = a.order[r];
    int64_t x = a.indptr[row], y = a.indptr[row + 1];
    const int64_t e0 = b * w.win;
    while (x < y) {
      const int64_t mid = (x + y) >> 1;
      if (__ldg(w.sorted_eids + mid) < e0) x = mid + 1; else y = mid;
    }
    w.bounds[i] = x;
  }
}

// one warp per (heavy row, column): lanes merge strided window partials,
// then a fixed xor tree combines the lanes (deterministic)
template <typename T, bool BWD>
__global__ void edge_softmax_window_merge(const SoftmaxArgs a, const WindowArgs w) {
  const int lane = threadIdx.x & 31;
  const int64_t total = a.n_heavy * (int64_t)a.H;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < total; i += nw) {
    const int64_t r = i / a.H;
    const int c = (int)(i - r * a.H);
    T mm = -INFINITY;
    double ll = 0.0;
    for (int64_t b = lane; b < w.n_windows; b += 32) {
      const int64_t at = (b * a.n_heavy + r) * a.H + c;
      if constexpr (BWD) ll += w.pl[at];
      else sm_merge<T>(mm, ll, static_cast<const T*>(w.pm)[at], w.pl[at]);
    }
    for (int off = 1; off < 32; off <<= 1) {
      const double ol = __shfl_xor_sync(kFull, ll, off);
      if constexpr (BWD) {
        ll += ol;
      } else {
        const T om = __shfl_xor_sync(kFull, mm, off);
        sm_merge<T>(mm, ll, om, ol);
      }
    }
    if (lane != 0) continue;
    const int64_t row = a.order[r];
    T* st = static_cast<T*>(a.stat) + row * 2 * (int64_t)a.H + c;
    if constexpr (BWD) {
      const T hi = (T)ll;
      st[0] = hi;
      st[a.H] = (T)(ll - (double)hi);
    } else {
      st[0] = mm;
      st[a.H] = (T)(1.0 / ll);
    }
  }
}

// Segmented statistics for the heavy rows (edge-keyed scores; replaces the
// (window, row) work items above when a gmp_segplan is given). The heavy
// rows' in-edges are laid out once per graph in window-major order - edge
// ids sorted by (eid / win, heavy row, eid) - each (window, row) segment
// padded with -1 to a multiple of the lane-group count E, so a warp sub-step
// (E positions, one per lane group) never straddles two segments. Pieces =
// segments cut every kSegChunkSub sub-steps (a chunk). A warp claims chunks
// in order (the warps in flight sweep about one window of score rows, which
// L2 holds while each 128 B line is touched by its four edges' rows); lane
// groups read consecutive positions (coalesced), a batch of U sub-steps is
// loaded at once, and the piece starts inside a chunk are warp-uniform bits.
// Batches without a piece start take the group update (one max, one
// rescale, U exps per column); the rest a rolled per-sub-step loop that
// closes a piece (fixed xor-tree fold, one partial per piece) at each start.
// A merge kernel folds each row's pieces in piece (= window) order, so the
// result is deterministic.
constexpr int kSegChunkSub = 16;  // sub-steps per chunk (GMP_SEG_CHUNK_SUB)
// sub-steps per load batch (Reddit H=8 backward: 8 -> 3.78 ms, 4 -> 3.96 ms)
template <bool BWD> struct SegBatch { static constexpr int value = 8; };

struct SegArgs {
  const int32_t* perm;         // n_pos edge ids, window-major, -1 = padding
  const uint32_t* starts;      // bit j: sub-step j starts a piece
  const int32_t* chunk_piece;  // piece id of each chunk's first sub-step
  const int64_t* row_ptr;      // n_heavy + 1: pieces of heavy row r
  const int32_t* row_pieces;   // piece ids grouped by heavy row, ascending
  int64_t n_pos, n_chunks, n_pieces;
  unsigned long long* counter; // chunk counter (zeroed by the launcher)
  void* pm;                    // (n_pieces, H) T: partial max (fwd)
  double* pl;                  // (n_pieces, H): partial sum
};

// Fold of one piece across the warp's lane groups: the common maximum
// first (order-free), then every lane group rescales its own compensated sum
// once and a fixed xor tree adds the fp64 values (deterministic). Cheaper than
// a pairwise online merge at each tree level (one exp per lane, no branches).
template <typename T, int V, bool BWD>
__device__ __forceinline__ void seg_fold(int G, T (&m)[V], const ColSum<T> (&acc)[V],
                                         double (&l)[V]) {
#pragma unroll
  for (int k = 0; k < V; ++k) {
    if constexpr (BWD) {
      l[k] = acc[k].value();
    } else {
      T M = m[k];
      for (int off = G; off < 32; off <<= 1) M = fmax(M, __shfl_xor_sync(kFull, M, off));
      l[k] = m[k] == T(-INFINITY) ? 0.0 : acc[k].value() * (double)sm_exp(m[k], M);
      m[k] = M;
    }
    for (int off = G; off < 32; off <<= 1) l[k] += __shfl_xor_sync(kFull, l[k], off);
  }
}

// packed (f32x2) column-pair updates of the batch fast path
__device__ __forceinline__ float2 ex2_2(float2 d) {
  const float2 y = __fmul2_rn(d, f2(kLog2e, kLog2e));
  return f2(ex2_approx(y.x), ex2_approx(y.y));
}

// latency bound: Reddit H=8 fwd with 1 / 2 / 3 resident CTAs per SM 3.69 /
// 2.77 / 2.55 ms; forcing four (64 registers) spills and takes 2.71 ms
template <typename T, int V, bool BWD>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    edge_softmax_seg_kernel(const SoftmaxArgs a, const SegArgs sg) {
  constexpr int U = SegBatch<BWD>::value;
  constexpr bool PACK = sizeof(T) == 4 && V % 2 == 0;
  const int lane = threadIdx.x & 31;
  const int G = 1 << a.g_log2, E = 32 >> a.g_log2;
  const int slot = lane >> a.g_log2, gl = lane & (G - 1);
  const int col = gl * V;
  const bool valid = col < a.H;
  const int ccol = valid ? col : 0;
  const T* S = static_cast<const T*>(a.s) + ccol;
  const T* Gd = static_cast<const T*>(a.g) + ccol;
  const int32_t lds = (int32_t)a.lds, ldg = (int32_t)a.ldg;  // host-checked < 2^31
  T* PM = static_cast<T*>(sg.pm);
  const T pad = BWD ? T(0) : T(-INFINITY);  // padding: no max, exp 0 / product 0
  T m[V];
  ColSum<T> acc[V];
  int64_t piece = 0;
  auto reset = [&]() {
#pragma unroll
    for (int k = 0; k < V; ++k) { m[k] = -INFINITY; acc[k] = ColSum<T>(); }
  };
  auto flush = [&]() {
    double l[V];
    seg_fold<T, V, BWD>(G, m, acc, l);
    if (slot == 0 && valid) {
      const int64_t base = piece * a.H + col;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if constexpr (!BWD) PM[base + k] = m[k];
        sg.pl[base + k] = l[k];
      }
    }
    reset();
  };
  // the edge ids of the next batch are loaded one batch ahead (across chunk
  // boundaries: the next chunk is claimed one ahead), so each batch waits for
  // one memory latency (its score rows), not two (ids, then rows)
  int32_t ev[U];
  auto load_ids = [&](int64_t cc, int b) {
    const int32_t* pp = sg.perm + (cc * kSegChunkSub + b) * E + slot;  // whole chunks
#pragma unroll
    for (int u = 0; u < U; ++u) ev[u] = __ldg(pp + u * E);
  };
  unsigned long long nxt = 0;
  if (lane == 0) nxt = atomicAdd(sg.counter, 1ull);
  int64_t c = (int64_t)__shfl_sync(kFull, nxt, 0);
  if (c >= sg.n_chunks) return;
  if (lane == 0) nxt = atomicAdd(sg.counter, 1ull);
  load_ids(c, 0);
  for (;;) {
    const int64_t j0 = c * kSegChunkSub;  // first sub-step of the chunk
    const uint32_t cb = (__ldg(sg.starts + (j0 >> 5)) >> (j0 & 31)) & ((1u << kSegChunkSub) - 1u);
    piece = (int64_t)__ldg(sg.chunk_piece + c);  // bit 0 of cb is always set
    reset();
#pragma unroll 1
    for (int b = 0; b < kSegChunkSub; b += U) {
      T x[U][V], gg[U][V];
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int k = 0; k < V; ++k) { x[u][k] = pad; gg[u][k] = T(0); }
        if (ev[u] >= 0 && valid) {
          load_vec<T, V>(S + (int64_t)ev[u] * lds, x[u]);
          if constexpr (BWD) load_vec<T, V>(Gd + (int64_t)ev[u] * ldg, gg[u]);
        }
      }
      if (b + U < kSegChunkSub) {
        load_ids(c, b + U);
      } else {
        const int64_t cn = (int64_t)__shfl_sync(kFull, nxt, 0);
        if (cn < sg.n_chunks) load_ids(cn, 0);
      }
      const uint32_t bits = (cb >> b) & ((1u << U) - 1u);
      if ((bits >> 1) == 0) {
        // no piece start after this batch's first sub-step
        if (b > 0 && (bits & 1u)) { flush(); ++piece; }
        if constexpr (BWD) {
          if constexpr (PACK) {
#pragma unroll
            for (int k = 0; k < V; k += 2) {
              float2 s2 = f2(acc[k].s, acc[k + 1].s), c2 = f2(acc[k].c, acc[k + 1].c);
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const float2 xx = f2(x[u][k], x[u][k + 1]), yy = f2(gg[u][k], gg[u][k + 1]);
                const float2 pr = fmul2(xx, yy);
                two_sum2(s2, c2, pr);
                c2 = __fadd2_rn(c2, __ffma2_rn(xx, yy, f2(-pr.x, -pr.y)));
              }
              acc[k].s = s2.x; acc[k + 1].s = s2.y; acc[k].c = c2.x; acc[k + 1].c = c2.y;
            }
          } else {
#pragma unroll
            for (int k = 0; k < V; ++k) {
#pragma unroll
              for (int u = 0; u < U; ++u) acc[k].add_prod(x[u][k], gg[u][k]);
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < V; ++k) {
            T mx = m[k];
#pragma unroll
            for (int u = 0; u < U; ++u) mx = fmax(mx, x[u][k]);
            if (mx > m[k]) {
              if (m[k] != T(-INFINITY)) acc[k].scale(sm_exp(m[k], mx));
              m[k] = mx;
            }
          }
          if constexpr (PACK) {
#pragma unroll
            for (int k = 0; k < V; k += 2) {
              if (m[k] == T(-INFINITY) || m[k + 1] == T(-INFINITY)) {  // padding / -inf scores
#pragma unroll
                for (int h = k; h < k + 2; ++h) {
                  if (m[h] == T(-INFINITY)) continue;
#pragma unroll
                  for (int u = 0; u < U; ++u) acc[h].add(sm_exp(x[u][h], m[h]));
                }
                continue;
              }
              float2 s2 = f2(acc[k].s, acc[k + 1].s), c2 = f2(acc[k].c, acc[k + 1].c);
              const float2 m2 = f2(m[k], m[k + 1]);
#pragma unroll
              for (int u = 0; u < U; ++u) two_sum2(s2, c2, ex2_2(fsub2(f2(x[u][k], x[u][k + 1]), m2)));
              acc[k].s = s2.x; acc[k + 1].s = s2.y; acc[k].c = c2.x; acc[k + 1].c = c2.y;
            }
          } else {
#pragma unroll
            for (int k = 0; k < V; ++k) {
              if (m[k] == T(-INFINITY)) continue;
#pragma unroll
              for (int u = 0; u < U; ++u) acc[k].add(sm_exp(x[u][k], m[k]));
            }
          }
        }
      } else {
        // rolled: one sub-step per iteration, the batch shifted down a slot
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
          if (((bits >> u) & 1u) && (b > 0 || u > 0)) { flush(); ++piece; }
#pragma unroll
          for (int k = 0; k < V; ++k) {
            if constexpr (BWD) {
              acc[k].add_prod(x[0][k], gg[0][k]);
            } else if (x[0][k] != T(-INFINITY)) {
              if (x[0][k] > m[k]) {
                if (m[k] != T(-INFINITY)) acc[k].scale(sm_exp(m[k], x[0][k]));
                m[k] = x[0][k];
              }
              acc[k].add(sm_exp(x[0][k], m[k]));
            }
          }
#pragma unroll
          for (int w = 0; w + 1 < U; ++w) {
#pragma unroll
            for (int k = 0; k < V; ++k) { x[w][k] = x[w + 1][k]; gg[w][k] = gg[w + 1][k]; }
          }
        }
      }
    }
    flush();  // pieces never cross a chunk boundary
    c = (int64_t)__shfl_sync(kFull, nxt, 0);
    if (c >= sg.n_chunks) return;
    if (lane == 0) nxt = atomicAdd(sg.counter, 1ull);
  }
}

// one warp per (heavy row, column): lanes fold strided pieces of the row in
// piece order, then a fixed xor tree combines the lanes (deterministic)
template <typename T, bool BWD>
__global__ void edge_softmax_seg_merge(const SoftmaxArgs a, const SegArgs sg) {
  const int lane = threadIdx.x & 31;
  const int64_t total = a.n_heavy * (int64_t)a.H;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T* PM = static_cast<const T*>(sg.pm);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < total; i += nw) {
    const int64_t r = i / a.H;
    const int c = (int)(i - r * a.H);
    const int64_t q0 = sg.row_ptr[r], q1 = sg.row_ptr[r + 1];
    T mm = -INFINITY;
    double ll = 0.0;
    for (int64_t q = q0 + lane; q < q1; q += 32) {
      const int64_t at = (int64_t)__ldg(sg.row_pieces + q) * a.H + c;
      if constexpr (BWD) ll += sg.pl[at];
      else sm_merge<T>(mm, ll, PM[at], sg.pl[at]);
    }
    for (int off = 1; off < 32; off <<= 1) {
      const double ol = __shfl_xor_sync(kFull, ll, off);
      if constexpr (BWD) {
        ll += ol;
      } else {
        const T om = __shfl_xor_sync(kFull, mm, off);
        sm_merge<T>(mm, ll, om, ol);
      }
    }
    if (lane != 0) continue;
    const int64_t row = a.order[r];
    T* st = static_cast<T*>(a.stat) + row * 2 * (int64_t)a.H + c;
    if constexpr (BWD) {
      const T hi = (T)ll;
      st[0] = hi;
      st[a.H] = (T)(ll - (double)hi);
    } else {
      st[0] = mm;
      st[a.H] = (T)(1.0 / ll);
    }
  }
}

// alpha[e] = exp(s[e] - max[dst e]) * inv_sum[dst e]   (fwd)
// ds[e]    = alpha[e] * (g[e] - sum[dst e])            (bwd)
// Edge-id order: s / g / alpha / ds stream coalesced; the per-destination
// statistics (T pairs, (n, H)) are L2-resident gathers. The destination ids
// of a thread's next group are loaded while the current group computes, so
// the dependent statistics gather is not serialised behind a DRAM miss on
// dst[e].
// one vector per thread per step: with the destination ids pipelined, more
// vectors in flight per thread only cost occupancy (measured H=8: 1 -> 3.05
// ms, 2 -> 3.18, 4 -> 3.25, 8 -> 4.28)
constexpr int kApplyU = 1;

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
    T x[kApplyU][V], xl[kApplyU][V], gg[kApplyU][V], p0[kApplyU][V], p1[kApplyU][V];
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
        for (int k = 0; k < V; ++k) uv_score(x[u][k], xr[k], x[u][k], xl[u][k]);
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
          if constexpr (UV) r[k] = sm_exp(x[u][k], xl[u][k], p0[u][k]) * p1[u][k];
          else r[k] = sm_exp(x[u][k], p0[u][k]) * p1[u][k];
        }
      }
      store_vec<T, V>(static_cast<T*>(a.out) + ev[u] * a.ldo + cv[u], r);
    }
  }
}

cudaError_t launch_edge_softmax(int dtype_is_f64, int V, bool bwd, bool uv, const SoftmaxArgs& a,
                                int64_t grid, cudaStream_t s);
cudaError_t launch_edge_softmax_slots(int dtype_is_f64, int V, bool bwd, bool uv,
                                      const SoftmaxArgs& a, cudaStream_t s);
cudaError_t launch_edge_softmax_window(int dtype_is_f64, int V, bool bwd, const SoftmaxArgs& a,
                                       const WindowArgs& w, cudaStream_t s);
cudaError_t launch_edge_softmax_apply(int dtype_is_f64, int V, bool bwd, bool uv,
                                      const SoftmaxArgs& a, cudaStream_t s);
cudaError_t launch_edge_softmax_seg(int dtype_is_f64, int V, bool bwd, const SoftmaxArgs& a,
                                    const SegArgs& sg, cudaStream_t s);

}  // namespace gmp
