// softmax.cuh - fused edge_softmax forward and backward.
//
// Forward replaces messaging.edge_softmax (messaging.py:105-126), which
// dispatches gspmm(copy_rhs(edge), max) -> gsddmm(sub(edge,dst)) -> exp ->
// gspmm(copy_rhs(edge), sum) -> gsddmm(div(edge,dst)) and keeps four (m,H) /
// (n,H) temporaries. Here one kernel walks each destination's in-edges twice:
//   pass 1: online (max, sum of exp) per head column, fp64 sum;
//   pass 2: alpha = exp(s - max) / sum, written at the edge id.
// Backward (the composition of those four kernel backwards, autodiff.py:398-418)
// is the closed form  ds = alpha * (g - sum_{in-edges} alpha * g), again two
// passes per destination. Same row schedule as spmm_rows.cuh (degree-sorted,
// CTA per heavy row, warp per light row); columns tiled when H > 32 * V.
#pragma once

#include "gmp_common.cuh"
#include "spmm_rows.cuh"

namespace gmp {

struct SoftmaxArgs {
  const int64_t* indptr;
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
};

__device__ __forceinline__ float exp_t(float x) { return expf(x); }
__device__ __forceinline__ double exp_t(double x) { return exp(x); }

// (m, l) online-softmax merge; empty partials carry m = -inf, l = 0.
template <typename T>
__device__ __forceinline__ void sm_merge(T& m, double& l, T om, double ol) {
  if (om == -INFINITY) return;
  if (m == -INFINITY) { m = om; l = ol; return; }
  if (om > m) { l = l * (double)exp_t(T(m - om)) + ol; m = om; }
  else        { l += ol * (double)exp_t(T(om - m)); }
}

template <typename T, int V, bool BWD>
__global__ void __launch_bounds__(kWarpsPerCta * 32) edge_softmax_kernel(const SoftmaxArgs a) {
  __shared__ double s_l[kWarpsPerCta][32 * V];
  __shared__ T s_m[kWarpsPerCta][32 * V];
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
  if (pe == pb) return;  // no in-edges: nothing keyed to this row (block-uniform when heavy)
  const int col = c0 + gl * V;
  const bool valid = col < c1;
  const T* S = static_cast<const T*>(a.s);
  const T* Gd = static_cast<const T*>(a.g);
  T* O = static_cast<T*>(a.out);
  const int64_t first = heavy ? (int64_t)warp * 32 : 0;
  const int64_t stride = heavy ? 32 * kWarpsPerCta : 32;

  // ---- pass 1 ----
  T m[V];
  double l[V];
#pragma unroll
  for (int k = 0; k < V; ++k) { m[k] = -INFINITY; l[k] = 0.0; }
  for (int64_t base = pb + first; base < pe; base += stride) {
    const int cnt = batch_count(pe - base);
    const int32_t eb = lane < cnt ? __ldg(a.eids + base + lane) : 0;
    for (int t = 0; t < cnt; t += E) {
      const int j = t + slot;
      const int32_t e = __shfl_sync(kFull, eb, j & 31);
      if (j < cnt && valid) {
        T x[V];
        load_vec<T, V>(S + (int64_t)e * a.lds + col, x);
        if constexpr (BWD) {
          T gg[V];
          load_vec<T, V>(Gd + (int64_t)e * a.ldg + col, gg);
#pragma unroll
          for (int k = 0; k < V; ++k) l[k] += (double)x[k] * (double)gg[k];
        } else {
#pragma unroll
          for (int k = 0; k < V; ++k) {
            if (x[k] > m[k]) { l[k] = l[k] * (double)exp_t(T(m[k] - x[k])) + 1.0; m[k] = x[k]; }
            else             { l[k] += (double)exp_t(T(x[k] - m[k])); }
          }
        }
      }
    }
  }
  for (int off = G; off < 32; off <<= 1) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const double ol = shfl_xor_d(l[k], off);
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

  // ---- pass 2 ----
  T inv[V];
#pragma unroll
  for (int k = 0; k < V; ++k) inv[k] = BWD ? T(0) : (T)(1.0 / l[k]);
  for (int64_t base = pb + first; base < pe; base += stride) {
    const int cnt = batch_count(pe - base);
    const int32_t eb = lane < cnt ? __ldg(a.eids + base + lane) : 0;
    for (int t = 0; t < cnt; t += E) {
      const int j = t + slot;
      const int32_t e = __shfl_sync(kFull, eb, j & 31);
      if (j < cnt && valid) {
        T x[V], r[V];
        load_vec<T, V>(S + (int64_t)e * a.lds + col, x);
        if constexpr (BWD) {
          T gg[V];
          load_vec<T, V>(Gd + (int64_t)e * a.ldg + col, gg);
#pragma unroll
          for (int k = 0; k < V; ++k) r[k] = (T)((double)x[k] * ((double)gg[k] - l[k]));
        } else {
#pragma unroll
          for (int k = 0; k < V; ++k) r[k] = exp_t(T(x[k] - m[k])) * inv[k];
        }
        store_vec<T, V>(O + (int64_t)e * a.ldo + col, r);
      }
    }
  }
}

cudaError_t launch_edge_softmax(int dtype_is_f64, int V, bool bwd, const SoftmaxArgs& a,
                                int64_t grid, cudaStream_t s);

}  // namespace gmp
