// spmm_dot.cuh - g-SpMM with a dot-product message (d_out == 1).
//
// Replaces gspmm for phi = dot(a, b) (kernels.py:290-293: the message is the
// row sum of a*b, one column). Same row schedule as spmm_rows.cuh; inside a
// warp, G lanes cooperate on one edge's dot (fp64 partials, xor-shuffle tree),
// E = 32 / G edges run side by side, then rho reduces across edge slots.
#pragma once

#include "gmp_common.cuh"
#include "spmm_rows.cuh"
#include "softmax.cuh"

namespace gmp {

struct SpmmDotArgs {
  const int64_t* indptr;
  const int32_t* indices;
  const int32_t* eids;
  const int32_t* order;
  int64_t n_rows;
  int64_t n_heavy;
  int64_t n_medium;       // rows [n_heavy, n_medium): one warp each; the rest one per lane group
  int64_t medium_blocks;  // CTAs covering the warp rows
  int32_t dim;     // operand width
  int32_t g_log2;  // lanes per edge
  int32_t mean;
  OperandDev lhs, rhs;
  void* Z;
  int64_t ldz;
  int64_t* arg;
  int64_t* counts;
  int32_t cluster;  // CTAs per heavy row (thread-block cluster), 1 = one CTA
};

template <typename T, int V>
__device__ __forceinline__ double dot_partial(const OperandDev& a, const OperandDev& b, int64_t row,
                                              int32_t nbr, int32_t eid, int gl, int G, int dim) {
  const int64_t ra = a.target == T_SRC ? nbr : (a.target == T_DST ? row : eid);
  const int64_t rb = b.target == T_SRC ? nbr : (b.target == T_DST ? row : eid);
  const T* pa = static_cast<const T*>(a.data) + ra * a.ld;
  const T* pb = static_cast<const T*>(b.data) + rb * b.ld;
  ColSum<T> cs;
  for (int c = gl * V; c < dim; c += G * V) {
    T xa[V], xb[V];
    load_vec<T, V>(pa + c, xa);
    load_vec<T, V>(pb + c, xb);
#pragma unroll
    for (int k = 0; k < V; ++k) cs.add_prod(xa[k], xb[k]);
  }
  const double s = cs.value();
  return s;
}

template <typename T, int RHO, int V>
__global__ void __launch_bounds__(kWarpsPerCta * 32) spmm_dot_kernel(const SpmmDotArgs a) {
  __shared__ double s_acc[kWarpsPerCta];
  __shared__ int32_t s_arg[kWarpsPerCta];
  const int64_t local = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = 1 << a.g_log2, E = 32 >> a.g_log2;
  const int slot = lane >> a.g_log2, gl = lane & (G - 1);
  const int ncl = a.cluster > 1 ? a.cluster : 1;
  const int64_t heavy_blocks = a.n_heavy * ncl;
  const bool heavy = local < heavy_blocks;
  const int crank = heavy ? (int)(local % ncl) : 0;
  const bool light = local >= heavy_blocks + a.medium_blocks;  // block-uniform
  int64_t row;
  if (heavy) {
    row = a.order[local / ncl];
  } else if (!light) {
    const int64_t r = a.n_heavy + (local - heavy_blocks) * kWarpsPerCta + warp;
    if (r >= a.n_medium) return;
    row = a.order ? (int64_t)a.order[r] : r;
  } else {
    // short rows (<= light threshold in-edges): each lane group owns a row
    // and walks its edges itself, E rows per warp
    const int64_t r = a.n_medium +
                      ((local - heavy_blocks - a.medium_blocks) * kWarpsPerCta + warp) * E + slot;
    if (__all_sync(kFull, r >= a.n_rows)) return;
    row = r < a.n_rows ? (a.order ? (int64_t)a.order[r] : r) : -1;
  }
  const int64_t pb = row >= 0 ? a.indptr[row] : 0, pe = row >= 0 ? a.indptr[row + 1] : 0;
  const int64_t deg = pe - pb;
  double acc = (RHO == RHO_SUM) ? 0.0 : ext_init<RHO>();
  int32_t arg = 0x7fffffff;
  if (light) {
    const int max_deg = (int)__reduce_max_sync(kFull, (unsigned)deg);
    for (int j = 0; j < max_deg; ++j) {
      const bool ok = j < deg;
      const int32_t uu = ok ? __ldg(a.indices + pb + j) : 0;
      const int32_t ee = ok ? __ldg(a.eids + pb + j) : 0;
      double s = 0.0;
      if (ok) s = dot_partial<T, V>(a.lhs, a.rhs, row, uu, ee, gl, G, a.dim);
      for (int off = 1; off < G; off <<= 1) s += shfl_xor_d(s, off);
      if (ok) {
        if constexpr (RHO == RHO_SUM) acc += s;
        else ext_update<RHO>(acc, arg, s, ee);
      }
    }
    if (row < 0 || gl != 0) return;
    T* z = static_cast<T*>(a.Z) + row * a.ldz;
    if (a.counts) a.counts[row] = deg;
    if constexpr (RHO == RHO_SUM) {
      double v = acc;
      if (a.mean && deg > 0) v = v / (double)deg;
      *z = (T)v;
    } else {
      *z = deg > 0 ? (T)acc : T(0);
      a.arg[row] = deg > 0 ? arg : -1;
    }
    return;
  }
  const int64_t first = heavy ? ((int64_t)crank * kWarpsPerCta + warp) * 32 : 0;
  const int64_t stride = heavy ? (int64_t)32 * kWarpsPerCta * ncl : 32;
  // kDotU batches per iteration: their index loads and dot products are
  // independent, so a lane keeps kDotU edges in flight (hub rows would
  // otherwise walk one dependent load chain per 32 edges)
  constexpr int kDotU = 4;
  for (int64_t base0 = pb + first; base0 < pe; base0 += stride * kDotU) {
    int nb[kDotU], eb[kDotU], cnt[kDotU];
#pragma unroll
    for (int u = 0; u < kDotU; ++u) {
      const int64_t base = base0 + u * stride;
      cnt[u] = base < pe ? batch_count(pe - base) : 0;
      nb[u] = lane < cnt[u] ? __ldg(a.indices + base + lane) : 0;
      eb[u] = lane < cnt[u] ? __ldg(a.eids + base + lane) : 0;
    }
    for (int t = 0; t < 32; t += E) {
      double sv[kDotU];
      int32_t ev[kDotU];
#pragma unroll
      for (int u = 0; u < kDotU; ++u) {
        const int j = t + slot;
        const int32_t uu = __shfl_sync(kFull, nb[u], j & 31);
        ev[u] = __shfl_sync(kFull, eb[u], j & 31);
        sv[u] = 0.0;
        if (j < cnt[u]) sv[u] = dot_partial<T, V>(a.lhs, a.rhs, row, uu, ev[u], gl, G, a.dim);
      }
#pragma unroll
      for (int u = 0; u < kDotU; ++u) {
        double s = sv[u];
        for (int off = 1; off < G; off <<= 1) s += shfl_xor_d(s, off);
        if (t + slot < cnt[u]) {
          if constexpr (RHO == RHO_SUM) acc += s;
          else ext_update<RHO>(acc, arg, s, ev[u]);
        }
      }
    }
  }
  for (int off = G; off < 32; off <<= 1) {
    const double o = shfl_xor_d(acc, off);
    if constexpr (RHO == RHO_SUM) acc += o;
    else ext_update<RHO>(acc, arg, o, __shfl_xor_sync(kFull, arg, off));
  }
  if (heavy) {
    if (lane == 0) { s_acc[warp] = acc; s_arg[warp] = arg; }
    __syncthreads();
    if (threadIdx.x == 0) {
      acc = s_acc[0]; arg = s_arg[0];
      for (int w = 1; w < kWarpsPerCta; ++w) {
        if constexpr (RHO == RHO_SUM) acc += s_acc[w];
        else ext_update<RHO>(acc, arg, s_acc[w], s_arg[w]);
      }
    }
    if (ncl > 1) {
      // the row's CTAs form a cluster: rank 0 merges the ranks' partials
      // from their shared memory (DSMEM) in rank order
      namespace cg = cooperative_groups;
      cg::cluster_group cluster = cg::this_cluster();
      if (threadIdx.x == 0) { s_acc[0] = acc; s_arg[0] = arg; }
      cluster.sync();
      if (threadIdx.x == 0 && crank == 0) {
        for (int r = 1; r < ncl; ++r) {
          const double o = *cluster.map_shared_rank(&s_acc[0], r);
          const int32_t oa = *cluster.map_shared_rank(&s_arg[0], r);
          if constexpr (RHO == RHO_SUM) acc += o;
          else ext_update<RHO>(acc, arg, o, oa);
        }
      }
      cluster.sync();
      if (crank != 0) return;
    }
    if (threadIdx.x != 0) return;
  } else if (lane != 0) {
    return;
  }
  T* z = static_cast<T*>(a.Z) + row * a.ldz;
  if (a.counts) a.counts[row] = deg;
  if constexpr (RHO == RHO_SUM) {
    double v = acc;
    if (a.mean && deg > 0) v = v / (double)deg;
    *z = (T)v;
  } else {
    *z = deg > 0 ? (T)acc : T(0);
    a.arg[row] = deg > 0 ? arg : -1;
  }
}

cudaError_t launch_spmm_dot(int dtype_is_f64, int rho, int V, const SpmmDotArgs& a, int64_t grid,
                            cudaStream_t s);

}  // namespace gmp
