// spmm_rows.cuh - the g-SpMM row kernel (elementwise messages).
//
// Replaces the reference's default gspmm strategy, node_parallel over the
// in-adjacency (kernels.py:473-482) and its per-destination segment walk
// _GroupedWalk (kernels.py:340-466): for every destination row v,
//   Z[v, c] = rho_{(u,e,v)} phi(lhs[., c], rhs[., c])
// with the message formed in registers and never materialised.
//
// Work decomposition:
//  * columns are split into tiles of `tile_cols` (the reference's
//    feature_parallel column split, kernels.py:485-513) so that one column
//    slice of the gathered source matrix stays L2-resident; tiles are the
//    slowest-varying grid index, so concurrently running CTAs share a slice;
//  * rows come in degree-descending order (gmp_sched). The first n_heavy rows
//    (degree > heavy threshold) are reduced by a whole CTA (warps interleave
//    32-edge batches, partials merged through shared memory in warp order);
//    the rest are reduced by one warp each;
//  * inside a warp, 32 lanes = E edge slots x G feature lanes; each feature
//    lane owns P vectors of V elements (128/64-bit loads). Edge indices are
//    loaded 32 at a time, coalesced, and broadcast by shuffle; the next batch
//    is prefetched while the current one is gathered.
//  * slot partials are combined by a fixed xor-shuffle tree: results are
//    deterministic run to run.
#pragma once

#include "gmp_common.cuh"

namespace gmp {

constexpr int kWarpsPerCta = 8;

struct SpmmArgs {
  const int64_t* indptr;
  const int32_t* indices;
  const int32_t* eids;
  const int32_t* order;  // nullable: identity order
  int64_t n_rows;
  int64_t n_heavy;
  int64_t blocks_per_tile;
  int32_t d_out;
  int32_t tile_cols;
  int32_t g_log2;  // feature lanes per edge slot = 1 << g_log2
  int32_t mean;
  OperandDev lhs, rhs;
  void* Z;
  int64_t ldz;
  int64_t* arg;
  int64_t* counts;
  int32_t* err_pos;
};

template <typename T, int V, int P>
__device__ __forceinline__ void load_hoisted(const OperandDev& o, int64_t row, const int (&colv)[P],
                                             const bool (&valid)[P], T (&h)[P][V]) {
  const T* base = static_cast<const T*>(o.data) + row * o.ld;
  if (o.bcast) {
    const T s = __ldg(base);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int k = 0; k < V; ++k) h[p][k] = s;
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (valid[p]) load_vec<T, V>(base + colv[p], h[p]);
      else
#pragma unroll
        for (int k = 0; k < V; ++k) h[p][k] = T(0);
    }
  }
}

template <typename T, int V, int P>
__device__ __forceinline__ void load_operand(const OperandDev& o, int32_t nbr, int32_t eid,
                                             const int (&colv)[P], const bool (&valid)[P],
                                             const T (&hoisted)[P][V], T (&out)[P][V]) {
  if (o.target == T_DST) {
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int k = 0; k < V; ++k) out[p][k] = hoisted[p][k];
    return;
  }
  const int64_t r = (o.target == T_SRC) ? nbr : eid;
  const T* base = static_cast<const T*>(o.data) + r * o.ld;
  if (o.bcast) {
    const T s = __ldg(base);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int k = 0; k < V; ++k) out[p][k] = s;
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p)
      if (valid[p]) load_vec<T, V>(base + colv[p], out[p]);
  }
}

// Accumulate the messages of edges [pb, pe) of one row owned by this warp:
// 32-edge batches starting at pb + first, advancing by `stride` edges.
template <typename T, int OP, int RHO, int V, int P, int U>
__device__ __forceinline__ void spmm_accumulate(const SpmmArgs& a, int64_t pb, int64_t pe,
                                                int64_t first, int64_t stride, int lane, int slot,
                                                int E, const int (&colv)[P], const bool (&valid)[P],
                                                const T (&ha)[P][V], const T (&hb)[P][V],
                                                double (&acc)[P][V], int32_t (&arg)[P][V]) {
  constexpr bool BIN = OP != OP_COPY;
  const bool need_eid = (a.lhs.target == T_EDGE) || (BIN && a.rhs.target == T_EDGE) ||
                        (RHO != RHO_SUM);
  const int32_t* __restrict__ indices = a.indices;
  const int32_t* __restrict__ eids = a.eids;

  int64_t base = pb + first;
  int nb = 0, eb = 0;
  if (base < pe && lane < pe - base) {
    nb = __ldg(indices + base + lane);
    if (need_eid) eb = __ldg(eids + base + lane);
  }
  for (; base < pe; base += stride) {
    const int cnt = batch_count(pe - base);
    // prefetch the next batch's indices while this one is gathered
    const int64_t nbase = base + stride;
    int nb_next = 0, eb_next = 0;
    if (nbase < pe && lane < pe - nbase) {
      nb_next = __ldg(indices + nbase + lane);
      if (need_eid) eb_next = __ldg(eids + nbase + lane);
    }
    for (int t = 0; t < cnt; t += E * U) {
      T va[U][P][V];
      T vb[U][P][V];
      int32_t ee[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = t + slot + E * u;
        ok[u] = j < cnt;
        const int src_lane = j & 31;
        const int32_t uu = __shfl_sync(kFull, nb, src_lane);
        ee[u] = need_eid ? __shfl_sync(kFull, eb, src_lane) : 0;
        if (ok[u]) {
          load_operand<T, V, P>(a.lhs, uu, ee[u], colv, valid, ha, va[u]);
          if constexpr (BIN) load_operand<T, V, P>(a.rhs, uu, ee[u], colv, valid, hb, vb[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
        if constexpr (OP == OP_DIV) {
          bool zero = false;
#pragma unroll
          for (int p = 0; p < P; ++p)
            if (valid[p])
#pragma unroll
              for (int k = 0; k < V; ++k) zero |= (vb[u][p][k] == T(0));
          if (zero) atomicMin(a.err_pos, (int32_t)(base + t + slot + E * u));
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
          if (!valid[p]) continue;
#pragma unroll
          for (int k = 0; k < V; ++k) {
            const double x = apply_op<OP>((double)va[u][p][k], BIN ? (double)vb[u][p][k] : 0.0);
            if constexpr (RHO == RHO_SUM) acc[p][k] += x;
            else ext_update<RHO>(acc[p][k], arg[p][k], x, ee[u]);
          }
        }
      }
    }
    nb = nb_next;
    eb = eb_next;
  }
}

template <int RHO, int V, int P>
__device__ __forceinline__ void combine_slots(int g_log2, double (&acc)[P][V], int32_t (&arg)[P][V]) {
  for (int off = 1 << g_log2; off < 32; off <<= 1) {
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const double o = shfl_xor_d(acc[p][k], off);
        if constexpr (RHO == RHO_SUM) {
          acc[p][k] += o;
        } else {
          const int32_t oa = __shfl_xor_sync(kFull, arg[p][k], off);
          ext_update<RHO>(acc[p][k], arg[p][k], o, oa);
        }
      }
  }
}

template <typename T, int RHO, int V, int P>
__device__ __forceinline__ void write_row(const SpmmArgs& a, int64_t row, int64_t deg,
                                          const int (&colv)[P], const bool (&valid)[P],
                                          const double (&acc)[P][V], const int32_t (&arg)[P][V]) {
  T* z = static_cast<T*>(a.Z) + row * a.ldz;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    if (!valid[p]) continue;
    T out[V];
    if constexpr (RHO == RHO_SUM) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        double v = acc[p][k];
        if (a.mean && deg > 0) v = v / (double)deg;  // kernels.py:719-722
        out[k] = (T)v;
      }
      store_vec<T, V>(z + colv[p], out);
    } else {
      int32_t ar[V];
#pragma unroll
      for (int k = 0; k < V; ++k) {
        out[k] = deg > 0 ? (T)acc[p][k] : T(0);
        ar[k] = deg > 0 ? arg[p][k] : -1;
      }
      store_vec<T, V>(z + colv[p], out);
      store_arg<V>(a.arg + row * (int64_t)a.d_out + colv[p], ar);
    }
  }
}

template <typename T, int OP, int RHO, int V, int P>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
spmm_rows_kernel(const SpmmArgs a) {
  constexpr int U = (16 / (P * V)) < 2 ? 2 : (16 / (P * V));
  constexpr int kCols = 32 * V * P;  // widest tile one warp covers
  __shared__ double s_acc[kWarpsPerCta][kCols];
  __shared__ int32_t s_arg[RHO == RHO_SUM ? 1 : kWarpsPerCta][kCols];

  const int64_t bid = blockIdx.x;
  const int tile = (int)(bid / a.blocks_per_tile);
  const int64_t local = bid - (int64_t)tile * a.blocks_per_tile;
  const int c0 = tile * a.tile_cols;
  const int c1 = min(a.d_out, c0 + a.tile_cols);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int G = 1 << a.g_log2;
  const int E = 32 >> a.g_log2;
  const int slot = lane >> a.g_log2;
  const int gl = lane & (G - 1);
  const bool heavy = local < a.n_heavy;  // block-uniform

  int64_t row;
  if (heavy) {
    row = a.order[local];
  } else {
    const int64_t r = a.n_heavy + (local - a.n_heavy) * kWarpsPerCta + warp;
    if (r >= a.n_rows) return;  // light mode never synchronises the CTA
    row = a.order ? (int64_t)a.order[r] : r;
  }
  const int64_t pb = a.indptr[row];
  const int64_t pe = a.indptr[row + 1];
  const int64_t deg = pe - pb;

  int colv[P];
  bool valid[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    colv[p] = c0 + (gl + G * p) * V;
    valid[p] = colv[p] < c1;
  }

  T ha[P][V], hb[P][V];
  if (a.lhs.target == T_DST && deg > 0) load_hoisted<T, V, P>(a.lhs, row, colv, valid, ha);
  if (OP != OP_COPY && a.rhs.target == T_DST && deg > 0) {
    load_hoisted<T, V, P>(a.rhs, row, colv, valid, hb);
    if constexpr (OP == OP_DIV) {
      bool zero = false;
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (valid[p])
#pragma unroll
          for (int k = 0; k < V; ++k) zero |= (hb[p][k] == T(0));
      if (zero) atomicMin(a.err_pos, (int32_t)pb);
    }
  }

  double acc[P][V];
  int32_t arg[P][V];
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int k = 0; k < V; ++k) {
      acc[p][k] = (RHO == RHO_SUM) ? 0.0 : ext_init<RHO>();
      arg[p][k] = 0x7fffffff;
    }

  if (heavy) {
    spmm_accumulate<T, OP, RHO, V, P, U>(a, pb, pe, (int64_t)warp * 32, 32 * kWarpsPerCta, lane,
                                         slot, E, colv, valid, ha, hb, acc, arg);
  } else {
    spmm_accumulate<T, OP, RHO, V, P, U>(a, pb, pe, 0, 32, lane, slot, E, colv, valid, ha, hb,
                                         acc, arg);
  }
  combine_slots<RHO, V, P>(a.g_log2, acc, arg);

  if (a.counts && tile == 0 && ((heavy && threadIdx.x == 0) || (!heavy && lane == 0)))
    a.counts[row] = deg;

  if (!heavy) {
    if (slot == 0) write_row<T, RHO, V, P>(a, row, deg, colv, valid, acc, arg);
    return;
  }
  // CTA mode: merge the warp partials in warp order through shared memory.
  if (slot == 0) {
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int cl = (gl + G * p) * V + k;
        s_acc[warp][cl] = acc[p][k];
        if constexpr (RHO != RHO_SUM) s_arg[warp][cl] = arg[p][k];
      }
  }
  __syncthreads();
  if (warp == 0 && slot == 0) {
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int cl = (gl + G * p) * V + k;
        double v = s_acc[0][cl];
        int32_t ar = 0x7fffffff;
        if constexpr (RHO != RHO_SUM) ar = s_arg[0][cl];
        for (int w = 1; w < kWarpsPerCta; ++w) {
          if constexpr (RHO == RHO_SUM) v += s_acc[w][cl];
          else ext_update<RHO>(v, ar, s_acc[w][cl], s_arg[w][cl]);
        }
        acc[p][k] = v;
        arg[p][k] = ar;
      }
    write_row<T, RHO, V, P>(a, row, deg, colv, valid, acc, arg);
  }
}

template <typename T, int OP, int RHO, int V, int P>
cudaError_t launch_spmm_rows_t(const SpmmArgs& a, int64_t grid, cudaStream_t s) {
  spmm_rows_kernel<T, OP, RHO, V, P><<<(unsigned)grid, kWarpsPerCta * 32, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int OP, int RHO, int V>
cudaError_t launch_spmm_rows_p(int P, const SpmmArgs& a, int64_t grid, cudaStream_t s) {
  if (P == 1) return launch_spmm_rows_t<T, OP, RHO, V, 1>(a, grid, s);
  return launch_spmm_rows_t<T, OP, RHO, V, 2>(a, grid, s);
}

template <typename T, int OP, int RHO>
cudaError_t launch_spmm_rows_v(int V, int P, const SpmmArgs& a, int64_t grid, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if (V == 4) return launch_spmm_rows_p<T, OP, RHO, 4>(P, a, grid, s);
  }
  if (V == 2) return launch_spmm_rows_p<T, OP, RHO, 2>(P, a, grid, s);
  return launch_spmm_rows_p<T, OP, RHO, 1>(P, a, grid, s);
}

// Instantiated once per OP in spmm_op_<op>.cu so the op families compile in
// parallel.
template <int OP>
cudaError_t launch_spmm_rows(int dtype_is_f64, int rho, int V, int P, const SpmmArgs& a,
                             int64_t grid, cudaStream_t s) {
  if (dtype_is_f64) {
    if (rho == RHO_SUM) return launch_spmm_rows_v<double, OP, RHO_SUM>(V, P, a, grid, s);
    if (rho == RHO_MAX) return launch_spmm_rows_v<double, OP, RHO_MAX>(V, P, a, grid, s);
    return launch_spmm_rows_v<double, OP, RHO_MIN>(V, P, a, grid, s);
  }
  if (rho == RHO_SUM) return launch_spmm_rows_v<float, OP, RHO_SUM>(V, P, a, grid, s);
  if (rho == RHO_MAX) return launch_spmm_rows_v<float, OP, RHO_MAX>(V, P, a, grid, s);
  return launch_spmm_rows_v<float, OP, RHO_MIN>(V, P, a, grid, s);
}

}  // namespace gmp
