// sddmm.cuh - g-SDDMM, edge-parallel over the COO list.
//
// Replaces kernels.gsddmm's default edge_parallel strategy over COO
// (kernels.py:744-836, hot loop _gsddmm_chunked kernels.py:732-741): one
// output row per edge, in edge-id order. A warp takes 32 consecutive edges,
// loads their (src, dst) ids coalesced, and E = 32 / G edge slots of G lanes
// each write whole output rows with vector stores (coalesced in edge order).
// dot messages reduce over the operand width with an fp64 xor-shuffle tree.
#pragma once

#include "gmp_common.cuh"
#include "softmax.cuh"

namespace gmp {

struct SddmmArgs {
  const int32_t* src;
  const int32_t* dst;
  int64_t m;
  int32_t d_out;  // output width (1 for dot)
  int32_t dim;    // operand width for dot
  int32_t g_log2;
  OperandDev lhs, rhs;
  void* M;
  int64_t ldm;
  int32_t* err_eid;
};

__device__ __forceinline__ int64_t operand_row(const OperandDev& o, int32_t u, int32_t v, int64_t e) {
  return o.target == T_SRC ? (int64_t)u : (o.target == T_DST ? (int64_t)v : e);
}

template <typename T, int V>
__device__ __forceinline__ void load_elem(const OperandDev& o, int64_t r, int c, T (&out)[V]) {
  const T* base = static_cast<const T*>(o.data) + r * o.ld;
  if (o.bcast) {
    const T s = __ldg(base);
#pragma unroll
    for (int k = 0; k < V; ++k) out[k] = s;
  } else {
    load_vec<T, V>(base + c, out);
  }
}

template <typename T, int OP, int V>
__global__ void __launch_bounds__(256) sddmm_kernel(const SddmmArgs a) {
  constexpr bool BIN = OP != OP_COPY;
  const int lane = threadIdx.x & 31;
  const int G = 1 << a.g_log2, E = 32 >> a.g_log2;
  const int slot = lane >> a.g_log2, gl = lane & (G - 1);
  const int64_t warp_id = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp_id * 32; b < a.m; b += n_warps * 32) {
    const int cnt = batch_count(a.m - b);
    int32_t su = 0, sv = 0;
    if (lane < cnt) {
      su = __ldg(a.src + b + lane);
      sv = __ldg(a.dst + b + lane);
    }
    for (int t = 0; t < cnt; t += E) {
      const int j = t + slot;
      const int32_t u = __shfl_sync(kFull, su, j & 31);
      const int32_t v = __shfl_sync(kFull, sv, j & 31);
      const int64_t e = b + j;
      if constexpr (OP == OP_DOT) {
        ColSum<T> cs;
        if (j < cnt) {
          const T* pa = static_cast<const T*>(a.lhs.data) + operand_row(a.lhs, u, v, e) * a.lhs.ld;
          const T* pb = static_cast<const T*>(a.rhs.data) + operand_row(a.rhs, u, v, e) * a.rhs.ld;
          for (int c = gl * V; c < a.dim; c += G * V) {
            T xa[V], xb[V];
            load_vec<T, V>(pa + c, xa);
            load_vec<T, V>(pb + c, xb);
#pragma unroll
            for (int k = 0; k < V; ++k) cs.add_prod(xa[k], xb[k]);
          }
        }
        double s = cs.value();
        for (int off = 1; off < G; off <<= 1) s += shfl_xor_d(s, off);
        if (j < cnt && gl == 0) static_cast<T*>(a.M)[e * a.ldm] = (T)s;
      } else {
        if (j >= cnt) continue;
        const int64_t ra = operand_row(a.lhs, u, v, e);
        const int64_t rb = BIN ? operand_row(a.rhs, u, v, e) : 0;
        T* out = static_cast<T*>(a.M) + e * a.ldm;
        bool zero = false;
        for (int c = gl * V; c < a.d_out; c += G * V) {
          T xa[V], xb[V], r[V];
          load_elem<T, V>(a.lhs, ra, c, xa);
          if constexpr (BIN) load_elem<T, V>(a.rhs, rb, c, xb);
#pragma unroll
          for (int k = 0; k < V; ++k) {
            if constexpr (OP == OP_DIV) zero |= (xb[k] == T(0));
            // an IEEE op on T operands == the fp64 op rounded to T (no double
            // rounding issue for + - * /), so the reference's fp64 message
            // cast to T is reproduced bit-exactly without conversions
            r[k] = apply_op_t<OP, T>(xa[k], BIN ? xb[k] : T(0));
          }
          store_vec<T, V>(out + c, r);
        }
        if constexpr (OP == OP_DIV) {
          if (zero) atomicMin(a.err_eid, (int32_t)e);
        }
      }
    }
  }
}

// Narrow dot messages (dim <= 32 floats / 16 doubles): one edge per lane.
// Consecutive lanes own consecutive edges, so the (src, dst) loads and the
// M stores are coalesced; each lane reads its two operand rows with vector
// loads (one 128 B line each at most) and forms the exact dot product as a
// compensated fp32 pair (TwoProduct + TwoSum on packed FFMA2 / FADD2),
// rounded once through fp64 - no shuffles and no per-element conversions.
template <typename T, int V>
__global__ void __launch_bounds__(256) sddmm_dot_lane_kernel(const SddmmArgs a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // the next edge's (src, dst) are loaded while the current edge's rows are
  // gathered and reduced: the DRAM read of the ids leaves the dependent chain
  int32_t un = 0, vn = 0;
  if (e < a.m) { un = __ldg(a.src + e); vn = __ldg(a.dst + e); }
  for (; e < a.m; e += stride) {
    const int32_t u = un, v = vn;
    if (e + stride < a.m) { un = __ldg(a.src + e + stride); vn = __ldg(a.dst + e + stride); }
    const T* pa = static_cast<const T*>(a.lhs.data) + operand_row(a.lhs, u, v, e) * a.lhs.ld;
    const T* pb = static_cast<const T*>(a.rhs.data) + operand_row(a.rhs, u, v, e) * a.rhs.ld;
    double r;
    if constexpr (sizeof(T) == 4 && V >= 2) {
      float2 S = f2(0.f, 0.f), C = f2(0.f, 0.f);
#pragma unroll 4
      for (int c = 0; c < a.dim; c += V) {
        T xa[V], xb[V];
        load_vec<T, V>(pa + c, xa);
        load_vec<T, V>(pb + c, xb);
#pragma unroll
        for (int k = 0; k < V; k += 2) {
          const float2 x = f2(xa[k], xa[k + 1]), y = f2(xb[k], xb[k + 1]);
          two_sum_prod2(S, C, x, y);  // spmm_rows.cuh: exact products, no contraction
        }
      }
      r = ((double)S.x + (double)S.y) + ((double)C.x + (double)C.y);
    } else {
      ColSum<T> cs;
#pragma unroll 4
      for (int c = 0; c < a.dim; c += V) {
        T xa[V], xb[V];
        load_vec<T, V>(pa + c, xa);
        load_vec<T, V>(pb + c, xb);
#pragma unroll
        for (int k = 0; k < V; ++k) cs.add_prod(xa[k], xb[k]);
      }
      r = cs.value();
    }
    static_cast<T*>(a.M)[e * a.ldm] = (T)r;
  }
}

cudaError_t launch_sddmm(int dtype_is_f64, int op, int V, const SddmmArgs& a, int64_t grid,
                         cudaStream_t s);

}  // namespace gmp
