// gmp_common.cuh - device helpers shared by every libgmp kernel.
//
// Numerics contract: every per-edge message is formed in
// fp64 from the (exactly up-cast) operands, which is bit-identical to the
// reference's float64 arithmetic on the same inputs (kernels.py:216 coerces
// every operand to float64, kernels.py:281-293 applies the op). Sums, means and
// dots accumulate in fp64 and round once on store. max/min compare the fp64
// messages, so values and arg edges equal the reference's exactly.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gmp {

constexpr unsigned kFull = 0xffffffffu;

// op codes after host canonicalisation (copy_rhs is turned into copy of lhs)
enum { OP_COPY = 0, OP_ADD = 2, OP_SUB = 3, OP_MUL = 4, OP_DIV = 5, OP_DOT = 6 };
enum { RHO_SUM = 0, RHO_MAX = 1, RHO_MIN = 2 };
enum { T_SRC = 0, T_DST = 1, T_EDGE = 2 };

struct OperandDev {
  const void* data;
  int64_t ld;
  int32_t dim;
  int32_t target;  // T_SRC / T_DST / T_EDGE
  int32_t bcast;   // 1: single column broadcast over d_out
};

// ---- vector loads (read-only path) -----------------------------------------

template <typename T, int V> struct Vec;
template <> struct Vec<float, 1> { using type = float; };
template <> struct Vec<float, 2> { using type = float2; };
template <> struct Vec<float, 4> { using type = float4; };
template <> struct Vec<double, 1> { using type = double; };
template <> struct Vec<double, 2> { using type = double2; };

template <typename T, int V>
__device__ __forceinline__ void load_vec(const T* __restrict__ p, T (&out)[V]) {
  if constexpr (V == 1) {
    out[0] = __ldg(p);
  } else if constexpr (V == 2) {
    auto v = __ldg(reinterpret_cast<const typename Vec<T, 2>::type*>(p));
    out[0] = v.x; out[1] = v.y;
  } else {
    auto v = __ldg(reinterpret_cast<const typename Vec<T, 4>::type*>(p));
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  }
}

template <typename T, int V>
__device__ __forceinline__ void store_vec(T* p, const T (&in)[V]) {
  if constexpr (V == 1) {
    *p = in[0];
  } else if constexpr (V == 2) {
    typename Vec<T, 2>::type v; v.x = in[0]; v.y = in[1];
    *reinterpret_cast<typename Vec<T, 2>::type*>(p) = v;
  } else {
    typename Vec<T, 4>::type v; v.x = in[0]; v.y = in[1]; v.z = in[2]; v.w = in[3];
    *reinterpret_cast<typename Vec<T, 4>::type*>(p) = v;
  }
}

template <int V>
__device__ __forceinline__ void store_arg(int64_t* p, const int32_t (&a)[V]) {
  if constexpr (V == 1) {
    *p = a[0];
  } else if constexpr (V == 2) {
    longlong2 v; v.x = a[0]; v.y = a[1];
    *reinterpret_cast<longlong2*>(p) = v;
  } else {
    longlong2 v0, v1; v0.x = a[0]; v0.y = a[1]; v1.x = a[2]; v1.y = a[3];
    reinterpret_cast<longlong2*>(p)[0] = v0;
    reinterpret_cast<longlong2*>(p)[1] = v1;
  }
}

// ---- message ops (fp64; kernels.py:281-293) ---------------------------------

template <int OP>
__device__ __forceinline__ double apply_op(double a, double b) {
  if constexpr (OP == OP_ADD) return a + b;
  else if constexpr (OP == OP_SUB) return a - b;
  else if constexpr (OP == OP_MUL || OP == OP_DOT) return a * b;  // dot: one product term
  else if constexpr (OP == OP_DIV) return a / b;  // IEEE division (no fast-math)
  else return a;                                  // OP_COPY
}

template <int OP, typename T>
__device__ __forceinline__ T apply_op_t(T a, T b) {
  if constexpr (OP == OP_ADD) return a + b;
  else if constexpr (OP == OP_SUB) return a - b;
  else if constexpr (OP == OP_MUL) return a * b;
  else if constexpr (OP == OP_DIV) return a / b;
  else return a;
}

// ---- extrema combine: strictly better value wins; ties keep the smaller edge
// id (kernels.py:402-408 masked min-reduce over edge ids).
template <int RHO>
__device__ __forceinline__ void ext_update(double& cur, int32_t& arg, double x, int32_t e) {
  const bool better = (RHO == RHO_MAX) ? (x > cur) : (x < cur);
  if (better) { cur = x; arg = e; }
  else if (x == cur && e < arg) { arg = e; }
}

template <int RHO>
__device__ __forceinline__ double ext_init() {
  return (RHO == RHO_MAX) ? -__longlong_as_double(0x7ff0000000000000ll)
                          : __longlong_as_double(0x7ff0000000000000ll);
}

// edges left in a 32-edge batch
__device__ __forceinline__ int batch_count(int64_t rem) { return rem < 32 ? (int)rem : 32; }

__device__ __forceinline__ double shfl_xor_d(double v, int off) {
  return __shfl_xor_sync(kFull, v, off);
}

}  // namespace gmp
