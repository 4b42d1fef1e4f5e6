// spmm_op_attn.cu - the fused GAT attention aggregation through the g-SpMM
// row kernel: u_mul_e + sum whose per-edge weight is the edge_softmax of the
// u_add_v scores, recomputed from node-keyed data (el, er and the per-
// destination max / 1/sum) instead of being read from an (m, H) array.
// Forward (MP_AF) over destination rows; backward (MP_AB) over the reverse
// graph's rows (= sources), see gmp_gat_aggregate in include/gmp.h.
#include "spmm_rows.cuh"

namespace gmp {

template <typename T, int MP>
static cudaError_t attn_v(int V, const SpmmArgs& a, int64_t grid, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if (V == 4) return launch_spmm_rows_t<T, OP_MUL, RHO_SUM, 4, MP>(a, grid, s);
  }
  if (V == 2) return launch_spmm_rows_t<T, OP_MUL, RHO_SUM, 2, MP>(a, grid, s);
  return launch_spmm_rows_t<T, OP_MUL, RHO_SUM, 1, MP>(a, grid, s);
}

cudaError_t launch_spmm_rows_attn(int dtype_is_f64, int V, bool backward, const SpmmArgs& a,
                                  int64_t grid, cudaStream_t s) {
  if (dtype_is_f64)
    return backward ? attn_v<double, MP_AB>(V, a, grid, s) : attn_v<double, MP_AF>(V, a, grid, s);
  return backward ? attn_v<float, MP_AB>(V, a, grid, s) : attn_v<float, MP_AF>(V, a, grid, s);
}

}  // namespace gmp
