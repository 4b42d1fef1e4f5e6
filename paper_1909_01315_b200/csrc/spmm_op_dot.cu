// spmm_op_dot.cu - g-SpMM with dot messages under sum / mean through the row
// kernel (products accumulated per column, columns reduced at the end); the
// max / min of dot messages stay on spmm_dot.cuh (they need each edge's dot).
#include "spmm_rows.cuh"

namespace gmp {

cudaError_t launch_spmm_rows_dot_sum(int dtype_is_f64, int V, int mp, const SpmmArgs& a,
                                     int64_t grid, cudaStream_t s) {
  if (dtype_is_f64) return launch_spmm_rows_v<double, OP_DOT, RHO_SUM>(V, mp, a, grid, s);
  return launch_spmm_rows_v<float, OP_DOT, RHO_SUM>(V, mp, a, grid, s);
}

}  // namespace gmp
