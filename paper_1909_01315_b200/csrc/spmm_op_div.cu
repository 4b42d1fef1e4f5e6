// spmm_op_div.cu - instantiates the g-SpMM row kernel for OP_DIV (one op
// family per translation unit so the families compile in parallel).
#include "spmm_rows.cuh"

namespace gmp {
template cudaError_t launch_spmm_rows<OP_DIV>(int, int, int, int, const SpmmArgs&, int64_t,
                                               cudaStream_t);
}  // namespace gmp
