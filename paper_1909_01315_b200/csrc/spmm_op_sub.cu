// spmm_op_sub.cu - instantiates the g-SpMM row kernel for OP_SUB (one op
// family per translation unit so the families compile in parallel).
#include "spmm_rows.cuh"

namespace gmp {
template cudaError_t launch_spmm_rows<OP_SUB>(int, int, int, int, const SpmmArgs&, int64_t,
                                               cudaStream_t);
}  // namespace gmp
