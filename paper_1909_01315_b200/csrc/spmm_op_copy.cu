// spmm_op_copy.cu - instantiates the g-SpMM row kernel for OP_COPY (one op
// family per translation unit so the families compile in parallel).
#include "spmm_rows.cuh"

namespace gmp {
template cudaError_t launch_spmm_rows<OP_COPY>(int, int, int, int, const SpmmArgs&, int64_t,
                                               cudaStream_t);
}  // namespace gmp
