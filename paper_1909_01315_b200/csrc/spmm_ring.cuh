// spmm_ring.cuh - arguments of the heavy-row TMA gather4 ring (spmm_ring.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace gmp {

struct RingArgs {
  const int64_t* indptr;
  const int32_t* indices;
  const int32_t* order;      // heavy rows = order[0 .. n_heavy)
  int64_t n_heavy;
  const int32_t* item_start; // (n_heavy + 1): first item of each heavy row
  unsigned long long* counter;
  double* partial;           // (items, 64)
  const float* X;            // packed tile: rows of 64 floats (256 B), 16 B aligned
  const float* W;            // per-CSC-position scalar (u_mul_e) or null (copy_u)
  float* Z;
  int64_t ldz;
  int32_t width;             // columns of this tile stored into Z (<= 64); the bulk
                             // copies fetch width * 4 B rounded up to 16 B per row
  int32_t mean;
  int32_t row_bytes;          // gathered bytes per row (set by launch_ring: 128 or 256)
};

size_t ring_workspace_bytes(int64_t n_heavy, int64_t m);
cudaError_t launch_ring_prepare(const int64_t* indptr, const int32_t* order, int64_t n_heavy,
                                void* ws, cudaStream_t s);
cudaError_t launch_ring(int op_mul, const RingArgs& a, int64_t n_src_rows, void* ws,
                        cudaStream_t s);

}  // namespace gmp
