// TMA request rate for small random copies: W warps per CTA, each with its own
// 2-stage buffer of 32 rows x 256 B, each lane one cp.async.bulk (UBLKCP) per
// row (mode 0) or lanes 0-7 one tile::gather4 of 4 rows (mode 1), waiting on
// the stage's mbarrier before reusing it. Measures whether more issuing warps
// raise the per-SM rate (vs the LDG gather at the same occupancy).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tmaissue.cu -o tmaissue -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void issue(const float4* __restrict__ data, const __grid_constant__ CUtensorMap map,
                      uint32_t rows, int64_t per_warp, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[32][2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* buf = sm + (size_t)w * 2 * 32 * 256;
  if (lane == 0) {
    for (int s = 0; s < 2; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[w][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t ph[2] = {0, 0};
  uint32_t x = (blockIdx.x * 131 + w * 7 + lane) * 2654435761u;
  for (int64_t it = 0; it < per_warp; ++it) {
    const int s = it & 1;
    if (it >= 2) {
      asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
                   ::"r"(su(&bar[w][s])), "r"(ph[s]) : "memory");
      ph[s] ^= 1;
    }
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[w][s])),
                   "r"(32 * 256) : "memory");
    __syncwarp();
    x = x * 1664525u + 1013904223u;
    const uint32_t r = __umulhi(x, rows);
    uint8_t* dst = buf + s * 32 * 256;
    if (MODE == 0) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                   ::"r"(su(dst + lane * 256)), "l"(data + (int64_t)r * 16), "r"(su(&bar[w][s])) : "memory");
    } else if (lane < 8) {
      const uint32_t r1 = __umulhi(x * 3u + 7u, rows), r2 = __umulhi(x * 5u + 11u, rows),
                     r3 = __umulhi(x * 9u + 13u, rows);
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   ::"r"(su(dst + lane * 1024)), "l"(&map), "r"(0), "r"(r), "r"(r1), "r"(r2), "r"(r3),
                   "r"(su(&bar[w][s])) : "memory");
    }
  }
  for (int s = 0; s < 2; ++s)
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
                 ::"r"(su(&bar[w][s])), "r"(ph[s]) : "memory");
  if (lane == 0 && buf[0] == 123) out[0] = 1.f;
}

int main() {
  float4* data; float* out;
  cudaMalloc(&data, 64ull << 20); cudaMalloc(&out, 4);
  cudaMemset(data, 0, 64ull << 20);
  const uint32_t rows = (uint32_t)((60ull << 20) / 256);
  CUtensorMap map;
  cuuint64_t gdim[2] = {64, rows}; cuuint64_t gstride[1] = {256};
  cuuint32_t box[2] = {64, 1}; cuuint32_t es[2] = {1, 1};
  cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, data, gdim, gstride, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode)
    for (int W : {1, 4, 8, 13}) {
      const int smem = W * 2 * 32 * 256;
      auto k = mode ? issue<1> : issue<0>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int64_t per_warp = 2000;
      k<<<148, W * 32, smem>>>(data, map, rows, per_warp, out);
      cudaEventRecord(a);
      k<<<148, W * 32, smem>>>(data, map, rows, per_warp, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double bytes = 148.0 * W * per_warp * 32 * 256;
      printf("%s warps/SM %2d: %.3f ms %.1f GB/s  %.1f cycles per request per SM @1.9GHz %s\n",
             mode ? "gather4" : "bulk256", W, ms, bytes / ms / 1e6,
             ms * 1e-3 * 1.9e9 / (W * per_warp * (mode ? 8 : 32)),
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
