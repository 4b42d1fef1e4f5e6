// Random 256 B row gathers from an L2-resident slice (the packed column tile
// of the g-SpMM row kernel), three ways, to decide how the row kernel should
// move its gathers on sm_100a:
//   ldg     : 16 lanes x LDG.128 per row, 8 rows in flight per lane group
//             (the current row kernel's scheme, full occupancy);
//   bulk    : persistent CTA per SM, one producer warp issuing one
//             cp.async.bulk (256 B, UBLKCP) per row into an smem ring guarded
//             by mbarriers (complete_tx), 8 consumer warps summing from smem;
//   gather4 : the same ring fed by cp.async.bulk.tensor.2d.tile::gather4
//             (4 rows x 256 B per instruction, UTMALDG) through a tensor map.
// Indices are read from an HBM array as the row kernel reads its CSC.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tmagather.cu -o tmagather -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void gen_idx(uint32_t* idx, int64_t n, uint32_t rows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    idx[i] = (uint32_t)(x % rows);
  }
}

template <int U>
__global__ void __launch_bounds__(256) ldg_gather(const float4* __restrict__ data,
                                                  const uint32_t* __restrict__ idx, int64_t n,
                                                  float* out) {
  const int lane = threadIdx.x & 15;
  const int64_t groups = (int64_t)gridDim.x * blockDim.x / 16;
  float acc = 0.f;
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 16; g * U < n; g += groups) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = g * U + u;
      const uint32_t r = e < n ? __ldg(idx + e) : 0;
      v[u] = __ldg(data + (int64_t)r * 16 + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int c0, int r0, int r1,
                                        int r2, int r3, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(b))
      : "memory");
}

constexpr int kConsumers = 8;
constexpr int kRows = 64;  // rows per stage (16 KB)

template <int MODE, int S>
__global__ void __launch_bounds__((kConsumers + 1) * 32) ring_gather(
    const float4* __restrict__ data, const __grid_constant__ CUtensorMap map,
    const uint32_t* __restrict__ idx, int64_t n, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float4* ring = reinterpret_cast<float4*>(smem);
  __shared__ uint64_t full[S], empty[S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kConsumers); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t chunks = (n + kRows - 1) / kRows;
  if (warp == kConsumers) {  // producer
    int s = 0;
    uint32_t ph = 0;
    for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
      if (lane == 0) mbar_wait(&empty[s], ph ^ 1);
      __syncwarp();
      const int64_t e0 = c * kRows;
      const int cnt = (int)min((int64_t)kRows, n - e0);
      if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)(kRows * 256));
      __syncwarp();
      float4* st = ring + (int64_t)s * kRows * 16;
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < kRows / 32; ++i) {
          const int j = i * 32 + lane;
          const uint32_t r = __ldg(idx + e0 + (j < cnt ? j : 0));
          bulk_g2s(st + j * 16, data + (int64_t)r * 16, 256, &full[s]);
        }
      } else {
        if (lane < kRows / 4) {
          const int j = lane * 4;
          uint32_t r[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) r[k] = __ldg(idx + e0 + (j + k < cnt ? j + k : 0));
          gather4(st + j * 16, &map, 0, r[0], r[1], r[2], r[3], &full[s]);
        }
      }
      if (++s == S) { s = 0; ph ^= 1; }
    }
    return;
  }
  float acc = 0.f;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    mbar_wait(&full[s], ph);
    const float4* st = ring + (int64_t)s * kRows * 16;
    // 8 rows per consumer warp: 2 rows per warp step, 16 lanes x float4 each
#pragma unroll
    for (int i = 0; i < kRows / kConsumers / 2; ++i) {
      const int j = warp * (kRows / kConsumers) + i * 2 + (lane >> 4);
      const float4 v = st[j * 16 + (lane & 15)];
      acc += v.x + v.y + v.z + v.w;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) { s = 0; ph ^= 1; }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const int64_t n = 64ll << 20;  // gathers
  uint32_t* idx; float4* data; float* out;
  cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
  cudaMalloc(&data, 256ull << 20);
  cudaMemset(data, 0, 256ull << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  constexpr int S = 12;
  const int smem = S * kRows * 256;
  cudaFuncSetAttribute(ring_gather<0, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(ring_gather<1, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mb : {32, 60, 96}) {
    const uint32_t rows = (uint32_t)(((int64_t)mb << 20) / 256);
    CUtensorMap map;
    cuuint64_t gdim[2] = {64, rows};
    cuuint64_t gstride[1] = {256};
    cuuint32_t box[2] = {64, 1};
    cuuint32_t estride[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, data, gdim,
                                         gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                         CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) printf("tensor map encode failed %d\n", (int)cr);
    gen_idx<<<1184, 256>>>(idx, n, rows);
    for (int mode = 0; mode < 3; ++mode) {
      auto run = [&]() {
        if (mode == 0) ldg_gather<8><<<sms * 8, 256>>>(data, idx, n, out);
        else if (mode == 1)
          ring_gather<0, S><<<sms, (kConsumers + 1) * 32, smem>>>(data, map, idx, n, out);
        else ring_gather<1, S><<<sms, (kConsumers + 1) * 32, smem>>>(data, map, idx, n, out);
      };
      run();
      cudaEventRecord(a);
      for (int rep = 0; rep < 5; ++rep) run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaError_t e = cudaGetLastError();
      float ms; cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      const char* nm[3] = {"ldg", "bulk", "gather4"};
      printf("slice %3d MB %-8s: %.3f ms  %.1f GB/s of 256 B rows gathered %s\n", mb, nm[mode], ms,
             n * 256.0 / ms / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
