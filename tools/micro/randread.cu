// Random-chunk read microbenchmark: how many DRAM bytes does a random
// 32 / 64 / 128 B read cost on this part? (sizing the edge_softmax stats pass)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a randread.cu -o randread
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void gen_idx(uint32_t* idx, int64_t n, uint32_t nchunks) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    idx[i] = (uint32_t)(x % nchunks);
  }
}

// each group of L lanes reads one chunk of L*16 bytes
template <int L>
__global__ void rd(const float4* __restrict__ data, const uint32_t* __restrict__ idx, int64_t n,
                   float* out) {
  const int lane = threadIdx.x % L;
  float acc = 0.f;
  const int64_t groups = (int64_t)gridDim.x * blockDim.x / L;
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / L; g < n; g += groups) {
    const uint32_t c = __ldg(idx + g);
    const float4 v = __ldg(data + (int64_t)c * L + lane);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const size_t bytes = 4ull << 30;
  float4* data; uint32_t* idx; float* out;
  cudaMalloc(&data, bytes); cudaMemset(data, 0, bytes);
  const int64_t n = 64 << 20;
  cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int L) {
    const uint32_t nchunks = (uint32_t)(bytes / (16 * L));
    gen_idx<<<1184, 256>>>(idx, n, nchunks);
    kern<<<148 * 8, 256>>>(data, idx, n, out);
    cudaEventRecord(a);
    kern<<<148 * 8, 256>>>(data, idx, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("chunk %4d B: %.3f ms, useful %.1f GB/s, %.2f Gchunks/s\n", 16 * L, ms,
           n * 16.0 * L / ms / 1e6, n / ms / 1e6);
  };
  run(rd<2>, 2); run(rd<4>, 4); run(rd<8>, 8); run(rd<16>, 16);
  return 0;
}
