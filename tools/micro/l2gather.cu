// L2-resident random gather bandwidth: the ceiling of the g-SpMM row kernel
// once its column tile of X is L2-resident (each edge gathers one 256 B tile
// row at a random source). 16 lanes x float4 per 256 B row, 8 rows in flight
// per lane group, slice sizes around the row kernel's 60 MB tile.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a l2gather.cu -o l2gather
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void gen_idx(uint32_t* idx, int64_t n, uint32_t rows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    idx[i] = (uint32_t)(x % rows);
  }
}

template <int U, int L = 16>
__global__ void __launch_bounds__(256) gather(const float4* __restrict__ data,
                                              const uint32_t* __restrict__ idx, int64_t n,
                                              float* out) {
  const int lane = threadIdx.x & (L - 1);  // L lanes x 16 B per row
  const int64_t groups = (int64_t)gridDim.x * blockDim.x / L;
  float acc = 0.f;
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / L; g * U < n; g += groups) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = g * U + u;
      const uint32_t r = e < n ? __ldg(idx + e) : 0;
      v[u] = __ldg(data + (int64_t)r * L + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
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
  for (int mb : {16, 32, 48, 60, 96, 192}) {
    const uint32_t rows = (uint32_t)(((int64_t)mb << 20) / 256);
    gen_idx<<<1184, 256>>>(idx, n, rows);
    gather<8><<<sms * 8, 256>>>(data, idx, n, out);
    cudaEventRecord(a);
    for (int rep = 0; rep < 5; ++rep) gather<8><<<sms * 8, 256>>>(data, idx, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("slice %4d MB: %.3f ms  %.1f GB/s of 256 B rows gathered\n", mb, ms, n * 256.0 / ms / 1e6);
  }
  // 64 B rows (d = 16 fp32: the GCN hidden layer), X of the Reddit shape (15 MB)
  for (int mb : {15, 60}) {
    const uint32_t rows = (uint32_t)(((int64_t)mb << 20) / 64);
    gen_idx<<<1184, 256>>>(idx, n, rows);
    gather<8, 4><<<sms * 8, 256>>>(data, idx, n, out);
    cudaEventRecord(a);
    for (int rep = 0; rep < 5; ++rep) gather<8, 4><<<sms * 8, 256>>>(data, idx, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("slice %4d MB: %.3f ms  %.1f GB/s of 64 B rows gathered\n", mb, ms, n * 64.0 / ms / 1e6);
  }
  return 0;
}
