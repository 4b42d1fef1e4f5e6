// L2 gather bandwidth of 256 B rows for a given index sequence (a binary
// file of uint32 row ids): the row kernel's exact access stream (CSC-ordered
// sources of the Reddit-shaped graph) against the same multiset shuffled.
// 16 lanes x float4 per row, U rows in flight per lane group, full occupancy.
//   l2gather_file idx.bin rows
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) gather(const float4* __restrict__ data,
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

// contiguous chunks: group g reads idx[g*chunk .. (g+1)*chunk) (like a warp
// walking its own part of a row)
template <int U>
__global__ void __launch_bounds__(256) gather_chunk(const float4* __restrict__ data,
                                                    const uint32_t* __restrict__ idx, int64_t n,
                                                    float* out) {
  const int lane = threadIdx.x & 15;
  const int64_t groups = (int64_t)gridDim.x * blockDim.x / 16;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 16;
  const int64_t chunk = (n + groups - 1) / groups;
  const int64_t b = g * chunk, e = b + chunk < n ? b + chunk : n;
  float acc = 0.f;
  for (int64_t p = b; p < e; p += U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t r = p + u < e ? __ldg(idx + p + u) : 0;
      v[u] = __ldg(data + (int64_t)r * 16 + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  const int64_t rows = atoll(argv[2]);
  fseek(f, 0, SEEK_END);
  const int64_t n = ftell(f) / 4;
  fseek(f, 0, SEEK_SET);
  std::vector<uint32_t> h(n);
  if (fread(h.data(), 4, n, f) != (size_t)n) return 1;
  fclose(f);
  uint32_t* idx; float4* data; float* out;
  cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
  cudaMalloc(&data, rows * 256);
  cudaMemset(data, 0, rows * 256);
  cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    for (int bps : {3, 8}) {
      auto launch = [&]() {
        if (mode == 0) gather<8><<<sms * bps, 256>>>(data, idx, n, out);
        else gather_chunk<8><<<sms * bps, 256>>>(data, idx, n, out);
      };
      launch();
      cudaEventRecord(a);
      for (int rep = 0; rep < 5; ++rep) launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      printf("%s %s, %d CTAs/SM: %.3f ms  %.1f GB/s of 256 B rows\n", argv[1],
             mode ? "chunked" : "interleaved", bps, ms, n * 256.0 / ms / 1e6);
    }
  }
  return 0;
}
