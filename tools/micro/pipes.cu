// Issue throughput of the instructions the row kernel's accumulation uses:
// packed FADD2 (sub.rn.f32x2 / add.rn.f32x2), scalar FADD, IADD3/LOP3/SHF
// (integer ALU), DADD, F2F.F64.F32. Each thread runs 8 independent chains
// (latency hidden), 64 warps/SM; result = warp-instructions per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__global__ void k_fadd2(unsigned long long* out, unsigned long long s) {
  unsigned long long a[8];
  for (int i = 0; i < 8; ++i) a[i] = s + threadIdx.x + i;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = add2(a[i], s);
  unsigned long long r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_fadd(float* out, float s) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = s + threadIdx.x + i;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(s));
  float r = 0;
  for (int i = 0; i < 8; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_iadd(unsigned* out, unsigned s) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) a[i] = s + threadIdx.x + i;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("xor.b32 %0, %0, %1;" : "+r"(a[i]) : "r"(s + i));
  unsigned r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_shf(unsigned* out, unsigned s) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) a[i] = s + threadIdx.x + i;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(a[i]) : "r"(s));
  unsigned r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_dadd(double* out, double s) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = s + threadIdx.x + i;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a[i]) : "d"(s));
  double r = 0;
  for (int i = 0; i < 8; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k_f2f(double* out, float s) {
  double a[8];
  float f[8];
  for (int i = 0; i < 8; ++i) { a[i] = 0; f[i] = s + threadIdx.x + i; }
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double t;
      asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[i]));
      a[i] = t;  // dependency-free conversions
      f[i] = __int_as_float(__float_as_int(f[i]) ^ 1);
    }
  double r = 0;
  for (int i = 0; i < 8; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <typename K, typename P, typename S>
void run(const char* name, K k, P* buf, S s, int sms, int insts_per_iter) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  int blocks = sms * 8, threads = 256;  // 64 warps / SM
  k<<<blocks, threads>>>(buf, s);
  cudaEventRecord(a);
  k<<<blocks, threads>>>(buf, s);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double warp_insts = (double)blocks * threads / 32 * N * insts_per_iter;
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-6s %8.3f ms  %.2f warp-inst/clk/SM (clock %d MHz)\n", name, ms, warp_insts / cycles / sms, clk / 1000);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* buf; cudaMalloc(&buf, (size_t)sms * 8 * 256 * 8);
  run("FADD2", k_fadd2, (unsigned long long*)buf, 1ull, sms, 8);
  run("FADD", k_fadd, (float*)buf, 1.0f, sms, 8);
  run("LOP3", k_iadd, (unsigned*)buf, 1u, sms, 8);
  run("SHF", k_shf, (unsigned*)buf, 3u, sms, 8);
  run("DADD", k_dadd, (double*)buf, 1.0, sms, 8);
  run("F2F64", k_f2f, (double*)buf, 1.0f, sms, 8);
  return 0;
}
