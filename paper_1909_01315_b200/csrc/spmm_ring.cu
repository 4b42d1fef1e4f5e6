// spmm_ring.cu - heavy-row g-SpMM over one packed 256 B column tile, fed by
// the Blackwell bulk-copy engine (cp.async.bulk -> UBLKCP) through a shared
// memory ring.
//
// The packed-tile path (kernels._gspmm_tiled; the Reddit-shaped headline and
// every wide copy_u / u_mul_e aggregation) reduces, per column tile, every
// destination row over 256 B source rows that are L2-resident. In the row
// kernel (spmm_rows.cuh) those gathers sit in registers: 8 float4 in flight
// per lane, 24 warps per SM (80 registers), ~98 KB in flight per SM, which
// measured 63 % of the L2 gather ceiling. Here the heavy rows (degree >
// heavy threshold; 96 % of Reddit's edges) are instead streamed through
// shared memory:
//  * one persistent CTA per SM: a producer warp and 8 consumer warps;
//  * work items = (heavy row, chunk of kChunk CSC positions), claimed through
//    an atomic counter in schedule order (largest rows first); the producer
//    reads the chunk's neighbour ids (coalesced, one batch of 512 ahead) and
//    issues one 256 B cp.async.bulk per edge into a stage of the ring, the
//    stage's mbarrier counting the bytes (complete_tx) - the ring holds
//    kStages x 64 rows = 192 KB in flight per SM, twice the register path;
//  * consumer warps wait on the stage's mbarrier, each takes 8 of its 64
//    rows (16 lanes x float4 per row, two rows per step), accumulates the
//    exact message into compensated fp32 pairs (as spmm_rows.cuh), folds to
//    fp64 at least every 32 edges, and releases the stage (empty mbarrier);
//  * at an item's last stage the consumers reduce their partials (half-warp
//    shuffle, then the 8 warps in warp order through shared memory) and
//    write one fp64 partial row per item; the merge kernel sums a row's item
//    partials in item order and rounds once into Z. Everything is
//    order-fixed: results are deterministic and equal to fp64 accumulation
//    of the exact messages (the same contract as the row kernel).
// The light and medium rows run the row kernel (gmp_api.cu skips the heavy
// prefix of the schedule for them).
#include <cstdint>
#include <cuda_runtime.h>

#include "gmp_common.cuh"
#include "spmm_rows.cuh"
#include "spmm_ring.cuh"

namespace gmp {

constexpr int kRingRows = 64;         // rows (edges) per stage: 16 KB
constexpr int kRingStages = 12;       // 192 KB of ring per CTA
constexpr int kRingConsumers = 8;     // consumer warps
constexpr int kRingThreads = (kRingConsumers + 1) * 32;
constexpr int64_t kRingChunk = 8192;  // CSC positions per work item
constexpr int kRingBatch = 512;       // neighbour ids the producer loads ahead (16 per lane)


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
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kRingConsumers * 32) : "memory");
}

struct RingMeta {
  int64_t q;     // first CSC position of the stage
  int32_t item;  // work item, -1 = exit
  int32_t cnt;   // rows in the stage
  int32_t last;  // last stage of the item
};

template <int OP>
__global__ void __launch_bounds__(kRingThreads, 1) spmm_ring_kernel(const RingArgs a) {
  extern __shared__ __align__(128) uint8_t ring_smem[];
  float4* ring = reinterpret_cast<float4*>(ring_smem);
  __shared__ uint64_t full[kRingStages], empty[kRingStages];
  __shared__ RingMeta meta[kRingStages];
  __shared__ double red[kRingConsumers][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRingStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kRingConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n_items = a.item_start[a.n_heavy];

  if (warp == kRingConsumers) {
    // ---------------------------------------------------------- producer ---
    // bytes copied per row: the tile's columns rounded up to 16 B (a narrow
    // last tile does not fetch the unused sectors)
    const uint32_t rb16 = (uint32_t)((a.width * 4 + 15) & ~15);
    int s = 0;
    uint32_t ph = 0;
    for (;;) {
      unsigned long long it = 0;
      if (lane == 0) it = atomicAdd(a.counter, 1ull);
      it = __shfl_sync(kFull, it, 0);
      if ((int64_t)it >= n_items) break;
      // heavy row of the item: last r with item_start[r] <= it
      int lo = 0, hi = (int)a.n_heavy - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(a.item_start + mid) <= (int)it) lo = mid; else hi = mid - 1;
      }
      const int64_t row = __ldg(a.order + lo);
      const int64_t rb = __ldg(a.indptr + row), re = __ldg(a.indptr + row + 1);
      const int64_t p0 = rb + ((int64_t)it - __ldg(a.item_start + lo)) * kRingChunk;
      const int64_t p1 = min(p0 + kRingChunk, re);
      int32_t nb[kRingBatch / 32];
      auto load_batch = [&](int64_t b0) {
#pragma unroll
        for (int i = 0; i < kRingBatch / 32; ++i) {
          const int64_t p = b0 + i * 32 + lane;
          nb[i] = p < p1 ? __ldg(a.indices + p) : 0;
        }
      };
      load_batch(p0);
      for (int64_t b0 = p0; b0 < p1; b0 += kRingBatch) {
        int32_t cur[kRingBatch / 32];
#pragma unroll
        for (int i = 0; i < kRingBatch / 32; ++i) cur[i] = nb[i];
        if (b0 + kRingBatch < p1) load_batch(b0 + kRingBatch);
#pragma unroll
        for (int k = 0; k < kRingBatch / kRingRows; ++k) {
          const int64_t q = b0 + k * kRingRows;
          if (q >= p1) continue;
          const int cnt = (int)min((int64_t)kRingRows, p1 - q);
          if (lane == 0) {
            mbar_wait(&empty[s], ph ^ 1);
            meta[s].q = q;
            meta[s].item = (int)it;
            meta[s].cnt = cnt;
            meta[s].last = q + kRingRows >= p1;
            mbar_expect_tx(&full[s], (uint32_t)cnt * rb16);
          }
          __syncwarp();
          float4* st = ring + (int64_t)s * kRingRows * 16;
#pragma unroll
          for (int i = 0; i < kRingRows / 32; ++i) {
            const int j = i * 32 + lane;
            if (j < cnt)
              bulk_row(st + j * 16, a.X + (int64_t)cur[k * (kRingRows / 32) + i] * 64, rb16,
                       &full[s]);
          }
          if (++s == kRingStages) { s = 0; ph ^= 1; }
        }
      }
    }
    if (lane == 0) {
      mbar_wait(&empty[s], ph ^ 1);
      meta[s].item = -1;
      mbar_arrive(&full[s]);
    }
    return;
  }

  // ------------------------------------------------------------ consumers ---
  // lane -> (half h = row parity, column group c4 = 4 columns)
  const int h = lane >> 4, c4 = lane & 15;
  float sc[4] = {0.f, 0.f, 0.f, 0.f}, cc[4] = {0.f, 0.f, 0.f, 0.f};
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int since_fold = 0;
  int s = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&full[s], ph);
    const RingMeta md = meta[s];
    if (md.item < 0) break;
    const float4* st = ring + (int64_t)s * kRingRows * 16;
    constexpr int kPer = kRingRows / kRingConsumers;  // rows per warp per stage
#pragma unroll
    for (int i = 0; i < kPer / 2; ++i) {
      const int j = warp * kPer + 2 * i + h;
      if (j < md.cnt) {
        const float4 v = st[j * 16 + c4];
        float2 S0 = f2(sc[0], sc[1]), C0 = f2(cc[0], cc[1]);
        float2 S1 = f2(sc[2], sc[3]), C1 = f2(cc[2], cc[3]);
        if constexpr (OP == OP_COPY) {
          two_sum2(S0, C0, f2(v.x, v.y));
          two_sum2(S1, C1, f2(v.z, v.w));
        } else {  // OP_MUL: exact product x*w = pr + (fma(x, w, -pr)) (TwoProduct)
          const float w = __ldg(a.W + md.q + j);
          const float2 ww = f2(w, w);
          const float2 x0 = f2(v.x, v.y), x1 = f2(v.z, v.w);
          const float2 pr0 = __fmul2_rn(x0, ww), pr1 = __fmul2_rn(x1, ww);
          two_sum2(S0, C0, pr0);
          two_sum2(S1, C1, pr1);
          C0 = __fadd2_rn(C0, __ffma2_rn(x0, ww, f2(-pr0.x, -pr0.y)));
          C1 = __fadd2_rn(C1, __ffma2_rn(x1, ww, f2(-pr1.x, -pr1.y)));
        }
        sc[0] = S0.x; sc[1] = S0.y; sc[2] = S1.x; sc[3] = S1.y;
        cc[0] = C0.x; cc[1] = C0.y; cc[2] = C1.x; cc[3] = C1.y;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == kRingStages) { s = 0; ph ^= 1; }
    since_fold += kPer / 2;
    if (since_fold >= 32 || md.last) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[k] += (double)sc[k];
        acc[k] += (double)cc[k];
        sc[k] = cc[k] = 0.f;
      }
      since_fold = 0;
    }
    if (md.last) {
      // halves (rows of even / odd slot) -> one partial per column, then warps
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[k] += __shfl_xor_sync(kFull, acc[k], 16);
        if (h == 0) red[warp][c4 * 4 + k] = acc[k];
        acc[k] = 0.0;
      }
      consumers_sync();
      if (warp == 0) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int col = lane * 2 + k;
          double t = red[0][col];
#pragma unroll
          for (int w = 1; w < kRingConsumers; ++w) t += red[w][col];
          a.partial[(int64_t)md.item * 64 + col] = t;
        }
      }
      consumers_sync();
    }
  }
}

// item_start[r] = sum_{r' < r} ceil(deg(order[r']) / kRingChunk), one block
__global__ void ring_items_kernel(const int64_t* indptr, const int32_t* order, int64_t n_heavy,
                                  int32_t* item_start) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = 0; base < n_heavy; base += blockDim.x) {
    const int64_t r = base + threadIdx.x;
    int32_t c = 0;
    if (r < n_heavy) {
      const int64_t row = order[r];
      c = (int32_t)((indptr[row + 1] - indptr[row] + kRingChunk - 1) / kRingChunk);
    }
    int32_t x = c;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int32_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(kFull, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const int32_t before = carry + (warp ? warp_tot[warp - 1] : 0) + x - c;
    if (r < n_heavy) item_start[r] = before;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = before + c;
    __syncthreads();
  }
  if (threadIdx.x == 0) item_start[n_heavy] = carry;
}

// Z[row, :width] = round(sum of the row's item partials in item order)
// (mean: / in-degree); one warp per heavy row, two columns per lane.
__global__ void ring_merge_kernel(const RingArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= a.n_heavy) return;
  const int64_t row = a.order[r];
  const int i0 = a.item_start[r], i1 = a.item_start[r + 1];
  double t0 = 0.0, t1 = 0.0;
  for (int i = i0; i < i1; ++i) {
    const double2 p = reinterpret_cast<const double2*>(a.partial + (int64_t)i * 64)[lane];
    t0 += p.x;
    t1 += p.y;
  }
  if (a.mean) {
    const double deg = (double)(a.indptr[row + 1] - a.indptr[row]);
    t0 /= deg;
    t1 /= deg;
  }
  float* z = a.Z + row * a.ldz;
  const int c = lane * 2;
  if (c < a.width) z[c] = (float)t0;
  if (c + 1 < a.width) z[c + 1] = (float)t1;
}

size_t ring_workspace_bytes(int64_t n_heavy, int64_t m) {
  const int64_t items = m / kRingChunk + n_heavy + 1;
  return 256 + (size_t)(n_heavy + 1) * 4 + 256 + (size_t)items * 64 * 8;
}

// workspace layout: [counter (256 B)] [item_start (n_heavy + 1 int32), padded] [partials]
void ring_layout(void* ws, int64_t n_heavy, unsigned long long** counter, int32_t** item_start,
                 double** partial) {
  uint8_t* p = static_cast<uint8_t*>(ws);
  *counter = reinterpret_cast<unsigned long long*>(p);
  *item_start = reinterpret_cast<int32_t*>(p + 256);
  const size_t off = 256 + (((size_t)(n_heavy + 1) * 4 + 255) / 256) * 256;
  *partial = reinterpret_cast<double*>(p + off);
}

cudaError_t launch_ring_prepare(const int64_t* indptr, const int32_t* order, int64_t n_heavy,
                                void* ws, cudaStream_t s) {
  unsigned long long* counter;
  int32_t* item_start;
  double* partial;
  ring_layout(ws, n_heavy, &counter, &item_start, &partial);
  ring_items_kernel<<<1, 1024, 0, s>>>(indptr, order, n_heavy, item_start);
  return cudaGetLastError();
}

cudaError_t launch_ring(int op_mul, const RingArgs& a_in, void* ws, cudaStream_t s) {
  RingArgs a = a_in;
  ring_layout(ws, a.n_heavy, &a.counter, const_cast<int32_t**>(&a.item_start), &a.partial);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int smem = kRingStages * kRingRows * 256;
  cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (op_mul) {
    cudaFuncSetAttribute(spmm_ring_kernel<OP_MUL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    spmm_ring_kernel<OP_MUL><<<sms, kRingThreads, smem, s>>>(a);
  } else {
    cudaFuncSetAttribute(spmm_ring_kernel<OP_COPY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    spmm_ring_kernel<OP_COPY><<<sms, kRingThreads, smem, s>>>(a);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t warps = a.n_heavy;
  ring_merge_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace gmp
