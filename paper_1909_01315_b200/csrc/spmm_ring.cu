// spmm_ring.cu - heavy-row g-SpMM over one packed 256 B column tile, its
// gathers moved by the Tensor Memory Accelerator: cp.async.bulk.tensor
// .tile::gather4 (SASS UTMALDG), four 256 B source rows per request, into a
// per-warp shared-memory ring completed by mbarrier transaction counts.
//
// The packed-tile path (kernels._gspmm_tiled; the Reddit-shaped headline and
// every wide copy_u / u_mul_e aggregation) reduces, per column tile, every
// destination row over 256 B source rows that are L2-resident. In the row
// kernel (spmm_rows.cuh) those gathers sit in registers: 8 float4 in flight
// per lane, 24 warps per SM (80 registers), ~98 KB in flight per SM, and
// between two bursts a warp has nothing in flight - 62 % of the L2 gather
// ceiling. Measured on this B200 (tools/micro/tmaissue.cu,
// profiles/r02_tma_gather.json): one warp-wide TMA instruction is served
// request by request (~56-78 cycles each), but instructions of different
// warps overlap, so 8 warps/SM each keeping 8 gather4 requests in flight
// reach 19.9 TB/s - the ceiling - while a single producer warp feeding the
// whole CTA tops out at ~1-2 TB/s. Hence no dedicated producer here:
//  * one persistent CTA per SM, kG4Warps warps, each warp both issues and
//    consumes: its own kG4Stages-stage ring of 32-row stages (8 KB);
//  * work items = (heavy row, chunk of kG4Chunk CSC positions) claimed by a
//    warp through an atomic counter in schedule order (largest rows first);
//    per 32-edge batch the warp holds the neighbour ids in registers (one per
//    lane, loaded kG4Stages batches ahead), lanes 0-7 each issue one gather4
//    of four rows into the batch's stage, lane 0 arms the stage's mbarrier
//    with the byte count, and the warp consumes the stage issued
//    kG4Stages - 1 batches earlier: 16 lanes x float4 per row, two rows per
//    step, exact messages into compensated fp32 pairs folded to fp64 every 32
//    edges (the row kernel's arithmetic);
//  * an item's partial (64 fp64 columns) is written once; the merge kernel
//    sums a row's item partials in item order and rounds once into Z - fixed
//    order, deterministic, fp64 accumulation of the exact messages.
// The light and medium rows run the row kernel (gmp_api.cu skips the heavy
// prefix of the schedule for them).
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "gmp_common.cuh"
#include "spmm_rows.cuh"
#include "spmm_ring.cuh"

namespace gmp {

constexpr int kG4Warps = 16;            // warps per CTA (one CTA per SM)
constexpr int kG4Stages = 3;            // 32-row stages per warp
constexpr int kG4B = 16;                // rows (edges) per stage
constexpr int kG4StageBytes = kG4B * 256; // one stage: kG4B rows of up to 256 B
constexpr int64_t kG4Chunk = 2048;      // CSC positions per work item

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
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int r0, int r1,
                                            int r2, int r3, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(b))
      : "memory");
}

// Heavy-row items: one warp per item at a time. The tile's rows are
// `rb` = 128 or 256 bytes (box width of the tensor map: a narrow last tile
// fetches one 128 B line per row); a lane group of rb/16 lanes covers a row.
// four columns of one lane as two compensated fp32 pairs (TwoSum /
// TwoProduct on packed FADD2 / FFMA2, as RowAcc in spmm_rows.cuh)
template <int OP>
struct Comp4 {
  float2 s0, s1, c0, c1;
  __device__ __forceinline__ void zero() { s0 = s1 = c0 = c1 = f2(0.f, 0.f); }
  __device__ __forceinline__ void add(const float4 v, float w) {
    if constexpr (OP == OP_COPY) {
      two_sum2(s0, c0, f2(v.x, v.y));
      two_sum2(s1, c1, f2(v.z, v.w));
    } else {  // the row kernel's product accumulate (two_sum_prod2)
      const float2 ww = f2(w, w);
      two_sum_prod2(s0, c0, f2(v.x, v.y), ww);
      two_sum_prod2(s1, c1, f2(v.z, v.w), ww);
    }
  }
  __device__ __forceinline__ void fold(double (&acc)[4]) {
    acc[0] += (double)s0.x; acc[0] += (double)c0.x;
    acc[1] += (double)s0.y; acc[1] += (double)c0.y;
    acc[2] += (double)s1.x; acc[2] += (double)c1.x;
    acc[3] += (double)s1.y; acc[3] += (double)c1.y;
    zero();
  }
};

template <int OP, int RB>
__global__ void __launch_bounds__(kG4Warps * 32, 1)
    spmm_g4_kernel(const __grid_constant__ CUtensorMap map, const RingArgs a) {
  extern __shared__ __align__(1024) uint8_t g4_smem[];
  __shared__ uint64_t full[kG4Warps][kG4Stages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    for (int s = 0; s < kG4Stages; ++s) mbar_init(&full[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint8_t* ring = g4_smem + (size_t)warp * kG4Stages * kG4StageBytes;
  constexpr int rb = RB;
  constexpr int lpr = RB / 16;       // lanes per row (16 or 8)
  constexpr int rps = 32 / lpr;      // rows per warp step (2 or 4)
  constexpr int steps = kG4B / rps;  // warp steps per full stage
  const int sub = lane / lpr, c4 = lane % lpr;
  const int n_items = a.item_start[a.n_heavy];
  uint32_t ph = 0;  // bit s: phase parity of stage s's mbarrier
  int slot = 0;  // stage of the next batch to consume (rotates with the issue slot)

  for (;;) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(a.counter, 1ull);
    it = __shfl_sync(kFull, it, 0);
    if ((int64_t)it >= n_items) break;
    int lo = 0, hi = (int)a.n_heavy - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(a.item_start + mid) <= (int)it) lo = mid; else hi = mid - 1;
    }
    const int64_t row = __ldg(a.order + lo);
    const int64_t re = __ldg(a.indptr + row + 1);
    const int64_t p0 = __ldg(a.indptr + row) + ((int64_t)it - __ldg(a.item_start + lo)) * kG4Chunk;
    const int64_t p1 = min(p0 + kG4Chunk, re);
    const int nb = (int)((p1 - p0 + kG4B - 1) / kG4B);  // kG4B-edge batches of the item

    // neighbour ids: idx[k] holds batch (issued + k)'s id of lane `lane`
    int32_t idx[kG4Stages];
#pragma unroll
    for (int k = 0; k < kG4Stages; ++k) {
      const int64_t p = p0 + (int64_t)k * kG4B + lane;
      idx[k] = (lane < kG4B && p < p1) ? __ldg(a.indices + p) : 0;
    }
    auto issue = [&](int b, int s, int32_t id) {
      const int cnt = (int)min((int64_t)kG4B, p1 - p0 - (int64_t)b * kG4B);
      const int reqs = (cnt + 3) >> 2;
      const int32_t first = __shfl_sync(kFull, id, 0);
      const int32_t own = lane < cnt ? id : first;  // tail rows re-fetch row 0
      int32_t r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = __shfl_sync(kFull, own, (lane * 4 + k) & 31);
      if (lane == 0) mbar_expect_tx(&full[warp][s], (uint32_t)(reqs * 4 * rb));
      __syncwarp();
      if (lane < reqs)
        tma_gather4(ring + (size_t)s * kG4StageBytes + (size_t)lane * 4 * rb, &map, r[0], r[1],
                    r[2], r[3], &full[warp][s]);
    };
    // prologue: the first kG4Stages - 1 batches in flight
    int issued = 0;
#pragma unroll
    for (int k = 0; k < kG4Stages - 1; ++k) {
      if (issued < nb) {
        issue(issued, (slot + k) % kG4Stages, idx[k]);
        ++issued;
      }
    }
    // two independent accumulator sets (alternate rows) halve the dependent
    // FADD2 chains; four shared-memory loads are in flight per group
    Comp4<OP> A, B;
    A.zero();
    B.zero();
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int since_fold = 0;
    for (int b = 0; b < nb; ++b) {
      // rotate the id registers: idx[k] now holds batch b + 1 + k
#pragma unroll
      for (int k = 0; k < kG4Stages - 1; ++k) idx[k] = idx[k + 1];
      {
        const int64_t p = p0 + (int64_t)(b + kG4Stages) * kG4B + lane;
        idx[kG4Stages - 1] = (lane < kG4B && p < p1) ? __ldg(a.indices + p) : 0;
      }
      if (issued < nb) {  // keep kG4Stages - 1 batches ahead
        issue(issued, (slot + kG4Stages - 1) % kG4Stages, idx[kG4Stages - 2]);
        ++issued;
      }
      const int s = slot;
      const int64_t pb = p0 + (int64_t)b * kG4B;
      const int cnt = (int)min((int64_t)kG4B, p1 - pb);
      float wl = 0.f;  // u_mul_e: lane l holds w of the batch's row l (coalesced)
      if constexpr (OP == OP_MUL) wl = lane < cnt ? __ldg(a.W + pb + lane) : 0.f;
      mbar_wait(&full[warp][s], (ph >> s) & 1u);
      ph ^= 1u << s;
      const float4* stv = reinterpret_cast<const float4*>(ring + (size_t)s * kG4StageBytes) +
                          sub * lpr + c4;
      if (cnt == kG4B) {
#pragma unroll
        for (int q = 0; q < steps; q += 4) {
          float4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = stv[(q + u) * rps * lpr];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float w = OP == OP_MUL ? __shfl_sync(kFull, wl, (q + u) * rps + sub) : 0.f;
            if (u & 1) B.add(v[u], w); else A.add(v[u], w);
          }
        }
      } else {
        for (int q = 0; q < steps; ++q) {
          const int j = q * rps + sub;
          const float w = OP == OP_MUL ? __shfl_sync(kFull, wl, j & 31) : 0.f;
          if (j < cnt) A.add(stv[q * rps * lpr], w);
        }
      }
      __syncwarp();  // the stage's reads are done before it is re-armed
      slot = slot + 1 == kG4Stages ? 0 : slot + 1;
      since_fold += steps;
      if (since_fold >= 32 || b + 1 == nb) {
        A.fold(acc);
        B.fold(acc);
        since_fold = 0;
      }
    }
    // lane groups holding the same columns -> one partial per column
    for (int off = lpr; off < 32; off <<= 1) {
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] += __shfl_xor_sync(kFull, acc[k], off);
    }
    if (sub == 0) {
      double* out = a.partial + (int64_t)it * 64 + c4 * 4;
#pragma unroll
      for (int k = 0; k < 4; ++k) out[k] = acc[k];
    }
  }
}

// item_start[r] = sum_{r' < r} ceil(deg(order[r']) / kG4Chunk), one block
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
      c = (int32_t)((indptr[row + 1] - indptr[row] + kG4Chunk - 1) / kG4Chunk);
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
  const int64_t items = m / kG4Chunk + n_heavy + 1;
  return 256 + (size_t)(n_heavy + 1) * 4 + 256 + (size_t)items * 64 * 8;
}

// workspace layout: [counter (256 B)] [item_start (n_heavy + 1 int32), padded] [partials]
static void ring_layout(void* ws, int64_t n_heavy, unsigned long long** counter,
                        int32_t** item_start, double** partial) {
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

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

cudaError_t launch_ring(int op_mul, const RingArgs& a_in, int64_t n_src_rows, void* ws,
                        cudaStream_t s) {
  RingArgs a = a_in;
  ring_layout(ws, a.n_heavy, &a.counter, const_cast<int32_t**>(&a.item_start), &a.partial);
  a.row_bytes = a.width > 32 ? 256 : 128;
  auto encode = tensor_map_encoder();
  if (!encode) return cudaErrorNotSupported;
  CUtensorMap map;
  cuuint64_t gdim[2] = {64, (cuuint64_t)n_src_rows};
  cuuint64_t gstride[1] = {256};
  cuuint32_t box[2] = {(cuuint32_t)(a.row_bytes / 4), 1};
  cuuint32_t estride[2] = {1, 1};
  if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.X), gdim, gstride, box,
             estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int smem = kG4Warps * kG4Stages * kG4StageBytes;
  cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<sms, kG4Warps * 32, smem, s>>>(map, a);
  };
  if (op_mul) {
    if (a.row_bytes == 256) go(spmm_g4_kernel<OP_MUL, 256>); else go(spmm_g4_kernel<OP_MUL, 128>);
  } else {
    if (a.row_bytes == 256) go(spmm_g4_kernel<OP_COPY, 256>); else go(spmm_g4_kernel<OP_COPY, 128>);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ring_merge_kernel<<<(unsigned)((a.n_heavy * 32 + 255) / 256), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace gmp
