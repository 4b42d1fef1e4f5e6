// kernels_misc.cu - launchers for the dot / SDDMM / softmax kernels, the
// extrema gradient kernels and the degree-binned schedule builder.
#include <cub/device/device_radix_sort.cuh>
#include <cstdlib>

#include "sddmm.cuh"
#include "softmax.cuh"
#include "spmm_dot.cuh"

namespace gmp {

// a.cluster > 1: thread-block clusters of a.cluster CTAs (heavy-row merge via DSMEM)
template <typename Kern>
static void launch_dot_cfg(Kern kern, const SpmmDotArgs& a, int64_t grid, cudaStream_t s) {
  if (a.cluster <= 1) {
    kern<<<(unsigned)grid, kWarpsPerCta * 32, 0, s>>>(a);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid, 1, 1);
  cfg.blockDim = dim3(kWarpsPerCta * 32, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a);
}

cudaError_t launch_spmm_dot(int f64, int rho, int V, const SpmmDotArgs& a, int64_t grid,
                            cudaStream_t s) {
#define GMP_DOT(T, R, VV) launch_dot_cfg(spmm_dot_kernel<T, R, VV>, a, grid, s)
#define GMP_DOT_V(T, R)            \
  do {                             \
    if (V == 4 && sizeof(T) == 4)  \
      GMP_DOT(float, R, 4);        \
    else if (V == 2)               \
      GMP_DOT(T, R, 2);            \
    else                           \
      GMP_DOT(T, R, 1);            \
  } while (0)
  if (f64) {
    if (rho == RHO_SUM) GMP_DOT_V(double, RHO_SUM);
    else if (rho == RHO_MAX) GMP_DOT_V(double, RHO_MAX);
    else GMP_DOT_V(double, RHO_MIN);
  } else {
    if (rho == RHO_SUM) GMP_DOT_V(float, RHO_SUM);
    else if (rho == RHO_MAX) GMP_DOT_V(float, RHO_MAX);
    else GMP_DOT_V(float, RHO_MIN);
  }
#undef GMP_DOT_V
#undef GMP_DOT
  return cudaGetLastError();
}

template <typename T, int OP>
static void sddmm_v(int V, const SddmmArgs& a, int64_t grid, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if (V == 4) { sddmm_kernel<T, OP, 4><<<(unsigned)grid, 256, 0, s>>>(a); return; }
  }
  if (V == 2) { sddmm_kernel<T, OP, 2><<<(unsigned)grid, 256, 0, s>>>(a); return; }
  sddmm_kernel<T, OP, 1><<<(unsigned)grid, 256, 0, s>>>(a);
}

template <typename T>
static void sddmm_op(int op, int V, const SddmmArgs& a, int64_t grid, cudaStream_t s) {
  switch (op) {
    case OP_COPY: sddmm_v<T, OP_COPY>(V, a, grid, s); break;
    case OP_ADD: sddmm_v<T, OP_ADD>(V, a, grid, s); break;
    case OP_SUB: sddmm_v<T, OP_SUB>(V, a, grid, s); break;
    case OP_MUL: sddmm_v<T, OP_MUL>(V, a, grid, s); break;
    case OP_DIV: sddmm_v<T, OP_DIV>(V, a, grid, s); break;
    default: sddmm_v<T, OP_DOT>(V, a, grid, s); break;
  }
}

template <typename T>
static void sddmm_dot_lane(int V, const SddmmArgs& a, cudaStream_t s) {
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((a.m + 255) / 256, 148 * 8));
  if constexpr (sizeof(T) == 4) {
    if (V == 4) { sddmm_dot_lane_kernel<T, 4><<<(unsigned)grid, 256, 0, s>>>(a); return; }
  }
  if (V == 2) { sddmm_dot_lane_kernel<T, 2><<<(unsigned)grid, 256, 0, s>>>(a); return; }
  sddmm_dot_lane_kernel<T, 1><<<(unsigned)grid, 256, 0, s>>>(a);
}

cudaError_t launch_sddmm(int f64, int op, int V, const SddmmArgs& a, int64_t grid, cudaStream_t s) {
  if (op == OP_DOT && a.dim * (f64 ? 8 : 4) <= 128) {  // one operand row per 128 B line
    if (f64) sddmm_dot_lane<double>(V, a, s);
    else sddmm_dot_lane<float>(V, a, s);
    return cudaGetLastError();
  }
  if (f64) sddmm_op<double>(op, V, a, grid, s);
  else sddmm_op<float>(op, V, a, grid, s);
  return cudaGetLastError();
}

template <typename T, bool BWD, bool UV>
static void softmax_v(int V, const SoftmaxArgs& a, int64_t grid, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if (V == 4) { edge_softmax_kernel<T, 4, BWD, UV><<<(unsigned)grid, kWarpsPerCta * 32, 0, s>>>(a); return; }
  }
  if (V == 2) { edge_softmax_kernel<T, 2, BWD, UV><<<(unsigned)grid, kWarpsPerCta * 32, 0, s>>>(a); return; }
  edge_softmax_kernel<T, 1, BWD, UV><<<(unsigned)grid, kWarpsPerCta * 32, 0, s>>>(a);
}

cudaError_t launch_edge_softmax(int f64, int V, bool bwd, bool uv, const SoftmaxArgs& a,
                                int64_t grid, cudaStream_t s) {
  if (f64) {
    if (bwd) softmax_v<double, true, false>(V, a, grid, s);
    else if (uv) softmax_v<double, false, true>(V, a, grid, s);
    else softmax_v<double, false, false>(V, a, grid, s);
  } else {
    if (bwd) softmax_v<float, true, false>(V, a, grid, s);
    else if (uv) softmax_v<float, false, true>(V, a, grid, s);
    else softmax_v<float, false, false>(V, a, grid, s);
  }
  return cudaGetLastError();
}

template <typename T, bool BWD, bool UV>
static void softmax_slot_v(int V, const SoftmaxArgs& a, int64_t grid, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if (V == 4) { edge_softmax_slot_kernel<T, 4, BWD, UV><<<(unsigned)grid, kWarpsPerCta * 32, 0, s>>>(a); return; }
  }
  if (V == 2) { edge_softmax_slot_kernel<T, 2, BWD, UV><<<(unsigned)grid, kWarpsPerCta * 32, 0, s>>>(a); return; }
  edge_softmax_slot_kernel<T, 1, BWD, UV><<<(unsigned)grid, kWarpsPerCta * 32, 0, s>>>(a);
}

// short rows, one per lane group: a.n_rows rows of a.order, one column tile
cudaError_t launch_edge_softmax_slots(int f64, int V, bool bwd, bool uv, const SoftmaxArgs& a,
                                      cudaStream_t s) {
  const int64_t per_cta = (int64_t)kWarpsPerCta * (32 >> a.g_log2);
  const int64_t grid = (a.n_rows + per_cta - 1) / per_cta;
  if (grid == 0) return cudaSuccess;
  if (f64) {
    if (bwd) softmax_slot_v<double, true, false>(V, a, grid, s);
    else if (uv) softmax_slot_v<double, false, true>(V, a, grid, s);
    else softmax_slot_v<double, false, false>(V, a, grid, s);
  } else {
    if (bwd) softmax_slot_v<float, true, false>(V, a, grid, s);
    else if (uv) softmax_slot_v<float, false, true>(V, a, grid, s);
    else softmax_slot_v<float, false, false>(V, a, grid, s);
  }
  return cudaGetLastError();
}

template <typename T, bool BWD>
static void softmax_window_v(int V, const SoftmaxArgs& a, const WindowArgs& w, unsigned grid,
                             cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if (V == 4) { edge_softmax_window_kernel<T, 4, BWD><<<grid, kWarpsPerCta * 32, 0, s>>>(a, w); return; }
  }
  if (V == 2) { edge_softmax_window_kernel<T, 2, BWD><<<grid, kWarpsPerCta * 32, 0, s>>>(a, w); return; }
  edge_softmax_window_kernel<T, 1, BWD><<<grid, kWarpsPerCta * 32, 0, s>>>(a, w);
}

// resident warps of the window kernel on this device (for window sizing)
int softmax_window_resident_ctas(int f64, int V, bool bwd) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const void* fn;
  if (f64) {
    fn = bwd ? (V == 2 ? (const void*)edge_softmax_window_kernel<double, 2, true>
                       : (const void*)edge_softmax_window_kernel<double, 1, true>)
             : (V == 2 ? (const void*)edge_softmax_window_kernel<double, 2, false>
                       : (const void*)edge_softmax_window_kernel<double, 1, false>);
  } else {
    fn = bwd ? (V == 4 ? (const void*)edge_softmax_window_kernel<float, 4, true>
                       : V == 2 ? (const void*)edge_softmax_window_kernel<float, 2, true>
                                : (const void*)edge_softmax_window_kernel<float, 1, true>)
             : (V == 4 ? (const void*)edge_softmax_window_kernel<float, 4, false>
                       : V == 2 ? (const void*)edge_softmax_window_kernel<float, 2, false>
                                : (const void*)edge_softmax_window_kernel<float, 1, false>);
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kWarpsPerCta * 32, 0);
  return std::max(1, per) * sms;
}

cudaError_t launch_edge_softmax_window(int f64, int V, bool bwd, const SoftmaxArgs& a,
                                       const WindowArgs& w, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(w.counter, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  {
    const int64_t nb = a.n_heavy * (w.n_windows + 1);
    edge_softmax_window_bounds<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((nb + 255) / 256, 148 * 16)),
                                 256, 0, s>>>(a, w);
  }
  const unsigned grid = (unsigned)softmax_window_resident_ctas(f64, V, bwd);
  if (f64) {
    if (bwd) softmax_window_v<double, true>(V, a, w, grid, s);
    else softmax_window_v<double, false>(V, a, w, grid, s);
  } else {
    if (bwd) softmax_window_v<float, true>(V, a, w, grid, s);
    else softmax_window_v<float, false>(V, a, w, grid, s);
  }
  const int64_t total = a.n_heavy * (int64_t)a.H;  // one warp each
  const unsigned mg = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 7) / 8, 148 * 16));
  if (f64) {
    if (bwd) edge_softmax_window_merge<double, true><<<mg, 256, 0, s>>>(a, w);
    else edge_softmax_window_merge<double, false><<<mg, 256, 0, s>>>(a, w);
  } else {
    if (bwd) edge_softmax_window_merge<float, true><<<mg, 256, 0, s>>>(a, w);
    else edge_softmax_window_merge<float, false><<<mg, 256, 0, s>>>(a, w);
  }
  return cudaGetLastError();
}

template <typename T, bool BWD>
static const void* seg_kernel_fn(int V) {
  if constexpr (sizeof(T) == 4) {
    if (V == 4) return (const void*)edge_softmax_seg_kernel<T, 4, BWD>;
  }
  if (V == 2) return (const void*)edge_softmax_seg_kernel<T, 2, BWD>;
  return (const void*)edge_softmax_seg_kernel<T, 1, BWD>;
}

template <typename T, bool BWD>
static void softmax_seg_v(int V, const SoftmaxArgs& a, const SegArgs& sg, unsigned grid,
                          cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if (V == 4) { edge_softmax_seg_kernel<T, 4, BWD><<<grid, kWarpsPerCta * 32, 0, s>>>(a, sg); return; }
  }
  if (V == 2) { edge_softmax_seg_kernel<T, 2, BWD><<<grid, kWarpsPerCta * 32, 0, s>>>(a, sg); return; }
  edge_softmax_seg_kernel<T, 1, BWD><<<grid, kWarpsPerCta * 32, 0, s>>>(a, sg);
}

// segmented heavy-row statistics (softmax.cuh): persistent warps claiming
// chunks in order, then the per-row piece merge
cudaError_t launch_edge_softmax_seg(int f64, int V, bool bwd, const SoftmaxArgs& a,
                                    const SegArgs& sg, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(sg.counter, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const void* fn = f64 ? (bwd ? seg_kernel_fn<double, true>(V) : seg_kernel_fn<double, false>(V))
                       : (bwd ? seg_kernel_fn<float, true>(V) : seg_kernel_fn<float, false>(V));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kWarpsPerCta * 32, 0);
  static const int cap = [] {
    const char* v = getenv("GMP_SOFTMAX_SEG_CTAS");  // resident CTAs per SM (tuning)
    return v ? std::max(0, atoi(v)) : 0;  // 0 / unset: occupancy limit only
  }();
  if (cap) per = std::min(per, cap);
  const unsigned grid = (unsigned)(std::max(1, per) * sms);
  if (f64) {
    if (bwd) softmax_seg_v<double, true>(V, a, sg, grid, s);
    else softmax_seg_v<double, false>(V, a, sg, grid, s);
  } else {
    if (bwd) softmax_seg_v<float, true>(V, a, sg, grid, s);
    else softmax_seg_v<float, false>(V, a, sg, grid, s);
  }
  const int64_t total = a.n_heavy * (int64_t)a.H;  // one warp each
  const unsigned mg = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 7) / 8, 148 * 16));
  if (f64) {
    if (bwd) edge_softmax_seg_merge<double, true><<<mg, 256, 0, s>>>(a, sg);
    else edge_softmax_seg_merge<double, false><<<mg, 256, 0, s>>>(a, sg);
  } else {
    if (bwd) edge_softmax_seg_merge<float, true><<<mg, 256, 0, s>>>(a, sg);
    else edge_softmax_seg_merge<float, false><<<mg, 256, 0, s>>>(a, sg);
  }
  return cudaGetLastError();
}

template <typename T, bool BWD, bool UV>
static void softmax_apply_v(int V, const SoftmaxArgs& a, cudaStream_t s) {
  const int64_t total = a.m * (int64_t)(a.H / V);
  const unsigned grid = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((total + 256 * kApplyU - 1) / (256 * kApplyU), 148 * 64));
  if constexpr (sizeof(T) == 4) {
    if (V == 4) { edge_softmax_apply_kernel<T, 4, BWD, UV><<<grid, 256, 0, s>>>(a); return; }
  }
  if (V == 2) { edge_softmax_apply_kernel<T, 2, BWD, UV><<<grid, 256, 0, s>>>(a); return; }
  edge_softmax_apply_kernel<T, 1, BWD, UV><<<grid, 256, 0, s>>>(a);
}

cudaError_t launch_edge_softmax_apply(int f64, int V, bool bwd, bool uv, const SoftmaxArgs& a,
                                      cudaStream_t s) {
  if (f64) {
    if (bwd) softmax_apply_v<double, true, false>(V, a, s);
    else if (uv) softmax_apply_v<double, false, true>(V, a, s);
    else softmax_apply_v<double, false, false>(V, a, s);
  } else {
    if (bwd) softmax_apply_v<float, true, false>(V, a, s);
    else if (uv) softmax_apply_v<float, false, true>(V, a, s);
    else softmax_apply_v<float, false, false>(V, a, s);
  }
  return cudaGetLastError();
}

// ---- extrema gradient routing (kernels.py:843-857) --------------------------

template <typename T>
__global__ void route_extrema_kernel(int64_t n, int32_t d, const int64_t* __restrict__ arg,
                                     const T* __restrict__ dZ, int64_t lddz, T* dM, int64_t ldm) {
  const int64_t total = n * (int64_t)d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / d;
    const int k = (int)(i - v * d);
    const int64_t e = arg[i];
    if (e >= 0) dM[e * ldm + k] = dZ[v * lddz + k];
  }
}

// ---- deterministic many-writer accumulation ----------------------------------
// Cells whose gradient row has several writers (a source row that wins
// several (row, column) cells, a broadcast operand) emit (key = out row *
// cols + out column, fp64 value) pairs; a stable radix sort groups them by
// key in cell order and one thread per key sums its run in fp64 and stores
// the rounded result once. Same terms, same order every run - no float
// atomics, one rounding (the reference routes then reduces in float64,
// kernels.py:843-857 + autodiff.py:398-412).
struct CellSink {
  uint64_t* keys;  // null: single-writer targets store directly
  double* vals;
};

int key_bits(uint64_t max_key) {
  int b = 1;
  while (b < 64 && (max_key >> b)) ++b;
  return b;
}

template <typename T>
__global__ void segment_sum_kernel(int64_t total, const uint64_t* __restrict__ ks,
                                   const double* __restrict__ vs, uint64_t inv, int64_t cols,
                                   T* out, int64_t ldo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = ks[i];
    if (key == inv || (i > 0 && ks[i - 1] == key)) continue;  // invalid, or not a run head
    double acc = 0.0;
    for (int64_t j = i; j < total && ks[j] == key; ++j) acc += vs[j];
    const int64_t row = (int64_t)(key / (uint64_t)cols), col = (int64_t)(key % (uint64_t)cols);
    out[row * ldo + col] = (T)acc;
  }
}

size_t extrema_cub_bytes(int64_t cells) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs((void*)nullptr, bytes, (const uint64_t*)nullptr,
                                  (uint64_t*)nullptr, (const double*)nullptr, (double*)nullptr,
                                  (int)std::max<int64_t>(cells, 1));
  return bytes;
}

static size_t al256(size_t x) { return (x + 255) / 256 * 256; }

size_t extrema_workspace_bytes(int64_t cells) {
  if (cells <= 0) return 0;
  return 4 * al256((size_t)cells * 8) + al256(extrema_cub_bytes(cells));
}

// sort the emitted pairs and store one fp64 sum per key
template <typename T>
cudaError_t sort_and_sum(int64_t cells, void* ws, size_t ws_bytes, uint64_t inv, int64_t cols,
                         T* out, int64_t ldo, cudaStream_t s) {
  char* p = static_cast<char*>(ws);
  uint64_t* k0 = reinterpret_cast<uint64_t*>(p);
  double* v0 = reinterpret_cast<double*>(p + al256((size_t)cells * 8));
  uint64_t* k1 = reinterpret_cast<uint64_t*>(p + 2 * al256((size_t)cells * 8));
  double* v1 = reinterpret_cast<double*>(p + 3 * al256((size_t)cells * 8));
  char* tmp = p + 4 * al256((size_t)cells * 8);
  size_t tmp_bytes = ws_bytes - 4 * al256((size_t)cells * 8);
  // invalid cells carry inv (all ones over the sorted bits): they land last
  const int bits = key_bits(inv);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, (int)cells, 0,
                                                  bits, s);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)std::min<int64_t>((cells + 255) / 256, 148 * 32);
  segment_sum_kernel<T><<<grid, 256, 0, s>>>(cells, k1, v1, inv, cols, out, ldo);
  return cudaGetLastError();
}

template <typename T>
__global__ void extrema_bwd_copy_kernel(int64_t n, int32_t d, const int64_t* __restrict__ arg,
                                        const T* __restrict__ dZ, int64_t lddz,
                                        const int32_t* __restrict__ tindex, T* dOut, int64_t ldo,
                                        CellSink sink, uint64_t max_key) {
  const int64_t total = n * (int64_t)d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / d;
    const int k = (int)(i - v * d);
    const int64_t e = arg[i];
    if (tindex) {  // dX[src[e]]: many writers
      // keys of invalid cells: all ones in the sorted bit range (> every real key)
      sink.keys[i] = e < 0 ? max_key : (uint64_t)tindex[e] * (uint64_t)d + (uint64_t)k;
      sink.vals[i] = e < 0 ? 0.0 : (double)dZ[v * lddz + k];
      continue;
    }
    if (e >= 0) dOut[e * ldo + k] = dZ[v * lddz + k];  // one winner per (edge, column)
  }
}

cudaError_t launch_route_extrema(int f64, int64_t n, int32_t d, const int64_t* arg, const void* dZ,
                                 int64_t lddz, void* dM, int64_t ldm, cudaStream_t s) {
  const int64_t total = n * (int64_t)d;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32);
  if (total == 0) return cudaSuccess;
  if (f64) route_extrema_kernel<double><<<grid, 256, 0, s>>>(n, d, arg, (const double*)dZ, lddz, (double*)dM, ldm);
  else route_extrema_kernel<float><<<grid, 256, 0, s>>>(n, d, arg, (const float*)dZ, lddz, (float*)dM, ldm);
  return cudaGetLastError();
}

// max_key: an upper bound on real keys (target rows * d); invalid cells get
// the all-ones pattern of the sorted bit range so they sort last
static uint64_t invalid_key(uint64_t max_key) {
  const int bits = key_bits(max_key + 1);
  return bits >= 64 ? ~0ull : ((1ull << bits) - 1);
}

cudaError_t launch_extrema_bwd_copy(int f64, int64_t n, int32_t d, const int64_t* arg,
                                    const void* dZ, int64_t lddz, const int32_t* tindex,
                                    int64_t n_target_rows, void* dOut, int64_t ldo, void* ws,
                                    size_t ws_bytes, cudaStream_t s) {
  const int64_t total = n * (int64_t)d;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32);
  if (total == 0) return cudaSuccess;
  CellSink sink{nullptr, nullptr};
  const uint64_t max_key = (uint64_t)n_target_rows * (uint64_t)d;
  const uint64_t inv = invalid_key(max_key);
  if (tindex) {
    sink.keys = static_cast<uint64_t*>(ws);
    sink.vals = reinterpret_cast<double*>(static_cast<char*>(ws) + al256((size_t)total * 8));
  }
  if (f64) extrema_bwd_copy_kernel<double><<<grid, 256, 0, s>>>(n, d, arg, (const double*)dZ, lddz, tindex, (double*)dOut, ldo, sink, inv);
  else extrema_bwd_copy_kernel<float><<<grid, 256, 0, s>>>(n, d, arg, (const float*)dZ, lddz, tindex, (float*)dOut, ldo, sink, inv);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !tindex) return e;
  return f64 ? sort_and_sum<double>(total, ws, ws_bytes, inv, d, (double*)dOut, ldo, s)
             : sort_and_sum<float>(total, ws, ws_bytes, inv, d, (float*)dOut, ldo, s);
}

// Fused max/min backward of a binary message (add / sub / mul / div of two
// operands): the gradient of one operand straight from the winning edges,
// without route_extrema_grad's dense (m, d) matrix (kernels.py:843-857 then
// autodiff.py:289-372). Cell (v, k) with winner e = arg[v, k] contributes
// dZ[v, k] * d phi / d operand, evaluated in fp64 on the winner's operands
// (the reference's fp64 expression order), to the operand's row: src[e]
// (several cells can hit one source row: the cells go to a CellSink as
// (row, column) keyed fp64 values, sorted and summed in fp64 in key order by
// sort_and_sum - deterministic, no float atomics), v or e (one cell per
// (row, column): plain store, bit-exact) - a broadcast operand (own_dim == 1)
// sums its cells the same way.
struct ExtBinArgs {
  int64_t n;
  int32_t d;
  const int64_t* arg;
  const void* dZ;
  int64_t lddz;
  const int32_t* src;
  int32_t op, role, target;
  OperandDev lhs, rhs;
  void* out;
  int64_t ldo;
  int32_t own_dim;
};

__device__ __forceinline__ int64_t ext_row(int32_t t, int64_t u, int64_t v, int64_t e) {
  return t == T_SRC ? u : (t == T_DST ? v : e);
}

// dot messages (d_out == 1): cell (v, c) for every operand column c adds
// dZ[v] * other[c] to the operand's row (d(a.b)/da = b)
template <typename T>
__global__ void extrema_bwd_dot_kernel(const ExtBinArgs a, CellSink sink, uint64_t inv) {
  const int64_t total = a.n * (int64_t)a.own_dim;
  T* out = static_cast<T*>(a.out);
  const OperandDev& other = a.role == 0 ? a.rhs : a.lhs;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / a.own_dim;
    const int c = (int)(i - v * a.own_dim);
    const int64_t e = a.arg[v];
    if (e < 0) {
      if (sink.keys) { sink.keys[i] = inv; sink.vals[i] = 0.0; }
      continue;
    }
    const int64_t u = __ldg(a.src + e);
    const double dz = (double)static_cast<const T*>(a.dZ)[v * a.lddz];
    const double ov = (double)static_cast<const T*>(other.data)[
        ext_row(other.target, u, v, e) * other.ld + c];
    if (sink.keys) {  // source rows: many writers
      sink.keys[i] = (uint64_t)u * (uint64_t)a.own_dim + (uint64_t)c;
      sink.vals[i] = dz * ov;
    } else {
      out[ext_row(a.target, u, v, e) * a.ldo + c] = (T)(dz * ov);
    }
  }
}

template <typename T>
__global__ void extrema_bwd_binary_kernel(const ExtBinArgs a, CellSink sink, uint64_t inv) {
  const int64_t total = a.n * (int64_t)a.d;
  T* out = static_cast<T*>(a.out);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / a.d;
    const int k = (int)(i - v * a.d);
    const int64_t e = a.arg[i];
    if (e < 0) {
      if (sink.keys) { sink.keys[i] = inv; sink.vals[i] = 0.0; }
      continue;
    }
    const int64_t u = __ldg(a.src + e);
    const double dz = (double)static_cast<const T*>(a.dZ)[v * a.lddz + k];
    const double av = (double)static_cast<const T*>(a.lhs.data)[
        ext_row(a.lhs.target, u, v, e) * a.lhs.ld + (a.lhs.dim == 1 ? 0 : k)];
    const double bv = (double)static_cast<const T*>(a.rhs.data)[
        ext_row(a.rhs.target, u, v, e) * a.rhs.ld + (a.rhs.dim == 1 ? 0 : k)];
    double g;
    switch (a.op) {
      case OP_ADD: g = dz; break;
      case OP_SUB: g = a.role == 0 ? dz : -dz; break;
      case OP_MUL: g = dz * (a.role == 0 ? bv : av); break;
      default:  // OP_DIV: d(a/b)/da = 1/b, d(a/b)/db = -a/b^2 (0 where b == 0)
        if (bv == 0.0) g = 0.0;
        else g = a.role == 0 ? dz / bv : -((dz * av) / (bv * bv));
        break;
    }
    const int64_t row = ext_row(a.target, u, v, e);
    const int col = a.own_dim == 1 ? 0 : k;
    if (sink.keys) {  // source rows / broadcast operands: many writers
      sink.keys[i] = (uint64_t)row * (uint64_t)a.own_dim + (uint64_t)col;
      sink.vals[i] = g;
    } else {
      out[row * a.ldo + col] = (T)g;  // one cell per (row, column)
    }
  }
}

cudaError_t launch_extrema_bwd_binary(int f64, const ExtBinArgs& a, int64_t n_target_rows,
                                      void* ws, size_t ws_bytes, cudaStream_t s) {
  const bool dot = a.op == OP_DOT;
  const int64_t total = a.n * (int64_t)(dot ? a.own_dim : a.d);
  if (total == 0) return cudaSuccess;
  const bool many = a.target == T_SRC || (!dot && a.own_dim == 1);
  CellSink sink{nullptr, nullptr};
  const uint64_t inv = invalid_key((uint64_t)n_target_rows * (uint64_t)a.own_dim);
  if (many) {
    sink.keys = static_cast<uint64_t*>(ws);
    sink.vals = reinterpret_cast<double*>(static_cast<char*>(ws) + al256((size_t)total * 8));
  }
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32);
  if (dot) {
    if (f64) extrema_bwd_dot_kernel<double><<<grid, 256, 0, s>>>(a, sink, inv);
    else extrema_bwd_dot_kernel<float><<<grid, 256, 0, s>>>(a, sink, inv);
  } else {
    if (f64) extrema_bwd_binary_kernel<double><<<grid, 256, 0, s>>>(a, sink, inv);
    else extrema_bwd_binary_kernel<float><<<grid, 256, 0, s>>>(a, sink, inv);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !many) return e;
  return f64 ? sort_and_sum<double>(total, ws, ws_bytes, inv, a.own_dim, (double*)a.out, a.ldo, s)
             : sort_and_sum<float>(total, ws, ws_bytes, inv, a.own_dim, (float*)a.out, a.ldo, s);
}

// ---- row dot products: out[v * os] = sum_c A[v,c] B[v,c] - sub[v] (fp64) ---------
// The fused GAT backward's node-level epilogue (S_v = dZ[v].Z[v] into the
// pack; d el[u] = X[u].dX[u] - t[u]) in one pass each instead of a chain of
// elementwise / reduction launches.
template <typename T, typename TB>
__global__ void rowdot_kernel(int64_t n, int32_t d, const T* __restrict__ A, int64_t lda,
                              const TB* __restrict__ B, int64_t ldb,
                              const double* __restrict__ sub, T* out, int64_t os, int pair) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    const T* a = A + v * lda;
    const TB* b = B + v * ldb;
    for (int c = 0; c < d; ++c) acc += (double)__ldg(a + c) * (double)__ldg(b + c);
    if (sub) acc -= sub[v];
    const T hi = (T)acc;
    out[v * os] = hi;
    if (pair) out[v * os + 1] = (T)(acc - (double)hi);  // fp64 value as hi + lo
  }
}

// B may be fp64 for an fp32 A: the unrounded fp64 rows of an aggregation
// (gmp_gat_aggregate's z64), so a dot that cancels is not limited by the
// fp32 rounding of B
cudaError_t launch_rowdot(int f64, int b_f64, int64_t n, int32_t d, const void* A, int64_t lda,
                          const void* B, int64_t ldb, const double* sub, void* out, int64_t os,
                          int pair, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (f64) rowdot_kernel<double, double><<<grid, 256, 0, s>>>(n, d, (const double*)A, lda, (const double*)B, ldb, sub, (double*)out, os, pair);
  else if (b_f64) rowdot_kernel<float, double><<<grid, 256, 0, s>>>(n, d, (const float*)A, lda, (const double*)B, ldb, sub, (float*)out, os, pair);
  else rowdot_kernel<float, float><<<grid, 256, 0, s>>>(n, d, (const float*)A, lda, (const float*)B, ldb, sub, (float*)out, os, pair);
  return cudaGetLastError();
}

// ---- row gather: dst[i] = src[idx[i]] ------------------------------------------

template <typename T>
__global__ void gather_rows_kernel(int64_t n, int32_t dim, const int32_t* __restrict__ idx,
                                   const T* __restrict__ src, int64_t lds, T* dst, int64_t ldd) {
  const int64_t total = n * (int64_t)dim;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / dim;
    const int c = (int)(i - r * dim);
    dst[r * ldd + c] = __ldg(src + (int64_t)__ldg(idx + r) * lds + c);
  }
}

// ---- windowed adjacency-order gather: dst[p] = src[eids[p]] -----------------
// A per-edge operand laid out in adjacency (CSC) order once per call so every
// column tile of a u_op_e g-SpMM streams it. The plain gather reads src at
// random edge ids: on the Reddit-shaped graph 114.5 M random 4 B reads, each a
// 128 B DRAM line (12.6 GB for a 458 MB array, 2.2 ms). When every row's edge
// ids ascend (CSC of an edge list grouped by source, the reference's
// generators), a heavy row's positions inside one window of consecutive edge
// ids form one contiguous run: items (window b, heavy row r) are walked
// window-major by persistent warps, so the window's src lines are fetched
// from DRAM about once and reused from L2 by every row that reads them; the
// light rows (few edges each, 4 % of Reddit's) gather directly.
struct GatherAdjArgs {
  const int64_t* indptr;
  const int32_t* eids;
  const int32_t* order;
  int64_t n_heavy, n_nonempty, n_windows, win;
  const int64_t* bounds;  // (n_heavy, n_windows + 1)
  int32_t dim;
  int64_t lds, ldd;
};

static __global__ void gather_adj_bounds(GatherAdjArgs a, int64_t* bounds) {
  const int64_t per = a.n_windows + 1;
  const int64_t total = a.n_heavy * per;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per, b = i - r * per;
    const int64_t row = a.order[r];
    int64_t x = a.indptr[row], y = a.indptr[row + 1];
    const int64_t e0 = b * a.win;
    while (x < y) {
      const int64_t mid = (x + y) >> 1;
      if (__ldg(a.eids + mid) < e0) x = mid + 1; else y = mid;
    }
    bounds[i] = x;
  }
}

template <typename T>
__global__ void __launch_bounds__(256, 4) gather_adj_kernel(GatherAdjArgs a, const T* __restrict__ src,
                                                             T* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t heavy_items = a.n_windows * a.n_heavy;
  const int64_t items = heavy_items + (a.n_nonempty - a.n_heavy);
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
       it += nwarps) {
    int64_t lo, hi;
    if (it < heavy_items) {  // window-major: warps in flight share a window
      const int64_t b = it / a.n_heavy, r = it - b * a.n_heavy;
      const int64_t* bd = a.bounds + r * (a.n_windows + 1) + b;
      lo = __ldg(bd);
      hi = __ldg(bd + 1);
    } else {
      const int64_t row = a.order[a.n_heavy + (it - heavy_items)];
      lo = a.indptr[row];
      hi = a.indptr[row + 1];
    }
    if (a.dim == 1) {
      // 8 positions per lane in flight: the eid loads, then the dependent
      // src loads, then the stores
      constexpr int U = 8;
      for (int64_t p0 = lo; p0 < hi; p0 += 32 * U) {
        int32_t e[U];
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t p = p0 + u * 32 + lane;
          e[u] = p < hi ? __ldg(a.eids + p) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = e[u] >= 0 ? __ldg(src + (int64_t)e[u] * a.lds) : T(0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t p = p0 + u * 32 + lane;
          if (p < hi) dst[p * a.ldd] = v[u];
        }
      }
    } else {
      for (int64_t p = lo; p < hi; ++p) {
        const int64_t e = __ldg(a.eids + p);
        for (int c = lane; c < a.dim; c += 32) dst[p * a.ldd + c] = __ldg(src + e * a.lds + c);
      }
    }
  }
}

size_t gather_adj_workspace(int64_t n_heavy, int64_t m, int32_t dim, size_t F, int64_t* nw_out,
                            int64_t* win_out) {
  // windows of edge ids whose src rows take 2 MB: warps take items
  // window-major but heavy-row items differ in size by ~100x, so many
  // windows are in flight at once next to the streamed eids / dst. Reddit
  // u_mul_e (458 MB of w): 2 / 4 / 8 / 16 / 32 MB windows read 1.5 / 2.4 /
  // 4.7 / 6.1 / 5.5 GB of DRAM in 1.12 / 1.10 / 1.33 / 1.52 / 1.48 ms; the
  // plain gather 12.6 GB in 2.2 ms (GMP_GATHER_WIN_MB overrides the size)
  static const int64_t win_mb = getenv("GMP_GATHER_WIN_MB") ? atoll(getenv("GMP_GATHER_WIN_MB")) : 2;
  const int64_t per_edge = std::max<int64_t>(1, (int64_t)dim * (int64_t)F);
  const int64_t win = std::max<int64_t>(1 << 14, (std::max<int64_t>(win_mb, 1) << 20) / per_edge);
  const int64_t nw = (m + win - 1) / win;
  if (nw_out) *nw_out = nw;
  if (win_out) *win_out = win;
  return (size_t)(n_heavy * (nw + 1)) * sizeof(int64_t);
}

cudaError_t launch_gather_adj(int f64, const int64_t* indptr, const int32_t* eids,
                              const int32_t* order, int64_t n_heavy, int64_t n_nonempty, int64_t m,
                              int32_t dim, const void* src, int64_t lds, void* dst, int64_t ldd,
                              void* ws, cudaStream_t s) {
  GatherAdjArgs a{};
  a.indptr = indptr; a.eids = eids; a.order = order;
  a.n_heavy = n_heavy; a.n_nonempty = n_nonempty;
  gather_adj_workspace(n_heavy, m, dim, f64 ? 8 : 4, &a.n_windows, &a.win);
  a.bounds = static_cast<const int64_t*>(ws);
  a.dim = dim; a.lds = lds; a.ldd = ldd;
  if (n_heavy > 0) {
    const int64_t total = n_heavy * (a.n_windows + 1);
    gather_adj_bounds<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, s>>>(
        a, static_cast<int64_t*>(ws));
  }
  // persistent: every warp resident at once (the static window-major item
  // striding assumes it; a second wave would re-walk every window)
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const unsigned grid = (unsigned)sms * 4;
  if (f64) gather_adj_kernel<double><<<grid, 256, 0, s>>>(a, (const double*)src, (double*)dst);
  else gather_adj_kernel<float><<<grid, 256, 0, s>>>(a, (const float*)src, (float*)dst);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(int f64, int64_t n, int32_t dim, const int32_t* idx, const void* src,
                               int64_t lds, void* dst, int64_t ldd, cudaStream_t s) {
  const int64_t total = n * (int64_t)dim;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32);
  if (f64) gather_rows_kernel<double><<<grid, 256, 0, s>>>(n, dim, idx, (const double*)src, lds, (double*)dst, ldd);
  else gather_rows_kernel<float><<<grid, 256, 0, s>>>(n, dim, idx, (const float*)src, lds, (float*)dst, ldd);
  return cudaGetLastError();
}

// ---- column-tile packing ------------------------------------------------------
// packed[t][r][c] = src[r][t*tw + c] (0 past column d): every column tile of a
// row becomes one aligned tw-element run, so the row kernel's per-edge gather
// of a tile is whole 32 B sectors with 128-bit loads whatever the caller's ld.

// grid.y = tile; x = (row, column pair) with shifts only (power-of-two tile
// width); adjacent threads touch adjacent columns, so loads and stores are
// coalesced on both sides.
template <typename T>
__global__ void pack_tiles_kernel(int64_t n, int32_t d, int32_t tw, const T* __restrict__ src,
                                  int64_t lds, T* __restrict__ dst) {
  const int t = blockIdx.y;
  const int half = tw >> 1;  // column pairs per tile row (a power of two)
  const int hl = __ffs(half) - 1;
  const int64_t total = n * half;
  const int c_base = t * tw;
  T* out = dst + (int64_t)t * n * tw;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i >> hl;
    const int c = (int)(i & (half - 1)) * 2;
    const int col = c_base + c;
    const T* sp = src + r * lds + col;
    const T v0 = col < d ? sp[0] : T(0);
    const T v1 = col + 1 < d ? sp[1] : T(0);
    out[r * tw + c] = v0;
    out[r * tw + c + 1] = v1;
  }
}

template <typename T>
__global__ void unpack_tiles_kernel(int64_t n, int32_t d, int32_t tw, const T* __restrict__ src,
                                    T* __restrict__ dst, int64_t ldd) {
  const int t = blockIdx.y;
  const int half = tw >> 1;
  const int hl = __ffs(half) - 1;
  const int64_t total = n * half;
  const int c_base = t * tw;
  const T* in = src + (int64_t)t * n * tw;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i >> hl;
    const int c = (int)(i & (half - 1)) * 2;
    const int col = c_base + c;
    if (col < d) dst[r * ldd + col] = in[r * tw + c];
    if (col + 1 < d) dst[r * ldd + col + 1] = in[r * tw + c + 1];
  }
}

cudaError_t launch_pack_tiles(int f64, bool unpack, int64_t n, int32_t d, int32_t tw,
                              const void* src, int64_t lds, void* dst, int64_t ldd,
                              cudaStream_t s) {
  const int32_t ntiles = (d + tw - 1) / tw;
  if (tw < 2 || (tw & (tw - 1))) return cudaErrorInvalidValue;  // a power-of-two tile
  const int64_t total = n * (int64_t)(tw / 2);
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 4)),
                  (unsigned)ntiles);
  if (f64) {
    if (unpack) unpack_tiles_kernel<double><<<grid, 256, 0, s>>>(n, d, tw, (const double*)src, (double*)dst, ldd);
    else pack_tiles_kernel<double><<<grid, 256, 0, s>>>(n, d, tw, (const double*)src, lds, (double*)dst);
  } else {
    if (unpack) unpack_tiles_kernel<float><<<grid, 256, 0, s>>>(n, d, tw, (const float*)src, (float*)dst, ldd);
    else pack_tiles_kernel<float><<<grid, 256, 0, s>>>(n, d, tw, (const float*)src, lds, (float*)dst);
  }
  return cudaGetLastError();
}

// ---- degree-binned schedule ---------------------------------------------------

__global__ void degree_kernel(int64_t n, const int64_t* __restrict__ indptr, int32_t* deg,
                              int32_t* rows, int32_t thr, int32_t light,
                              unsigned long long* counters) {
  unsigned long long heavy = 0, nonempty = 0, medium = 0, dmax = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t dg = indptr[r + 1] - indptr[r];
    deg[r] = (int32_t)dg;
    rows[r] = (int32_t)r;
    heavy += dg > thr;
    nonempty += dg > 0;
    medium += dg > light;
    dmax = dmax > (unsigned long long)dg ? dmax : (unsigned long long)dg;
  }
  for (int off = 16; off > 0; off >>= 1) {
    heavy += __shfl_xor_sync(kFull, heavy, off);
    nonempty += __shfl_xor_sync(kFull, nonempty, off);
    medium += __shfl_xor_sync(kFull, medium, off);
    const unsigned long long o = __shfl_xor_sync(kFull, dmax, off);
    dmax = dmax > o ? dmax : o;
  }
  if ((threadIdx.x & 31) == 0) {
    if (heavy) atomicAdd(counters, heavy);
    if (nonempty) atomicAdd(counters + 1, nonempty);
    if (medium) atomicAdd(counters + 2, medium);
    if (dmax) atomicMax(counters + 3, dmax);
  }
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t schedule_cub_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending((void*)nullptr, bytes, (const int32_t*)nullptr,
                                            (int32_t*)nullptr, (const int32_t*)nullptr,
                                            (int32_t*)nullptr, (int)n);
  return bytes;
}

size_t schedule_workspace_bytes(int64_t n) {
  return align256(32) + 3 * align256((size_t)n * 4) + align256(schedule_cub_bytes(n));
}

cudaError_t build_schedule(int64_t n, const int64_t* indptr, int32_t thr, int32_t light,
                           int32_t* order_out, void* ws, size_t ws_bytes, int64_t* n_heavy,
                           int64_t* n_medium, int64_t* n_nonempty, int64_t* max_degree,
                           cudaStream_t s) {
  char* p = static_cast<char*>(ws);
  auto* counters = reinterpret_cast<unsigned long long*>(p);
  p += align256(32);
  auto* deg = reinterpret_cast<int32_t*>(p);
  p += align256((size_t)n * 4);
  auto* deg_sorted = reinterpret_cast<int32_t*>(p);
  p += align256((size_t)n * 4);
  auto* rows = reinterpret_cast<int32_t*>(p);
  p += align256((size_t)n * 4);
  size_t cub_bytes = ws_bytes - (size_t)(p - static_cast<char*>(ws));
  cudaError_t err = cudaMemsetAsync(counters, 0, 32, s);
  if (err != cudaSuccess) return err;
  if (n > 0) {
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
    degree_kernel<<<grid, 256, 0, s>>>(n, indptr, deg, rows, thr, light, counters);
    err = cub::DeviceRadixSort::SortPairsDescending(p, cub_bytes, deg, deg_sorted, rows, order_out,
                                                    (int)n, 0, 32, s);
    if (err != cudaSuccess) return err;
  }
  unsigned long long host[4] = {0, 0, 0, 0};
  err = cudaMemcpyAsync(host, counters, 32, cudaMemcpyDeviceToHost, s);
  if (err != cudaSuccess) return err;
  err = cudaStreamSynchronize(s);
  *n_heavy = (int64_t)host[0];
  *n_nonempty = (int64_t)host[1];
  *n_medium = (int64_t)host[2];
  *max_degree = (int64_t)host[3];
  return err;
}


// ---- L2 gather probe -----------------------------------------------------------
// The ceiling the row kernel's gathers run against once a column tile of X is
// L2-resident: n random rows of row_bytes (64 or 256) gathered from a slice
// of `rows` rows, L = row_bytes / 16 lanes x float4 per row, 8 rows in flight
// per lane group, full occupancy. Indices come from a 32-bit hash of the
// gather number (no index array: the row kernel's indices stream from HBM,
// which this probe does not charge). bench.py times it live beside the
// kernel it bounds.
template <int L>
__global__ void __launch_bounds__(256) l2_gather_probe_kernel(const float4* __restrict__ data,
                                                              uint32_t rows, int64_t n,
                                                              float* sink) {
  constexpr int U = 8;
  const int lane = threadIdx.x & (L - 1);
  const int64_t groups = (int64_t)gridDim.x * blockDim.x / L;
  float acc = 0.f;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / L; g * U < n; g += groups) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // 32-bit murmur finaliser + multiply-high range reduction: a few
      // integer ops per gather (a 64-bit modulo is ~100 instructions and made
      // an earlier version of this probe issue-bound far below the ceiling)
      uint32_t x = (uint32_t)(g * U + u) * 0x9E3779B1u + 0x7F4A7C15u;
      x ^= x >> 16; x *= 0x85EBCA6Bu; x ^= x >> 13; x *= 0xC2B2AE35u; x ^= x >> 16;
      const uint32_t r = __umulhi(x, rows);
      v[u] = __ldg(data + (int64_t)r * L + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) sink[0] = acc;  // keeps the loads live
}

cudaError_t launch_l2_gather_probe(const void* data, int64_t rows, int32_t row_bytes, int64_t n,
                                   float* sink, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (row_bytes == 256)
    l2_gather_probe_kernel<16><<<sms * 8, 256, 0, s>>>((const float4*)data, (uint32_t)rows, n, sink);
  else
    l2_gather_probe_kernel<4><<<sms * 8, 256, 0, s>>>((const float4*)data, (uint32_t)rows, n, sink);
  return cudaGetLastError();
}

}  // namespace gmp
