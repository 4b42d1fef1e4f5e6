// sampling.cu - neighbour sampling for mini-batch training (replaces
// graph.neighbor_sample, /root/reference/pkg/src/graphmp/graph.py:231-286).
//
// The reference walks the seeds in order on one numpy Generator and, per
// seed, runs a partial Fisher-Yates pass over a copy of the seed's in-edge
// segment (graph.py:259-266), then sorts the k picks. Here one warp owns one
// seed: k = min(fanout, deg) distinct offsets in [0, deg) are drawn with
// Floyd's algorithm (uniform over k-subsets, like the partial shuffle), the
// membership test of each draw is a warp-wide scan + ballot over the picks so
// far, and the picks are written ascending by rank (distinct values -> unique
// ranks). Randomness is counter-based (splitmix64 of rng_seed, node id, draw
// index), so a sample is a pure function of (graph, seed node, fanout,
// rng_seed): independent of the batch it is drawn in and of the launch shape.
#include <cstdint>

#include <cuda_runtime.h>

namespace gmp {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// uniform integer in [0, bound) (Lemire multiply-high; bias < bound / 2^64)
__device__ __forceinline__ int64_t draw_below(uint64_t key, uint64_t draw, uint64_t bound) {
  const uint64_t h = splitmix64(key ^ splitmix64(draw));
  return (int64_t)__umul64hi(h, bound);
}

constexpr int kSampleWarps = 4;

__global__ void __launch_bounds__(kSampleWarps * 32)
    neighbor_sample_kernel(const int64_t* __restrict__ indptr, const int64_t* __restrict__ seeds,
                           int64_t n_seeds, const int64_t* __restrict__ out_off,
                           uint64_t rng_seed, int64_t* __restrict__ scratch,
                           int64_t* __restrict__ out_pos) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * kSampleWarps + (threadIdx.x >> 5);
  if (w >= n_seeds) return;
  const int64_t node = seeds[w];
  const int64_t lo = indptr[node], deg = indptr[node + 1] - lo;
  const int64_t off = out_off[w], k = out_off[w + 1] - off;
  if (k == 0) return;
  if (k == deg) {  // every in-edge is taken, already ascending
    for (int64_t j = lane; j < k; j += 32) out_pos[off + j] = lo + j;
    return;
  }
  const uint64_t key = splitmix64(rng_seed ^ splitmix64((uint64_t)node * 0xD1B54A32D192ED03ull));
  int64_t* picks = scratch + off;
  // Floyd: for j in [deg-k, deg): t = U[0, j]; insert t unless taken, else j
  for (int64_t i = 0; i < k; ++i) {
    const int64_t j = deg - k + i;
    const int64_t t = draw_below(key, (uint64_t)i, (uint64_t)j + 1);
    bool hit = false;
    for (int64_t q = lane; q < i; q += 32) hit |= picks[q] == t;
    hit = __any_sync(0xffffffffu, hit);
    if (lane == 0) picks[i] = hit ? j : t;
    __syncwarp();
  }
  // ascending output: rank of each pick among the k distinct picks
  for (int64_t a = lane; a < k; a += 32) {
    const int64_t v = picks[a];
    int64_t rank = 0;
    for (int64_t b = 0; b < k; ++b) rank += picks[b] < v;
    out_pos[off + rank] = lo + v;
  }
}

cudaError_t launch_neighbor_sample(const int64_t* indptr, const int64_t* seeds, int64_t n_seeds,
                                   const int64_t* out_off, uint64_t rng_seed, int64_t* scratch,
                                   int64_t* out_pos, cudaStream_t s) {
  const int64_t grid = (n_seeds + kSampleWarps - 1) / kSampleWarps;
  neighbor_sample_kernel<<<(unsigned)grid, kSampleWarps * 32, 0, s>>>(
      indptr, seeds, n_seeds, out_off, rng_seed, scratch, out_pos);
  return cudaGetLastError();
}

}  // namespace gmp
