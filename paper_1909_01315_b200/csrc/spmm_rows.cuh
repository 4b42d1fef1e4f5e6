// spmm_rows.cuh - the g-SpMM row kernel (elementwise messages).
//
// Replaces the reference's default gspmm strategy, node_parallel over the
// in-adjacency (kernels.py:473-482) and its per-destination segment walk
// _GroupedWalk (kernels.py:340-466): for every destination row v,
//   Z[v, c] = rho_{(u,e,v)} phi(lhs[., c], rhs[., c])
// with the message formed in registers and never materialised.
//
// Work decomposition:
//  * columns are split into tiles of <= 32*V columns (the reference's
//    feature_parallel column split, kernels.py:485-513), sized so one column
//    slice of the gathered source matrix stays L2-resident; tiles are the
//    slowest-varying grid index, so concurrently running CTAs share a slice;
//  * rows come in degree-descending order (gmp_sched). The first n_heavy rows
//    (degree > heavy threshold) are reduced by a whole CTA (warps interleave
//    32-edge batches, partials merged through shared memory in warp order);
//    the rest are reduced by one warp each;
//  * inside a warp, 32 lanes = E edge slots x G feature lanes; each feature
//    lane owns one V-vector (128/64-bit loads). Edge indices (and per-edge
//    scalar operands such as an attention weight) are loaded 32 at a time,
//    coalesced, ahead of use, and broadcast by shuffle. The gather loop is
//    branch-free: masked lanes load a clamped in-bounds address and select 0;
//  * operand access modes (per-edge vector gather / per-edge scalar /
//    row-constant) are template parameters for the hot combinations
//    (copy_u/copy_e, u_op_e, u_op_v, e_op_v) and runtime for the rest;
//  * slot partials are combined by a fixed xor-shuffle tree: results are
//    deterministic run to run.
//
// Numerics: fp32 sums are carried as an exact
// compensated pair (TwoSum / TwoProduct on packed FADD2/FFMA2) and folded
// into an fp64 accumulator every 32 edges - equivalent to fp64 accumulation
// of the exact fp64 messages the reference forms, without per-element
// F2F.F64.F32 conversions (those run on the slow XU pipe). max/min of copy
// messages compare the fp32 values directly (exact); max/min of binary
// messages compare the fp64 message, so arg edges equal the reference's.
#pragma once

#include <cstdlib>
#include <type_traits>

#include <cooperative_groups.h>

#include "gmp_common.cuh"

namespace gmp {

constexpr int kWarpsPerCta = 8;
#ifndef GMP_PIPE_MIN_BLOCKS
#define GMP_PIPE_MIN_BLOCKS 3
#endif
#ifndef GMP_PIPE_NB
#define GMP_PIPE_NB 4
#endif
#ifndef GMP_PIPE_NB_NARROW
#define GMP_PIPE_NB_NARROW 4
#endif
#ifndef GMP_ROW_MIN_BLOCKS
#define GMP_ROW_MIN_BLOCKS 3
#endif

// operand access modes inside the row kernel
enum { M_FULL = 0, M_SCALAR = 1, M_HOIST = 2, M_NONE = 3 };
// compile-time (lhs, rhs) mode pairs; MP_GEN reads the modes at run time.
// MP_AF / MP_AB: fused GAT attention (edge_softmax of u_add_v scores times a
// gathered vector, see gmp_gat_aggregate): lhs is a gathered vector and the
// per-edge scalar is the attention weight, recomputed from node-keyed data
//   alpha = exp((el[src] + er[dst]) - max[dst]) * inv_sum[dst]
// MP_AF walks destination rows (el gathered per edge, (er, max, inv) of the
// row constant); MP_AB walks source rows of the reverse graph ((er, max, inv)
// gathered per edge as one packed row, el of the row constant).
enum { MP_F = 0, MP_FF = 1, MP_FS = 2, MP_FH = 3, MP_GEN = 4, MP_AF = 5, MP_AB = 6 };

template <int MP>
struct IsAttn {
  static constexpr bool value = MP == MP_AF || MP == MP_AB;
};

struct RowOperand {
  const void* data;
  uint32_t ld;
  int32_t mode;      // M_FULL / M_SCALAR / M_HOIST
  int32_t from_eid;  // gathered by edge id (EDGE target) instead of neighbour id (SRC target)
  int32_t bcast;     // hoisted operand is a single column
  int32_t from_pos;  // edge operand already permuted to adjacency order: row = position
};

enum { kAccRead = 1, kAccZ = 2, kAccStore = 4 };

struct SpmmArgs {
  const int64_t* indptr;
  const int32_t* indices;
  const int32_t* eids;
  const int32_t* order;  // nullable: identity order
  int64_t n_rows;
  int64_t n_heavy;
  int64_t n_medium;       // rows [n_heavy, n_medium) of `order`: one warp each
  int64_t medium_blocks;  // CTAs covering them (kWarpsPerCta rows per CTA)
  int64_t blocks_per_tile;
  int32_t d_out;
  int32_t tile_cols;
  int32_t g_log2;  // feature lanes per edge slot = 1 << g_log2
  int32_t mean;
  int32_t need_eid;
  RowOperand lhs, rhs;
  void* Z;
  int64_t ldz;
  int64_t* arg;
  int64_t* counts;
  int32_t* err_pos;
  // fused attention (MP_AF / MP_AB only)
  const void* attn_el;    // (n) el column, stride attn_lde
  uint32_t attn_lde;
  const void* attn_pack;  // (n, PackW<T>) 32 B rows [er, max, inv_sum, w (, w_lo)]
  double* attn_t;         // MP_AB: t[u] = sum_{u->v} alpha_e w[v] (nullable)
  int32_t cluster;        // CTAs per heavy row (a thread-block cluster), 1 = one CTA
  int32_t z_split;        // 1: Z rows only 8 B aligned: store a 4-vector as two 8 B halves;
                          // 2: 4 B aligned: element stores
  // fp64 row sums (sum / mean only; null acc64: plain store of Z). acc_mode
  // bits: kAccRead - add acc64[row] first (staged sums over several edge
  // blocks of the same rows, gmp_gspmm_staged); kAccZ - round once into Z
  // (mean divides by deg_full[row] when given); kAccStore - store the fp64
  // sum into acc64 (a later stage, or an exact copy of Z for the fused GAT
  // backward's row dots).
  double* acc64;
  int64_t ldacc;
  int32_t acc_mode;
  const int64_t* deg_full;
};

// per-node pack of the fused attention: one 32 B row (a single sector per
// gathered edge): fp32 [er, max, inv_sum, w_hi, w_lo, -, -, -], fp64
// [er, max, inv_sum, w]. w = S_v (backward only) is carried to fp64
// accuracy: t[u] = sum alpha_e S_v feeds d el = X.dX - t, which cancels.
template <typename T>
struct PackW {
  static constexpr int value = sizeof(T) == 4 ? 8 : 4;
};

template <typename T>
__device__ __forceinline__ void load_pack4(const T* p, T& a, T& b, T& c, T& d) {
  if constexpr (sizeof(T) == 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    a = v.x; b = v.y; c = v.z; d = v.w;
  } else {
    const double2 v0 = __ldg(reinterpret_cast<const double2*>(p));
    const double2 v1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
    a = v0.x; b = v0.y; c = v1.x; d = v1.y;
  }
}

// row constants of the fused attention: (er, max, inv) of a destination row
// (MP_AF) or el of a source row (MP_AB, in rc[0])
template <typename T, int MP>
__device__ __forceinline__ void attn_row_consts(const SpmmArgs& a, int64_t row, T (&rc)[3]) {
  rc[0] = rc[1] = rc[2] = T(0);
  if (row < 0) return;
  if constexpr (MP == MP_AF) {
    T w;
    load_pack4<T>(static_cast<const T*>(a.attn_pack) + row * PackW<T>::value, rc[0], rc[1], rc[2],
                  w);
  } else if constexpr (MP == MP_AB) {
    rc[0] = __ldg(static_cast<const T*>(a.attn_el) + (uint64_t)row * a.attn_lde);
  }
}

// exp(x - m) of a softmax term / attention weight. fp32: 2^((x - m) log2 e)
// on the SFU (ex2.approx.ftz, max rel. error 2^-22). The argument is formed
// as (x - m) first and then scaled, so its rounding error is relative to
// |x - m| (x - m is exact by Sterbenz whenever x and m are within a factor 2
// of each other, i.e. for every term that is not negligible), never to |m|:
// rounding -m*log2e first would put an absolute exponent error of
// ulp(m log2e)/2 on every term, 2.4e-5 relative at |m| ~ 1000, which does not
// cancel once partials with different maxima are merged. u_add_v scores
// (GAT) are carried as the exact TwoSum pair hi + lo of el + er and enter as
// ((hi - m) + lo), so the fp32 rounding of the score itself (|s| 2^-24) does
// not leak into the exponent either. Every fp32 softmax term in the library
// (statistics, rescale, merges, normalisation, fused GAT weights) uses these
// formulas, so a recomputed weight equals the stored one bit for bit.
constexpr float kLog2e = 1.4426950408889634f;
__device__ __forceinline__ float ex2_approx(float a) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a));
  return y;
}
__device__ __forceinline__ float sm_exp(float x, float m) {
  return ex2_approx(__fmul_rn(__fsub_rn(x, m), kLog2e));
}
__device__ __forceinline__ float sm_exp(float hi, float lo, float m) {
  return ex2_approx(__fmul_rn(__fadd_rn(__fsub_rn(hi, m), lo), kLog2e));
}
__device__ __forceinline__ double sm_exp(double x, double m) { return exp(x - m); }
__device__ __forceinline__ double sm_exp(double hi, double lo, double m) { return exp((hi - m) + lo); }

// u_add_v score a + b as the exact pair hi + lo (TwoSum; order-independent)
__device__ __forceinline__ void uv_score(float a, float b, float& hi, float& lo) {
  hi = __fadd_rn(a, b);
  const float bb = __fsub_rn(hi, a);
  lo = __fadd_rn(__fsub_rn(a, __fsub_rn(hi, bb)), __fsub_rn(b, bb));
}
__device__ __forceinline__ void uv_score(double a, double b, double& hi, double& lo) {
  hi = __dadd_rn(a, b);
  const double bb = __dsub_rn(hi, a);
  lo = __dadd_rn(__dsub_rn(a, __dsub_rn(hi, bb)), __dsub_rn(b, bb));
}

// attention weight of the edge to/from neighbour nb; same fp operation
// order as the fused softmax (softmax.cuh: s = el + er; exp(s - max) * inv).
// MP_AB also returns the neighbour's pack w (the backward's per-destination
// sum S_v, fp64) in w.
template <typename T, int MP>
__device__ __forceinline__ T attn_alpha(const SpmmArgs& a, uint32_t nb, const T (&rc)[3],
                                        double& w) {
  T hi, lo;
  if constexpr (MP == MP_AF) {
    w = 0.0;
    uv_score(__ldg(static_cast<const T*>(a.attn_el) + (uint64_t)nb * a.attn_lde), rc[0], hi, lo);
    return sm_exp(hi, lo, rc[1]) * rc[2];
  } else {
    T er, mx, inv, wh;
    const T* p = static_cast<const T*>(a.attn_pack) + (uint64_t)nb * PackW<T>::value;
    load_pack4<T>(p, er, mx, inv, wh);
    w = (double)wh;
    if constexpr (sizeof(T) == 4) w += (double)__ldg(p + 4);  // same 32 B sector
    uv_score(rc[0], er, hi, lo);
    return sm_exp(hi, lo, mx) * inv;
  }
}

// per-edge scalar operand: a stored scalar, or the recomputed attention
// weight (MP_AB adds alpha * w of the edge into tsum)
template <typename T, int MP>
__device__ __forceinline__ T rhs_scalar(const SpmmArgs& a, uint32_t row, const T (&rc)[3],
                                        double& tsum) {
  if constexpr (IsAttn<MP>::value) {
    double w;
    const T al = attn_alpha<T, MP>(a, row, rc, w);
    if constexpr (MP == MP_AB) tsum += (double)al * w;
    return al;
  } else {
    return __ldg(static_cast<const T*>(a.rhs.data) + (uint64_t)row * a.rhs.ld);
  }
}

// ---- accumulation policies ---------------------------------------------------

enum { POL_COMP = 0, POL_DBL = 1, POL_EXT_T = 2, POL_EXT_D = 3 };

template <typename T, int OP, int RHO>
struct Policy {
  static constexpr int value =
      (RHO != RHO_SUM)
          ? ((OP == OP_COPY || sizeof(T) == 8) ? POL_EXT_T : POL_EXT_D)
          : ((sizeof(T) == 4 && OP != OP_DIV) ? POL_COMP : POL_DBL);
};

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// a - b on packed fp32x2: FADD2 with a negated operand (two register
// sources; an FFMA2 by -1 has three and issues at half the rate)
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}

// x * y on packed fp32x2 as its own rounded FMUL2 (with fadd2 below: a
// product contracted into the following add breaks TwoSum's premise that
// the addend is a float)
// ptxas fuses mul.rn.f32x2 into a following add.rn.f32x2 (FFMA2 in the
// SASS, contrary to the .rn no-contraction rule), so the rounded product is
// formed by two scalar FMULs, which it keeps
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
}

// a + b as its own rounded FADD2: ptxas contracts __fadd2_rn(s, x * y) into
// an FFMA2 even when the product comes from mul.rn.f32x2 (seen in the SASS)
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}

// s + c += x exactly (TwoSum, Knuth); packed fp32x2, seven FADD2.
__device__ __forceinline__ void two_sum2(float2& s, float2& c, float2 x) {
  const float2 t = fadd2(s, x);  // never contracted with a producer of x
  const float2 bb = fsub2(t, s);               // t - s
  const float2 e1 = fsub2(s, fsub2(t, bb));    // s - (t - bb)
  const float2 e2 = fsub2(x, bb);              // x - bb
  c = __fadd2_rn(c, __fadd2_rn(e1, e2));
  s = t;
}

// s + x*y accumulated exactly to second order: TwoSum of the rounded product
// pr with its two error parts fused - (pr - bb) + (x*y - pr) = x*y - bb in
// one FMA (rounded once, 2^-24 of a term already ~2^-24 of |t|) - 8 packed
// ops per column pair instead of TwoProduct + TwoSum's 10
__device__ __forceinline__ void two_sum_prod2(float2& s, float2& c, float2 x, float2 y) {
  const float2 pr = fmul2(x, y);
  const float2 t = fadd2(s, pr);
  const float2 bb = fsub2(t, s);                        // t - s
  const float2 e1 = fsub2(s, fsub2(t, bb));             // s - (t - bb)
  const float2 e2 = __ffma2_rn(x, y, f2(-bb.x, -bb.y));  // x*y - bb
  c = __fadd2_rn(c, __fadd2_rn(e1, e2));
  s = t;
}
__device__ __forceinline__ void two_sum_prod1(float& s, float& c, float x, float y) {
  const float pr = __fmul_rn(x, y);
  const float t = __fadd_rn(s, pr);
  const float bb = __fsub_rn(t, s);
  const float e1 = __fsub_rn(s, __fsub_rn(t, bb));
  const float e2 = __fmaf_rn(x, y, -bb);
  c = __fadd_rn(c, __fadd_rn(e1, e2));
  s = t;
}

__device__ __forceinline__ void two_sum1(float& s, float& c, float x) {
  const float t = __fadd_rn(s, x);
  const float bb = __fsub_rn(t, s);
  const float e = __fadd_rn(__fsub_rn(s, __fsub_rn(t, bb)), __fsub_rn(x, bb));
  c = __fadd_rn(c, e);
  s = t;
}

// Per-lane accumulator for the V output elements a feature lane owns.
template <typename T, int OP, int RHO, int V>
struct RowAcc {
  static constexpr int POL = Policy<T, OP, RHO>::value;
  using ExtT = typename std::conditional<POL == POL_EXT_D, double, T>::type;
  double acc[V];
  float s[V], c[V];
  ExtT cur[V];
  int32_t arg[V];
  double tsum;  // MP_AB only: sum of alpha_e * w over the edges this lane prefetched

  __device__ __forceinline__ void init() {
    tsum = 0.0;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      acc[k] = 0.0;
      s[k] = 0.f;
      c[k] = 0.f;
      cur[k] = (ExtT)ext_init<RHO == RHO_SUM ? RHO_MAX : RHO>();
      arg[k] = 0x7fffffff;
    }
  }

  // fold the compensated fp32 pair into fp64 (every <= 32 edges)
  __device__ __forceinline__ void fold() {
    if constexpr (POL == POL_COMP) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        acc[k] += (double)s[k];
        acc[k] += (double)c[k];
        s[k] = 0.f;
        c[k] = 0.f;
      }
    }
  }

  // add the message op(a, b) of one edge; masked lanes carry zeros for the
  // sum policies and are excluded by `ok` for extrema
  __device__ __forceinline__ void add(const T (&a)[V], const T (&b)[V], bool ok, int32_t e) {
    if constexpr (POL == POL_COMP) {
      if constexpr (V == 1) {
        const float x = (float)a[0], y = (float)b[0];
        if constexpr (OP == OP_COPY) {
          two_sum1(s[0], c[0], x);
        } else if constexpr (OP == OP_MUL || OP == OP_DOT) {
          two_sum_prod1(s[0], c[0], x, y);
        } else {  // ADD / SUB: the exact message is itself a TwoSum pair
          const float yy = OP == OP_SUB ? -y : y;
          const float t = __fadd_rn(x, yy);
          const float bb = __fsub_rn(t, x);
          const float r = __fadd_rn(__fsub_rn(x, __fsub_rn(t, bb)), __fsub_rn(yy, bb));
          two_sum1(s[0], c[0], t);
          c[0] = __fadd_rn(c[0], r);
        }
      } else {
#pragma unroll
        for (int k = 0; k < V; k += 2) {
          float2 S = f2(s[k], s[k + 1]), C = f2(c[k], c[k + 1]);
          const float2 x = f2((float)a[k], (float)a[k + 1]);
          if constexpr (OP == OP_COPY) {
            two_sum2(S, C, x);
          } else if constexpr (OP == OP_MUL || OP == OP_DOT) {
            two_sum_prod2(S, C, x, f2((float)b[k], (float)b[k + 1]));
          } else {
            float2 y = f2((float)b[k], (float)b[k + 1]);
            if constexpr (OP == OP_SUB) y = f2(-y.x, -y.y);
            // exact message x + y = t + r, then accumulate both parts
            const float2 t = __fadd2_rn(x, y);
            const float2 bb = fsub2(t, x);
            const float2 r = __fadd2_rn(fsub2(x, fsub2(t, bb)), fsub2(y, bb));
            two_sum2(S, C, t);
            C = __fadd2_rn(C, r);
          }
          s[k] = S.x; s[k + 1] = S.y;
          c[k] = C.x; c[k + 1] = C.y;
        }
      }
    } else if constexpr (POL == POL_DBL) {
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] += apply_op<OP>((double)a[k], (double)b[k]);
    } else {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        ExtT x;
        if constexpr (POL == POL_EXT_T && OP == OP_COPY) x = a[k];
        else x = (ExtT)apply_op<OP>((double)a[k], (double)b[k]);
        const bool better = (RHO == RHO_MAX) ? (x > cur[k]) : (x < cur[k]);
        const bool tie = (x == cur[k]) && (e < arg[k]);
        if (ok && better) cur[k] = x;
        if (ok && (better || tie)) arg[k] = e;
      }
    }
  }

  // combine with the partial of another lane/warp (fixed order => deterministic)
  __device__ __forceinline__ void merge(int k, double oacc, ExtT ocur, int32_t oarg) {
    if constexpr (POL == POL_COMP || POL == POL_DBL) {
      acc[k] += oacc;
    } else {
      const bool better = (RHO == RHO_MAX) ? (ocur > cur[k]) : (ocur < cur[k]);
      if (better) { cur[k] = ocur; arg[k] = oarg; }
      else if (ocur == cur[k] && oarg < arg[k]) arg[k] = oarg;
    }
  }

  __device__ __forceinline__ void combine_slots(int g_log2) {
    for (int off = 1 << g_log2; off < 32; off <<= 1) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if constexpr (POL == POL_COMP || POL == POL_DBL) {
          merge(k, __shfl_xor_sync(kFull, acc[k], off), ExtT(0), 0);
        } else {
          const ExtT oc = __shfl_xor_sync(kFull, cur[k], off);
          const int32_t oa = __shfl_xor_sync(kFull, arg[k], off);
          merge(k, 0.0, oc, oa);
        }
      }
    }
  }
};

template <typename T, int V>
__device__ __forceinline__ void load_hoisted(const RowOperand& o, int64_t row, int col, bool valid,
                                             T (&h)[V]) {
  const T* base = static_cast<const T*>(o.data) + (uint64_t)row * o.ld;
  if (o.bcast) {
    const T s = __ldg(base);
#pragma unroll
    for (int k = 0; k < V; ++k) h[k] = s;
  } else {
#pragma unroll
    for (int k = 0; k < V; ++k) h[k] = T(0);
    if (valid) load_vec<T, V>(base + col, h);
  }
}

template <typename T>
__device__ __forceinline__ T scalar_at(const RowOperand& o, uint32_t row) {
  return __ldg(static_cast<const T*>(o.data) + (uint64_t)row * o.ld);
}

// Branch-free vector gather: `colbase` already points at this lane's (clamped,
// in-bounds) column of row 0; masked lanes read row 0 and select zero.
template <typename T, int V>
__device__ __forceinline__ void gather_full(const T* colbase, uint32_t ld_bytes, uint32_t row,
                                            bool use, T (&out)[V]) {
  const T* p = reinterpret_cast<const T*>(reinterpret_cast<const char*>(colbase) +
                                          (uint64_t)(use ? row : 0u) * ld_bytes);
  load_vec<T, V>(p, out);
}

// Accumulate the messages of edges [pb, pe) of one row owned by this warp:
// 32-edge batches starting at pb + first, advancing by `stride` edges.
template <typename T, int OP, int RHO, int V, int MP, int U>
__device__ __forceinline__ void spmm_accumulate(const SpmmArgs& a, int64_t pb, int64_t pe,
                                                int64_t first, int64_t stride, int lane, int slot,
                                                int E, int col, bool valid, const T (&ha)[V],
                                                const T (&hb)[V], const T (&rc)[3],
                                                RowAcc<T, OP, RHO, V>& acc) {
  constexpr bool BIN = OP != OP_COPY;
  const int32_t* __restrict__ indices = a.indices;
  const int32_t* __restrict__ eids = a.eids;
  const bool need_eid = a.need_eid;
  // operand modes: compile-time unless MP_GEN
  const int lm = (MP == MP_GEN) ? a.lhs.mode : M_FULL;
  const int rm = !BIN ? M_NONE
                      : (MP == MP_FF ? M_FULL
                                     : ((MP == MP_FS || IsAttn<MP>::value) ? M_SCALAR
                                                    : (MP == MP_FH ? M_HOIST : a.rhs.mode)));
  const bool l_eid = a.lhs.from_eid, r_eid = a.rhs.from_eid;
  // lane column base pointers (clamped in-bounds for masked columns)
  const int ccol = valid ? col : 0;
  const T* lcol = static_cast<const T*>(a.lhs.data) + ccol;
  const T* rcol = BIN ? static_cast<const T*>(a.rhs.data) + ccol : nullptr;
  const uint32_t lld = a.lhs.ld * (uint32_t)sizeof(T);
  const uint32_t rld = a.rhs.ld * (uint32_t)sizeof(T);

  // two-deep index prefetch, one-deep per-edge scalar prefetch
  int64_t base = pb + first;
  int32_t nb0 = 0, eb0 = 0, nb1 = 0, eb1 = 0;
  if (base + lane < pe) {
    nb0 = __ldg(indices + base + lane);
    if (need_eid) eb0 = __ldg(eids + base + lane);
  }
  if (base + stride + lane < pe) {
    nb1 = __ldg(indices + base + stride + lane);
    if (need_eid) eb1 = __ldg(eids + base + stride + lane);
  }
  const bool l_pos = a.lhs.from_pos, r_pos = a.rhs.from_pos;
  auto lrow = [&](int32_t nb, int32_t eb, int64_t at) -> uint32_t {
    return l_pos ? (uint32_t)(at + lane) : (uint32_t)(l_eid ? eb : nb);
  };
  auto rrow = [&](int32_t nb, int32_t eb, int64_t at) -> uint32_t {
    return r_pos ? (uint32_t)(at + lane) : (uint32_t)(r_eid ? eb : nb);
  };
  T sa0 = T(0), sb0 = T(0);
  if (base + lane < pe) {
    if (lm == M_SCALAR) sa0 = scalar_at<T>(a.lhs, lrow(nb0, eb0, base));
    if (rm == M_SCALAR) sb0 = rhs_scalar<T, MP>(a, rrow(nb0, eb0, base), rc, acc.tsum);
  }
  int since_fold = 0;
  for (; base < pe; base += stride) {
    const int cnt = batch_count(pe - base);
    // prefetch: indices two batches ahead, scalars one batch ahead
    const int64_t b2 = base + 2 * stride;
    int32_t nb2 = 0, eb2 = 0;
    if (b2 + lane < pe) {
      nb2 = __ldg(indices + b2 + lane);
      if (need_eid) eb2 = __ldg(eids + b2 + lane);
    }
    T sa1 = T(0), sb1 = T(0);
    if (base + stride + lane < pe) {
      if (lm == M_SCALAR) sa1 = scalar_at<T>(a.lhs, lrow(nb1, eb1, base + stride));
      if (rm == M_SCALAR) sb1 = rhs_scalar<T, MP>(a, rrow(nb1, eb1, base + stride), rc, acc.tsum);
    }
    const uint32_t ra_lane = lrow(nb0, eb0, base);
    const uint32_t rb_lane = rrow(nb0, eb0, base);
    // One 32-edge batch. FULLB: all 32 edges present and E*U <= 32, so no
    // edge masking at all (lanes with !valid columns accumulate junk that is
    // never stored) - the common case inside heavy rows.
    auto pass = [&](auto full_tag) {
      constexpr bool FULLB = decltype(full_tag)::value;
#pragma unroll 1
      for (int t = 0; t < cnt; t += E * U) {
        T va[U][V];
        T vb[U][V];
        int32_t ee[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = t + slot + E * u;
          ok[u] = FULLB ? true : (j < cnt);
          const int sl = FULLB ? j : (j & 31);
          const bool use = FULLB ? true : (ok[u] && valid);
          ee[u] = (RHO != RHO_SUM) ? __shfl_sync(kFull, eb0, sl) : 0;
          // lhs
          if (lm == M_FULL) {
            gather_full<T, V>(lcol, lld, __shfl_sync(kFull, ra_lane, sl), use, va[u]);
          } else {
            const T sa = (lm == M_SCALAR) ? __shfl_sync(kFull, sa0, sl) : T(0);
#pragma unroll
            for (int k = 0; k < V; ++k) va[u][k] = (lm == M_SCALAR) ? sa : ha[k];
          }
          // rhs
          if (rm == M_FULL) {
            gather_full<T, V>(rcol, rld, __shfl_sync(kFull, rb_lane, sl), use, vb[u]);
          } else if (rm == M_NONE) {
#pragma unroll
            for (int k = 0; k < V; ++k) vb[u][k] = T(0);
          } else {
            const T sb = (rm == M_SCALAR) ? __shfl_sync(kFull, sb0, sl) : T(0);
#pragma unroll
            for (int k = 0; k < V; ++k) vb[u][k] = (rm == M_SCALAR) ? sb : hb[k];
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if constexpr (OP == OP_DIV) {
            bool zero = false;
#pragma unroll
            for (int k = 0; k < V; ++k) zero |= valid && (vb[u][k] == T(0));
            if (ok[u] && zero) atomicMin(a.err_pos, (int32_t)(base + t + slot + E * u));
          }
          if constexpr (!FULLB) {
            // masked lanes contribute exactly nothing: a = 0 and b = 0 (1 for div)
            const bool use = ok[u] && valid;
#pragma unroll
            for (int k = 0; k < V; ++k) {
              va[u][k] = use ? va[u][k] : T(0);
              vb[u][k] = use ? vb[u][k] : (OP == OP_DIV ? T(1) : T(0));
            }
          }
          acc.add(va[u], vb[u], ok[u], ee[u]);
        }
      }
    };
    if (cnt == 32 && E * U <= 32) pass(std::true_type{});
    else pass(std::false_type{});
    if (++since_fold >= E) {  // each slot has seen <= 32 edges since the last fold
      acc.fold();
      since_fold = 0;
    }
    nb0 = nb1; eb0 = eb1; nb1 = nb2; eb1 = eb2;
    sa0 = sa1; sb0 = sb1;
  }
  acc.fold();
}

// Software-pipelined accumulate, one float4 per lane: G = 2^GL lanes per
// edge (64 / 128 / 256 B rows for GL = 2 / 3 / 4), E = 32 / G edge slots per
// warp step. spmm_accumulate issues a burst of U gathers, waits for all of
// them and then runs the compensated sums, so a warp has nothing in flight
// while it computes. Here every lane keeps a ring of NB float4 registers:
// step t consumes ring slot t % NB and immediately refills it with the gather
// of step t + NB (taken from the next iteration's neighbour ids near the end
// of an iteration), so gathers stay in flight through the arithmetic.
// An iteration covers R 32-edge index registers (R = 1 for 256 / 128 B rows,
// 2 for 64 B rows): T = R * G steps of E edges.
// For GL = 4 the edge order per slot and the fold points (every 32 edges per
// slot) equal spmm_accumulate's, so the sums are bit-identical to it.
// Operands: lhs gathered by neighbour id; rhs none (copy), a per-edge scalar
// addressed by position or neighbour id, or the recomputed attention weight
// (MP_AF / MP_AB) - no edge ids needed.
// ring depth (float4 registers per lane) and index registers per iteration
// of the pipelined accumulate, by log2 of the lanes per edge
template <int GL>
struct PipeR {
  static constexpr int value = (1 << GL) >= 8 ? 1 : 8 / (1 << GL);
};
template <int GL>
struct PipeNB {
  static constexpr int value = GL >= 4 ? GMP_PIPE_NB : GMP_PIPE_NB_NARROW;
};

template <int OP, int RHO, int MP, int GL, int NB>
__device__ __forceinline__ void spmm_accumulate_pipe(const SpmmArgs& a, int64_t pb, int64_t pe,
                                                     int64_t first, int64_t stride, int lane,
                                                     int slot, int col, bool valid,
                                                     const float (&rc)[3],
                                                     RowAcc<float, OP, RHO, 4>& acc) {
  constexpr int G = 1 << GL, E = 32 >> GL;
  constexpr int R = G >= 8 ? 1 : 8 / G;  // 32-edge index registers per iteration
  constexpr int T = R * G;               // steps per iteration
  constexpr int FOLD = 32 / T > 0 ? 32 / T : 1;  // iterations per 32 edges of a slot
  static_assert(T % NB == 0 && NB <= T, "ring slots must be compile-time across an iteration");
  constexpr bool SC = OP != OP_COPY;  // per-edge scalar rhs
  constexpr bool EXT = RHO != RHO_SUM;  // max / min: edge ids for the arg
  // 32-bit offsets relative to the iteration start (a row has < 2^31 edges)
  if (pb + first >= pe) return;
  const int32_t* __restrict__ ip = a.indices + pb + first;
  const int32_t* __restrict__ ep = a.eids + pb + first;
  int32_t left = (int32_t)(pe - pb - first);  // edges from the current iteration start on
  const int32_t step = (int32_t)stride;
  const float* lcol = static_cast<const float*>(a.lhs.data) + (valid ? col : 0);
  const uint32_t lld = a.lhs.ld * (uint32_t)sizeof(float);
  const bool r_pos = a.rhs.from_pos;
  // lane L of index register q holds edge 32 q + E (L & (G-1)) + (L >> GL):
  // slot s reads edge 32 q + E k + s with a width-G shuffle from lane k (an
  // immediate lane, no per-step lane arithmetic); the loads stay coalesced
  const int pl = E * (lane & (G - 1)) + (lane >> GL);
  // index of edge pl of register q at iteration offset o (0 past the row:
  // row 0, loaded but never summed)
  auto ld_idx = [&](int32_t o) -> int32_t { return pl + o < left ? __ldg(ip + o + pl) : 0; };
  auto ld_eid = [&](int32_t o) -> int32_t {
    if constexpr (EXT) return pl + o < left ? __ldg(ep + o + pl) : 0;
    return 0;
  };
  auto ld_sc = [&](int32_t o, int32_t nb) -> float {
    if constexpr (SC) {
      if (pl + o < left) {
        const int64_t q = (ip - a.indices) + o + pl;  // CSC position
        return rhs_scalar<float, MP>(a, r_pos ? (uint32_t)q : (uint32_t)nb, rc, acc.tsum);
      }
    }
    return 0.f;
  };
  auto gather = [&](int32_t nbreg, int k) -> float4 {
    const uint32_t r = (uint32_t)__shfl_sync(kFull, nbreg, k, G);
    return __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const char*>(lcol) +
                                                 (uint64_t)r * lld));
  };
  int32_t cur[R], nxt[R], ecur[R], enxt[R];
  float wcur[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    cur[q] = ld_idx(32 * q);
    nxt[q] = ld_idx(step + 32 * q);
    ecur[q] = ld_eid(32 * q);
    enxt[q] = ld_eid(step + 32 * q);
  }
#pragma unroll
  for (int q = 0; q < R; ++q) wcur[q] = ld_sc(32 * q, cur[q]);
  float4 buf[NB];
#pragma unroll
  for (int t = 0; t < NB; ++t) buf[t] = gather(cur[t / G], t % G);

  for (int b = 0;; ++b) {
    int32_t nn[R], enn[R];
    float wnxt[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      nn[q] = ld_idx(2 * step + 32 * q);
      enn[q] = ld_eid(2 * step + 32 * q);
    }
#pragma unroll
    for (int q = 0; q < R; ++q) wnxt[q] = ld_sc(step + 32 * q, nxt[q]);
    auto steps = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int q = t / G, k = t % G;
        const bool use = FULL || 32 * q + E * k + slot < left;
        const float4 x = buf[t % NB];
        float va[4] = {x.x, x.y, x.z, x.w};
        float vb[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (SC) {
          const float w = __shfl_sync(kFull, wcur[q], k, G);
#pragma unroll
          for (int c = 0; c < 4; ++c) vb[c] = w;
        }
        if constexpr (!FULL && !EXT) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            va[c] = use ? va[c] : 0.f;
            vb[c] = use ? vb[c] : 0.f;
          }
        }
        const int32_t e = EXT ? __shfl_sync(kFull, ecur[q], k, G) : 0;
        // refill this ring slot with step t + NB (the next iteration's ids
        // near the end; past the last iteration they are 0: row 0, unused)
        const int tn = t + NB;
        buf[t % NB] = tn < T ? gather(cur[tn / G], tn % G) : gather(nxt[(tn - T) / G], (tn - T) % G);
        acc.add(va, vb, use, e);  // extrema: masked edges excluded by `use`
      }
    };
    if (left >= 32 * R) steps(std::true_type{});
    else steps(std::false_type{});
    if ((b + 1) % FOLD == 0) acc.fold();
    left -= step;
    if (left <= 0) break;
    ip += step;
    ep += step;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      cur[q] = nxt[q];
      nxt[q] = nn[q];
      ecur[q] = enxt[q];
      enxt[q] = enn[q];
      wcur[q] = wnxt[q];
    }
  }
  acc.fold();
}

// Narrow rows (E * U > 32 edge slots per warp step, i.e. d < 16): a 32-edge
// batch gives each lane fewer than U gathers, so edge ids are staged in
// shared memory kChunkE at a time (coalesced, one chunk ahead) and every
// lane keeps U independent gathers in flight.
constexpr int kChunkE = 256;

template <typename T, int OP, int RHO, int V, int MP, int U>
__device__ __forceinline__ void spmm_accumulate_chunked(
    const SpmmArgs& a, int64_t pb, int64_t pe, int64_t first, int64_t stride, int lane, int slot,
    int E, int col, bool valid, const T (&ha)[V], const T (&hb)[V], const T (&rc)[3],
    int32_t* sidx, int32_t* seid, RowAcc<T, OP, RHO, V>& acc) {
  constexpr bool BIN = OP != OP_COPY;
  constexpr int B = kChunkE / 32;
  const int lm = (MP == MP_GEN) ? a.lhs.mode : M_FULL;
  const int rm = !BIN ? M_NONE
                      : (MP == MP_FF ? M_FULL
                                     : ((MP == MP_FS || IsAttn<MP>::value) ? M_SCALAR
                                                    : (MP == MP_FH ? M_HOIST : a.rhs.mode)));
  const bool need_eid = a.need_eid;
  const int ccol = valid ? col : 0;
  const T* lcol = static_cast<const T*>(a.lhs.data) + ccol;
  const T* rcol = BIN ? static_cast<const T*>(a.rhs.data) + ccol : nullptr;
  const uint32_t lld = a.lhs.ld * (uint32_t)sizeof(T);
  const uint32_t rld = a.rhs.ld * (uint32_t)sizeof(T);
  int32_t pn[B], pe_[B];
  auto fetch = [&](int64_t cb) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const int64_t q = cb + i * 32 + lane;
      pn[i] = q < pe ? __ldg(a.indices + q) : 0;
      pe_[i] = (q < pe && need_eid) ? __ldg(a.eids + q) : 0;
    }
  };
  fetch(pb + first);
  int since_fold = 0;
  for (int64_t cb = pb + first; cb < pe; cb += stride) {
    const int cnt = (int)min((int64_t)kChunkE, pe - cb);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < B; ++i) {
      sidx[i * 32 + lane] = pn[i];
      if constexpr (IsAttn<MP>::value && sizeof(T) == 4) {
        // the attention weight of each staged edge, computed once per edge
        // (not once per feature lane) and kept in the edge-id slot
        float al = 0.f;
        if (cb + i * 32 + lane < pe) al = rhs_scalar<T, MP>(a, (uint32_t)pn[i], rc, acc.tsum);
        seid[i * 32 + lane] = __float_as_int(al);
      } else {
        seid[i * 32 + lane] = pe_[i];
      }
    }
    __syncwarp();
    fetch(cb + stride);
#pragma unroll 1
    for (int t = 0; t < cnt; t += E * U) {
      T va[U][V], vb[U][V];
      int32_t ee[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = t + slot + E * u;
        ok[u] = j < cnt;
        const int jj = ok[u] ? j : 0;
        const int32_t nb = sidx[jj];
        const int32_t eb = seid[jj];
        ee[u] = eb;
        const int64_t p = cb + jj;
        const uint32_t ra = a.lhs.from_pos ? (uint32_t)p : (uint32_t)(a.lhs.from_eid ? eb : nb);
        const uint32_t rb = a.rhs.from_pos ? (uint32_t)p : (uint32_t)(a.rhs.from_eid ? eb : nb);
        const bool use = ok[u] && valid;
        if (lm == M_FULL) {
          gather_full<T, V>(lcol, lld, ra, use, va[u]);
        } else {
          const T sa = (lm == M_SCALAR && ok[u]) ? scalar_at<T>(a.lhs, ra) : T(0);
#pragma unroll
          for (int k = 0; k < V; ++k) va[u][k] = (lm == M_SCALAR) ? sa : ha[k];
        }
        if (rm == M_FULL) {
          gather_full<T, V>(rcol, rld, rb, use, vb[u]);
        } else if (rm == M_NONE) {
#pragma unroll
          for (int k = 0; k < V; ++k) vb[u][k] = T(0);
        } else {
          T sb;
          if constexpr (IsAttn<MP>::value && sizeof(T) == 4) {
            sb = __int_as_float(eb);  // staged attention weight
          } else {
            double dummy = 0.0;
            sb = (rm == M_SCALAR && ok[u]) ? rhs_scalar<T, MP>(a, rb, rc, dummy) : T(0);
          }
#pragma unroll
          for (int k = 0; k < V; ++k) vb[u][k] = (rm == M_SCALAR) ? sb : hb[k];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool use = ok[u] && valid;
        if constexpr (OP == OP_DIV) {
          bool zero = false;
#pragma unroll
          for (int k = 0; k < V; ++k) zero |= valid && (vb[u][k] == T(0));
          if (ok[u] && zero) atomicMin(a.err_pos, (int32_t)(cb + t + slot + E * u));
        }
#pragma unroll
        for (int k = 0; k < V; ++k) {
          va[u][k] = use ? va[u][k] : T(0);
          vb[u][k] = use ? vb[u][k] : (OP == OP_DIV ? T(1) : T(0));
        }
        acc.add(va[u], vb[u], ok[u], ee[u]);
      }
    }
    since_fold += (cnt + E - 1) / E;  // edges each slot added from this chunk
    if (since_fold + kChunkE / E > 32) {  // fold before a slot could pass 32 edges
      acc.fold();
      since_fold = 0;
    }
  }
  acc.fold();
}

// Short rows (<= light threshold edges): each lane group (slot) of the warp
// owns one row and walks its edges itself - E rows per warp, so a warp is not
// tied up by a row of a handful of edges. Rows arrive degree-sorted, so the
// slots of a warp have near-equal lengths.
template <typename T, int OP, int RHO, int V, int MP, int U>
__device__ __forceinline__ void spmm_accumulate_slot(const SpmmArgs& a, int64_t pb, int64_t pe,
                                                     int col, bool valid, const T (&ha)[V],
                                                     const T (&hb)[V], const T (&rc)[3],
                                                     RowAcc<T, OP, RHO, V>& acc) {
  constexpr bool BIN = OP != OP_COPY;
  const int lm = (MP == MP_GEN) ? a.lhs.mode : M_FULL;
  const int rm = !BIN ? M_NONE
                      : (MP == MP_FF ? M_FULL
                                     : ((MP == MP_FS || IsAttn<MP>::value) ? M_SCALAR
                                                    : (MP == MP_FH ? M_HOIST : a.rhs.mode)));
  const bool need_eid = a.need_eid;
  const int ccol = valid ? col : 0;
  const T* lcol = static_cast<const T*>(a.lhs.data) + ccol;
  const T* rcol = BIN ? static_cast<const T*>(a.rhs.data) + ccol : nullptr;
  const uint32_t lld = a.lhs.ld * (uint32_t)sizeof(T);
  const uint32_t rld = a.rhs.ld * (uint32_t)sizeof(T);
  const int cnt = (int)(pe - pb);
  const int max_cnt = __reduce_max_sync(kFull, (unsigned)cnt);
  // every lane of a slot computes the same edge's weight; one lane sums alpha*w
  const bool t_owner = ((threadIdx.x & 31) & ((1 << a.g_log2) - 1)) == 0;
  for (int t = 0; t < max_cnt; t += U) {
    T va[U][V], vb[U][V];
    int32_t ee[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = t + u;
      ok[u] = j < cnt;
      const int64_t p = pb + (ok[u] ? j : 0);
      const int32_t nb = ok[u] ? __ldg(a.indices + p) : 0;
      const int32_t eb = (ok[u] && need_eid) ? __ldg(a.eids + p) : 0;
      ee[u] = eb;
      const uint32_t ra = a.lhs.from_pos ? (uint32_t)p : (uint32_t)(a.lhs.from_eid ? eb : nb);
      const uint32_t rb = a.rhs.from_pos ? (uint32_t)p : (uint32_t)(a.rhs.from_eid ? eb : nb);
      const bool use = ok[u] && valid;
      if (lm == M_FULL) {
        gather_full<T, V>(lcol, lld, ra, use, va[u]);
      } else {
        const T sa = (lm == M_SCALAR && ok[u]) ? scalar_at<T>(a.lhs, ra) : T(0);
#pragma unroll
        for (int k = 0; k < V; ++k) va[u][k] = (lm == M_SCALAR) ? sa : ha[k];
      }
      if (rm == M_FULL) {
        gather_full<T, V>(rcol, rld, rb, use, vb[u]);
      } else if (rm == M_NONE) {
#pragma unroll
        for (int k = 0; k < V; ++k) vb[u][k] = T(0);
      } else {
        double tdummy = 0.0;
        const T sb = (rm == M_SCALAR && ok[u])
                         ? rhs_scalar<T, MP>(a, rb, rc, t_owner ? acc.tsum : tdummy)
                         : T(0);
#pragma unroll
        for (int k = 0; k < V; ++k) vb[u][k] = (rm == M_SCALAR) ? sb : hb[k];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool use = ok[u] && valid;
      if constexpr (OP == OP_DIV) {
        bool zero = false;
#pragma unroll
        for (int k = 0; k < V; ++k) zero |= valid && (vb[u][k] == T(0));
        if (ok[u] && zero) atomicMin(a.err_pos, (int32_t)(pb + t + u));
      }
#pragma unroll
      for (int k = 0; k < V; ++k) {
        va[u][k] = use ? va[u][k] : T(0);
        vb[u][k] = use ? vb[u][k] : (OP == OP_DIV ? T(1) : T(0));
      }
      acc.add(va[u], vb[u], ok[u], ee[u]);
    }
  }
  acc.fold();
}

template <typename T, int OP, int RHO, int V>
__device__ __forceinline__ void write_row(const SpmmArgs& a, int64_t row, int64_t deg, int col,
                                          bool valid, const RowAcc<T, OP, RHO, V>& acc) {
  if constexpr (OP == OP_DOT) {
    // dot message, sum/mean: the row sum of products over every column the
    // lane group covers (one tile), reduced across the group's lanes
    double v = 0.0;
    if (valid)
#pragma unroll
      for (int k = 0; k < V; ++k) v += acc.acc[k];
    const unsigned mask = __activemask();
    for (int off = 1; off < (1 << a.g_log2); off <<= 1) v += __shfl_xor_sync(mask, v, off);
    if ((threadIdx.x & ((1 << a.g_log2) - 1)) == 0) {
      if (a.mean && deg > 0) v = v / (double)deg;
      static_cast<T*>(a.Z)[row * a.ldz] = (T)v;
    }
    return;
  }
  if (!valid) return;
  T* z = static_cast<T*>(a.Z) + row * a.ldz;
  T out[V];
  if constexpr (RHO == RHO_SUM) {
    // columns of this lane's vector inside the output: < V only for the last
    // vector of a width that is not a multiple of V (tail-masked float4s)
    const int nv = min(V, a.d_out - col);
    int64_t dg = deg;
    double vs[V];
#pragma unroll
    for (int k = 0; k < V; ++k) vs[k] = acc.acc[k];
    if (a.acc64) {
      double* ap = a.acc64 + row * a.ldacc + col;
      if (a.acc_mode & kAccRead) {
#pragma unroll
        for (int k = 0; k < V; ++k)
          if (k < nv) vs[k] += ap[k];
      }
      if (a.acc_mode & kAccStore) {
#pragma unroll
        for (int k = 0; k < V; ++k)
          if (k < nv) ap[k] = vs[k];
      }
      if (!(a.acc_mode & kAccZ)) return;
      if (a.deg_full) dg = a.deg_full[row];
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double v = vs[k];
      if (a.mean && dg > 0) v = v / (double)dg;  // kernels.py:719-722
      out[k] = (T)v;
    }
    if (nv < V || a.z_split == 2) {  // element stores (tail, or 4 B-aligned rows)
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (k < nv) z[col + k] = out[k];
      return;
    }
    if constexpr (V == 4) {
      if (a.z_split) {  // e.g. a 64-column tile written straight into Z with ld 602
        const T lo[2] = {out[0], out[1]}, hi[2] = {out[2], out[3]};
        store_vec<T, 2>(z + col, lo);
        store_vec<T, 2>(z + col + 2, hi);
        return;
      }
    }
    store_vec<T, V>(z + col, out);
  } else {
    int32_t ar[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      out[k] = deg > 0 ? (T)acc.cur[k] : T(0);
      ar[k] = deg > 0 ? acc.arg[k] : -1;
    }
    store_vec<T, V>(z + col, out);
    store_arg<V>(a.arg + row * (int64_t)a.d_out + col, ar);
  }
}

template <int V>
struct Unroll {
  static constexpr int value = 8;  // gathers in flight per lane (measured: 8 beats 4 for V=4 too)
};

// NARROW: rows use few lanes (E > 1 and E*U > 32, i.e. d < 16): short rows
// share a warp and longer rows stage edge ids in shared memory. Wide kernels
// (every d >= 16 with V=4, and all fp64 launches) compile without those paths
// so their main loop is scheduled on its own.
template <typename T, int OP, int RHO, int V, int MP, bool NARROW, int PGL = 0>
__global__ void __launch_bounds__(kWarpsPerCta * 32, PGL ? GMP_PIPE_MIN_BLOCKS : GMP_ROW_MIN_BLOCKS)
spmm_rows_kernel(const SpmmArgs a) {
  using Acc = RowAcc<T, OP, RHO, V>;
  using ExtT = typename Acc::ExtT;
  // run-time operand modes and max/min of binary messages carry more live
  // state per gather (fp64 messages, both operands, arg): 4 gathers in
  // flight per lane keeps them in registers (op sweep: div 1.3-2.4x, binary
  // max/min 1.1-1.4x faster than with 8, which spilled); the narrow / wide
  // launch split still follows Unroll<V>
  constexpr int U = (MP == MP_GEN || (RHO != RHO_SUM && OP != OP_COPY)) ? 4 : Unroll<V>::value;
  constexpr int kCols = 32 * V;  // widest tile one warp covers
  __shared__ double s_acc[RHO == RHO_SUM ? kWarpsPerCta : 1][kCols];
  __shared__ ExtT s_cur[RHO == RHO_SUM ? 1 : kWarpsPerCta][kCols];
  __shared__ int32_t s_arg[RHO == RHO_SUM ? 1 : kWarpsPerCta][kCols];
  extern __shared__ int32_t s_chunk[];  // [2][kWarpsPerCta][kChunkE], only for chunked launches

  const int64_t bid = blockIdx.x;
  const int tile = (int)(bid / a.blocks_per_tile);
  const int64_t local = bid - (int64_t)tile * a.blocks_per_tile;
  const int c0 = tile * a.tile_cols;
  const int c1 = min(a.d_out, c0 + a.tile_cols);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int G = 1 << a.g_log2;
  const int E = 32 >> a.g_log2;
  const int slot = lane >> a.g_log2;
  const int gl = lane & (G - 1);
  // heavy rows: `cl` CTAs each (one thread-block cluster, rank crank)
  const int ncl = a.cluster > 1 ? a.cluster : 1;
  const int64_t heavy_blocks = a.n_heavy * ncl;
  const bool heavy = local < heavy_blocks;  // block-uniform
  const int crank = heavy ? (int)(local % ncl) : 0;
  // light rows share a warp, one per lane group (NARROW kernels and the
  // pipelined ones: PGL = log2 of the lanes per edge)
  constexpr bool PIPE = PGL != 0;
  const bool light = (NARROW || PIPE) && local >= heavy_blocks + a.medium_blocks;  // block-uniform

  int64_t row;
  if (heavy) {
    row = a.order[local / ncl];
  } else if (!light) {
    const int64_t r = a.n_heavy + (local - heavy_blocks) * kWarpsPerCta + warp;
    if (r >= a.n_medium) return;  // warp rows never synchronise the CTA
    row = a.order ? (int64_t)a.order[r] : r;
  } else {
    const int64_t r = a.n_medium +
                      ((local - heavy_blocks - a.medium_blocks) * kWarpsPerCta + warp) * E + slot;
    if (__all_sync(kFull, r >= a.n_rows)) return;
    row = r < a.n_rows ? (a.order ? (int64_t)a.order[r] : r) : -1;  // -1: idle slot
  }
  const int64_t pb = row >= 0 ? a.indptr[row] : 0;
  const int64_t pe = row >= 0 ? a.indptr[row + 1] : 0;
  const int64_t deg = pe - pb;
  const int col = c0 + gl * V;
  const bool valid = col < c1;

  T ha[V], hb[V];
#pragma unroll
  for (int k = 0; k < V; ++k) ha[k] = hb[k] = T(0);
  if (MP == MP_GEN && a.lhs.mode == M_HOIST && deg > 0) load_hoisted<T, V>(a.lhs, row, col, valid, ha);
  if (OP != OP_COPY && (MP == MP_FH || (MP == MP_GEN && a.rhs.mode == M_HOIST)) && deg > 0) {
    load_hoisted<T, V>(a.rhs, row, col, valid, hb);
    if constexpr (OP == OP_DIV) {
      bool zero = false;
#pragma unroll
      for (int k = 0; k < V; ++k) zero |= valid && (hb[k] == T(0));
      if (zero) atomicMin(a.err_pos, (int32_t)pb);
    }
  }

  T rc[3] = {T(0), T(0), T(0)};
  if constexpr (IsAttn<MP>::value) {
    if (deg > 0) attn_row_consts<T, MP>(a, row, rc);
  }

  Acc acc;
  acc.init();
  // copy of the destination's own row (copy_lhs(dst) / copy_rhs(dst)): every
  // message of the row is Y[v], so sum = deg * Y[v] - exact in fp64 for
  // deg < 2^29, equal to the reference's fp64 accumulation - and no edge
  // needs to be read (one writer per row: slot 0, warp 0 of a heavy CTA)
  bool row_const = false;
  if constexpr (OP == OP_COPY && RHO == RHO_SUM && MP == MP_GEN) {
    if (a.lhs.mode == M_HOIST) {
      row_const = true;
      const bool own = NARROW && light ? true
                                       : (slot == 0 && (!heavy || (warp == 0 && crank == 0)));
      if (own && deg > 0) {
#pragma unroll
        for (int k = 0; k < V; ++k) acc.acc[k] = (double)deg * (double)ha[k];
      }
    }
  }
  if constexpr (PIPE) {
    if (light) {
      spmm_accumulate_slot<T, OP, RHO, V, MP, GMP_PIPE_NB>(a, pb, pe, col, valid, ha, hb, rc, acc);
      if (row < 0) return;
      if constexpr (MP == MP_AB) {
        if (a.attn_t && tile == 0 && gl == 0) a.attn_t[row] = acc.tsum;
      }
      if (a.counts && tile == 0 && gl == 0) a.counts[row] = deg;
      write_row<T, OP, RHO, V>(a, row, deg, col, valid, acc);
      return;
    }
  }
  if (row_const) {
    if constexpr (NARROW) {
      if (light) {
        if (row < 0) return;
        if (a.counts && tile == 0 && gl == 0) a.counts[row] = deg;
        write_row<T, OP, RHO, V>(a, row, deg, col, valid, acc);
        return;
      }
    }
  } else if constexpr (NARROW) {
    if (light) {
      spmm_accumulate_slot<T, OP, RHO, V, MP, U>(a, pb, pe, col, valid, ha, hb, rc, acc);
      if (row < 0) return;
      if constexpr (MP == MP_AB) {
        if (a.attn_t && tile == 0 && gl == 0) a.attn_t[row] = acc.tsum;
      }
      if (a.counts && tile == 0 && gl == 0) a.counts[row] = deg;
      write_row<T, OP, RHO, V>(a, row, deg, col, valid, acc);
      return;
    }
    spmm_accumulate_chunked<T, OP, RHO, V, MP, U>(
        a, pb, pe, heavy ? ((int64_t)crank * kWarpsPerCta + warp) * kChunkE : 0,
        heavy ? (int64_t)kChunkE * kWarpsPerCta * ncl : kChunkE, lane, slot, E, col, valid, ha, hb, rc,
        s_chunk + warp * kChunkE, s_chunk + (kWarpsPerCta + warp) * kChunkE, acc);
  } else if (row_const) {
    // nothing to accumulate
  } else if (heavy) {
    if constexpr (PIPE)
      spmm_accumulate_pipe<OP, RHO, MP, PGL, PipeNB<PGL>::value>(
          a, pb, pe, ((int64_t)crank * kWarpsPerCta + warp) * 32 * PipeR<PGL>::value,
          (int64_t)32 * PipeR<PGL>::value * kWarpsPerCta * ncl, lane, slot, col, valid, rc, acc);
    else
      spmm_accumulate<T, OP, RHO, V, MP, U>(a, pb, pe, ((int64_t)crank * kWarpsPerCta + warp) * 32,
                                            (int64_t)32 * kWarpsPerCta * ncl, lane, slot, E, col,
                                            valid, ha, hb, rc, acc);
  } else {
    if constexpr (PIPE)
      spmm_accumulate_pipe<OP, RHO, MP, PGL, PipeNB<PGL>::value>(a, pb, pe, 0, 32 * PipeR<PGL>::value,
                                                             lane, slot, col, valid, rc, acc);
    else
      spmm_accumulate<T, OP, RHO, V, MP, U>(a, pb, pe, 0, 32, lane, slot, E, col, valid, ha, hb,
                                            rc, acc);
  }
  acc.combine_slots(a.g_log2);
  if constexpr (MP == MP_AB) {  // every lane summed alpha*w of its own edges
    for (int off = 16; off > 0; off >>= 1) acc.tsum += __shfl_xor_sync(kFull, acc.tsum, off);
  }

  if (a.counts && tile == 0 && ((heavy && crank == 0 && threadIdx.x == 0) || (!heavy && lane == 0)))
    a.counts[row] = deg;

  if (!heavy) {
    if (slot == 0) write_row<T, OP, RHO, V>(a, row, deg, col, valid, acc);
    if constexpr (MP == MP_AB) {
      if (a.attn_t && tile == 0 && lane == 0) a.attn_t[row] = acc.tsum;
    }
    return;
  }
  __shared__ double s_t[IsAttn<MP>::value ? kWarpsPerCta : 1];
  if constexpr (MP == MP_AB) {
    if (lane == 0) s_t[warp] = acc.tsum;
  }
  // CTA mode: merge the warp partials in warp order through shared memory.
  if (slot == 0) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int cl = gl * V + k;
      if constexpr (RHO == RHO_SUM) {
        s_acc[warp][cl] = acc.acc[k];
      } else {
        s_cur[warp][cl] = acc.cur[k];
        s_arg[warp][cl] = acc.arg[k];
      }
    }
  }
  __syncthreads();
  if (warp == 0 && slot == 0) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int cl = gl * V + k;
      if constexpr (RHO == RHO_SUM) {
        double v = s_acc[0][cl];
        for (int w = 1; w < kWarpsPerCta; ++w) v += s_acc[w][cl];
        acc.acc[k] = v;
      } else {
        acc.cur[k] = s_cur[0][cl];
        acc.arg[k] = s_arg[0][cl];
        for (int w = 1; w < kWarpsPerCta; ++w) acc.merge(k, 0.0, s_cur[w][cl], s_arg[w][cl]);
      }
    }
    double t = 0.0;
    if constexpr (MP == MP_AB) {
      if (lane == 0) {
        t = s_t[0];
        for (int w = 1; w < kWarpsPerCta; ++w) t += s_t[w];
      }
    }
    if (ncl == 1) {
      write_row<T, OP, RHO, V>(a, row, deg, col, valid, acc);
      if constexpr (MP == MP_AB) {
        if (a.attn_t && tile == 0 && lane == 0) a.attn_t[row] = t;
      }
    } else {
      // this CTA's partial of the row, for the cluster merge below
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int cl = gl * V + k;
        if constexpr (RHO == RHO_SUM) {
          s_acc[0][cl] = acc.acc[k];
        } else {
          s_cur[0][cl] = acc.cur[k];
          s_arg[0][cl] = acc.arg[k];
        }
      }
      if constexpr (MP == MP_AB) {
        if (lane == 0) s_t[0] = t;
      }
    }
  }
  if (ncl > 1) {
    // the row's CTAs form one cluster: rank 0 reads the other ranks'
    // partials from their shared memory (DSMEM) and merges them in rank order
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    if (crank == 0 && warp == 0 && slot == 0) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int cl = gl * V + k;
        for (int r = 1; r < ncl; ++r) {
          if constexpr (RHO == RHO_SUM) {
            acc.acc[k] += *cluster.map_shared_rank(&s_acc[0][cl], r);
          } else {
            acc.merge(k, 0.0, *cluster.map_shared_rank(&s_cur[0][cl], r),
                      *cluster.map_shared_rank(&s_arg[0][cl], r));
          }
        }
      }
      write_row<T, OP, RHO, V>(a, row, deg, col, valid, acc);
      if constexpr (MP == MP_AB) {
        if (a.attn_t && tile == 0 && lane == 0) {
          double t = s_t[0];
          for (int r = 1; r < ncl; ++r) t += *cluster.map_shared_rank(&s_t[0], r);
          a.attn_t[row] = t;
        }
      }
    }
    cluster.sync();  // the partials stay readable until rank 0 is done
  }
}

template <int V>
__host__ __device__ constexpr bool narrow_launch(int g_log2) {
  return (32 >> g_log2) > 1 && (32 >> g_log2) * Unroll<V>::value > 32;
}

// a.cluster > 1: launched as thread-block clusters of a.cluster CTAs (grid a
// multiple of it) so a heavy row's CTAs can merge through DSMEM
template <typename Kern>
cudaError_t launch_rows_cfg(Kern kern, const SpmmArgs& a, int64_t grid, size_t smem,
                            cudaStream_t s) {
  if (a.cluster <= 1) {
    kern<<<(unsigned)grid, kWarpsPerCta * 32, smem, s>>>(a);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid, 1, 1);
  cfg.blockDim = dim3(kWarpsPerCta * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// fp32 launches that take the pipelined gather ring (spmm_accumulate_pipe):
// sum / mean of copy_u, u_mul_e (per-edge scalar) or the fused GAT attention
// (MP_AF / MP_AB) with one float4 per lane and 4, 8 or 16 lanes per edge
// (64 / 128 / 256 B rows), no edge ids. The host sizes the grid by the same
// predicate (light rows several per warp). GMP_NO_PIPE=1 disables it.
// lhs_by_nb: the gathered operand is keyed by the neighbour (source) id -
// the pipelined ring gathers rows by `indices` only (an edge-keyed copy
// operand, max / min of copy_lhs(edge), takes the row kernel)
inline bool pipe_launch(int V, int rho, int op, int mp, int g_log2, int need_eid, bool lhs_by_nb) {
  static const bool off = getenv("GMP_NO_PIPE") != nullptr;
  if (off || !lhs_by_nb || V != 4 || g_log2 < 2 || g_log2 > 4) return false;
  if (rho != RHO_SUM)  // max / min of copy_u: edge ids only for the arg
    return op == OP_COPY && mp == MP_F;
  return !need_eid && ((op == OP_COPY && mp == MP_F) ||
                       (op == OP_MUL && (mp == MP_FS || mp == MP_AF || mp == MP_AB)));
}

template <typename T, int OP, int RHO, int V, int MP>
cudaError_t launch_spmm_rows_t(const SpmmArgs& a, int64_t grid, cudaStream_t s) {
  if constexpr (sizeof(T) == 4 && V == 4 &&
                ((OP == OP_COPY && MP == MP_F) ||
                 (RHO == RHO_SUM && OP == OP_MUL &&
                  (MP == MP_FS || MP == MP_AF || MP == MP_AB)))) {
    if (pipe_launch(V, RHO, OP, MP, a.g_log2, a.need_eid, !a.lhs.from_eid && !a.lhs.from_pos)) {
      if (a.g_log2 == 4)
        return launch_rows_cfg(spmm_rows_kernel<T, OP, RHO, V, MP, false, 4>, a, grid, 0, s);
      if (a.g_log2 == 3)
        return launch_rows_cfg(spmm_rows_kernel<T, OP, RHO, V, MP, false, 3>, a, grid, 0, s);
      return launch_rows_cfg(spmm_rows_kernel<T, OP, RHO, V, MP, false, 2>, a, grid, 0, s);
    }
  }
  if constexpr (sizeof(T) == 4) {
    if (narrow_launch<V>(a.g_log2))
      return launch_rows_cfg(spmm_rows_kernel<T, OP, RHO, V, MP, true>, a, grid,
                             2 * kWarpsPerCta * kChunkE * sizeof(int32_t), s);
  }
  return launch_rows_cfg(spmm_rows_kernel<T, OP, RHO, V, MP, false>, a, grid, 0, s);
}

// float: hot mode pairs get their own kernels; double (the parity
// instantiation) always uses the run-time-mode kernel.
template <typename T, int OP, int RHO, int V>
cudaError_t launch_spmm_rows_mp(int mp, const SpmmArgs& a, int64_t grid, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if constexpr (OP == OP_COPY) {
      if (mp == MP_F) return launch_spmm_rows_t<T, OP, RHO, V, MP_F>(a, grid, s);
    } else if constexpr (OP != OP_DIV) {  // add / sub / mul / dot
      if (mp == MP_FF) return launch_spmm_rows_t<T, OP, RHO, V, MP_FF>(a, grid, s);
      if (mp == MP_FS) return launch_spmm_rows_t<T, OP, RHO, V, MP_FS>(a, grid, s);
      if (mp == MP_FH) return launch_spmm_rows_t<T, OP, RHO, V, MP_FH>(a, grid, s);
    }
  }
  return launch_spmm_rows_t<T, OP, RHO, V, MP_GEN>(a, grid, s);
}

template <typename T, int OP, int RHO>
cudaError_t launch_spmm_rows_v(int V, int mp, const SpmmArgs& a, int64_t grid, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if (V == 4) return launch_spmm_rows_mp<T, OP, RHO, 4>(mp, a, grid, s);
  }
  if (V == 2) return launch_spmm_rows_mp<T, OP, RHO, 2>(mp, a, grid, s);
  return launch_spmm_rows_mp<T, OP, RHO, 1>(mp, a, grid, s);
}

// fused GAT attention aggregation (u_mul_e + sum with recomputed weights):
// spmm_op_attn.cu. backward = MP_AB on the reverse graph.
cudaError_t launch_spmm_rows_attn(int dtype_is_f64, int V, bool backward, const SpmmArgs& a,
                                  int64_t grid, cudaStream_t s);

// dot messages under sum/mean (single column tile): spmm_op_dot.cu
cudaError_t launch_spmm_rows_dot_sum(int dtype_is_f64, int V, int mp, const SpmmArgs& a,
                                     int64_t grid, cudaStream_t s);

// Instantiated once per OP in spmm_op_<op>.cu so the op families compile in
// parallel.
template <int OP>
cudaError_t launch_spmm_rows(int dtype_is_f64, int rho, int V, int mp, const SpmmArgs& a,
                             int64_t grid, cudaStream_t s) {
  if (dtype_is_f64) {
    if (rho == RHO_SUM) return launch_spmm_rows_v<double, OP, RHO_SUM>(V, mp, a, grid, s);
    if (rho == RHO_MAX) return launch_spmm_rows_v<double, OP, RHO_MAX>(V, mp, a, grid, s);
    return launch_spmm_rows_v<double, OP, RHO_MIN>(V, mp, a, grid, s);
  }
  if (rho == RHO_SUM) return launch_spmm_rows_v<float, OP, RHO_SUM>(V, mp, a, grid, s);
  if (rho == RHO_MAX) return launch_spmm_rows_v<float, OP, RHO_MAX>(V, mp, a, grid, s);
  return launch_spmm_rows_v<float, OP, RHO_MIN>(V, mp, a, grid, s);
}

}  // namespace gmp
