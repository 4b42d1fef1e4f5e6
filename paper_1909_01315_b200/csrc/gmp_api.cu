// gmp_api.cu - the extern "C" boundary of libgmp.so (declared in include/gmp.h).
//
// Host-side validation mirrors the reference's operand checks
// (kernels.py:224-252, _operands_for) so that a caller gets the same class of
// error for the same mistake; shape checks that need row counts stay in the
// Python mirror (paper_1909_01315_b200/kernels.py), which owns the tensors.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/gmp.h"
#include "sddmm.cuh"
#include "softmax.cuh"
#include "spmm_dot.cuh"
#include "spmm_rows.cuh"
#include "spmm_ring.cuh"

namespace gmp {
template <int OP>
cudaError_t launch_spmm_rows(int, int, int, int, const SpmmArgs&, int64_t, cudaStream_t);  // (f64, rho, V, mode pair)
cudaError_t launch_route_extrema(int, int64_t, int32_t, const int64_t*, const void*, int64_t, void*,
                                 int64_t, cudaStream_t);
cudaError_t launch_extrema_bwd_copy(int, int64_t, int32_t, const int64_t*, const void*, int64_t,
                                    const int32_t*, int64_t, void*, int64_t, void*, size_t,
                                    cudaStream_t);
size_t extrema_workspace_bytes(int64_t cells);
cudaError_t launch_l2_gather_probe(const void*, int64_t, int32_t, int64_t, float*, cudaStream_t);
size_t schedule_workspace_bytes(int64_t n);
size_t gather_adj_workspace(int64_t n_heavy, int64_t m, int32_t dim, size_t F, int64_t* nw_out,
                            int64_t* win_out);
cudaError_t launch_gather_adj(int f64, const int64_t* indptr, const int32_t* eids,
                              const int32_t* order, int64_t n_heavy, int64_t n_nonempty, int64_t m,
                              int32_t dim, const void* src, int64_t lds, void* dst, int64_t ldd,
                              void* ws, cudaStream_t s);
cudaError_t launch_gather_rows(int, int64_t, int32_t, const int32_t*, const void*, int64_t, void*,
                               int64_t, cudaStream_t);
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
cudaError_t launch_extrema_bwd_binary(int, const ExtBinArgs&, int64_t, void*, size_t, cudaStream_t);
cudaError_t launch_rowdot(int, int, int64_t, int32_t, const void*, int64_t, const void*, int64_t,
                          const double*, void*, int64_t, int, cudaStream_t);
cudaError_t launch_pack_tiles(int, bool, int64_t, int32_t, int32_t, const void*, int64_t, void*,
                              int64_t, cudaStream_t);
cudaError_t launch_neighbor_sample(const int64_t*, const int64_t*, int64_t, const int64_t*, uint64_t,
                                   int64_t*, int64_t*, cudaStream_t);
int softmax_window_resident_ctas(int f64, int V, bool bwd);

cudaError_t build_schedule(int64_t n, const int64_t* indptr, int32_t thr, int32_t light,
                           int32_t* order_out, void* ws, size_t ws_bytes, int64_t* n_heavy,
                           int64_t* n_medium, int64_t* n_nonempty, int64_t* max_degree,
                           cudaStream_t s);
}  // namespace gmp

using namespace gmp;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return GMP_OK;
  return fail(GMP_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

const char* op_name(int op) {
  static const char* n[] = {"copy_lhs", "copy_rhs", "add", "sub", "mul", "div", "dot"};
  return (op >= 0 && op <= 6) ? n[op] : "?";
}

bool aligned(const void* p, size_t bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; }

// mirrors narrow_launch<V> in spmm_rows.cuh
bool narrow_launch_host(int V, int g_log2) {
  const int E = 32 >> g_log2;
  const int U = Unroll<4>::value;  // Unroll<V> is 8 for every V
  return E > 1 && E * U > 32;
}

int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

int log2i(int x) {
  int l = 0;
  while ((1 << l) < x) ++l;
  return l;
}

struct Opnd {
  OperandDev dev;
  bool present;
};

Opnd to_dev(const gmp_operand* o, int d_out) {
  Opnd r{};
  if (!o || !o->data) return r;
  r.present = true;
  r.dev.data = o->data;
  r.dev.ld = o->ld;
  r.dev.dim = o->dim;
  r.dev.target = o->target;
  r.dev.bcast = (o->dim == 1 && d_out > 1) ? 1 : 0;
  return r;
}

// CTAs per heavy row: a thread-block cluster of 8 when the largest row alone
// holds more than half of one SM's share of the edges (otherwise that row's
// single CTA is the kernel's tail) and an edge carries enough work (width >=
// 4 columns; below that the extra CTAs cost more than the tail, op sweep);
// GMP_NO_CLUSTER=1 disables it.
int hub_cluster(const gmp_adj* adj, const gmp_sched* sched, int width) {
  static const bool off = getenv("GMP_NO_CLUSTER") != nullptr;
  if (off || !sched || sched->n_heavy <= 0 || adj->m <= 0 || width < 4) return 1;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  static const int forced = getenv("GMP_CLUSTER") ? atoi(getenv("GMP_CLUSTER")) : 0;
  if (forced == 1 || forced == 2 || forced == 4 || forced == 8) return forced;
  return sched->max_degree * 2 * (int64_t)sms > adj->m ? 8 : 1;
}

int64_t round_up(int64_t x, int64_t k) { return (x + k - 1) / k * k; }

// Largest vector width every full-width operand, the output and arg support.
int pick_v(size_t F, int width, const Opnd* ops, int nops, const void* out, int64_t ldo,
           const void* arg) {
  const int cands[3] = {4, 2, 1};
  for (int V : cands) {
    if (F == 8 && V == 4) continue;
    if (width % V) continue;
    bool ok = true;
    for (int i = 0; i < nops; ++i) {
      if (!ops[i].present || ops[i].dev.bcast) continue;
      ok &= (ops[i].dev.ld % V == 0) && aligned(ops[i].dev.data, V * F);
    }
    if (out) ok &= (ldo % V == 0) && aligned(out, V * F);
    if (arg && V > 1) ok &= aligned(arg, 16);
    if (ok) return V;
  }
  return 1;
}

// every full-width operand's rows are 16 B aligned runs of whole float4s
// (ld % 4 == 0, 16 B-aligned base), so 16 B gathers stay in bounds of the row
// even past a width that is not a multiple of 4
bool gathers_v4(const Opnd* ops, int nops) {
  bool any = false;
  for (int i = 0; i < nops; ++i) {
    if (!ops[i].present || ops[i].dev.bcast) continue;
    if (ops[i].dev.ld % 4 != 0 || !aligned(ops[i].dev.data, 16)) return false;
    any = true;
  }
  return any;
}

// Validate phi's operands and derive d_out (kernels.py:224-252).
int check_operands(int op, const gmp_operand* lhs, const gmp_operand* rhs, int32_t* d_out_expected) {
  if (op < GMP_COPY_LHS || op > GMP_DOT) return fail(GMP_EINVAL, "unknown op %d", op);
  const bool binary = op >= GMP_ADD;
  const gmp_operand* used = (op == GMP_COPY_RHS) ? rhs : lhs;
  if (!used || !used->data) return fail(GMP_EINVAL, "phi %s needs its operand", op_name(op));
  if (used->target < GMP_SRC || used->target > GMP_EDGE_POS)
    return fail(GMP_EINVAL, "bad operand target %d", used->target);
  if (used->dim < 0 || used->ld < used->dim) return fail(GMP_EINVAL, "bad operand dim/ld");
  if (!binary) {
    *d_out_expected = used->dim;
    return GMP_OK;
  }
  if (!rhs || !rhs->data) return fail(GMP_EINVAL, "phi %s needs its rhs operand", op_name(op));
  if (rhs->target < GMP_SRC || rhs->target > GMP_EDGE_POS)
    return fail(GMP_EINVAL, "bad operand target %d", rhs->target);
  if (lhs->target == rhs->target) return fail(GMP_EINVAL, "binary op targets must differ");
  if (rhs->dim < 0 || rhs->ld < rhs->dim) return fail(GMP_EINVAL, "bad operand dim/ld");
  const int dl = lhs->dim, dr = rhs->dim;
  if (op == GMP_DOT) {
    if (dl != dr) return fail(GMP_EINVAL, "dot needs equal operand dims, got %d and %d", dl, dr);
    *d_out_expected = 1;
    return GMP_OK;
  }
  if (dl != dr && dl != 1 && dr != 1)
    return fail(GMP_EINVAL, "operand dims %d and %d are not broadcastable", dl, dr);
  *d_out_expected = dl > dr ? dl : dr;
  return GMP_OK;
}

int kernel_op(int op) {
  switch (op) {
    case GMP_COPY_LHS:
    case GMP_COPY_RHS: return OP_COPY;
    case GMP_ADD: return OP_ADD;
    case GMP_SUB: return OP_SUB;
    case GMP_MUL: return OP_MUL;
    case GMP_DIV: return OP_DIV;
    default: return OP_DOT;
  }
}

// Column-tile width: the whole row when the gathered source slice fits the
// L2 budget, otherwise the widest multiple of one full warp pass (32 * V
// columns) that does; then balanced over the resulting tile count.
int pick_tile(const gmp_tuning* tun, int d_out, int V, size_t F, int64_t n_src_rows, bool src_full,
              int max_tw) {
  int tw;
  if (tun && tun->tile_cols > 0) {
    tw = ((tun->tile_cols + V - 1) / V) * V;
  } else {
    tw = d_out;
    if (src_full) {
      const int64_t budget = (int64_t)((tun && tun->l2_budget_mb > 0) ? tun->l2_budget_mb : 64) << 20;
      const int64_t per_col = n_src_rows * (int64_t)F;
      const int64_t fit = per_col > 0 ? budget / per_col : d_out;
      if (fit < d_out) {
        const int unit = 32 * V;
        tw = (int)std::max<int64_t>(unit, (fit / unit) * unit);
      }
    }
  }
  if (tw > max_tw) tw = max_tw;
  if (tw >= d_out) return d_out;
  if (tw < 1) tw = 1;
  const int ntiles = (d_out + tw - 1) / tw;
  tw = (d_out + ntiles - 1) / ntiles;
  tw = ((tw + V - 1) / V) * V;
  return tw;
}

RowOperand row_operand(const Opnd& o) {
  RowOperand r{};
  if (!o.present) return r;
  r.data = o.dev.data;
  r.ld = (uint32_t)o.dev.ld;
  r.from_eid = o.dev.target == GMP_EDGE;
  r.from_pos = o.dev.target == GMP_EDGE_POS;
  r.bcast = o.dev.bcast;
  r.mode = o.dev.target == GMP_DST ? M_HOIST : (o.dev.bcast ? M_SCALAR : M_FULL);
  return r;
}

}  // namespace

extern "C" {

const char* gmp_last_error(void) { return g_last_error.c_str(); }

const char* gmp_strerror(int status) {
  switch (status) {
    case GMP_OK: return "ok";
    case GMP_EINVAL: return "invalid argument";
    case GMP_ECUDA: return "CUDA error";
    case GMP_EUNSUPPORTED: return "unsupported configuration";
    default: return "unknown status";
  }
}

uint64_t gmp_launch_count(void) { return g_launches.load(); }

int gmp_version(void) { return 1; }

size_t gmp_schedule_workspace_size(int64_t n_rows) { return schedule_workspace_bytes(n_rows); }

int gmp_build_schedule(const gmp_adj* adj, int32_t heavy_threshold, int32_t light_threshold,
                       int32_t* order_out, void* workspace, size_t workspace_bytes,
                       gmp_sched* sched_out, void* stream) {
  if (!adj || !sched_out) return fail(GMP_EINVAL, "null adjacency or schedule");
  if (adj->n_rows < 0 || adj->n_rows >= (1ll << 31)) return fail(GMP_EINVAL, "n_rows out of range");
  if (adj->n_rows > 0 && (!order_out || !adj->indptr)) return fail(GMP_EINVAL, "null arrays");
  if (workspace_bytes < schedule_workspace_bytes(adj->n_rows))
    return fail(GMP_EINVAL, "workspace too small: %zu < %zu", workspace_bytes,
                schedule_workspace_bytes(adj->n_rows));
  if (light_threshold < 0 || light_threshold > heavy_threshold)
    return fail(GMP_EINVAL, "light threshold must be in [0, heavy threshold]");
  int64_t nh = 0, nm = 0, nn = 0, dmax = 0;
  cudaError_t e = build_schedule(adj->n_rows, adj->indptr, heavy_threshold, light_threshold,
                                 order_out, workspace, workspace_bytes, &nh, &nm, &nn, &dmax,
                                 (cudaStream_t)stream);
  g_launches += adj->n_rows > 0 ? 2 : 0;
  if (e != cudaSuccess) return cuda_status(e, "gmp_build_schedule");
  sched_out->order = order_out;
  sched_out->n_heavy = nh;
  sched_out->n_medium = nm;
  sched_out->n_nonempty = nn;
  sched_out->heavy_threshold = heavy_threshold;
  sched_out->light_threshold = light_threshold;
  sched_out->max_degree = dmax;
  return GMP_OK;
}

struct Staged {
  double* acc;
  int64_t ldacc;
  int mode;
  const int64_t* deg_full;
};

static int gspmm_impl(const gmp_adj* adj, const gmp_sched* sched, int op, int rho, int dtype,
                      const gmp_operand* lhs, const gmp_operand* rhs, void* Z, int64_t ldz,
                      int32_t d_out, int64_t* arg, int64_t* counts, int32_t* err_pos,
                      const gmp_tuning* tuning, void* stream, const Staged* stg) {
  if (!adj) return fail(GMP_EINVAL, "null adjacency");
  if (rho < GMP_SUM || rho > GMP_MEAN) return fail(GMP_EINVAL, "unknown reducer %d", rho);
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (adj->m < 0 || adj->m >= (1ll << 31)) return fail(GMP_EINVAL, "edge count out of int32 range");
  if (adj->n_rows < 0 || adj->n_rows >= (1ll << 31)) return fail(GMP_EINVAL, "row count out of range");
  int32_t want = 0;
  int st = check_operands(op, lhs, rhs, &want);
  if (st) return st;
  if (d_out != want) return fail(GMP_EINVAL, "d_out %d does not match phi's output width %d", d_out, want);
  if (ldz < d_out || (!Z && adj->n_rows > 0 && d_out > 0)) return fail(GMP_EINVAL, "bad output Z/ldz");
  const bool ext = (rho == GMP_MAX || rho == GMP_MIN);
  if (ext && !arg && adj->n_rows > 0 && d_out > 0) return fail(GMP_EINVAL, "max/min need the arg output");
  if (op == GMP_DIV && !err_pos) return fail(GMP_EINVAL, "div needs the err_pos slot");
  if (adj->n_rows == 0 || d_out == 0) return GMP_OK;
  if (adj->m > 0 && (!adj->indices || !adj->eids)) return fail(GMP_EINVAL, "null adjacency arrays");
  if (sched && sched->order == nullptr && sched->n_heavy > 0)
    return fail(GMP_EINVAL, "schedule has heavy rows but no order");

  if ((lhs && lhs->ld >= (1ll << 32)) || (rhs && rhs->ld >= (1ll << 32)))
    return fail(GMP_EUNSUPPORTED, "operand leading dimension must be < 2^32");
  const size_t F = dtype == GMP_F64 ? 8 : 4;
  const int kop = kernel_op(op);
  const int krho = rho == GMP_MAX ? RHO_MAX : (rho == GMP_MIN ? RHO_MIN : RHO_SUM);
  // copy_rhs reads only its rhs: canonicalise to a copy of "lhs"
  const gmp_operand* L = (op == GMP_COPY_RHS) ? rhs : lhs;
  const gmp_operand* R = (kop == OP_COPY) ? nullptr : rhs;
  Opnd ops[2] = {to_dev(L, d_out), to_dev(R, d_out)};
  const int64_t n_heavy = sched ? sched->n_heavy : 0;
  const int32_t* order = sched ? sched->order : nullptr;
  const int64_t light_blocks = (adj->n_rows - n_heavy + kWarpsPerCta - 1) / kWarpsPerCta;
  const int64_t bpt = n_heavy + light_blocks;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;

  if (kop == OP_DOT) {
    if (L->target == GMP_EDGE_POS || (R && R->target == GMP_EDGE_POS))
      return fail(GMP_EINVAL, "dot messages take edge operands in edge-id order");
    const int dim = L->dim;
    const int Vd = dim > 0 ? pick_v(F, dim, ops, 2, nullptr, 0, nullptr) : 1;
    if (!ext && dim > 0 && dim <= 32 * Vd) {
      // sum / mean of dots == sum of per-column products: the row kernel
      // accumulates them per column and reduces the columns at the end
      const int Gd = std::min(32, next_pow2((dim + Vd - 1) / Vd));
      const bool narrow = (F == 4) && narrow_launch_host(Vd, log2i(Gd));
      const int64_t n_med = (order && narrow) ? std::max(n_heavy, sched->n_medium) : adj->n_rows;
      const int64_t med_blocks = (n_med - n_heavy + kWarpsPerCta - 1) / kWarpsPerCta;
      const int64_t rows_per_light_cta = (int64_t)kWarpsPerCta * (32 / Gd);
      SpmmArgs a{};
      a.indptr = adj->indptr; a.indices = adj->indices; a.eids = adj->eids; a.order = order;
      a.n_rows = adj->n_rows; a.n_heavy = n_heavy; a.n_medium = n_med;
      a.medium_blocks = med_blocks;
      a.cluster = hub_cluster(adj, sched, dim);
      a.blocks_per_tile = round_up(
          n_heavy * a.cluster + med_blocks +
              (adj->n_rows - n_med + rows_per_light_cta - 1) / rows_per_light_cta,
          a.cluster);
      a.d_out = dim; a.tile_cols = dim; a.g_log2 = log2i(Gd); a.mean = rho == GMP_MEAN;
      a.lhs = row_operand(ops[0]);
      a.rhs = row_operand(ops[1]);
      a.lhs.bcast = a.rhs.bcast = 0;
      if (a.lhs.mode != M_FULL && a.rhs.mode == M_FULL) std::swap(a.lhs, a.rhs);  // dot commutes
      int mp = MP_GEN;
      if (F == 4 && a.lhs.mode == M_FULL)
        mp = a.rhs.mode == M_FULL ? MP_FF : (a.rhs.mode == M_HOIST ? MP_FH : MP_GEN);
      a.need_eid = (a.lhs.from_eid && a.lhs.mode != M_HOIST) ||
                   (a.rhs.from_eid && a.rhs.mode != M_HOIST);
      a.Z = Z; a.ldz = ldz; a.counts = counts;
      e = launch_spmm_rows_dot_sum(F == 8, Vd, mp, a, a.blocks_per_tile, s);
      g_launches++;
      return cuda_status(e, "gmp_gspmm(dot rows)");
    }
    SpmmDotArgs a{};
    a.indptr = adj->indptr; a.indices = adj->indices; a.eids = adj->eids; a.order = order;
    a.n_rows = adj->n_rows; a.n_heavy = n_heavy; a.dim = dim;
    const int V = dim > 0 ? pick_v(F, dim, ops, 2, nullptr, 0, nullptr) : 1;
    // at most 8 lanes per edge: wide dots loop over columns instead of
    // paying a 5-level fp64 shuffle tree per edge
    a.g_log2 = log2i(std::min(8, next_pow2(std::max(1, (dim + V - 1) / V))));
    {
      // short rows: one per lane group when a row uses fewer than 32 lanes
      const int Ed = 32 >> a.g_log2;
      const int64_t n_med = (order && Ed > 1) ? std::max(n_heavy, sched->n_medium) : adj->n_rows;
      a.n_medium = n_med;
      a.medium_blocks = (n_med - n_heavy + kWarpsPerCta - 1) / kWarpsPerCta;
      const int64_t per = (int64_t)kWarpsPerCta * Ed;
      a.cluster = hub_cluster(adj, sched, dim);
      const int64_t bpt_dot = round_up(
          n_heavy * a.cluster + a.medium_blocks + (adj->n_rows - n_med + per - 1) / per,
          a.cluster);
      a.Z = Z; a.ldz = ldz; a.arg = arg; a.counts = counts;
      a.mean = rho == GMP_MEAN; a.lhs = ops[0].dev; a.rhs = ops[1].dev;
      a.lhs.bcast = a.rhs.bcast = 0;
      e = launch_spmm_dot(F == 8, krho, V, a, bpt_dot, s);
      g_launches++;
      return cuda_status(e, "gmp_gspmm(dot)");
    }
  }

  int V = pick_v(F, d_out, ops, 2, Z, ldz, ext ? arg : nullptr);
  int z_split = 0;
  if (!ext && V < 4 && F == 4) {
    if (ldz % 2 == 0 && aligned(Z, 8) && pick_v(F, d_out, ops, 2, nullptr, 0, nullptr) == 4) {
      // sum / mean into an output whose rows are only 8 B aligned (a column
      // tile of a row-major Z): keep 16 B gathers, store each 4-vector as two
      // 8 B halves
      V = 4;
      z_split = 1;
    } else if (d_out % 4 && gathers_v4(ops, 2)) {
      // a width that is not a multiple of 4 over 16 B-aligned operand rows
      // (a padded projection, the last packed column tile): 16 B gathers, the
      // last vector of a row stored element by element
      V = 4;
      z_split = (ldz % 4 == 0 && aligned(Z, 16)) ? 0 : ((ldz % 2 == 0 && aligned(Z, 8)) ? 1 : 2);
    }
  }
  const bool src_full = (ops[0].dev.target == GMP_SRC && !ops[0].dev.bcast) ||
                        (ops[1].present && ops[1].dev.target == GMP_SRC && !ops[1].dev.bcast);
  const int max_tw = 32 * V;
  const int tw = pick_tile(tuning, d_out, V, F, adj->n_rows, src_full, max_tw);
  const int G = std::min(32, next_pow2((tw + V - 1) / V));
  const int ntiles = (d_out + tw - 1) / tw;

  // short rows share a warp (one per lane group) when a row uses fewer than
  // 32 lanes; otherwise every non-heavy row gets a warp
  const int E = 32 / G;
  const bool narrow = (F == 4) && narrow_launch_host(V, log2i(G));
  // a copy of the destination's own row reads no edges (row-constant path)
  const bool row_const = kop == OP_COPY && ops[0].dev.target == GMP_DST;
  const int ncl = hub_cluster(adj, sched, row_const ? 0 : tw);
  SpmmArgs a{};
  a.cluster = ncl;
  a.z_split = z_split;
  a.indptr = adj->indptr; a.indices = adj->indices; a.eids = adj->eids; a.order = order;
  a.n_rows = adj->n_rows; a.n_heavy = n_heavy;
  a.d_out = d_out; a.tile_cols = tw; a.g_log2 = log2i(G); a.mean = rho == GMP_MEAN;
  a.lhs = row_operand(ops[0]);
  a.rhs = row_operand(ops[1]);
  // compile-time mode pair for the hot shapes; add / mul commute, so a
  // gathered operand on the right is swapped to the left (bit-identical)
  int mp = MP_GEN;
  if (F == 4) {
    if (kop == OP_COPY) {
      mp = a.lhs.mode == M_FULL ? MP_F : MP_GEN;
    } else if (kop == OP_ADD || kop == OP_MUL || kop == OP_SUB) {
      if (a.lhs.mode != M_FULL && a.rhs.mode == M_FULL && kop != OP_SUB) std::swap(a.lhs, a.rhs);
      if (a.lhs.mode == M_FULL)
        mp = a.rhs.mode == M_FULL ? MP_FF : (a.rhs.mode == M_SCALAR ? MP_FS : MP_FH);
    }
  }
  a.need_eid = ext || (a.lhs.from_eid && a.lhs.mode != M_HOIST) ||
               (ops[1].present && a.rhs.from_eid && a.rhs.mode != M_HOIST);
  // light rows (degree <= the schedule's light threshold) share a warp, one
  // per lane group, in the narrow kernels and in the pipelined 256 B-row
  // kernel (launch_spmm_rows_t picks it by the same predicate)
  const bool pipe = F == 4 && pipe_launch(V, krho, kop, mp, a.g_log2, a.need_eid,
                                          !a.lhs.from_eid && !a.lhs.from_pos);
  const int64_t n_medium =
      (order && (narrow || pipe)) ? std::max(n_heavy, sched->n_medium) : adj->n_rows;
  const int64_t medium_blocks = (n_medium - n_heavy + kWarpsPerCta - 1) / kWarpsPerCta;
  const int64_t light_rows = adj->n_rows - n_medium;
  const int64_t bpt_rows = round_up(
      n_heavy * ncl + medium_blocks +
          (light_rows + (int64_t)kWarpsPerCta * E - 1) / ((int64_t)kWarpsPerCta * E),
      ncl);
  a.n_medium = n_medium;
  a.medium_blocks = medium_blocks;
  a.blocks_per_tile = bpt_rows;
  a.Z = Z; a.ldz = ldz; a.arg = arg; a.counts = counts; a.err_pos = err_pos;
  if (stg) {
    a.acc64 = stg->acc; a.ldacc = stg->ldacc; a.acc_mode = stg->mode; a.deg_full = stg->deg_full;
  }
  const int64_t grid = bpt_rows * ntiles;
  if (grid >= (1ll << 31)) return fail(GMP_EUNSUPPORTED, "grid too large");
  switch (kop) {
    case OP_COPY: e = launch_spmm_rows<OP_COPY>(F == 8, krho, V, mp, a, grid, s); break;
    case OP_ADD: e = launch_spmm_rows<OP_ADD>(F == 8, krho, V, mp, a, grid, s); break;
    case OP_SUB: e = launch_spmm_rows<OP_SUB>(F == 8, krho, V, mp, a, grid, s); break;
    case OP_MUL: e = launch_spmm_rows<OP_MUL>(F == 8, krho, V, mp, a, grid, s); break;
    default: e = launch_spmm_rows<OP_DIV>(F == 8, krho, V, mp, a, grid, s); break;
  }
  g_launches++;
  return cuda_status(e, "gmp_gspmm");
}

int gmp_gspmm(const gmp_adj* adj, const gmp_sched* sched, int op, int rho, int dtype,
              const gmp_operand* lhs, const gmp_operand* rhs, void* Z, int64_t ldz, int32_t d_out,
              int64_t* arg, int64_t* counts, int32_t* err_pos, const gmp_tuning* tuning,
              void* stream) {
  return gspmm_impl(adj, sched, op, rho, dtype, lhs, rhs, Z, ldz, d_out, arg, counts, err_pos,
                    tuning, stream, nullptr);
}

int gmp_gspmm_staged(const gmp_adj* adj, const gmp_sched* sched, int op, int rho, int dtype,
                     const gmp_operand* lhs, const gmp_operand* rhs, double* acc, int64_t ldacc,
                     int mode, const int64_t* deg_full, void* Z, int64_t ldz, int32_t d_out,
                     int32_t* err_pos, const gmp_tuning* tuning, void* stream) {
  if (rho != GMP_SUM && rho != GMP_MEAN)
    return fail(GMP_EINVAL, "staged g-SpMM takes sum / mean reducers");
  if (op == GMP_DOT) return fail(GMP_EUNSUPPORTED, "staged g-SpMM does not take dot messages");
  if (mode < GMP_STAGE_FIRST || mode > GMP_STAGE_LAST || mode == 2)
    return fail(GMP_EINVAL, "unknown stage mode %d", mode);
  if (!adj) return fail(GMP_EINVAL, "null adjacency");
  if (adj->n_rows > 0 && d_out > 0 && (!acc || ldacc < d_out))
    return fail(GMP_EINVAL, "bad fp64 accumulator / ldacc");
  const int flags = mode == GMP_STAGE_FIRST ? kAccStore
                  : mode == GMP_STAGE_MID ? (kAccRead | kAccStore) : (kAccRead | kAccZ);
  Staged st{acc, ldacc, flags, deg_full};
  return gspmm_impl(adj, sched, op, rho, dtype, lhs, rhs, Z, ldz, d_out, nullptr, nullptr,
                    err_pos, tuning, stream, &st);
}

size_t gmp_gspmm_ring_workspace_size(const gmp_adj* adj, const gmp_sched* sched) {
  if (!adj || !sched || sched->n_heavy <= 0) return 0;
  return ring_workspace_bytes(sched->n_heavy, adj->m);
}

int gmp_gspmm_ring_prepare(const gmp_adj* adj, const gmp_sched* sched, void* ws,
                           size_t ws_bytes, void* stream) {
  if (!adj || !sched) return fail(GMP_EINVAL, "null adjacency / schedule");
  if (sched->n_heavy <= 0) return GMP_OK;
  if (!sched->order) return fail(GMP_EINVAL, "schedule has heavy rows but no order");
  if (!ws || ws_bytes < gmp_gspmm_ring_workspace_size(adj, sched))
    return fail(GMP_EINVAL, "ring workspace too small");
  cudaError_t e = launch_ring_prepare(adj->indptr, sched->order, sched->n_heavy, ws,
                                      (cudaStream_t)stream);
  g_launches++;
  return cuda_status(e, "gmp_gspmm_ring_prepare");
}

int gmp_gspmm_ring(const gmp_adj* adj, const gmp_sched* sched, int op, int rho, int dtype,
                   const gmp_operand* lhs, const gmp_operand* rhs, int64_t n_src_rows, void* Z,
                   int64_t ldz, int32_t d_out, void* ws, size_t ws_bytes, void* stream) {
  if (!adj || !sched || !lhs) return fail(GMP_EINVAL, "null adjacency / schedule / operand");
  if (n_src_rows < 1 || n_src_rows >= (1ll << 31)) return fail(GMP_EINVAL, "bad n_src_rows");
  if (dtype != GMP_F32) return fail(GMP_EUNSUPPORTED, "the ring path is fp32");
  if (rho != GMP_SUM && rho != GMP_MEAN) return fail(GMP_EUNSUPPORTED, "the ring path is sum / mean");
  const bool mul = op == GMP_MUL;
  if (op != GMP_COPY_LHS && !mul) return fail(GMP_EUNSUPPORTED, "the ring path is copy_u / u_mul_e");
  if (lhs->target != GMP_SRC || lhs->ld != 64 || !aligned(lhs->data, 16))
    return fail(GMP_EINVAL, "ring lhs must be packed 64-float source rows, 16 B aligned");
  if (mul && (!rhs || rhs->target != GMP_EDGE_POS || rhs->dim != 1))
    return fail(GMP_EINVAL, "ring u_mul_e takes a per-position scalar rhs");
  if (d_out < 1 || d_out > 64 || ldz < d_out || !Z) return fail(GMP_EINVAL, "bad d_out / Z");
  const int64_t nh = sched->n_heavy;
  cudaStream_t s = (cudaStream_t)stream;
  if (nh > 0) {
    if (!ws || ws_bytes < gmp_gspmm_ring_workspace_size(adj, sched))
      return fail(GMP_EINVAL, "ring workspace too small");
    RingArgs a{};
    a.indptr = adj->indptr; a.indices = adj->indices; a.order = sched->order; a.n_heavy = nh;
    a.X = static_cast<const float*>(lhs->data);
    a.W = mul ? static_cast<const float*>(rhs->data) : nullptr;
    a.Z = static_cast<float*>(Z); a.ldz = ldz; a.width = d_out; a.mean = rho == GMP_MEAN;
    cudaError_t e = launch_ring(mul, a, n_src_rows, ws, s);
    g_launches += 2;
    if (e != cudaSuccess) return cuda_status(e, "gmp_gspmm_ring");
  }
  if (nh >= adj->n_rows) return GMP_OK;
  // the remaining rows: the row kernel over the schedule without its heavy prefix
  gmp_sched lt = *sched;
  lt.order = sched->order ? sched->order + nh : nullptr;
  lt.n_heavy = 0;
  lt.n_medium = std::max<int64_t>(0, sched->n_medium - nh);
  lt.n_nonempty = std::max<int64_t>(0, sched->n_nonempty - nh);
  gmp_adj la = *adj;
  la.n_rows = adj->n_rows - nh;
  return gspmm_impl(&la, &lt, op, rho, dtype, lhs, rhs, Z, ldz, d_out, nullptr, nullptr, nullptr,
                    nullptr, stream, nullptr);
}

int gmp_gsddmm(const gmp_coo* coo, int op, int dtype, const gmp_operand* lhs, const gmp_operand* rhs,
               void* M, int64_t ldm, int32_t d_out, int32_t* err_eid, void* stream) {
  if (!coo) return fail(GMP_EINVAL, "null coo");
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (coo->m < 0 || coo->m >= (1ll << 31)) return fail(GMP_EINVAL, "edge count out of int32 range");
  int32_t want = 0;
  int st = check_operands(op, lhs, rhs, &want);
  if (st) return st;
  if (d_out != want) return fail(GMP_EINVAL, "d_out %d does not match phi's output width %d", d_out, want);
  if (ldm < d_out || (!M && coo->m > 0 && d_out > 0)) return fail(GMP_EINVAL, "bad output M/ldm");
  if (op == GMP_DIV && !err_eid) return fail(GMP_EINVAL, "div needs the err_eid slot");
  if ((lhs && lhs->target == GMP_EDGE_POS) || (rhs && rhs->target == GMP_EDGE_POS))
    return fail(GMP_EINVAL, "GMP_EDGE_POS operands are g-SpMM only");
  if (coo->m == 0 || d_out == 0) return GMP_OK;
  if (!coo->src || !coo->dst) return fail(GMP_EINVAL, "null coo arrays");
  const size_t F = dtype == GMP_F64 ? 8 : 4;
  const int kop = kernel_op(op);
  const gmp_operand* L = (op == GMP_COPY_RHS) ? rhs : lhs;
  const gmp_operand* R = (kop == OP_COPY) ? nullptr : rhs;
  Opnd ops[2] = {to_dev(L, d_out), to_dev(R, d_out)};
  SddmmArgs a{};
  a.src = coo->src; a.dst = coo->dst; a.m = coo->m; a.d_out = d_out;
  a.lhs = ops[0].dev; a.rhs = ops[1].dev; a.M = M; a.ldm = ldm; a.err_eid = err_eid;
  int V, width;
  if (kop == OP_DOT) {
    width = L->dim;
    a.lhs.bcast = a.rhs.bcast = 0;
    V = width > 0 ? pick_v(F, width, ops, 2, nullptr, 0, nullptr) : 1;
  } else {
    width = d_out;
    V = pick_v(F, width, ops, 2, M, ldm, nullptr);
  }
  a.dim = width;
  a.g_log2 = log2i(std::min(32, next_pow2(std::max(1, (width + V - 1) / V))));
  const int64_t warps = (coo->m + 31) / 32;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 148 * 16));
  cudaError_t e = launch_sddmm(F == 8, kop, V, a, grid, (cudaStream_t)stream);
  g_launches++;
  return cuda_status(e, "gmp_gsddmm");
}

size_t gmp_edge_softmax_workspace_size(int64_t n_rows, int32_t H) {
  return (size_t)std::max<int64_t>(0, n_rows) * (size_t)std::max(0, H) * 2 * sizeof(double);
}

// Windowed statistics plan: windows of `win` edge ids whose score rows (both
// operands for the backward) of all in-flight windows fit an L2 budget.
struct WindowPlan {
  bool on;
  int64_t win, n_windows;
  size_t off_counter, off_pm, off_pl, off_bounds, bytes;
};

static WindowPlan window_plan(const gmp_adj* adj, const gmp_sched* sched, int32_t H, size_t F,
                              bool bwd, int V) {
  WindowPlan p{};
  const size_t base = gmp_edge_softmax_workspace_size(adj ? adj->n_rows : 0, H);
  p.bytes = base;
  if (!adj || !sched || !sched->sorted_eids || sched->n_heavy <= 0 || H <= 0 || H > 32 * V ||
      adj->m < (1 << 22))
    return p;
  const int64_t R = sched->n_heavy;
  const int64_t warps = (int64_t)softmax_window_resident_ctas(F == 8, V, bwd) * kWarpsPerCta;
  const int64_t inflight = (warps + R - 1) / R + 1;  // windows touched by the warps in flight
  const int64_t row_bytes = (int64_t)H * (int64_t)F * (bwd ? 2 : 1);
  static const int64_t budget_mb = [] {
    const char* v = getenv("GMP_SOFTMAX_L2_MB");
    return v ? std::max<int64_t>(8, atoll(v)) : 80;
  }();
  const int64_t budget = budget_mb << 20;
  const int64_t win = budget / (inflight * row_bytes);
  if (win < (1 << 15)) return p;
  p.win = win;
  p.n_windows = (adj->m + win - 1) / win;
  const size_t part = (size_t)p.n_windows * (size_t)R * (size_t)H;
  p.off_counter = (base + 255) / 256 * 256;
  p.off_pm = p.off_counter + 256;
  p.off_pl = (p.off_pm + part * F + 255) / 256 * 256;
  p.off_bounds = (p.off_pl + part * sizeof(double) + 255) / 256 * 256;
  p.bytes = p.off_bounds + (size_t)R * (size_t)(p.n_windows + 1) * sizeof(int64_t);
  p.on = true;
  return p;
}

static int softmax_vec(size_t F, int32_t H) {
  const int cands[3] = {4, 2, 1};
  for (int V : cands) {
    if (F == 8 && V == 4) continue;
    if (H % V == 0) return V;
  }
  return 1;
}

static_assert(GMP_SEG_CHUNK_SUB == kSegChunkSub, "gmp.h and softmax.cuh disagree on the chunk");

// Segmented statistics layout in the workspace: [stats | counter | pm | pl]
struct SegLayout {
  bool on;
  size_t off_counter, off_pm, off_pl, bytes;
};

static SegLayout seg_layout(const gmp_adj* adj, const gmp_sched* sched, int32_t H, size_t F) {
  SegLayout p{};
  p.bytes = gmp_edge_softmax_workspace_size(adj ? adj->n_rows : 0, H);
  const gmp_segplan* sp = sched ? sched->segplan : nullptr;
  if (!adj || !sp || sched->n_heavy <= 0 || sp->n_pos <= 0 || sp->n_pieces <= 0 || H <= 0 ||
      !sp->perm || !sp->starts || !sp->chunk_piece || !sp->row_ptr || !sp->row_pieces)
    return p;
  const size_t part = (size_t)sp->n_pieces * (size_t)H;
  p.off_counter = (p.bytes + 255) / 256 * 256;
  p.off_pm = p.off_counter + 256;
  p.off_pl = (p.off_pm + part * F + 255) / 256 * 256;
  p.bytes = p.off_pl + part * sizeof(double);
  p.on = true;
  return p;
}

size_t gmp_edge_softmax_workspace_size_ex(const gmp_adj* in_adj, const gmp_sched* sched, int32_t H,
                                          int dtype, int backward) {
  const size_t F = dtype == GMP_F64 ? 8 : 4;
  return std::max(window_plan(in_adj, sched, H, F, backward != 0, softmax_vec(F, H)).bytes,
                  seg_layout(in_adj, sched, H, F).bytes);
}

static int softmax_common(const gmp_adj* adj, const gmp_coo* coo, const gmp_sched* sched,
                          int dtype, const void* s, int64_t lds, const void* g, int64_t ldg,
                          int32_t H, void* out, int64_t ldo, void* ws, size_t ws_bytes, bool bwd,
                          void* stream, const void* el = nullptr, int64_t lde = 0,
                          const void* er = nullptr, int64_t ldr = 0, bool stats_only = false) {
  const bool uv = el != nullptr;
  if (!adj || (!coo && !stats_only)) return fail(GMP_EINVAL, "null adjacency or coo");
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (adj->m < 0 || adj->m >= (1ll << 31)) return fail(GMP_EINVAL, "edge count out of int32 range");
  if (coo && coo->m != adj->m) return fail(GMP_EINVAL, "coo and adjacency edge counts differ");
  if (H < 0 || (!uv && lds < H) || (!stats_only && ldo < H) || (bwd && ldg < H) || (uv && (lde < H || ldr < H || !er)))
    return fail(GMP_EINVAL, "bad head count / ld");
  if (adj->m == 0 || H == 0 || adj->n_rows == 0) return GMP_OK;
  if ((!s && !uv) || (!out && !stats_only) || (bwd && !g) || !adj->eids || !adj->indptr ||
      (!stats_only && !coo->dst) || (uv && (!adj->indices || (!stats_only && !coo->src))))
    return fail(GMP_EINVAL, "null arrays");
  const size_t F = dtype == GMP_F64 ? 8 : 4;
  const size_t ws_need = stats_only ? (size_t)adj->n_rows * 2 * (size_t)H * F
                                    : gmp_edge_softmax_workspace_size(adj->n_rows, H);
  if (!ws || ws_bytes < ws_need) return fail(GMP_EINVAL, "softmax workspace too small");
  Opnd ops[2] = {};
  ops[0].present = true; ops[0].dev.data = uv ? el : s; ops[0].dev.ld = uv ? lde : lds;
  if (bwd) { ops[1].present = true; ops[1].dev.data = g; ops[1].dev.ld = ldg; }
  if (uv) { ops[1].present = true; ops[1].dev.data = er; ops[1].dev.ld = ldr; }
  const int V = pick_v(F, H, ops, 2, stats_only ? nullptr : out, ldo, nullptr);
  int tw = std::min(H, 32 * V);
  const int ntiles = (H + tw - 1) / tw;
  tw = ((H + ntiles - 1) / ntiles + V - 1) / V * V;
  const int G = std::min(32, next_pow2((tw + V - 1) / V));
  const int64_t n_heavy = sched ? sched->n_heavy : 0;
  SoftmaxArgs a{};
  a.indptr = adj->indptr; a.indices = adj->indices; a.eids = adj->eids; a.order = sched ? sched->order : nullptr;
  a.n_rows = adj->n_rows; a.n_heavy = n_heavy;
  a.blocks_per_tile = n_heavy + (adj->n_rows - n_heavy + kWarpsPerCta - 1) / kWarpsPerCta;
  a.H = H; a.tile_cols = tw; a.g_log2 = log2i(G);
  a.s = s; a.lds = lds; a.g = g; a.ldg = ldg; a.out = out; a.ldo = ldo;
  a.dst = coo ? coo->dst : nullptr; a.m = adj->m;
  a.stat = ws;
  a.el = el; a.lde = lde; a.er = er; a.ldr = ldr; a.src = coo ? coo->src : nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  const WindowPlan wp = uv ? WindowPlan{} : window_plan(adj, sched, H, F, bwd, V);
  const SegLayout sgl = uv ? SegLayout{} : seg_layout(adj, sched, H, F);
  if (sgl.on && ntiles == 1 && sched->order && ws_bytes >= sgl.bytes &&
      sched->segplan->group == (32 >> a.g_log2) &&
      sched->segplan->n_pos % (kSegChunkSub * sched->segplan->group) == 0 && lds < (1ll << 31) &&
      ldg < (1ll << 31)) {
    // heavy rows: one chunked segmented pass over the window-major plan;
    // the rest as below
    const gmp_segplan* sp = sched->segplan;
    SegArgs sg{};
    sg.perm = sp->perm;
    sg.starts = sp->starts;
    sg.chunk_piece = sp->chunk_piece;
    sg.row_ptr = sp->row_ptr;
    sg.row_pieces = sp->row_pieces;
    sg.n_pos = sp->n_pos;
    const int64_t chunk_pos = (int64_t)kSegChunkSub * sp->group;
    sg.n_chunks = (sp->n_pos + chunk_pos - 1) / chunk_pos;
    sg.n_pieces = sp->n_pieces;
    sg.counter = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + sgl.off_counter);
    sg.pm = static_cast<char*>(ws) + sgl.off_pm;
    sg.pl = reinterpret_cast<double*>(static_cast<char*>(ws) + sgl.off_pl);
    e = launch_edge_softmax_seg(F == 8, V, bwd, a, sg, st);
    g_launches += 2;
    const int64_t n_med = std::max(n_heavy, std::min(sched->n_medium, sched->n_nonempty));
    SoftmaxArgs lt = a;
    lt.order = a.order + n_heavy;
    lt.n_rows = n_med - n_heavy;
    lt.n_heavy = 0;
    lt.blocks_per_tile = (lt.n_rows + kWarpsPerCta - 1) / kWarpsPerCta;
    if (e == cudaSuccess && lt.n_rows > 0) {
      e = launch_edge_softmax(F == 8, V, bwd, uv, lt, lt.blocks_per_tile, st);
      g_launches++;
    }
    SoftmaxArgs sl = a;
    sl.order = a.order + n_med;
    sl.n_rows = sched->n_nonempty - n_med;
    sl.n_heavy = 0;
    if (e == cudaSuccess && sl.n_rows > 0) {
      e = launch_edge_softmax_slots(F == 8, V, bwd, uv, sl, st);
      g_launches++;
    }
  } else if (wp.on && ntiles == 1 && V == softmax_vec(F, H) && ws_bytes >= wp.bytes) {
    // heavy rows: edge-id windows; the rest: the row kernel on the light rows
    WindowArgs w{};
    w.sorted_eids = sched->sorted_eids;
    w.win = wp.win;
    w.n_windows = wp.n_windows;
    w.counter = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + wp.off_counter);
    w.pm = static_cast<char*>(ws) + wp.off_pm;
    w.pl = reinterpret_cast<double*>(static_cast<char*>(ws) + wp.off_pl);
    w.bounds = reinterpret_cast<int64_t*>(static_cast<char*>(ws) + wp.off_bounds);
    e = launch_edge_softmax_window(F == 8, V, bwd, a, w, st);
    g_launches += 3;
    // rows [n_heavy, n_medium): one warp each; [n_medium, n_nonempty): one
    // per lane group (short rows); empty rows have no edge to normalise
    const int64_t n_med = std::max(n_heavy, std::min(sched->n_medium, sched->n_nonempty));
    SoftmaxArgs lt = a;
    lt.order = a.order + n_heavy;
    lt.n_rows = n_med - n_heavy;
    lt.n_heavy = 0;
    lt.blocks_per_tile = (lt.n_rows + kWarpsPerCta - 1) / kWarpsPerCta;
    if (e == cudaSuccess && lt.n_rows > 0) {
      e = launch_edge_softmax(F == 8, V, bwd, uv, lt, lt.blocks_per_tile, st);
      g_launches++;
    }
    SoftmaxArgs sl = a;
    sl.order = a.order + n_med;
    sl.n_rows = sched->n_nonempty - n_med;
    sl.n_heavy = 0;
    if (e == cudaSuccess && sl.n_rows > 0) {
      e = launch_edge_softmax_slots(F == 8, V, bwd, uv, sl, st);
      g_launches++;
    }
  } else if (sched && sched->order && ntiles == 1) {
    // rows [0, n_medium) of the schedule: CTA / warp per row; the short rows
    // after them one per lane group; empty rows are not launched
    const int64_t n_med = std::max(n_heavy, std::min(sched->n_medium, sched->n_nonempty));
    SoftmaxArgs hm = a;
    hm.n_rows = n_med;
    hm.blocks_per_tile = n_heavy + (n_med - n_heavy + kWarpsPerCta - 1) / kWarpsPerCta;
    e = hm.blocks_per_tile > 0 ? launch_edge_softmax(F == 8, V, bwd, uv, hm, hm.blocks_per_tile, st)
                               : cudaSuccess;
    g_launches++;
    SoftmaxArgs sl = a;
    sl.order = a.order + n_med;
    sl.n_rows = sched->n_nonempty - n_med;
    sl.n_heavy = 0;
    if (e == cudaSuccess && sl.n_rows > 0) {
      e = launch_edge_softmax_slots(F == 8, V, bwd, uv, sl, st);
      g_launches++;
    }
  } else {
    e = launch_edge_softmax(F == 8, V, bwd, uv, a, a.blocks_per_tile * ntiles, st);
    g_launches++;
  }
  if (e == cudaSuccess && !stats_only) {
    e = launch_edge_softmax_apply(F == 8, V, bwd, uv, a, st);
    g_launches++;
  }
  return cuda_status(e, bwd ? "gmp_edge_softmax_bwd" : "gmp_edge_softmax_fwd");
}

int gmp_edge_softmax_fwd(const gmp_adj* in_adj, const gmp_coo* coo, const gmp_sched* sched,
                         int dtype, const void* scores, int64_t lds, int32_t H, void* alpha,
                         int64_t lda, void* workspace, size_t workspace_bytes, void* stream) {
  return softmax_common(in_adj, coo, sched, dtype, scores, lds, nullptr, 0, H, alpha, lda,
                        workspace, workspace_bytes, false, stream);
}

int gmp_edge_softmax_uv_fwd(const gmp_adj* in_adj, const gmp_coo* coo, const gmp_sched* sched,
                            int dtype, const void* el, int64_t lde, const void* er, int64_t ldr,
                            int32_t H, void* alpha, int64_t lda, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (!el || !er) return fail(GMP_EINVAL, "null el / er");
  return softmax_common(in_adj, coo, sched, dtype, nullptr, 0, nullptr, 0, H, alpha, lda,
                        workspace, workspace_bytes, false, stream, el, lde, er, ldr);
}

int gmp_edge_softmax_bwd(const gmp_adj* in_adj, const gmp_coo* coo, const gmp_sched* sched,
                         int dtype, const void* alpha, int64_t lda, const void* grad, int64_t ldg,
                         int32_t H, void* ds, int64_t ldds, void* workspace,
                         size_t workspace_bytes, void* stream) {
  return softmax_common(in_adj, coo, sched, dtype, alpha, lda, grad, ldg, H, ds, ldds, workspace,
                        workspace_bytes, true, stream);
}

size_t gmp_gather_adj_workspace_size(const gmp_adj* adj, const gmp_sched* sched, int32_t dim,
                                     int dtype) {
  if (!adj || !sched || dim <= 0) return 0;
  return gather_adj_workspace(sched->n_heavy, adj->m, dim, dtype == GMP_F64 ? 8 : 4, nullptr,
                              nullptr);
}

int gmp_gather_adj(const gmp_adj* adj, const gmp_sched* sched, int32_t dim, int dtype,
                   const void* src, int64_t lds, void* dst, int64_t ldd, void* workspace,
                   size_t workspace_bytes, void* stream) {
  if (!adj || !sched) return fail(GMP_EINVAL, "null adjacency / schedule");
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (dim < 1 || lds < dim || ldd < dim) return fail(GMP_EINVAL, "bad sizes");
  if (adj->m == 0) return GMP_OK;
  if (!src || !dst || !adj->indptr || !adj->eids) return fail(GMP_EINVAL, "null arrays");
  if (sched->n_heavy > 0 && (!sched->order || sched->sorted_eids != adj->eids))
    return fail(GMP_EINVAL, "windowed gather needs the schedule order and row-ascending edge ids "
                            "(sched->sorted_eids == adj->eids)");
  if (workspace_bytes < gmp_gather_adj_workspace_size(adj, sched, dim, dtype))
    return fail(GMP_EINVAL, "workspace too small");
  cudaError_t e = launch_gather_adj(dtype == GMP_F64, adj->indptr, adj->eids, sched->order,
                                    sched->n_heavy, sched->n_nonempty, adj->m, dim, src, lds, dst,
                                    ldd, workspace, (cudaStream_t)stream);
  g_launches += sched->n_heavy > 0 ? 2 : 1;
  return cuda_status(e, "gmp_gather_adj");
}

int gmp_gather_rows(int64_t n, int32_t dim, int dtype, const int32_t* idx, const void* src,
                    int64_t lds, void* dst, int64_t ldd, void* stream) {
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (n < 0 || dim < 0 || lds < dim || ldd < dim) return fail(GMP_EINVAL, "bad sizes");
  if (n == 0 || dim == 0) return GMP_OK;
  if (!idx || !src || !dst) return fail(GMP_EINVAL, "null arrays");
  cudaError_t e = launch_gather_rows(dtype == GMP_F64, n, dim, idx, src, lds, dst, ldd,
                                     (cudaStream_t)stream);
  g_launches++;
  return cuda_status(e, "gmp_gather_rows");
}

int gmp_route_extrema(int64_t n_rows, int32_t d, int dtype, const int64_t* arg, const void* dZ,
                      int64_t lddz, void* dM, int64_t ldm, void* stream) {
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (n_rows < 0 || d < 0 || lddz < d || ldm < d) return fail(GMP_EINVAL, "bad sizes");
  if (n_rows == 0 || d == 0) return GMP_OK;
  if (!arg || !dZ || !dM) return fail(GMP_EINVAL, "null arrays");
  cudaError_t e = launch_route_extrema(dtype == GMP_F64, n_rows, d, arg, dZ, lddz, dM, ldm,
                                       (cudaStream_t)stream);
  g_launches++;
  return cuda_status(e, "gmp_route_extrema");
}

size_t gmp_extrema_bwd_workspace_size(int64_t n_rows, int32_t cells_per_row) {
  if (n_rows <= 0 || cells_per_row <= 0) return 0;
  return extrema_workspace_bytes(n_rows * (int64_t)cells_per_row);
}

int gmp_extrema_bwd_copy(int64_t n_rows, int32_t d, int dtype, const int64_t* arg, const void* dZ,
                         int64_t lddz, const int32_t* target_index, int64_t n_target_rows,
                         void* dOut, int64_t ldo, void* workspace, size_t workspace_bytes,
                         void* stream) {
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (n_rows < 0 || d < 0 || lddz < d || ldo < d || n_target_rows < 0)
    return fail(GMP_EINVAL, "bad sizes");
  if (n_rows == 0 || d == 0) return GMP_OK;
  if (!arg || !dZ || !dOut) return fail(GMP_EINVAL, "null arrays");
  if (target_index && (!workspace || workspace_bytes < gmp_extrema_bwd_workspace_size(n_rows, d)))
    return fail(GMP_EINVAL, "workspace too small: %zu < %zu", workspace_bytes,
                gmp_extrema_bwd_workspace_size(n_rows, d));
  cudaError_t e = launch_extrema_bwd_copy(dtype == GMP_F64, n_rows, d, arg, dZ, lddz, target_index,
                                          n_target_rows, dOut, ldo, workspace, workspace_bytes,
                                          (cudaStream_t)stream);
  g_launches += target_index ? 3 : 1;
  return cuda_status(e, "gmp_extrema_bwd_copy");
}

int gmp_edge_softmax_uv_stats(const gmp_adj* in_adj, const gmp_sched* sched, int dtype,
                              const void* el, int64_t lde, const void* er, int64_t ldr, int32_t H,
                              void* stat, size_t stat_bytes, void* stream) {
  if (!el || !er) return fail(GMP_EINVAL, "null el / er");
  return softmax_common(in_adj, nullptr, sched, dtype, nullptr, 0, nullptr, 0, H, nullptr, 0, stat,
                        stat_bytes, false, stream, el, lde, er, ldr, true);
}

int gmp_gat_aggregate(const gmp_adj* adj, const gmp_sched* sched, int dtype, int backward,
                      const void* X, int64_t ldx, int32_t d, const void* el, int64_t lde,
                      const void* pack, void* Z, int64_t ldz, double* z64, int64_t ldz64,
                      double* t_out, const gmp_tuning* tuning, void* stream) {
  if (!adj) return fail(GMP_EINVAL, "null adjacency");
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (adj->m < 0 || adj->m >= (1ll << 31)) return fail(GMP_EINVAL, "edge count out of int32 range");
  if (adj->n_rows < 0 || adj->n_rows >= (1ll << 31)) return fail(GMP_EINVAL, "row count out of range");
  if (d < 0 || ldx < d || ldz < d || lde < 1 || ldx >= (1ll << 32) || lde >= (1ll << 32) ||
      (z64 && ldz64 < d))
    return fail(GMP_EINVAL, "bad sizes / leading dimensions");
  if (adj->n_rows == 0 || d == 0) return GMP_OK;
  if (!X || !el || !pack || !Z || !adj->indptr || (adj->m > 0 && !adj->indices))
    return fail(GMP_EINVAL, "null arrays");
  const size_t F = dtype == GMP_F64 ? 8 : 4;
  if (!aligned(pack, 32)) return fail(GMP_EINVAL, "pack must be aligned to its 32-byte rows");
  if (sched && sched->order == nullptr && sched->n_heavy > 0)
    return fail(GMP_EINVAL, "schedule has heavy rows but no order");
  Opnd ops[2] = {};
  ops[0].present = true; ops[0].dev.data = X; ops[0].dev.ld = ldx; ops[0].dev.dim = d;
  ops[0].dev.target = GMP_SRC;
  int V = pick_v(F, d, ops, 1, Z, ldz, nullptr);
  int z_split = 0;
  if (V < 4 && F == 4 && d % 4 && gathers_v4(ops, 1)) {
    // padded rows (ld a multiple of 4): 16 B gathers, tail-masked stores
    V = 4;
    z_split = (ldz % 4 == 0 && aligned(Z, 16)) ? 0 : ((ldz % 2 == 0 && aligned(Z, 8)) ? 1 : 2);
  }
  const int tw = pick_tile(tuning, d, V, F, adj->n_rows, true, 32 * V);
  const int G = std::min(32, next_pow2((tw + V - 1) / V));
  const int ntiles = (d + tw - 1) / tw;
  const int E = 32 / G;
  const int64_t n_heavy = sched ? sched->n_heavy : 0;
  const int32_t* order = sched ? sched->order : nullptr;
  const bool narrow = (F == 4) && narrow_launch_host(V, log2i(G));
  const int64_t n_medium = (order && narrow) ? std::max(n_heavy, sched->n_medium) : adj->n_rows;
  const int64_t medium_blocks = (n_medium - n_heavy + kWarpsPerCta - 1) / kWarpsPerCta;
  const int64_t light_rows = adj->n_rows - n_medium;
  const int ncl = hub_cluster(adj, sched, tw);
  const int64_t bpt_rows = round_up(
      n_heavy * ncl + medium_blocks +
          (light_rows + (int64_t)kWarpsPerCta * E - 1) / ((int64_t)kWarpsPerCta * E),
      ncl);
  SpmmArgs a{};
  a.cluster = ncl;
  a.indptr = adj->indptr; a.indices = adj->indices; a.eids = adj->eids; a.order = order;
  a.n_rows = adj->n_rows; a.n_heavy = n_heavy; a.n_medium = n_medium;
  a.medium_blocks = medium_blocks; a.blocks_per_tile = bpt_rows;
  a.z_split = z_split;
  a.d_out = d; a.tile_cols = tw; a.g_log2 = log2i(G); a.mean = 0;
  a.lhs = row_operand(ops[0]);
  a.rhs.data = backward ? pack : el; a.rhs.ld = 1; a.rhs.mode = M_SCALAR;
  a.need_eid = 0;
  a.Z = Z; a.ldz = ldz;
  a.attn_el = el; a.attn_lde = (uint32_t)lde; a.attn_pack = pack;
  a.attn_t = backward ? t_out : nullptr;
  if (z64) {  // the unrounded fp64 rows too (exact operand of the backward's row dots)
    a.acc64 = z64; a.ldacc = ldz64; a.acc_mode = kAccZ | kAccStore;
  }
  const int64_t grid = bpt_rows * ntiles;
  if (grid >= (1ll << 31)) return fail(GMP_EUNSUPPORTED, "grid too large");
  cudaError_t e = launch_spmm_rows_attn(F == 8, V, backward != 0, a, grid, (cudaStream_t)stream);
  g_launches++;
  return cuda_status(e, "gmp_gat_aggregate");
}

int gmp_pack_tiles(int64_t n, int32_t d, int dtype, int32_t tile, const void* src, int64_t lds,
                   void* packed, void* stream) {
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (n < 0 || d < 0 || tile < 1 || lds < d) return fail(GMP_EINVAL, "bad sizes");
  if (n == 0 || d == 0) return GMP_OK;
  if (!src || !packed) return fail(GMP_EINVAL, "null arrays");
  cudaError_t e = launch_pack_tiles(dtype == GMP_F64, false, n, d, tile, src, lds, packed, 0,
                                    (cudaStream_t)stream);
  g_launches++;
  return cuda_status(e, "gmp_pack_tiles");
}

int gmp_unpack_tiles(int64_t n, int32_t d, int dtype, int32_t tile, const void* packed, void* dst,
                     int64_t ldd, void* stream) {
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (n < 0 || d < 0 || tile < 1 || ldd < d) return fail(GMP_EINVAL, "bad sizes");
  if (n == 0 || d == 0) return GMP_OK;
  if (!dst || !packed) return fail(GMP_EINVAL, "null arrays");
  cudaError_t e = launch_pack_tiles(dtype == GMP_F64, true, n, d, tile, packed, 0, dst, ldd,
                                    (cudaStream_t)stream);
  g_launches++;
  return cuda_status(e, "gmp_unpack_tiles");
}

int gmp_extrema_bwd_binary(const gmp_coo* coo, int64_t n_rows, int32_t d, int dtype,
                           const int64_t* arg, const void* dZ, int64_t lddz, int op, int role,
                           const gmp_operand* lhs, const gmp_operand* rhs, void* out, int64_t ldo,
                           int32_t own_dim, int64_t n_target_rows, void* workspace,
                           size_t workspace_bytes, void* stream) {
  if (!coo || !lhs || !rhs) return fail(GMP_EINVAL, "null coo / operand");
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (op != GMP_ADD && op != GMP_SUB && op != GMP_MUL && op != GMP_DIV && op != GMP_DOT)
    return fail(GMP_EINVAL, "binary extrema backward takes add / sub / mul / div / dot, got %s",
                op_name(op));
  if (op == GMP_DOT && (d != 1 || lhs->dim != rhs->dim || own_dim != lhs->dim))
    return fail(GMP_EINVAL, "dot: d_out must be 1 and own_dim the operand width");
  if (role != 0 && role != 1) return fail(GMP_EINVAL, "role must be 0 (lhs) or 1 (rhs)");
  if (n_rows < 0 || d < 0 || lddz < d || ldo < own_dim ||
      (op != GMP_DOT && own_dim != 1 && own_dim != d))
    return fail(GMP_EINVAL, "bad sizes");
  const gmp_operand* own = role == 0 ? lhs : rhs;
  if (own->target < GMP_SRC || own->target > GMP_EDGE || lhs->target < GMP_SRC ||
      lhs->target > GMP_EDGE || rhs->target < GMP_SRC || rhs->target > GMP_EDGE)
    return fail(GMP_EINVAL, "operand targets must be src / dst / edge");
  if (n_rows == 0 || d == 0) return GMP_OK;
  if (!arg || !dZ || !out || !coo->src || !lhs->data || !rhs->data)
    return fail(GMP_EINVAL, "null arrays");
  ExtBinArgs a{};
  a.n = n_rows; a.d = d; a.arg = arg; a.dZ = dZ; a.lddz = lddz; a.src = coo->src;
  a.op = kernel_op(op); a.role = role; a.target = own->target;
  a.lhs = to_dev(lhs, op == GMP_DOT ? lhs->dim : d).dev;
  a.rhs = to_dev(rhs, op == GMP_DOT ? rhs->dim : d).dev;
  a.out = out; a.ldo = ldo; a.own_dim = own_dim;
  const bool many = own->target == GMP_SRC || (op != GMP_DOT && own_dim == 1);
  const int32_t cells = op == GMP_DOT ? own_dim : d;
  if (n_target_rows < 0) return fail(GMP_EINVAL, "bad sizes");
  if (many && (!workspace || workspace_bytes < gmp_extrema_bwd_workspace_size(n_rows, cells)))
    return fail(GMP_EINVAL, "workspace too small: %zu < %zu", workspace_bytes,
                gmp_extrema_bwd_workspace_size(n_rows, cells));
  cudaError_t e = launch_extrema_bwd_binary(dtype == GMP_F64, a, n_target_rows, workspace,
                                            workspace_bytes, (cudaStream_t)stream);
  g_launches += many ? 3 : 1;
  return cuda_status(e, "gmp_extrema_bwd_binary");
}

int gmp_rowdot(int64_t n, int32_t d, int dtype, const void* A, int64_t lda, int b_dtype,
               const void* B, int64_t ldb, const double* sub, void* out, int64_t out_stride,
               int out_pair, void* stream) {
  if (dtype != GMP_F32 && dtype != GMP_F64) return fail(GMP_EINVAL, "unknown dtype %d", dtype);
  if (b_dtype != dtype && b_dtype != GMP_F64) return fail(GMP_EINVAL, "B must be dtype or f64");
  if (n < 0 || d < 0 || lda < d || ldb < d || out_stride < 1) return fail(GMP_EINVAL, "bad sizes");
  if (n == 0) return GMP_OK;
  if ((d > 0 && (!A || !B)) || !out) return fail(GMP_EINVAL, "null arrays");
  cudaError_t e = launch_rowdot(dtype == GMP_F64, b_dtype == GMP_F64, n, d, A, lda, B, ldb, sub,
                                out, out_stride, out_pair ? 1 : 0, (cudaStream_t)stream);
  g_launches++;
  return cuda_status(e, "gmp_rowdot");
}

int gmp_neighbor_sample(const int64_t* indptr, int64_t n_rows, const int64_t* seeds,
                        int64_t n_seeds, const int64_t* out_off, uint64_t rng_seed,
                        int64_t* scratch, int64_t* out_pos, void* stream) {
  if (n_rows < 0 || n_seeds < 0) return fail(GMP_EINVAL, "bad sizes");
  if (n_seeds == 0) return GMP_OK;
  if (!indptr || !seeds || !out_off || !scratch || !out_pos) return fail(GMP_EINVAL, "null arrays");
  cudaError_t e = launch_neighbor_sample(indptr, seeds, n_seeds, out_off, rng_seed, scratch, out_pos,
                                         (cudaStream_t)stream);
  g_launches++;
  return cuda_status(e, "gmp_neighbor_sample");
}

int gmp_probe_l2_gather(const void* data, int64_t rows, int32_t row_bytes, int64_t n_gathers,
                        float* sink, void* stream) {
  if (row_bytes != 64 && row_bytes != 256) return fail(GMP_EINVAL, "row_bytes must be 64 or 256");
  if (rows <= 0 || rows >= (1ll << 32) || n_gathers < 0) return fail(GMP_EINVAL, "bad sizes");
  if (!data || !sink) return fail(GMP_EINVAL, "null arrays");
  if (!aligned(data, 16)) return fail(GMP_EINVAL, "data must be 16-byte aligned");
  cudaError_t e = launch_l2_gather_probe(data, rows, row_bytes, n_gathers, sink,
                                         (cudaStream_t)stream);
  g_launches++;
  return cuda_status(e, "gmp_probe_l2_gather");
}

}  // extern "C"
