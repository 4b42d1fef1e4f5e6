/*
 * gmp.h - C-ABI of libgmp.so, the B200 (sm_100a) g-SpMM / g-SDDMM /
 * edge_softmax engine.
 *
 * Every entry point replaces one function of the reference package's kernel
 * engine (graphmp 0.1.0, /root/reference/pkg/src/graphmp). The reference is
 * pure Python with no FFI, so the "binding" a maintainer adds is the ctypes
 * stub in INTEGRATION.md; paper_1909_01315_b200/_lib.py is that stub.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers; sizes/strides are in elements.
 *  - Outputs are caller-allocated (the paper's framework-allocates-outputs
 *    contract); the library never allocates device memory
 *    except inside gmp_build_schedule's caller-supplied workspace.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 *    stream-ordered and asynchronous; the host syncs only to read err slots.
 *  - Return value: GMP_OK (0) or an error code; gmp_last_error() returns a
 *    thread_local detail string for the last failing call on this thread.
 *  - Feature dtype: GMP_F32 or GMP_F64 (messages and sum/mean/dot
 *    accumulation are always carried out in fp64).
 *  - Edge count m must be < 2^31 (int32 indices / edge ids on device).
 */
#ifndef GMP_H_
#define GMP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
enum { GMP_OK = 0, GMP_EINVAL = 1, GMP_ECUDA = 2, GMP_EUNSUPPORTED = 3 };

/* message ops: kernels.py:43 OPS ("copy_lhs","copy_rhs","add","sub","mul","div","dot") */
enum { GMP_COPY_LHS = 0, GMP_COPY_RHS = 1, GMP_ADD = 2, GMP_SUB = 3,
       GMP_MUL = 4, GMP_DIV = 5, GMP_DOT = 6 };
/* operand targets: kernels.py:44 TARGETS ("src","dst","edge"); NONE for copy's unused side.
 * GMP_EDGE_POS is an edge operand already permuted into the adjacency's order
 * (row p holds edge eids[p]; see gmp_gather_rows) - g-SpMM only. */
enum { GMP_NONE = -1, GMP_SRC = 0, GMP_DST = 1, GMP_EDGE = 2, GMP_EDGE_POS = 3 };
/* reducers: kernels.py:45 REDUCERS ("sum","max","min","mean") */
enum { GMP_SUM = 0, GMP_MAX = 1, GMP_MIN = 2, GMP_MEAN = 3 };
/* feature dtypes */
enum { GMP_F32 = 0, GMP_F64 = 1 };

/* One grouped index (graph.py:23-32 Adjacency): for CSC (in-adjacency,
 * graph.py:137) rows are destinations and `indices` are sources; for the
 * reverse graph's CSC (== forward CSR, graph.py:203-215) rows are sources.
 * Within a row, indices ascend and parallel edges break ties by edge id. */
typedef struct {
  int64_t n_rows;          /* groups (num_nodes) */
  int64_t m;               /* edges */
  const int64_t* indptr;   /* n_rows + 1 */
  const int32_t* indices;  /* m: neighbour node id */
  const int32_t* eids;     /* m: edge id */
} gmp_adj;

/* Degree-binned row schedule for an adjacency (built by gmp_build_schedule).
 * order: row ids sorted by degree, descending (stable). Rows order[0..n_heavy)
 * have degree > heavy_threshold and are reduced by a whole CTA; rows
 * order[n_heavy..n_medium) (degree > light_threshold) by one warp each; the
 * rest (short rows, then empty rows) several per warp, one per lane group.
 * order == NULL means identity order, every row on the warp path.
 * sorted_eids (nullable): the adjacency's edge ids with each row's ids in
 * ascending order (equal to eids when they already ascend inside rows); when
 * given, edge-keyed passes over heavy rows (edge_softmax statistics) run in
 * L2-sized edge-id windows. When the largest row holds more than half of one
 * SM's share of the edges, heavy rows are reduced by a cluster of 8 CTAs
 * (partials merged through distributed shared memory, in rank order).
 * segplan (nullable): the window-major piece layout of the heavy rows'
 * in-edges (gmp_segplan below); when given, the edge_softmax statistics of
 * the heavy rows run as one chunked segmented pass over it. */
typedef struct gmp_segplan gmp_segplan;
typedef struct {
  const int32_t* order;
  int64_t n_heavy;
  int64_t n_medium;
  int64_t n_nonempty;
  int32_t heavy_threshold;
  int32_t light_threshold;
  const int32_t* sorted_eids;
  int64_t max_degree;      /* largest row degree (set by gmp_build_schedule) */
  const gmp_segplan* segplan;
} gmp_sched;

/* Window-major layout of the heavy rows' in-edges for the segmented
 * edge_softmax statistics (built once per graph, window and lane-group
 * count by the host, kernels._softmax_segplan). Replaces the reference's
 * per-destination walk of the in-adjacency (kernels.py:340-466 _GroupedWalk
 * under messaging.py:105-126) for the rows order[0..n_heavy) of the schedule:
 *   perm       n_pos entries: those rows' in-edge ids ordered by
 *              (eid / win, heavy row index r, eid), each (window, row)
 *              segment padded with -1 to a multiple of `group` positions
 *              (the lane groups of one warp sub-step: 32 / next_pow2(H / V));
 *   sub-steps  runs of `group` positions; pieces = the segments cut every
 *              GMP_SEG_CHUNK_SUB sub-steps (a chunk); piece ids ascend;
 *   starts     ceil(n_pos / group / 32) words, bit j set = sub-step j
 *              starts a piece;
 *   chunk_piece  one per chunk: the piece id of its first sub-step;
 *   row_ptr    n_heavy + 1, row_pieces n_pieces: the piece ids of heavy
 *              row r, ascending (window order).
 * win is sized so the score rows of about one window stay L2-resident. A
 * plan whose group does not match the launch's lane layout is ignored. */
#define GMP_SEG_CHUNK_SUB 16
struct gmp_segplan {
  int64_t n_pos;
  int64_t n_pieces;
  int64_t win;
  int64_t group;
  const int32_t* perm;
  const uint32_t* starts;
  const int32_t* chunk_piece;
  const int64_t* row_ptr;
  const int32_t* row_pieces;
};

/* COO edge list in edge-id order (graph.py:98-100). */
typedef struct {
  int64_t n_nodes;
  int64_t m;
  const int32_t* src;
  const int32_t* dst;
} gmp_coo;

/* One operand matrix: rows keyed by its target, row-major with leading
 * dimension ld (elements). dim == 1 with d_out > 1 broadcasts (kernels.py:247-251). */
typedef struct {
  const void* data;
  int64_t ld;
  int32_t dim;
  int32_t target; /* GMP_SRC / GMP_DST / GMP_EDGE */
} gmp_operand;

/* Tunables; pass NULL for defaults. tile_cols = column-tile width of the
 * row kernels (0 = auto: sized so one column slice of the gathered operand
 * stays L2-resident - the reference's feature_parallel split, kernels.py:485-513). */
typedef struct {
  int32_t tile_cols;
  int32_t warps_per_cta;
  int32_t l2_budget_mb;
} gmp_tuning;

/* ---- schedule ---------------------------------------------------------- */

/* Workspace bytes gmp_build_schedule needs for an n_rows adjacency. */
size_t gmp_schedule_workspace_size(int64_t n_rows);

/* Sort rows by in-degree (descending, stable) into order_out (n_rows int32,
 * device) and report the heavy/non-empty prefix lengths into *sched_out
 * (synchronises `stream` to read them back). Replaces nothing in the
 * reference (its _GroupedWalk.run walks rows in id order, kernels.py:361-373);
 * this is the degree-binned scheduling of the north star. */
int gmp_build_schedule(const gmp_adj* adj, int32_t heavy_threshold, int32_t light_threshold,
                       int32_t* order_out, void* workspace, size_t workspace_bytes,
                       gmp_sched* sched_out, void* stream);

/* ---- g-SpMM -------------------------------------------------------------
 * Replaces kernels.gspmm (kernels.py:685-725) with its default strategy
 * node_parallel (_gspmm_node_parallel + _GroupedWalk, kernels.py:340-482):
 *   Z[v] = rho_{(u,e,v) in adj row v} phi(lhs, rhs)
 * op/lhs/rhs follow MessageFunc (kernels.py:72-104): copy_lhs reads lhs only,
 * copy_rhs reads rhs only; the unused operand has target GMP_NONE.
 * Z: (n_rows, d_out) row-major with ldz. arg (max/min only, else NULL):
 * (n_rows, d_out) int64, ld = d_out, the winning edge id, ties -> smallest
 * edge id, -1 for empty rows (ArgExtrema, kernels.py:147-154). Empty rows get
 * Z = 0. Mean divides by in-degree (0/0 -> 0, kernels.py:719-722).
 * counts (nullable): int64 (n_rows,) in-degree.
 * err_pos (nullable unless op == DIV): device int32 slot the caller presets to
 * INT32_MAX; receives the smallest adjacency POSITION whose divisor row holds
 * an exact zero (kernels.py:263-268); the caller maps it to eids[pos]. */
int gmp_gspmm(const gmp_adj* adj, const gmp_sched* sched, int op, int rho, int dtype,
              const gmp_operand* lhs, const gmp_operand* rhs,
              void* Z, int64_t ldz, int32_t d_out,
              int64_t* arg, int64_t* counts, int32_t* err_pos,
              const gmp_tuning* tuning, void* stream);

/* Staged sum / mean g-SpMM: the rows' edges are split over several
 * adjacencies (blocks with the same rows - e.g. one per source owner of a
 * row-partitioned graph, aggregated as each owner's feature shard lands) and
 * accumulated in one fp64 buffer acc (n_rows, ldacc), rounded once at the
 * end - the same single rounding as one gmp_gspmm over the union (the
 * reference accumulates every row in float64, kernels.py:396). Generalises
 * the reference's node_parallel split of destination ranges
 * (kernels.py:473-482) to a split of each row's edges.
 *   GMP_STAGE_FIRST: acc = partial            (Z untouched)
 *   GMP_STAGE_MID:   acc += partial           (Z untouched)
 *   GMP_STAGE_LAST:  Z = round(acc + partial) (mean: / deg_full[row])
 * deg_full (nullable, mean only): the full in-degree of each row over all
 * stages; NULL = this block's degree. Messages as gmp_gspmm except dot. */
enum { GMP_STAGE_FIRST = 0, GMP_STAGE_MID = 1, GMP_STAGE_LAST = 3 };
int gmp_gspmm_staged(const gmp_adj* adj, const gmp_sched* sched, int op, int rho, int dtype,
                     const gmp_operand* lhs, const gmp_operand* rhs,
                     double* acc, int64_t ldacc, int mode, const int64_t* deg_full,
                     void* Z, int64_t ldz, int32_t d_out, int32_t* err_pos,
                     const gmp_tuning* tuning, void* stream);

/* ---- heavy rows over the TMA gather4 ring (one packed column tile) --------
 * The packed-tile aggregation of kernels._gspmm_tiled (the wide copy_u /
 * u_mul_e path; replaces the same _GroupedWalk segment reduction,
 * kernels.py:340-466, for one 256 B column slice): heavy rows (schedule
 * prefix, degree > heavy_threshold) stream their 256 B source rows through
 * per-warp shared-memory rings fed by cp.async.bulk.tensor tile::gather4,
 * one persistent CTA per SM, chunk partials merged in fixed order; the other
 * rows run the row kernel. n_src_rows = rows of the packed lhs (its tensor
 * map's extent).
 * Conditions: dtype GMP_F32; op GMP_COPY_LHS (lhs GMP_SRC) or GMP_MUL (lhs
 * GMP_SRC, rhs a GMP_EDGE_POS scalar); rho GMP_SUM / GMP_MEAN; lhs rows are
 * 64 floats (ld == 64, 16 B aligned); d_out <= 64. Results equal gmp_gspmm's
 * (fp64 accumulation of the exact messages, one rounding).
 * The workspace is sized by gmp_gspmm_ring_workspace_size and filled once
 * per (adjacency, schedule) by gmp_gspmm_ring_prepare; it is then reused by
 * every call on that adjacency (calls on one stream; not concurrently). */
size_t gmp_gspmm_ring_workspace_size(const gmp_adj* adj, const gmp_sched* sched);
int gmp_gspmm_ring_prepare(const gmp_adj* adj, const gmp_sched* sched, void* ws,
                           size_t ws_bytes, void* stream);
int gmp_gspmm_ring(const gmp_adj* adj, const gmp_sched* sched, int op, int rho, int dtype,
                   const gmp_operand* lhs, const gmp_operand* rhs, int64_t n_src_rows, void* Z,
                   int64_t ldz, int32_t d_out, void* ws, size_t ws_bytes, void* stream);

/* ---- g-SDDMM ------------------------------------------------------------
 * Replaces kernels.gsddmm (kernels.py:744-836), default strategy
 * edge_parallel over COO (_gsddmm_chunked, kernels.py:732-741):
 *   M[e] = phi(lhs, rhs)  for every edge e, in edge-id order.
 * dot yields d_out == 1 (kernels.py:242-246). err_eid (nullable unless DIV):
 * device int32 slot preset to INT32_MAX; receives the smallest edge id whose
 * divisor row holds an exact zero. */
int gmp_gsddmm(const gmp_coo* coo, int op, int dtype,
               const gmp_operand* lhs, const gmp_operand* rhs,
               void* M, int64_t ldm, int32_t d_out, int32_t* err_eid,
               void* stream);

/* ---- edge_softmax ---------------------------------------------------------
 * Replaces messaging.edge_softmax (messaging.py:105-126: gspmm max, gsddmm
 * sub, exp, gspmm sum, gsddmm div) with two fused kernels: a per-destination
 * statistics pass over the in-adjacency (max and sum of exp per head) and an
 * edge-parallel pass over the COO list writing
 *   alpha[e,h] = exp(s[e,h] - max_{e'->v} s[e',h]) / sum_{e'->v} exp(...)
 * scores/alpha: (m, H) row-major keyed by edge id, leading dims lds/lda.
 * workspace: gmp_edge_softmax_workspace_size(n_rows, H) bytes of device
 * memory for the per-destination statistics. */
size_t gmp_edge_softmax_workspace_size(int64_t n_rows, int32_t H);
/* Workspace that also enables the windowed statistics pass (sched->sorted_eids
 * set, heavy rows present, large edge count); >= the plain size. */
size_t gmp_edge_softmax_workspace_size_ex(const gmp_adj* in_adj, const gmp_sched* sched, int32_t H,
                                          int dtype, int backward);

int gmp_edge_softmax_fwd(const gmp_adj* in_adj, const gmp_coo* coo, const gmp_sched* sched,
                         int dtype, const void* scores, int64_t lds, int32_t H,
                         void* alpha, int64_t lda, void* workspace, size_t workspace_bytes,
                         void* stream);

/* Fused u_add_v scores + edge_softmax (GAT attention, layers.py:110-113):
 * alpha = edge_softmax(s) with s[e,h] = el[src e, h] + er[dst e, h] computed
 * on the fly - the (m, H) score matrix is never written or re-read.
 * el, er: (n, H) node-keyed, leading dims lde / ldr. */
int gmp_edge_softmax_uv_fwd(const gmp_adj* in_adj, const gmp_coo* coo, const gmp_sched* sched,
                            int dtype, const void* el, int64_t lde, const void* er, int64_t ldr,
                            int32_t H, void* alpha, int64_t lda, void* workspace,
                            size_t workspace_bytes, void* stream);

/* Fused backward of edge_softmax (the composition of the four kernel
 * backwards of messaging.py:117-121, autodiff.py:398-418):
 *   ds[e,h] = alpha[e,h] * (g[e,h] - sum_{e'->v} alpha[e',h] g[e',h]) */
int gmp_edge_softmax_bwd(const gmp_adj* in_adj, const gmp_coo* coo, const gmp_sched* sched,
                         int dtype, const void* alpha, int64_t lda, const void* grad,
                         int64_t ldg, int32_t H, void* ds, int64_t ldds, void* workspace,
                         size_t workspace_bytes, void* stream);

/* Statistics pass alone of the fused u_add_v + edge_softmax: stat (n_rows,
 * 2H) of the feature dtype receives [max_h | 1/sum_h] per destination row
 * (rows without in-edges are left untouched). stat_bytes >= n_rows * 2H *
 * sizeof(element). Consumed by gmp_gat_aggregate. */
int gmp_edge_softmax_uv_stats(const gmp_adj* in_adj, const gmp_sched* sched, int dtype,
                              const void* el, int64_t lde, const void* er, int64_t ldr, int32_t H,
                              void* stat, size_t stat_bytes, void* stream);

/* ---- fused GAT attention aggregation -----------------------------------------
 * One head of the reference's GAT aggregation (layers.py:110-115: u_add_v ->
 * edge_softmax -> u_mul_e + sum) with the attention weights never stored:
 *   alpha_e = exp((el[src e] + er[dst e]) - max[dst e]) * inv_sum[dst e]
 * pack: (n) 32-byte rows, one sector per gathered edge - fp32
 * [er, max, inv_sum, w_hi, w_lo, 0, 0, 0], fp64 [er, max, inv_sum, w]
 * (max / inv_sum from gmp_edge_softmax_uv_stats; w = w_hi + w_lo is read by
 * the backward only, carried to fp64 accuracy), el: (n) with stride lde.
 * backward == 0: adj = in-adjacency, Z[v] = sum_{(u,e)->v} alpha_e X[u]
 * backward == 1: adj = the reverse graph's in-adjacency (= forward CSR),
 *                Z[u] = sum_{(v,e): u->v} alpha_e X[v]  (X = upstream grad rows,
 *                the transposed aggregation of Theorem 1), and, when t_out is
 *                not NULL, t_out[u] = sum_{(v,e): u->v} alpha_e w[v] (fp64) -
 *                the softmax-backward term of d el.
 * X: (n, d) with ldx, Z: (n, d) with ldz. z64 (nullable, (n, d) fp64 with
 * ldz64): also receives the unrounded fp64 rows of Z, so the backward's row
 * dots (S_v = dZ[v].Z[v], d el[u] = X[u].dX[u] - t[u]) are formed from the
 * fp64 aggregate like the reference's float64 composition, not from Z
 * rounded to fp32 (a cancelling dot would inherit |Z| 2^-24 per term). */
int gmp_gat_aggregate(const gmp_adj* adj, const gmp_sched* sched, int dtype, int backward,
                      const void* X, int64_t ldx, int32_t d, const void* el, int64_t lde,
                      const void* pack, void* Z, int64_t ldz, double* z64, int64_t ldz64,
                      double* t_out, const gmp_tuning* tuning, void* stream);

/* Node-level epilogue of the fused GAT backward: out[v * out_stride] =
 * sum_c A[v,c] B[v,c] - sub[v] (fp64 accumulation, sub nullable), e.g.
 * S_v = dZ[v].Z[v] straight into the pack's 4th column, and
 * d el[u] = X[u].dX[u] - t[u]. A and out have `dtype`; B has b_dtype (dtype,
 * or GMP_F64 for an fp32 A: the z64 rows of gmp_gat_aggregate). out_pair != 0:
 * the fp64 result is stored as hi = out[v*out_stride], lo = out[v*out_stride+1]
 * (the pack's w_hi / w_lo). */
int gmp_rowdot(int64_t n, int32_t d, int dtype, const void* A, int64_t lda, int b_dtype,
               const void* B, int64_t ldb, const double* sub, void* out, int64_t out_stride,
               int out_pair, void* stream);

/* ---- extrema gradient routing ----------------------------------------------
 * Replaces kernels.route_extrema_grad (kernels.py:843-857): dM[arg[v,k], k] =
 * dZ[v,k] for every cell with arg >= 0. dM (m, d) must be zero-filled by the
 * caller (ldm). */
int gmp_route_extrema(int64_t n_rows, int32_t d, int dtype, const int64_t* arg,
                      const void* dZ, int64_t lddz, void* dM, int64_t ldm, void* stream);

/* Workspace bytes of the extrema backward entry points below for n_rows
 * output rows of cells_per_row cells (d; the operand width for dot). */
size_t gmp_extrema_bwd_workspace_size(int64_t n_rows, int32_t cells_per_row);

/* Fused max/min backward for copy messages: scatters dZ straight into the
 * gradient of the copied operand without the (m, d) intermediate
 * (autodiff.py:398-412 + _route for copy_lhs/copy_rhs). target_index: for
 * GMP_SRC the COO src array (dX[src[arg]] += dZ), for GMP_EDGE NULL
 * (dW[arg] = dZ, one writer per cell). n_target_rows: rows of dOut. dOut
 * must be zero-filled. Source rows have several writers: their cells are
 * grouped by a stable radix sort (workspace, gmp_extrema_bwd_workspace_size)
 * and each (row, column) summed in fp64 in cell order and stored once -
 * deterministic, no float atomics, one rounding. */
int gmp_extrema_bwd_copy(int64_t n_rows, int32_t d, int dtype, const int64_t* arg,
                         const void* dZ, int64_t lddz, const int32_t* target_index,
                         int64_t n_target_rows, void* dOut, int64_t ldo, void* workspace,
                         size_t workspace_bytes, void* stream);

/* Fused max/min backward for binary messages (add / sub / mul / div / dot): the
 * gradient of the lhs (role 0) or rhs (role 1) operand, straight from the
 * winning edges arg (n_rows, d), without route_extrema_grad's (m, d) matrix
 * (kernels.py:843-857 + autodiff.py:289-372). Cell (v, k) with winner e adds
 * dZ[v,k] * dphi/doperand (fp64, the reference's expression order; 0 where a
 * divisor is 0) to the operand's row src[e] / v / e. own_dim: 1 for a
 * broadcast operand (its cells sum) else d. out (zero-filled by the caller,
 * rows of the operand's target, ldo; n_target_rows of them). Source rows
 * and broadcast operands have several writers: summed deterministically in
 * fp64 (sort-grouped as gmp_extrema_bwd_copy; workspace sized by
 * gmp_extrema_bwd_workspace_size(n_rows, d or own_dim for dot));
 * destination and edge rows of full-width operands are written once
 * (bit-exact; workspace may be NULL). dot: d == 1 and own_dim is the operand
 * width (the gradient row is dZ[v] * the other row). */
int gmp_extrema_bwd_binary(const gmp_coo* coo, int64_t n_rows, int32_t d, int dtype,
                           const int64_t* arg, const void* dZ, int64_t lddz, int op, int role,
                           const gmp_operand* lhs, const gmp_operand* rhs, void* out, int64_t ldo,
                           int32_t own_dim, int64_t n_target_rows, void* workspace,
                           size_t workspace_bytes, void* stream);

/* ---- row gather ------------------------------------------------------------
 * dst[i, :] = src[idx[i], :] for i < n (dim columns). Used to lay an edge
 * operand out in adjacency order once (idx = the adjacency's eids) so that a
 * multi-tile g-SpMM reads it coalesced instead of gathering it per tile. */
int gmp_gather_rows(int64_t n, int32_t dim, int dtype, const int32_t* idx, const void* src,
                    int64_t lds, void* dst, int64_t ldd, void* stream);

/* dst[p, :] = src[eids[p], :] for every position p of the adjacency (the
 * same result as gmp_gather_rows with idx = adj->eids), reading src one
 * L2-sized window of consecutive edge ids at a time: heavy rows are walked
 * per (window, row) - their positions inside a window are one contiguous run
 * when every row's edge ids ascend - so each src line is fetched from DRAM
 * about once; rows after the heavy prefix (through n_nonempty) gather
 * directly. Requires sched->sorted_eids == adj->eids when sched->n_heavy > 0
 * (callers use gmp_gather_rows otherwise). workspace: per-(heavy row, window)
 * bounds, gmp_gather_adj_workspace_size bytes. Replaces the per-call
 * fancy-index gather of an edge operand into chunk order
 * (kernels.py:255-296, _gather of W by edge id). */
size_t gmp_gather_adj_workspace_size(const gmp_adj* adj, const gmp_sched* sched, int32_t dim,
                                     int dtype);
int gmp_gather_adj(const gmp_adj* adj, const gmp_sched* sched, int32_t dim, int dtype,
                   const void* src, int64_t lds, void* dst, int64_t ldd, void* workspace,
                   size_t workspace_bytes, void* stream);

/* ---- column-tile packing ----------------------------------------------------
 * tile: a power of two >= 2.
 * packed (ceil(d/tile), n, tile): packed[t][r][c] = src[r][t*tile + c], zero
 * past column d. A g-SpMM over a wide src operand then runs one launch per
 * column tile on packed[t] (ld = tile): each per-edge gather is an aligned
 * run of whole sectors read with 128-bit loads, whatever src's ld (the
 * reference's feature_parallel column split, kernels.py:485-513, laid out
 * for L2 residency). gmp_unpack_tiles writes dst[r][c] for c < d back. */
int gmp_pack_tiles(int64_t n, int32_t d, int dtype, int32_t tile, const void* src, int64_t lds,
                   void* packed, void* stream);
int gmp_unpack_tiles(int64_t n, int32_t d, int dtype, int32_t tile, const void* packed, void* dst,
                     int64_t ldd, void* stream);

/* ---- neighbour sampling ------------------------------------------------------
 * Replaces graph.neighbor_sample's per-seed draw (graph.py:231-266): for seed
 * i (node seeds[i], in-edges indptr[seeds[i]] .. indptr[seeds[i]+1] of the
 * in-adjacency), k_i = out_off[i+1] - out_off[i] (= min(fanout, deg), computed
 * by the caller) distinct adjacency positions, uniform over k-subsets, written
 * ascending to out_pos[out_off[i] .. out_off[i+1]). The draw is a pure
 * function of (rng_seed, node id, k, deg). scratch: out_off[n_seeds] int64. */
int gmp_neighbor_sample(const int64_t* indptr, int64_t n_rows, const int64_t* seeds,
                        int64_t n_seeds, const int64_t* out_off, uint64_t rng_seed,
                        int64_t* scratch, int64_t* out_pos, void* stream);

/* ---- diagnostics ------------------------------------------------------------ */
const char* gmp_last_error(void);
const char* gmp_strerror(int status);
/* Number of kernel launches issued by this library since load (all threads). */
uint64_t gmp_launch_count(void);
int gmp_version(void);

/* ---- measurement ------------------------------------------------------------
 * L2 gather probe (no reference counterpart; the roofline denominator of the
 * row kernel): n_gathers random rows of row_bytes (64 or 256) from data
 * (rows x row_bytes, 16 B aligned), 8 rows in flight per lane group at full
 * occupancy. Time it with events on `stream`; GB/s = n_gathers * row_bytes / t.
 * sink: one float the kernel may write (keeps the loads live). */
int gmp_probe_l2_gather(const void* data, int64_t rows, int32_t row_bytes, int64_t n_gathers,
                        float* sink, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GMP_H_ */
