/*
 * mwu.h — C ABI of the B200-native MWU positive-LP hot path.
 *
 * Implements the per-iteration sweep of the multiplicative-weight-update solver of
 * Ju, Yesil, Sun, Chekuri, Solomonik (arXiv 2307.03307) for the normalised mixed
 * packing/covering feasibility LP  P x <= 1, C x >= 1, x >= 0 with nonnegative P, C
 * (PAPER.md eq:NormFeasibleLP), i.e. Alg. 2 with the Alg. 3 step
 * search, plus the outer bisection over the objective bound of the pure
 * packing / covering embeddings and over the density D of the densest-
 * subgraph dual.  "P:n" = line n of PAPER.md; readings Qn are in DESIGN.md.
 *
 * Conventions for every entry point
 *  - Every call returns an mwu_status; no C++ exception crosses the ABI and nothing aborts.
 *    On failure, mwu_last_error(ctx) (or mwu_last_error(NULL) for create failures, thread-
 *    local) holds a one-line message.  A CUDA error poisons the context: later calls on it
 *    return MWU_ERR_CUDA.
 *  - Input arrays are BORROWED for the duration of the call only and may be host or device
 *    pointers (the library copies them with cudaMemcpyDefault / UVA).  The context owns all
 *    device memory it allocates; mwu_destroy frees it.
 *  - Output arrays are caller memory, host or device.
 *  - All floating point is IEEE fp64.  All integer structure is built bit-exactly.
 *  - A context is not thread-safe; distinct contexts may be used from distinct threads.
 *  - A solve or probe that ends INFEASIBLE or ITER_LIMIT is a successful call (MWU_OK);
 *    the outcome is reported through the out-parameter / mwu_stats.
 */
#ifndef MWU_H
#define MWU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mwu_ctx mwu_ctx;

typedef enum {
  MWU_OK = 0,
  MWU_ERR_ARG = 1,      /* invalid argument (sizes, indices, negative values, duplicates ...) */
  MWU_ERR_CUDA = 2,     /* CUDA runtime error (sticky for the context)                       */
  MWU_ERR_OOM = 3,      /* device allocation failed                                          */
  MWU_ERR_NCCL = 4,     /* NCCL library missing or a collective failed                       */
  MWU_ERR_STATE = 5,    /* call out of order (e.g. mwu_step before mwu_probe_begin)           */
  MWU_ERR_NUMERIC = 6   /* non-finite weight sums (should not happen; reported, not masked)  */
} mwu_status;

/* Probe / solve outcome: FEASIBLE once min(Cx) >= 1 (reading Q6). */
typedef enum { MWU_RUNNING = 0, MWU_FEASIBLE = 1, MWU_INFEASIBLE = 2, MWU_ITER_LIMIT = 3 } mwu_outcome;

/* Why a probe stopped. MAXD_ZERO: max(d) = 0; ALPHA_LT_1: step search returned
 * alpha < 1; EMPTY_COVER_ROW: a covering row has no entries (Q17). */
typedef enum {
  MWU_REASON_NONE = 0, MWU_REASON_MAXD_ZERO = 1, MWU_REASON_ALPHA_LT_1 = 2,
  MWU_REASON_EMPTY_COVER_ROW = 3, MWU_REASON_ITER_LIMIT = 4, MWU_REASON_MIN_Z = 5
} mwu_reason;

/* Problem mode of an explicit CSR instance. PURE_PACKING: maximise <1,x> s.t.
 * Px <= 1 (C is ignored; the objective row (1/M)1^T x >= 1 is embedded per P:322).
 * PURE_COVERING: minimise <1,x> s.t. Cx >= 1 (P ignored; (1/M)1^T x <= 1 embedded). */
typedef enum { MWU_MIXED = 0, MWU_PURE_PACKING = 1, MWU_PURE_COVERING = 2 } mwu_mode;

/* Graph LPs of §3 over an implicit edge-list representation:
 *  BMATCH / MATCH: variables = edges, P = M (vertex-edge incidence, eq:incidence P:349-354),
 *                  pure packing; BMATCH expects a bipartite list (left ids < n_left).
 *  VCOVER:  variables = vertices, C = M^T, pure covering.
 *  DOMSET:  variables = vertices, C = I + A stored as an explicit symmetric CSR.
 *  DENSEST: variables = vertex-edge pairs z_{2e+b} (b = 0 for src[e], 1 for dst[e]),
 *           P = O/D (eq:oddshifted_incidence P:489-499), C = W (eq:interweaved P:483-485),
 *           mixed, with an outer search over D. */
typedef enum {
  MWU_G_BMATCH = 0, MWU_G_MATCH = 1, MWU_G_VCOVER = 2, MWU_G_DOMSET = 3, MWU_G_DENSEST = 4
} mwu_graph_kind;

/* Explicit sparse matrix in CSR form (canonical: column indices strictly increasing within a
 * row, values >= 0).  rowptr[rows+1] with rowptr[0] = 0, rowptr[rows] = nnz; vals may be NULL
 * meaning all entries are 1.0.  Pointers are host or device, borrowed during create. */
typedef struct {
  int64_t rows, cols, nnz;
  const int64_t *rowptr;
  const int32_t *colidx;
  const double *vals;
} mwu_csr;

/* Graph descriptor: n_edges undirected edges (src[e], dst[e]), 0 <= ids < n_vertices, no
 * self-loops, no duplicate edges.  Edge id e = position in the list (stable ids, Q29): the
 * variables of BMATCH/MATCH are indexed by e, of DENSEST by 2e+b.  n_left > 0 marks a
 * bipartite graph (BMATCH).  Pointers are host or device, borrowed during create. */
typedef struct {
  mwu_graph_kind kind;
  int64_t n_vertices, n_edges, n_left;
  const int32_t *src;
  const int32_t *dst;
} mwu_graph;

typedef struct {
  double eta_factor;     /* eta = eta_factor * ln(m) / eps (Q1); default 10             */
  int64_t max_iter;      /* MWU iterations per probe; default 5000                */
  int tol_prose;         /* Alg. 3 stop: 1 = ub-lb <= eps*lb (default, Q9);           */
                         /*              0 = ub-lb <= (1-eps)*lb (listing P:819)                 */
  int max_evals;         /* cap on f(alpha) evaluations per step search; 200        */
  double outer_rel_tol;  /* outer bisection stops at H <= (1+tol)L; <= 0 means eps/4 (Q14)       */
  int use_graph;         /* 1: whole probe = one CUDA-graph launch (conditional WHILE nodes);    */
                         /* 0: host-driven loop (debug)                                           */
  int bisect_depth;      /* bisection levels evaluated per search pass (1..3); default 3         */
  int device;            /* CUDA device ordinal; -1 = current device                             */
  int world, rank;       /* multi-GPU: number of ranks and this rank (1, 0 for one GPU)          */
  const void *nccl_id;   /* 128-byte ncclUniqueId from mwu_get_unique_id on rank 0 (world > 1)   */
  void *comm_group;      /* in-process rank group from mwu_simgroup_create (tests), or NULL       */
  int deterministic;     /* 1: every reduction in a fixed order (run-to-run bit-identical); 0     */
                         /* (default): the forward product of graph kinds is scattered with fp64 */
                         /* atomics into the L2-resident vertex vector (summation order varies   */
                         /* run to run at the 1e-16 level)                          */
  void *stream;          /* cudaStream_t on which the caller produces the input buffers and       */
                         /* consumes the outputs (e.g. torch.cuda.current_stream()); NULL = the    */
                         /* legacy default stream.  Every call that reads or writes caller memory */
                         /* first makes the library's internal stream wait for work queued on it,  */
                         /* and returns only once its outputs are complete (mwu_set_stream moves   */
                         /* a context to another stream).                                          */
  int block_l, block_r;  /* L2-blocked internal edge order of the fast edge-variable path         */
                         /* (the paper's CSB tiles P:901-923 at L2 scale): source /  */
                         /* destination row blocks of 2^block_l / 2^block_r packing rows; 0 =     */
                         /* per-kind defaults (densest 22 / 20, matching one source block / 22).  */
                         /* Result-neutral up to summation order; tests force small blocks so     */
                         /* multi-block orders run under the parity checks.                        */
  int compact_cover;     /* vcover / domset on one rank: the forward product compacts the covering */
                         /* rows with d^(z) > 0 for the search passes (1, default); 0 streams all  */
                         /* covering rows.  Result-neutral up to summation order.   */
  int step_rule;         /* step size of each MWU iteration (MWU_STEP_*):                          */
                         /*  BINARY (default) Alg. 3; NEWTON: Newton's method on        */
                         /*  f(alpha) - 1 warm-started from the previous step, (1 - eps)^p back-off */
                         /*  (readings Q34-Q36); STANDARD: alpha = 1 (Alg. 1) */
} mwu_options;

enum { MWU_STEP_BINARY = 0, MWU_STEP_NEWTON = 1, MWU_STEP_STANDARD = 2 };

typedef struct {
  int32_t outcome, reason;           /* last probe (or solve) outcome / reason                   */
  int64_t probes;                    /* outer-search probes run by the last mwu_solve            */
  int64_t iters_total;               /* MWU iterations summed over those probes (Q26)            */
  int64_t iters_last;                /* iterations of the last probe                             */
  int64_t search_evals, search_passes;/* f(alpha) evaluations / HBM passes (all probes)          */
  double bound;                      /* final M (pure modes) or D (densest)                      */
  double objective;                  /* <1, x_out> (pure modes) or D (densest); NaN for MIXED     */
  double certificate;                /* rho = max(Px)/min(Cx) of the returned x (Q6); NaN if none */
  double eta, alpha_last;
  int64_t n, m_P, m_C, nnz_P, nnz_C, empty_rows_dropped;
  double t_create_ms, t_solve_ms, t_loop_ms;
  double bytes_alg_per_iter;         /* algorithmic HBM bytes of one MWU iteration   */
  int64_t kernel_launches;           /* kernels launched by the last solve / probe run            */
  /* ---- SURVEY §8(b) additions */
  int64_t near_tie_count;            /* decisions taken within 1e-12 relative of their threshold   */
                                     /* (f(alpha) >= 1, min z >= 1, rho <= 1+eps; Q22), all probes */
  double t_phase_ms[4];              /* device time by phase, all probes of the last solve / run:  */
                                     /* [0] column (transposed products, direction; fused scatter  */
                                     /* of d^(y) on the fast paths), [1] step (forward products),  */
                                     /* [2] step search passes, [3] update (y, z, weights); from    */
                                     /* %globaltimer at the end of each phase, gaps included        */
  double max_Px_raw, min_Cx_raw;     /* max y and min z of the feasible probe's final iterate x    */
  double max_Px, min_Cx;             /* the same for the returned x_out = x / min(Cx) (Q15):        */
                                     /* max_Px = certificate, min_Cx = 1; NaN if none               */
  int64_t probe_graph;               /* 1: the probe loop ran as one CUDA-graph launch per probe   */
                                     /* (one GPU, or sharded over NCCL); 0: host-driven iterations  */
} mwu_stats;

/* Vector ids for mwu_get_vec (per-iteration parity, BASELINE north_star): */
enum {
  MWU_VEC_X = 0,   /* x [n]                         (x after the last update)          */
  MWU_VEC_D = 1,   /* d [n]        step direction of the last iteration              */
  MWU_VEC_Y = 2,   /* y = Px [m_P] cached; length 1 if P is the embedded row  */
  MWU_VEC_Z = 3,   /* z = Cx [m_C] cached; length 1 if C is the embedded row                 */
  MWU_VEC_DY = 4,  /* d^(y) = Pd [m_P]                                                */
  MWU_VEC_DZ = 5,  /* d^(z) = Cd [m_C]                                                         */
  MWU_VEC_WP = 6,  /* w_p = grad smax(y) [m_P] of the current y                   */
  MWU_VEC_WC = 7,  /* w_c = grad smin(z) [m_C] of the current z                   */
  MWU_VEC_G = 8,   /* g = P^T w_p [n] of the last iteration; needs mwu_set_record(1)  */
  MWU_VEC_H = 9,   /* h = C^T w_c [n]; needs mwu_set_record(1)                        */
  MWU_VEC_XBEST = 10 /* the solve's answer x_out (Q15), same as mwu_get_x                       */
};

/* Integer structure ids for mwu_get_structure (bit-exact tests, BASELINE north_star). */
enum {
  MWU_ST_INC_ROWPTR = 0,  /* int64 [n_vertices+1]: vertex -> incident slots CSR       */
  MWU_ST_INC_SLOTS = 1,   /* uint32 [2E]: slot 2e+b, sorted within each vertex                 */
  MWU_ST_DEGREE = 2,      /* int32 [n_vertices]                                                 */
  MWU_ST_PROW_OF_VERTEX = 3,/* int32 [n_vertices]: compacted packing row id or -1 (Q17)         */
  MWU_ST_C_ROWPTR = 4,    /* int64 [m_C+1]: CSR of C (DOMSET I+A, or CSR instances)             */
  MWU_ST_C_COLIDX = 5,    /* int32 [nnz_C]                                                      */
  MWU_ST_CT_ROWPTR = 6,   /* int64 [n+1]: CSC of C (transposed copy for the column side)        */
  MWU_ST_CT_ROWIDX = 7,   /* int32 [nnz_C]                                                      */
  MWU_ST_PT_ROWPTR = 8,   /* int64 [n+1]: CSC of P                                              */
  MWU_ST_PT_ROWIDX = 9,   /* int32 [nnz_P]                                                      */
  MWU_ST_P_ROWPTR = 10,   /* int64 [m_P+1]: CSR of P after dropping empty rows                  */
  MWU_ST_P_COLIDX = 11    /* int32 [nnz_P]                                                      */
};

/* Fill *opt with the defaults listed above. */
void mwu_default_options(mwu_options *opt);

/* Build a context for an explicit instance.  P is required for MIXED / PURE_PACKING and C for
 * MIXED / PURE_COVERING (the other may be NULL).  Builds the CSC copies (transposes) for the
 * column side, drops empty packing rows (Q17), records empty covering rows (solve then returns
 * INFEASIBLE / EMPTY_COVER_ROW) and column maxima ||P_{:,i}||_inf.  Errors
 * (MWU_ERR_ARG): negative values, column index out of range or not strictly increasing in a row,
 * P.cols != C.cols, an all-zero packing column in MIXED / PURE_PACKING mode (init undefined). */
mwu_status mwu_create_csr(const mwu_csr *P, const mwu_csr *C, mwu_mode mode,
                          const mwu_options *opt, mwu_ctx **out);

/* Build a context for a graph LP (see mwu_graph_kind) over the implicit edge-list storage:
 * vertex -> incident-slot CSR (sorted), compacted packing rows (isolated vertices dropped, Q17),
 * degrees; DOMSET additionally builds I + A as CSR.  Errors (MWU_ERR_ARG): ids out of range,
 * self-loops, duplicate edges, BMATCH endpoints not split by n_left. */
mwu_status mwu_create_graph(const mwu_graph *g, const mwu_options *opt, mwu_ctx **out);

/* Generalized matching: the mixed feasibility LP
 * l <= M x <= u, x >= 0 over the edge variables of g (M = vertex-edge incidence, eq:incidence), as
 * P = diag(1/u) M (rows of the vertices with finite u) and C = diag(1/l) M (rows with l > 0), both
 * built on device from the vertex -> incident-edge CSR, then solved by the explicit-CSR engine as
 * one MIXED probe (mwu_solve; x indexed by edge id, Q29).  lb, ub: [n_vertices] doubles, host or
 * device, borrowed; need 0 <= lb <= ub, ub > 0 (+inf = no upper bound), lb finite.  Errors
 * (MWU_ERR_ARG): graph errors as mwu_create_graph, bad bounds, no finite u or no positive l, an
 * edge with both endpoints unbounded above (x_e unbounded).  A vertex with l > 0 and no edges makes
 * the LP infeasible (solve returns INFEASIBLE / EMPTY_COVER_ROW). */
mwu_status mwu_create_gmatch(const mwu_graph *g, const double *lb, const double *ub, const mwu_options *opt,
                             mwu_ctx **out);

/* Full solve: outer geometric bisection over the bound (Q14) with a fresh Alg. 2 probe per
 * bound (pure modes / DENSEST), or a single probe (MIXED CSR).  max_iter <= 0 keeps the option.
 * *outcome receives the outcome (pure modes always end FEASIBLE with the best certified x or the
 * bracket witness; see mwu_stats.certificate). */
mwu_status mwu_solve(mwu_ctx *ctx, double eps, int64_t max_iter, int32_t *outcome);

/* Copy the answer x_out [n] (original variable order, Q29) into caller memory (host or device). */
mwu_status mwu_get_x(mwu_ctx *ctx, double *x, int64_t len);

mwu_status mwu_get_stats(mwu_ctx *ctx, mwu_stats *out);

/* Free everything the context owns (device memory, streams, graphs, NCCL communicator). */
void mwu_destroy(mwu_ctx *ctx);

/* Last error message of ctx, or of the calling thread's last failed create when ctx == NULL. */
const char *mwu_last_error(const mwu_ctx *ctx);

/* ---- probe-level hooks (fixed-step parity tests, step-strategy studies, benchmarks) ---- */

/* Start a probe at bound M (pure modes) or D (DENSEST); ignored for MIXED.  Initialises eta,
 * x, y = Px, z = Cx and the shifted weights. */
mwu_status mwu_probe_begin(mwu_ctx *ctx, double bound, double eps);

/* One MWU iteration of the current probe.  alpha > 0: fixed step (no search); alpha <= 0: the
 * Alg. 3 search.  *state receives MWU_RUNNING or the probe outcome. */
mwu_status mwu_step(mwu_ctx *ctx, double alpha, int32_t *state);

/* Run the current probe to completion (one CUDA-graph launch when use_graph = 1). */
mwu_status mwu_run_probe(mwu_ctx *ctx, int32_t *state);

/* Run exactly k more iterations of the current probe (or fewer if it ends) — benchmarking. */
mwu_status mwu_run_iters(mwu_ctx *ctx, int64_t k, int32_t *state);

/* Copy vector `which` (MWU_VEC_*) into caller memory; len must equal its length. */
mwu_status mwu_get_vec(mwu_ctx *ctx, int which, double *out, int64_t len);
/* Length of vector `which` in the current probe (0 if unavailable). */
int64_t mwu_vec_len(mwu_ctx *ctx, int which);

/* Make the context order its caller-memory reads / writes after `stream` (see mwu_options). */
mwu_status mwu_set_stream(mwu_ctx *ctx, void *stream);

/* Record g and h in every iteration (parity tests); costs 16 bytes/variable/iteration. */
mwu_status mwu_set_record(mwu_ctx *ctx, int on);

/* Copy integer structure `which` (MWU_ST_*) into caller memory; *bytes is in: capacity,
 * out: size written.  Returns MWU_ERR_ARG if the structure does not exist for this kind. */
mwu_status mwu_get_structure(mwu_ctx *ctx, int which, void *out, int64_t *bytes);

/* Run up to k iterations host-driven with CUDA events around every phase (benchmarks):
 * out10[2p] = total ms and out10[2p+1] = kernel launches of phase p in {0 column, 1 step
 * (forward products), 2 search passes, 3 update}; out10[8] = iterations, out10[9] = passes. */
mwu_status mwu_profile_iters(mwu_ctx *ctx, int64_t k, double *out10);

/* Scalars of the current probe: [eta, sigma, sP, SP, sC, SC, t, alpha_last, evals, passes]. */
mwu_status mwu_get_scalars(mwu_ctx *ctx, double *out10);

/* ---- multi-GPU ----
 * Edge-sharded kinds (BMATCH / MATCH / DENSEST with deterministic = 0): every rank passes the
 * SAME full graph to mwu_create_graph with opt.world = W, opt.rank = r; the library orders the
 * edges (L2-blocked internal order) and keeps the contiguous internal range mwu_shard_range(E,
 * W, r); the packing (vertex) rows are replicated and the scattered forward product is
 * sum-allreduced once per iteration.  Every later call (solve, probe hooks, vector hooks,
 * mwu_get_x) is collective: all ranks call it in the same order; vectors are returned whole on
 * every rank.  Other kinds return MWU_ERR_ARG for W > 1. */
/* Write a 128-byte ncclUniqueId (rank 0) to share through torch.distributed.  MWU_ERR_NCCL if
 * the NCCL library (libnccl.so.2 or $MWU_NCCL_LIB) cannot be loaded. */
mwu_status mwu_get_unique_id(void *out128);
/* [*e0, *e1): the internal edge range rank `rank` of `world` owns (host-only, no device work). */
mwu_status mwu_shard_range(int64_t n_edges, int world, int rank, int64_t *e0, int64_t *e1);
/* In-process group of `world` ranks on one device (one host thread per rank, host barriers; for
 * testing the sharded engine without several GPUs).  Pass it as opt.comm_group. */
mwu_status mwu_simgroup_create(int world, void **group);
void mwu_simgroup_destroy(void *group);

#ifdef __cplusplus
}
#endif
#endif /* MWU_H */
