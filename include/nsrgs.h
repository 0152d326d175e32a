/*
 * nsrgs.h — C-ABI of the B200-native NS-RGS hot path (libnsrgs.so).
 *
 * NS-RGS = "Newton-Schulz based Riemannian Gradient Scheme" for orthogonal group
 * synchronization, arxiv 2604.07372.  Citations "PAPER.md:L" are lines of the
 * paper's LaTeX source, with the section / equation / algorithm they fall in.
 *
 * Problem (PAPER.md:192-194 Eq. def:f problem, :232-235 Alg. 2 "Input"): given the
 * symmetric block measurement matrix A = [A_ij] in R^{nd x nd} with A_ii = 0
 * (PAPER.md:225-230 Eq. def:measurements), estimate X = (X_1; ...; X_n), X_i in O(d),
 * minimising F(X) = sum_{i != j} 1/2 ||X_i X_j^T - A_ij||_F^2.
 *
 * Conventions (all entry points):
 *  - Every call returns an nsrgs_status; 0 = success.  On failure the context keeps a
 *    message readable with nsrgs_last_error().  No call aborts the process.
 *  - Calls are SYNCHRONOUS with respect to the context's CUDA stream: they return after the
 *    device work they enqueue has completed (so device-side error words can be reported).
 *  - Multi-GPU (world > 1): one context per process/GPU; every call except
 *    nsrgs_plan / nsrgs_get_nccl_unique_id / nsrgs_last_error / nsrgs_version is
 *    COLLECTIVE — all ranks must make the same sequence of calls with the same scalar
 *    arguments (NCCL semantics).  A is row-block sharded by node: rank g owns nodes
 *    [g n/world, (g+1) n/world), i.e. A rows [g N/world, (g+1) N/world), N = n d, all N
 *    columns.  X is replicated on every rank.
 *  - Matrices are row-major.  "block stack" = n blocks of d x d, block i at offset i*d*d,
 *    i.e. the nd x d matrix (X_1; ...; X_n) of PAPER.md:128 (§1.4) in row-major order.
 *  - Element type of every matrix argument = the context dtype (float or double).
 *  - Pointers marked "host" are host memory (pinned or pageable); "device" are CUDA device
 *    pointers on the context's device.  The library never frees caller memory.
 *  - Update rule: Jacobi — every block of X^{t+1} is computed from X^t.
 */
#ifndef NSRGS_H
#define NSRGS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NSRGS_VERSION 1

typedef struct nsrgs_ctx nsrgs_ctx; /* opaque; one per (process, GPU) */

typedef enum {
  NSRGS_OK = 0,
  NSRGS_ERR_INVALID_ARG = 1,       /* bad size / pointer / unsupported (d, dtype) combination   */
  NSRGS_ERR_STATE = 2,             /* call out of order (e.g. step before A or X is set)        */
  NSRGS_ERR_CUDA = 3,              /* CUDA runtime/driver error (message has cudaGetErrorString) */
  NSRGS_ERR_NCCL = 4,              /* NCCL error or NCCL library not loadable                    */
  NSRGS_ERR_OOM = 5,               /* device allocation failed                                  */
  NSRGS_ERR_DIVERGENCE = 6,        /* retraction left the NS region: non-finite X or
                                      ||S||_F > 10 sqrt(d) after Algorithm 1       */
  NSRGS_ERR_SINGULAR = 7,          /* init polar sgn(Y_i) did not converge: sigma_min(Y_i) ~ 0
                                      (PAPER.md:141 needs full rank), or Cholesky of Y^T Y failed */
  NSRGS_ERR_EIG_NOT_CONVERGED = 8, /* spectral subspace iteration hit max_sweeps above tol      */
  NSRGS_ERR_NONFINITE = 9          /* objective / metric evaluated to NaN or Inf                */
} nsrgs_status;

typedef enum { NSRGS_F32 = 0, NSRGS_F64 = 1 } nsrgs_dtype;

/* Context description. */
typedef struct {
  int64_t n;                    /* number of nodes (group elements), n >= 2                     */
  int32_t d;                    /* block size; supported: 2..16, 20, 24, 25, 32 (F32), 2..6 (F64) */
  int32_t dtype;                /* nsrgs_dtype: storage + arithmetic type of A, X (fp64 partials) */
  int32_t rank, world;          /* world >= 1, 0 <= rank < world, n % world == 0; for world > 1
                                   also (n/world)*d*sizeof(dtype) % 16 == 0 (TMA row-segment
                                   alignment of the per-rank column slices)                      */
  int32_t device;               /* CUDA device ordinal the context binds to                      */
  const void *nccl_unique_id;   /* host, 128 bytes from nsrgs_get_nccl_unique_id() on rank 0,
                                   broadcast by the caller; must be NULL iff world == 1 (test-only
                                   exception: env NSRGS_EMULATE_RANKS=1 allows world > 1 with NULL;
                                   collectives become no-ops, for rank-by-rank kernel tests)     */
  void *cuda_stream;            /* cudaStream_t to enqueue on; NULL = library-created stream    */
} nsrgs_desc;

/* Static sharding plan (pure host arithmetic; callable without a GPU). */
typedef struct {
  int64_t n_local;      /* nodes owned by this rank = n / world                               */
  int64_t node0;        /* first owned node = rank * n_local                                  */
  int64_t rows_local;   /* A rows owned = n_local * d (also the width of one rank's X slice)  */
  int64_t row0;         /* first owned A row = node0 * d                                      */
  int64_t col_tile;     /* X/A column tile width (elements) of the device layout = 128        */
  int64_t tiles_per_rank; /* ceil(rows_local / col_tile)                                       */
  int64_t x_elems;      /* elements of one device X buffer = world*tiles_per_rank*d*col_tile  */
  int64_t x_slice_elems;/* elements of one rank's contiguous X slice (NCCL all-gather count)  */
} nsrgs_plan_t;

int nsrgs_version(void);

/* Pure host: the sharding plan of (n, d, world, rank).  Returns INVALID_ARG if the
 * combination is not supported.  Device X layout ("tile layout"), with
 * g = c / rows_local the owning rank, cl = c % rows_local, T = col_tile:
 *   d <= 10: tile base b = (g*tiles_per_rank + cl/T) * d * T, o = cl % T; element (row c,
 *            component k) at b + (k & ~1)*T + 2*o + (k & 1), except for odd d and k = d-1:
 *            b + (d-1)*T + o;
 *   d > 10 : (g*tiles_per_rank*T + cl) * d + k   (row-major stack, rank slice padded to T rows);
 * padding entries are zero.  */
int nsrgs_plan(int64_t n, int32_t d, int32_t world, int32_t rank, nsrgs_plan_t *out);

/* Pure host: convert between the nd x d row-major stack and the tile layout above
 * (host buffers, element type by dtype).  Used by tests of the sharded layout. */
int nsrgs_pack_host(int64_t n, int32_t d, int32_t world, int32_t dtype, const void *stack, void *tiled);
int nsrgs_unpack_host(int64_t n, int32_t d, int32_t world, int32_t dtype, const void *tiled, void *stack);

/* Rank 0 only: create an NCCL unique id (128 bytes, host) to broadcast to all ranks. */
int nsrgs_get_nccl_unique_id(void *out128);

/* Create / destroy a context.  Allocates the library-owned X buffers (2 x x_elems), partial
 * buffers and (world > 1) the NCCL communicator.  *out is NULL on failure. */
int nsrgs_create(const nsrgs_desc *desc, nsrgs_ctx **out);
int nsrgs_destroy(nsrgs_ctx *ctx);
const char *nsrgs_last_error(const nsrgs_ctx *ctx); /* never NULL; "" if no error */

/* Use a caller-owned A shard: device pointer to rows_local x (n d) elements, row stride lda
 * (elements, lda >= n d, lda*sizeof(dtype) % 16 == 0, pointer 16-byte aligned).  BORROWED:
 * read-only, must outlive the context (or the next attach/generate).  The diagonal blocks
 * A_ii of the owned rows must be zero; the library does not check symmetry.
 * Computes ||A||_F^2 (fp64, all-reduced) for the objective.  (Alg. 2 Input.) */
int nsrgs_attach_A(nsrgs_ctx *ctx, const void *A_shard_dev, int64_t lda);

/* Generate the synthetic instance of PAPER.md:59-66 / :225-230 on the device (library-OWNED
 * A shard; no host traffic): Z_i = Q of QR(G_i) with diag(R) > 0, G_i Gaussian from Philox
 * counter (i,0,q,1); W_ij (i<j) from counter (i,j,q,2); A_ij = round(Z_i Z_j^T + sigma W_ij),
 * A_ji = A_ij^T, A_ii = 0.  Each rank generates only its
 * own rows; the instance is independent of world.  Z_out: host, n*d*d elements of dtype,
 * nullable — receives the ground truth.  sigma >= 0. */
int nsrgs_generate(nsrgs_ctx *ctx, uint64_t seed, double sigma, void *Z_out_host);

/* As nsrgs_generate with incomplete observations (§4.1):
 * the unordered pair {i < j} is observed iff u < p, u = first uniform of Philox counter
 * (i, j, 0, 4); unobserved blocks A_ij = A_ji = 0 (stored densely — the bytes per pass do not
 * shrink).  Use eta = 1/(n p) in nsrgs_run.  p in (0, 1]. */
int nsrgs_generate_observed(nsrgs_ctx *ctx, uint64_t seed, double sigma, double p, void *Z_out_host);

/* Block-sparse (BSR) storage of an incompletely observed instance (
 * PAPER.md:300-310 §4.1: each pair {i, j} observed with probability p, unobserved A_ij = 0;
 * use eta = 1/(n p)).  Only observed blocks are stored, so an A pass reads ~p
 * of the dense bytes.  Layout (device, library-OWNED after generate, BORROWED after attach):
 *   rowptr[n_local + 1] (int64): local node row il owns blocks [rowptr[il], rowptr[il+1]);
 *   col[nnzb] (int32): global node j of block b (ascending within a row; a row may end with
 *                      zero blocks whose col is the row's own node — the generator pads each
 *                      row to a multiple of 4 blocks);
 *   vals[nnzb][d][d] (float, row-major): A_{node0+il, col[b]}.
 * The diagonal block A_ii must not be stored unless it is zero.
 * nsrgs_generate_observed_bsr builds the SAME instance as nsrgs_generate_observed (same
 * counters; every stored block is bitwise the dense block; the dense shard is released).
 * F32 contexts, every supported d, any world.  nsrgs_set_symmetric and nsrgs_copy_A_rows
 * return NSRGS_ERR_STATE while block-sparse storage is active; a dense generate / attach
 * switches back.  nsrgs_get_A_bsr copies the arrays to host (each pointer nullable;
 * *nnzb_out receives nnzb).  nsrgs_attach_A_bsr checks the structure on the device before
 * using it (rowptr[0] = 0, non-decreasing, rowptr[n_local] = nnzb, every col in [0, n)) and
 * returns NSRGS_ERR_INVALID_ARG otherwise, leaving the previous A in place; the values and
 * the column order within a row are not checked. */
int nsrgs_generate_observed_bsr(nsrgs_ctx *ctx, uint64_t seed, double sigma, double p, void *Z_out_host);
int nsrgs_attach_A_bsr(nsrgs_ctx *ctx, const int64_t *rowptr_dev, const int32_t *col_dev, const void *vals_dev,
                       int64_t nnzb);
int nsrgs_get_A_bsr(nsrgs_ctx *ctx, int64_t *nnzb_out, int64_t *rowptr_host, int32_t *col_host, void *vals_host);

/* Copy rows [row0, row0+nrows) of THIS rank's A shard (local row index) to host `out`
 * (nrows x n d, dense).  Diagnostic / sampled-parity helper. */
int nsrgs_copy_A_rows(nsrgs_ctx *ctx, int64_t row0, int64_t nrows, void *out_host);

/* Spectral initialisation (Alg. 2): Y = top-d eigenvectors of A
 * by subspace iteration Y <- A Y (the same panel A.X kernel as nsrgs_step) with Cholesky-QR,
 * Y_0 Gaussian from Philox counter (r,0,q,3), stopped when ||Y_new - Y_old(Y_old^T Y_new)||_F
 * < tol or after max_sweeps; then X^0 = sgn(Y) blockwise by scaled Newton-Schulz (no SVD).
 * A tol below the dtype's rounding floor of the change (50 sqrt(d) eps: fp32 6.7e-6 at d = 5)
 * is raised to that floor, and a change that stalls within 10x of the floor counts as
 * converged; a slowly contracting subspace keeps iterating.  Sets the current iterate.
 * sweeps_used: host, nullable (sweeps actually run; small instances read the change back every
 * 4 sweeps, so it may exceed the first sweep that met tol by up to 3).  Returns
 * NSRGS_ERR_EIG_NOT_CONVERGED (X^0 still set) if tol was not reached within max_sweeps,
 * NSRGS_ERR_SINGULAR if the Cholesky factor of Y^T Y or the polar factor of a block failed. */
int nsrgs_init_spectral(nsrgs_ctx *ctx, uint64_t seed, int max_sweeps, double tol, int *sweeps_used);

/* One NS-RGS iteration t -> t+1 of Algorithm 2:
 *   G_i = sum_{j!=i}(X_i - A_ij X_j),  F_i = X_i - eta P_{T_{X_i}}(G_i),  X_i <- S(F_i),
 * P_T(G) = (G - X G^T X)/2, S = K steps of Algorithm 1.
 * eta > 0 (paper: mu = 1/n); K >= 0.  objective_before: host, nullable —
 * receives F(X^t) computed from fp64 partials fused into the same A pass.
 * Arithmetic of B = A X: fp32 (F32) / fp64 (F64) FMAs on the CUDA cores for d <= 10; for d > 10
 * (and d = 10 on dense fp32 shards >= 4 GB at world 1) 3xTF32 on the tensor cores with exact
 * hi/lo splits and the accumulator drained into fp32 sums every column tile: per-step error
 * vs fp64 <= 3e-7 (same 1e-6 bar as the CUDA-core pass; stats.wide_tc tells which pass ran). */
int nsrgs_step(nsrgs_ctx *ctx, double eta, int K, double *objective_before);

/* T iterations of nsrgs_step.  objective_trace: host, nullable, length T, receives
 * F(X^0..X^{T-1}).  Returns NSRGS_ERR_DIVERGENCE if any iteration left the NS region. */
int nsrgs_run(nsrgs_ctx *ctx, int T, double eta, int K, double *objective_trace);

/* GPM, the paper's comparison method (§4.1; definition):
 * T iterations of X_i <- sgn(sum_{j!=i} A_ij X_j) on the same A pass, the sign taken by
 * Newton-Schulz from B_i/||B_i||_F to convergence (no SVD).  objective_trace as nsrgs_run.
 * Returns NSRGS_ERR_SINGULAR if a sign did not converge (rank-deficient B_i). */
int nsrgs_gpm_run(nsrgs_ctx *ctx, int T, double *objective_trace);

/* The paper's experimental protocol (§4.1): iterate `algorithm` from the
 * current X^0 until R^t = (F(X^t) - F(X^{t+1}))/F(X^{t+1}) < stop_tol or max_iter iterations.
 * On return X = X^{t_stop}; *iters_used = t_stop; objective_trace (host, nullable, length
 * max_iter + 1) receives F(X^0..X^{t_stop}).  eta, K are used by NSRGS_ALG_NSRGS only.
 * F32 contexts evaluate F with nsrgs_objective_fp64's pass (one extra A pass per iteration) so
 * that the stop is decided by the iteration rather than by fp32 rounding of F; F64 contexts use
 * the fp64 partials fused into the iteration's own pass. */
typedef enum { NSRGS_ALG_NSRGS = 0, NSRGS_ALG_GPM = 1 } nsrgs_algorithm;
int nsrgs_solve(nsrgs_ctx *ctx, int algorithm, int max_iter, double eta, int K, double stop_tol, int *iters_used,
                double *objective_trace);

/* F(X) of the current iterate (PAPER.md:70-72 Eq. def:f); one A pass. */
int nsrgs_objective(nsrgs_ctx *ctx, double *F_out);

/* F(X) of the current iterate with every product A_rc (X_r . X_c) formed and summed in fp64
 * (F32 contexts; dense or block-sparse A): exact to ~1e-16 relative for the stored fp32 iterate,
 * where nsrgs_objective's fp32-accumulated <X, A X> carries ~1e-7 relative error.  One extra A
 * pass (fp64 FMA bound for d >= 10).  This is the evaluator nsrgs_solve uses for the stopping
 * rule on F32 contexts.  INVALID_ARG for F64 contexts (use nsrgs_objective). */
int nsrgs_objective_fp64(nsrgs_ctx *ctx, double *F_out);

/* Recovery metrics of the current iterate against ground truth Z (n*d*d elements of dtype,
 * host if Z_on_device == 0 else device): out[0] = Rel.Err. = ||ZZ^T - XX^T||_F/||ZZ^T||_F
 * (PAPER.md:314-317), out[1] = d_F(X, Z) = min_Q ||X - ZQ||_F via
 * ||X||^2 + ||Z||^2 - 2||Z^T X||_* (PAPER.md:633-637), out[2] = MSE = d_F^2/n
 * (PAPER.md:369-372).  fp64 Grams on the device. */
int nsrgs_alignment_error(nsrgs_ctx *ctx, const void *Z, int Z_on_device, double out[3]);

/* Set / get the full current iterate X (n*d*d elements, block stack).  host if on_device==0. */
int nsrgs_set_X(nsrgs_ctx *ctx, const void *X, int on_device);
int nsrgs_get_X(nsrgs_ctx *ctx, void *X, int on_device);

/* Symmetric half-storage pass (A symmetric by PAPER.md:227): when enabled,
 * every A pass reads only the upper half of A (row panel p: columns >= its first row, tile
 * aligned) and forms B = A X from both A_ij X_j and the mirrored A_ij^T X_i — half the HBM
 * bytes, twice the FMAs per byte.  Requires the stored A to be exactly symmetric (true for
 * nsrgs_generate; the caller's responsibility for nsrgs_attach_A).  Supported: world == 1,
 * F32, d in [2, 6]; otherwise NSRGS_ERR_INVALID_ARG.  enable = 0 returns to the dense pass.
 * Results are deterministic but differ from the dense pass by fp32 summation order. */
int nsrgs_set_symmetric(nsrgs_ctx *ctx, int enable);

/* Launch configuration + measurement hooks (bench / tests).  */
typedef struct {
  int32_t grid, threads, stages, rows_per_panel;     /* panel kernel launch shape              */
  int32_t cut_panels;   /* panels split into column-range units by the work queue (combined in order) */
  int64_t panels, smem_bytes;
  double panel_ms_total;        /* summed CUDA-event time of panel kernel launches since reset */
  int64_t panel_launches;       /* number of panel kernel launches since reset                 */
  int64_t kernel_launches;      /* all library kernel launches since reset                     */
  double ns_region_max;         /* max over nodes of ||I - F_i^T F_i||_F seen since reset        */
  double a_fro2;                /* ||A||_F^2 (global)                                           */
  int32_t symmetric;            /* 1 if the symmetric half-storage pass is active               */
  int64_t a_bytes_per_pass;     /* A bytes one pass requests from memory (full shard, ~half for
                                   the symmetric pass; values + col + rowptr for block-sparse)    */
  int32_t p2p;                  /* 1 if X^{t+1} is exchanged by the fused NVLink-store path     */
  int32_t bsr;                  /* 1 if the block-sparse storage is active                      */
  int64_t bsr_nnzb;             /* stored blocks of this rank (incl. zero padding blocks)       */
  int32_t bsr_slab;             /* 1 if the block-sparse pass runs the column-group slab variant  */
  int32_t bsr_g4;               /* 1 if it gathers X records with TMA tile::gather4              */
  int32_t wide_tc;              /* d > 10: 2 if the A.X pass runs 3xTF32 on tcgen05 (default), 1 on
                                   mma.sync (NSRGS_WIDE_MMA=1), 0 on CUDA cores (=0); d = 10: 2 if
                                   it runs on the tcgen05 pass (dense fp32 shard >= 4 GB at world 1,
                                   NSRGS_NARROW_TC), else 0; 0 for d < 10                          */
} nsrgs_stats_t;
int nsrgs_get_stats(nsrgs_ctx *ctx, nsrgs_stats_t *out);
int nsrgs_reset_stats(nsrgs_ctx *ctx, int enable_panel_timing);

/* Debug: per-CTA phase timestamps (%globaltimer, ns) of the dense panel kernel.  max_iters > 0
 * arms a [max_iters][grid][16] buffer for the following launches (slots, per iteration: 0
 * producer's first unit, 1 X ready after the readiness wait, 2 consumers' first unit,
 * 3 partial sums flushed, 4 CTA exit, 5 last unit streamed, 6 its B rows complete, 11 SM id;
 * unused slots 0); max_iters == 0 copies it to out_host (host, may be NULL) and disarms. */
int nsrgs_debug_timestamps(nsrgs_ctx *ctx, int max_iters, unsigned long long *out_host);

/* Measurement: HBM read-stream ceiling of this GPU (bench.py's roofline denominator).  Streams
 * `bytes` (>= 32 KB; far larger than L2 for a DRAM figure) of the 16-byte-aligned DEVICE buffer
 * buf_dev with the dense pass's access pattern (one CTA per SM, 32 KB cp.async.bulk copies into
 * a 6-stage shared-memory ring, nothing written back), once to warm up and then `reps` times on
 * `cuda_stream` (NULL: legacy default stream) of the current device; *best_gbs = bytes read per
 * second of the fastest rep (1e9 B/s).  INVALID_ARG for bad arguments, CUDA / OOM on failure. */
int nsrgs_probe_read_stream(const void *buf_dev, int64_t bytes, void *cuda_stream, int reps, double *best_gbs);

/* Test-only: link `world` rank contexts created in ONE process with NSRGS_EMULATE_RANKS=1 (no
 * communicator) so that the fused P2P X exchange runs between them on one GPU: each rank's
 * epilogue stores X^{t+1} into every linked rank's buffer and bumps its arrival counters.  The
 * caller must step the ranks one after another (rank 0..world-1 for iteration t, then t+1):
 * a launch only waits for counters the previous round already completed, so no kernel ever
 * waits on another.  ctxs[r] must be rank r of the same (n, d, dtype), d <= 10.  Returns
 * INVALID_ARG otherwise.  Real multi-GPU contexts set this path up in nsrgs_create (CUDA IPC
 * mapping of every peer's X buffers over NVLink, verified by a write handshake; NCCL
 * all-gather fallback if any rank cannot map a peer; NSRGS_P2P=0 forces the fallback). */
int nsrgs_debug_link_peers(nsrgs_ctx **ctxs, int world);

/* Test-only: join `world` rank contexts created in ONE process with NSRGS_EMULATE_RANKS=1 into
 * an in-process rank group whose collectives exchange real data (the multi-GPU collectives of
 * nsrgs_generate, nsrgs_init_spectral, nsrgs_run / nsrgs_step / nsrgs_gpm_run / nsrgs_solve,
 * nsrgs_objective(_fp64) on one GPU): the all-reduce of fp64 partials sums every rank's buffer
 * in rank order, the X all-gather copies the other ranks' slices.  Each rank's calls must be
 * issued from its own host thread (every call is collective, as with NCCL); collectives are
 * host-synchronised, so no kernel waits for another rank.  A rank that does not reach a
 * collective within 120 s fails it (and every later one) with NSRGS_ERR_NCCL.  ctxs[r] must be
 * rank r of the same (n, d, dtype, device), not linked by nsrgs_debug_link_peers (the fused P2P
 * exchange needs concurrently running ranks, i.e. one GPU per rank).  Returns INVALID_ARG
 * otherwise.  The group lives until its last context is destroyed. */
int nsrgs_debug_group(nsrgs_ctx **ctxs, int world);

#ifdef __cplusplus
}
#endif
#endif /* NSRGS_H */
