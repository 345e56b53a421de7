/*
 * sn_reorder.h -- C ABI of libsn_b200.so, a B200-native (sm_100a) implementation of the
 * eigenvalue-reordering step of StarNEig (arXiv 1905.04975).
 *
 * The operation (Eq. (7)): given a real Schur form S (upper
 * quasi-triangular with 1x1 and 2x2 diagonal blocks) and Schur vectors Q, compute an
 * orthogonal Q3 with  S = Q3 Ŝ Q3^T  such that the selected eigenvalues appear in the
 * leading diagonal blocks of Ŝ; overwrite S <- Ŝ and Q <- Q*Q3.
 *
 * The method: chains of diagonal windows of at most w rows.  The
 * window task applies adjacent 1x1/2x2 block swaps (Givens rotations and 3x3 Householder
 * reflectors) to the diagonal window and accumulates them into a k x k orthogonal
 * Z; right/left update tasks apply Z with level-3 (here FP64 tensor-core DMMA) products
 * to the column panel above the window, the row panel to its right and the columns of Q.
 * Readings of what the paper leaves unstated (window schedule, swap conventions,
 * stability test) are listed in DESIGN.md §3.
 *
 * Conventions for every entry point:
 *   - matrices are FP64, column-major, element (i,j) at a[i + j*ld], 0-based;
 *   - S and Q may be DEVICE pointers (cudaMalloc / torch CUDA tensors: the fast path) or
 *     HOST pointers (pageable or pinned; staged through device memory inside the call: Q is
 *     uploaded while the first levels run, and the final columns of S and Q are copied back
 *     as they become final; the staging memory is kept, see sn_release_workspace);
 *   - the caller owns every buffer; S and Q are modified in place (LAPACK style);
 *   - `select` is a HOST int32 array of n entries, one per row: nonzero = selected.  A
 *     2x2 block is selected if either of its rows is (LAPACK DTRSEN convention).
 *     On return it holds the achieved per-row mask (1 for rows < m after a full run);
 *   - return codes (LAPACK INFO style): 0 success; -i argument i invalid (n < 0, null
 *     pointer, ld too small, -2 also when S is not upper quasi-triangular); SN_ERR_REJECTED
 *     (+1) a block swap failed the stability test: S and Q hold a valid, partially
 *     reordered Schur form and select/m describe it; SN_ERR_CUDA (+2) a CUDA error;
 *     SN_ERR_NCCL (+3) an NCCL error or no communicator (sharded entry points);
 *     SN_ERR_UNSUPPORTED (+4) an option outside the supported range.
 *   - No CPU fallback: every arithmetic step runs in the library's CUDA kernels.  Without
 *     a usable CUDA device the compute entry points return SN_ERR_CUDA.
 */
#ifndef SN_REORDER_H
#define SN_REORDER_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SN_OK 0
#define SN_ERR_REJECTED 1
#define SN_ERR_CUDA 2
#define SN_ERR_NCCL 3
#define SN_ERR_UNSUPPORTED 4

/* Options (sn_default_opts fills the defaults). */
typedef struct sn_opts {
  int64_t window;            /* w: maximum window rows, 4 <= w <= 256 (default 256).
                                SURVEY §8c-2: ks = w/2 rows of movers per chain group. */
  int64_t inner_window;      /* rows of the in-kernel inner windows (default 64, <= 64) */
  int64_t max_windows;       /* stop after this many windows (prefix runs); < 0 = all */
  int64_t force_reject_window; /* debug: window (schedule order) whose swap is rejected; a value
                                  <= -2 rejects in every window of DAG level -2 - value (several
                                  partial windows in one level); -1 none */
  int64_t force_reject_swap;   /* debug: swap index (execution order within that window) */
  int32_t validate_lower;    /* 1: also check that S is exactly 0 below the subdiagonal
                                (n^2/2 device reads); the subdiagonal is always checked */
  int32_t serialize;         /* 1: debug, synchronise after every launch */
  int32_t q_stream_overlap;  /* 1 (default): Q updates on a second stream, overlapping the
                                next level's window tasks */
  int32_t profile;           /* 1: bracket every kernel launch with CUDA events on its own
                                stream and report per-kernel-kind times in sn_stats */
  int32_t lookahead;         /* 1 (default): the next level's window kernel waits only for the
                                update strips it reads; the rest overlaps it on a third stream */
  int32_t fuse_chain;        /* row f1: 1 = fuse the Q updates of two
                                consecutive windows x, y of a chain (y at the next level, above x,
                                overlapping it; no other window of y's level touching x's
                                columns): x's Q update is deferred to y's level and one CTA pass
                                per Q strip applies Zx, then Zy.  Results are bitwise those of the
                                unfused run.  Needs TMA-describable Q (16-byte aligned, even
                                ldQ), else ignored.  Default 0 (measured slower). */
  int32_t pencil_cluster;    /* row f2 (sn_reorder_pencil_ex): CTAs per window task, run as one
                                thread-block cluster that splits the window's row / column
                                applications (every CTA evaluates the step's transforms, so the
                                results are bitwise those of one CTA).  0 (default) = auto (as many
                                as the level's windows leave SMs for, <= 8), 1 = one CTA, 2..8. */
} sn_opts;

/* Statistics of one call. */
typedef struct sn_stats {
  int64_t windows;           /* windows executed */
  int64_t levels;            /* dependency levels of the window DAG */
  int64_t swaps;             /* block swaps scheduled in executed windows */
  int64_t swaps_by_type[4];  /* index (n1-1)*2 + (n2-1) */
  int64_t inner_windows;     /* in-kernel inner windows */
  int64_t rejected_window;   /* -1 if none */
  int64_t rejected_row;      /* first row j of the rejected swap (blocks n1 at j, n2 at j+n1) */
  int32_t rejected_n1, rejected_n2;
  double eq_flops;           /* equivalent update flops: per window with >= 1
                                swap, 2k^2 (n - j2) + 2k^2 j1 + 2k^2 n (Q term only if Q) */
  double ms_schedule;        /* host: structure scan + schedule construction */
  double ms_device;          /* device time of the reordering (CUDA events) */
  double ms_total;           /* wall time of the call */
  double ms_h2d, ms_d2h;     /* host-pointer staging copies (0 for device pointers) */
  /* per kernel kind: 0 window, 1 left update, 2 right update, 3 Q update, 4 scan */
  int64_t launches[5];       /* kernel launches of this call */
  double ms_kernel[5];       /* summed event time per kind (opts.profile = 1, else 0) */
  double flops_kernel[5];    /* algorithmic flops per kind (updates: 2 k^2 x panel extent) */
  double bytes_kernel[5];    /* algorithmic HBM bytes per kind (panel read + write once) */
  double flops_exec_kernel[5]; /* flops the panel kernels execute: Z^T row groups skip the K
                                  steps where Z is structurally zero; one-GPU
                                  executor only, else 0 */
  double g3_max_ratio;       /* generalized path: the largest stability-test residual ratio
                                (residual / threshold, G3) among the accepted swaps -- the
                                decision margin; 0 elsewhere */
  int64_t fused_q_pairs;     /* opts.fuse_chain: window pairs whose Q updates ran fused */
} sn_stats;

void sn_default_opts(sn_opts* o);
const char* sn_strerror(int code);

/* Eq. (7) with default options.  n: order; S (n x n, ld ldS >= max(1,n)); Q (n x n, ldQ >=
 * max(1,n)) or NULL (do not accumulate, LAPACK COMPQ='N'); select: host int32[n] in/out;
 * m: out, number of selected rows.  Synchronous with respect to the host. */
int sn_reorder_schur(int64_t n, double* S, int64_t ldS, double* Q, int64_t ldQ,
                     int32_t* select, int64_t* m);

/* Same with options, an optional host int8[n] block map output (0 = 1x1 block, 1/2 = first
 * and second row of a 2x2 block), optional statistics, and a CUDA stream (cudaStream_t, or
 * NULL for the legacy default stream) on which the device work is ordered.  Still
 * synchronous with respect to the host on return. */
int sn_reorder_schur_ex(const sn_opts* opts, int64_t n, double* S, int64_t ldS, double* Q,
                        int64_t ldQ, int32_t* select, int64_t* m, int8_t* bmap_out,
                        sn_stats* stats, void* stream);

/* ---- host-only helpers (no GPU needed): the window schedule of SURVEY §8c-2 ----
 * From a block map (bmap as above) and a per-row selection (0/1, block consistent),
 * sn_schedule_build computes the windows the library executes, in schedule order:
 * win_j1[t], win_k[t] (rows [j1, j1+k)), win_level[t] (its dependency level) and
 * win_nswap[t].  Pass NULL arrays to query only *nwin and *nswap.  Returns 0 or -i. */
int sn_schedule_build(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w,
                      int64_t* nwin, int64_t* nswap, int64_t* nlevels,
                      int64_t* win_j1, int64_t* win_k, int64_t* win_level, int64_t* win_nswap);

/* Lookahead split of window t's update strips (width `strip` = 64 in the executor): the
 * first crit_l[t] left-update strips and the last crit_r[t] right-update strips are applied
 * before the next dependency level's window kernel; the others overlap it.
 * Arrays of *nwin entries (schedule order).  Returns 0 or -i. */
int sn_schedule_lookahead(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w, int64_t strip,
                          int32_t* crit_l, int32_t* crit_r);

/* The swaps of window t of the schedule above, in the library's execution order inside
 * the window (inner windows of `inner_window` rows): global row j, sizes n1 (block at j),
 * n2 (moving block at j+n1).  cap = capacity of the arrays; returns the number of swaps or
 * a negative error. */
int64_t sn_schedule_window_swaps(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w,
                                 int64_t inner_window, int64_t t, int64_t cap,
                                 int64_t* swap_j, int8_t* swap_n1, int8_t* swap_n2);

/* ---- sharded (multi-GPU) reordering; PAPER.md P:158 (concurrent windows),
 * P:163-165 and P:189 (distributed blocks, implicit communication), P:249-258 ----
 * One process per GPU.  S is distributed over column blocks of width col_block (bc >= w):
 * global column j belongs to block b = j / bc on rank b % P and is stored, with all n rows,
 * at local column (b / P) * bc + (j - b * bc) of S_loc (n x user_cols, ld ldS_loc >= n,
 * user_cols from sn_dist_layout; columns past n in the last block are ignored).  Q is
 * distributed over contiguous row blocks: rank r holds rows [q0, q1) of Q (sn_dist_layout)
 * as Q_loc ((q1-q0) x n, ld ldQ_loc >= q1-q0), or Q_loc = NULL on every rank.  `select` is
 * the full host int32[n] selection on every rank (in/out, identical on return); m, bmap_out
 * and stats as for sn_reorder_schur_ex (stats count this rank's launches).  Per dependency
 * level the window task runs on the owner of column j1, its Z is broadcast to all ranks
 * (NCCL), every rank applies the left update to its own columns and the Q update to its own
 * rows, the owner applies the right update; windows straddling a block boundary first pull
 * the partner's columns [c, j2) (rows 0..j2) and push them back after the right update.
 * Collective: every rank of the communicator must call it with the same n, col_block,
 * options and selection.  Device or host shard pointers (host: staged inside the call). */

/* NCCL unique id (128 bytes) for sn_dist_init; create on one rank, share by any means. */
int sn_dist_unique_id(void* id_out);
/* Create the library's NCCL communicator: rank of world, on CUDA device `device`. */
int sn_dist_init(int rank, int world, const void* unique_id, int device);
int sn_dist_finalize(void);
/* Shard shapes of rank `rank`: S_loc columns, Q_loc rows [q0, q1).  Host only. */
int sn_dist_layout(int64_t n, int64_t P, int64_t col_block, int64_t rank, int64_t* user_cols, int64_t* q0,
                   int64_t* q1);
int sn_reorder_schur_dist(const sn_opts* opts, int64_t n, int64_t col_block, double* S_loc, int64_t ldS_loc,
                          double* Q_loc, int64_t ldQ_loc, int32_t* select, int64_t* m, int8_t* bmap_out,
                          sn_stats* stats, void* stream);
/* The same program for P ranks whose shards all live on the current device, executed in one
 * process phase by phase (messages become device copies, the broadcast a shared buffer):
 * the sharded data path on one GPU.  S_locs[r], Q_locs[r] (or Q_locs = NULL) as above. */
int sn_reorder_schur_dist_local(const sn_opts* opts, int64_t P, int64_t n, int64_t col_block, double* const* S_locs,
                                int64_t ldS_loc, double* const* Q_locs, int64_t ldQ_loc, int32_t* select,
                                int64_t* m, int8_t* bmap_out, sn_stats* stats, void* stream);
/* Host only: rank `rank`'s program as records of 8 int64 (returns the record count; pass
 * rec = NULL to size).  The halo width is w.  Records:
 *   (0, nlevels, nwin, ext_cols, q0, q1, hc, 0)                      header
 *   (1, level, t, j1, k, owner, partner, coff)                       window (level-sorted)
 *   (2, level, w0, w1, npull, nL, nR, nQ)                            level, then its
 *   (3, w, src, dst, nrows, ncols, src_lcol, dst_lcol)  pulls, (4, wl, cnt, x0, 0..) L strips,
 *   (5, ...) R strips, (7, ...) pushes, (8, ...) remaining L strips, (9, ...) remaining R
 *   strips, (6, ...) Q strips.  Execution order per level: pulls, window tasks, Z broadcast,
 *   the previous level's remaining L then R strips, this level's (critical) L then R strips,
 *   pushes; Q strips any time after the broadcast.
 * Local columns are in the extended layout: block lb at [lb*(bc+w), lb*(bc+w)+bc), its halo
 * slot after it. */
int64_t sn_dist_program(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w, int64_t col_block, int64_t P,
                        int64_t rank, int64_t cap, int64_t* rec);

/* Frees the device workspace the one-GPU entry points keep between calls (descriptors, Z
 * slots and, after host-buffer calls, the 2 n^2 doubles that stage S and Q). */
void sn_release_workspace(void);

/* ---- generalized reordering of a pencil ----
 * Eq. (7), right form: (S, T) = Q3 (Ŝ, T̂) Z3^T with Q3, Z3 orthogonal and
 * the selected generalized eigenvalues moved to the leading diagonal blocks of (Ŝ, T̂);
 * Q <- Q Q3, Z <- Z Z3 (Table 1, lists it beside the standard case).  (S, T) must be in
 * generalized real Schur form: S upper quasi-triangular (as for sn_reorder_schur_ex), T upper
 * triangular (not checked) with a diagonal 2x2 block on every 2x2 block of S.  The swap
 * transform follows the readings G1-G6 of DESIGN.md §3.1; on output every 2x2 block of T is
 * diagonal with t11 >= t22 > 0 and every 1x1 block of T that took part in a swap is >= 0.
 * S, T, Q, Z: column-major fp64 (Q and/or Z may be NULL), ld >= max(1, n), each a device or
 * a host pointer: a host matrix is copied to a compact device copy before the reordering and
 * back after it (also after SN_ERR_REJECTED), the caller keeping ownership; stats.ms_h2d /
 * ms_d2h time those copies.  The call is ordered on `stream` (a cudaStream_t, NULL = legacy
 * default stream) and returns when it has completed.  select/m/bmap_out/stats as sn_reorder_schur_ex (stats.eq_flops per
 * window 2k^2 (2(n-j2) + 2 j1 + n_Q + n_Z)).  opts: window, inner_window, max_windows,
 * force_reject_window/_swap and validate_lower are honoured.  Returns SN_OK,
 * SN_ERR_REJECTED (a swap failed the stability test: (S, T, Q, Z) hold a valid partially
 * reordered form that select / bmap_out describe), SN_ERR_CUDA, SN_ERR_UNSUPPORTED (options
 * out of range), or -i for an invalid argument i (-2 also when S is not
 * quasi-triangular). */
int sn_reorder_pencil_ex(const sn_opts* opts, int64_t n, double* S, int64_t ldS, double* T, int64_t ldT,
                         double* Q, int64_t ldQ, double* Z, int64_t ldZ, int32_t* select, int64_t* m,
                         int8_t* bmap_out, sn_stats* stats, void* stream);

/* Library version string. */
const char* sn_version(void);

/* ---- eigenvectors ----
 * PAPER.md Eq. (5): for every selected eigenvalue lambda of the real Schur form S,
 * a vector y with (S - lambda I) y = 0, computed by back substitution "protected against
 * floating-point overflow"; Eq. (6): the back-transform x = Q y.
 * Readings E1-E6: one column per selected 1x1 block, two (real part,
 * imaginary part of the eigenvector of lambda = a + i w, w > 0) per selected 2x2 block, in
 * block order; the block's own entries as LAPACK xTREVC; overflow protection by power-of-two
 * scalings keeping every stored value <= 2^500; each column (pair) normalised so that
 * max_i (|re_i| + |im_i|) = 1 (xTREVC).
 *
 * n: order; S: DEVICE pointer, n x n, ldS >= n, upper quasi-triangular in standard form (2x2
 * blocks [a b; c a], bc < 0: the output of sn_reorder_schur); Q: DEVICE n x n (ldQ >= n) or
 * NULL (X = Y, the Schur-basis vectors); select: HOST int32[n] (nonzero = selected; a 2x2
 * block if either row is); X: DEVICE n x ncols (ldX >= n) output, or NULL to query *ncols
 * only; ncols: out; scale_exp: HOST int32[ncols] or NULL: per column the e of the
 * protective scaling 2^-e applied before the normalisation; stats: optional; stream: the
 * CUDA stream (NULL: legacy default).  Synchronous with respect to the host.  Returns 0, -i
 * for argument i (-2 also if S is not quasi-triangular or not a device pointer),
 * SN_ERR_CUDA.  The library owns an n x ncols FP64 workspace when Q is given. */
typedef struct sn_eig_stats {
  int64_t columns;           /* columns of X */
  int64_t vectors;           /* eigenvectors (a complex pair counts once) */
  int64_t tiles;             /* row tiles of the blocked back substitution */
  int64_t rescales;          /* protective power-of-two rescalings performed */
  int64_t launches;          /* kernel launches */
  double flops_solve;        /* diagonal-tile back substitution flops */
  double flops_update;       /* off-diagonal update GEMM flops (2 i0 x tile x columns) */
  double flops_backtransform;/* X = Q Y GEMM flops (2 n x K extent x columns) */
  double ms_backsubstitution, ms_backtransform, ms_normalize, ms_device, ms_total;
} sn_eig_stats;

int sn_eigenvectors(int64_t n, const double* S, int64_t ldS, const double* Q, int64_t ldQ,
                    const int32_t* select, double* X, int64_t ldX, int64_t* ncols,
                    int32_t* scale_exp, sn_eig_stats* stats, void* stream);

/* ---- one bulge-chasing sweep of the multishift QR algorithm ----
 * bulges created at the top of the upper Hessenberg H and chased down the
 * diagonal by overlapping 3 x 3 Householder reflectors to complete one pipelined QR iteration
 * (Table 1).  Readings B1-B5: nshift (even) shifts sr[j] + i si[j] in
 * pairs (two real shifts, or a complex conjugate pair with sr equal and si opposite); pair j
 * makes bulge j, introduced by the reflector of (H^2 - sigma H + pi I) e1; the reflectors
 * follow xLARFG; the entries they annihilate are set to exact zeros.  On return
 * H <- U^T H U (upper Hessenberg) and Q <- Q U.
 *
 * Execution: chains of up to bulges_per_chain bulges spaced 4 rows apart, chased through
 * overlapping diagonal windows of <= window rows; each window's reflectors are accumulated
 * into a window-sized U and applied to the row panel right of the window, the column panel
 * above it and the columns of Q by the reordering's DMMA panel kernels (Fig. 1b).
 *
 * n: order; H: DEVICE n x n, ldH >= n, upper Hessenberg (exact zeros below the subdiagonal,
 * checked: -2 otherwise); Q: DEVICE n x n (ldQ >= n) or NULL; sr, si: HOST arrays of nshift
 * doubles; opts: NULL for the defaults; stats: optional; stream: CUDA stream (NULL: legacy
 * default).  Synchronous with respect to the host.  Returns 0, -i for argument i,
 * SN_ERR_CUDA, SN_ERR_UNSUPPORTED (window < 16 or > 256, or a chain that does not fit:
 * 4 (bulges_per_chain - 1) + 8 > window). */
typedef struct sn_sweep_opts {
  int64_t window;            /* rows of a window, 16..256 (default 160: <= 160 rows are staged
                                in shared memory) */
  int64_t bulges_per_chain;  /* bulges chased together, 1..60 (default 16) */
  int32_t q_stream_overlap;  /* 1 (default): Q updates on a second stream */
  int32_t lookahead;         /* 1 (default): the next level's window kernel waits only for the
                                strips it reads; the rest overlaps it on a third stream */
} sn_sweep_opts;

typedef struct sn_sweep_stats {
  int64_t windows, levels, chains, bulges, launches;
  double eq_flops;           /* equivalent update flops: per window 2k^2 ((n-j2) + j1 + n_Q) */
  double flops_left, flops_right, flops_q;
  double ms_device, ms_total;
} sn_sweep_stats;

void sn_sweep_default_opts(sn_sweep_opts* o);
int sn_qr_sweep(int64_t n, double* H, int64_t ldH, double* Q, int64_t ldQ, int64_t nshift,
                const double* sr, const double* si, const sn_sweep_opts* opts,
                sn_sweep_stats* stats, void* stream);

/* Host-only: the windows of one sweep in sequential order: rows [w0, w0+k), DAG level, chain,
 * and the chain steps [tau0, tau1) the window executes (in chain step tau, bulge b of the chain
 * makes its reflector at row tau - 4b if that lies in [0, n-2]).  Pass NULL arrays to query
 * the counts (w0 == NULL: none of the arrays is written). */
int sn_sweep_schedule(int64_t n, int64_t nshift, int64_t window, int64_t bulges_per_chain,
                      int64_t* nwin, int64_t* nlevels, int64_t* w0, int64_t* k, int64_t* level,
                      int64_t* chain, int64_t* tau0, int64_t* tau1);

#ifdef __cplusplus
}
#endif
#endif
