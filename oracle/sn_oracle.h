/*
 * sn_oracle.h -- CPU oracle for Schur-form eigenvalue reordering.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the plain, slow, obviously-correct CPU
 * reference that the CUDA path is checked against.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It shares no code with paper_1905_04975_b200/ (the product),
 * and the product never calls it.
 *
 * What it computes (PAPER.md = P:n lines, SPEC.md = S:n lines):
 *   Eq. (7):  S = Q3 Ŝ Q3^T, the selected eigenvalues of the real
 *   Schur form S moved to the leading diagonal blocks of Ŝ, Q ← Q·Q3.
 *   The method: chains of diagonal windows; inside a
 *   window, adjacent 1x1/2x2 block swaps ("Givens rotations and 3x3
 *   Householder reflectors") are accumulated into Z and then applied
 *   to the row panel on the right (left update), the column panel
 *   above (right update) and the columns of Q.
 *
 * Conventions: column-major, 0-based indices, element (i,j) of a matrix with
 * leading dimension ld is a[i + j*ld].  All arithmetic is IEEE fp64.
 *
 * Error convention (LAPACK INFO style): 0 ok, <0 argument -i invalid,
 * +1 a swap was rejected (state consistent, see or_reorder).
 */
#ifndef SN_ORACLE_H
#define SN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- scalar transform constructions (readings c4 #2, #3) ---- */

/* Givens (a1): given f, g returns c, s, r with [c s; -s c][f; g] = [r; 0],
 * c >= 0, r = sign(f)*hypot(f,g) (LAPACK >= 3.10 xLARTG convention). */
void or_lartg(double f, double g, double* c, double* s, double* r);

/* 3-element Householder: H = I - tau*v*v^T, v = (1, x'), maps (alpha, x) to
 * (beta, 0, 0) with beta = -sign(alpha)*||(alpha,x)|| (xLARFG convention).
 * On return x[0..1] holds v(2:3), *alpha holds beta. */
void or_larfg3(double* alpha, double x[2], double* tau);

/* Standardise a 2x2 block (xLANV2 semantics):
 * [a b; c d] = [cs -sn; sn cs] [aa bb; cc dd] [cs sn; -sn cs], with either
 * cc == 0 (real eigenvalues) or aa == dd and bb*cc < 0 (complex pair).
 * In/out: a b c d.  Out: cs, sn. */
void or_lanv2(double* a, double* b, double* c, double* d, double* cs, double* sn);

/* Small Sylvester solve T11*X - X*T22 = scale*T12 (n1,n2 in {1,2}) by Gaussian
 * elimination with complete pivoting on the Kronecker system (c4 #4).
 * T11 n1xn1, T22 n2xn2, T12 n1xn2, X n1xn2, all column-major with ld 2.
 * Returns 1 if a pivot had to be perturbed (near-singular), else 0. */
int or_sylv(int n1, int n2, const double* T11, const double* T22, const double* T12,
            double* X, double* scale);

/* ---- adjacent block swap ----
 * Swap the adjacent diagonal blocks of sizes n1 (at row j) and n2 (at j+n1)
 * of the nt x nt quasi-triangular T.  The orthogonal factor is applied:
 *   from the left to rows j..j+n1+n2-1, columns j..nt-1,
 *   from the right to columns j..j+n1+n2-1, rows 0..j+n1+n2-1,
 *   from the right to columns j..j+n1+n2-1 of Qm (nq rows), if Qm != NULL.
 * Returns 0 if the swap was done, 1 if rejected (T and Qm untouched). */
int or_swap(int64_t nt, double* T, int64_t ldt, int64_t j, int n1, int n2,
            double* Qm, int64_t ldq, int64_t nq);

/* Diagnostics of the last or_swap call (not thread-safe): 0 accepted, 1 rejected by the
 * weak stability test (c4 #5), 2 rejected because a moved 2x2 block would split into two
 * real eigenvalues (reading R6). */
int or_swap_last_reject(void);

/* ---- structure and selection (row a1 of SURVEY §8a) ---- */

/* Block map: bmap[i] = 0 (1x1 block), 1 (first row of a 2x2), 2 (second row).
 * Returns 0, or -2 if S is not upper quasi-triangular (entry below the first
 * subdiagonal nonzero, or two consecutive nonzero subdiagonal entries). */
int or_scan(int64_t n, const double* S, int64_t lds, int8_t* bmap);

/* Per-row selection normalised per block: a 2x2 block is selected if either
 * of its rows is (c4 #8).  selrow[i] in {0,1}; *m = selected rows. */
void or_select(int64_t n, const int8_t* bmap, const int32_t* select, int8_t* selrow, int64_t* m);

/* ---- window schedule (row a2) ----
 * Windows of at most w rows, ks = floor(w/2) rows of movers per group.
 * Output: for window t, rows [win_j1[t], win_j2[t]) and swaps
 * swap_off[t] .. swap_off[t+1]-1, each swap = (global row j, n1, n2) with the
 * moving (selected) block of size n2 at row j+n1 moving above the block of
 * size n1 at row j.  Call with NULL outputs to get the counts. */
int or_schedule(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w,
                int64_t* nwin, int64_t* nswap,
                int64_t* win_j1, int64_t* win_j2, int64_t* swap_off,
                int64_t* swap_j, int8_t* swap_n1, int8_t* swap_n2);

/* ---- the reordering (Eq. (7)) ----
 * mode 0: unblocked, every swap applied at once to the full S and Q
 *         (Fig. 1a, "scalar updates");
 * mode 1: accumulated-naive: swaps applied to a copy of the window and to
 *         Z = I, then the left update S[j1:j2, j2:n] = Z^T * (.), the right
 *         update S[0:j1, j1:j2] = (.) * Z and Q[:, j1:j2] = (.) * Z by naive
 *         triple loops (Fig. 1b, "accumulated updates").
 * select: in = per-row selection, out = achieved per-row selection mask.
 * bmap_out (n bytes, may be NULL): final block map.
 * max_windows < 0: all windows; otherwise stop after that many (prefix runs).
 * force_reject_at >= 0: treat the swap with that global index as rejected
 * (debug knob exercising the failure path).
 * Returns 0, +1 on rejection (S and Q hold a valid, partially reordered form),
 * or -i for an invalid argument i (-2 also when S is not quasi-triangular). */
typedef struct {
  int64_t windows;        /* windows executed */
  int64_t swaps;          /* swaps executed */
  int64_t swaps_by_type[4]; /* index (n1-1)*2 + (n2-1) */
  int64_t rejected_window;  /* -1 if none */
  int64_t rejected_swap;    /* global swap index, -1 if none */
  int64_t rejected_row;     /* row j of the rejected swap */
  int32_t rejected_n1, rejected_n2;
  double  eq_flops;       /* equivalent update flops */
} or_stats;

int or_reorder(int mode, int64_t n, double* S, int64_t lds, double* Q, int64_t ldq,
               int32_t* select, int64_t* m, int64_t w, int64_t max_windows,
               int64_t force_reject_at, int8_t* bmap_out, or_stats* st);

/* The same with Q of nq <= n rows (ld >= nq): rows of Q are updated independently
 * (Q <- Q Q3 row by row), so a row sample of Q gives exactly those rows of the full
 * result -- prefix parity at sizes where a full copy of Q does not fit. */
int or_reorder_q(int mode, int64_t n, double* S, int64_t lds, double* Q, int64_t ldq, int64_t nq,
                 int32_t* select, int64_t* m, int64_t w, int64_t max_windows,
                 int64_t force_reject_at, int8_t* bmap_out, or_stats* st);

/* ---- generalized reordering (Eq. (7) right form; Table 1
 * P:216).  Readings G1-G6 in sn_oracle.c and DESIGN.md §3. ----
 *
 * Generalized Sylvester pair (G2): S11 R - L S22 = S12, T11 R - L T22 = T12 for
 * n1, n2 in {1, 2} (all blocks column-major with ld 2), by Gaussian elimination
 * with complete pivoting on the Kronecker system of order 2 n1 n2.  Returns 1 if a
 * pivot was perturbed (near-common eigenvalue), else 0. */
int or_gsylv(int n1, int n2, const double* A11, const double* A22, const double* A12,
             const double* B11, const double* B22, const double* B12, double* R, double* L);

/* Swap the adjacent diagonal blocks of sizes n1 (row j) and n2 (row j+n1) of the
 * nt x nt pencil (S, T) in generalized real Schur form (S quasi-triangular, T upper
 * triangular with diagonal 2x2 blocks).  (S, T) <- U^T (S, T) V on rows/columns
 * j..j+n1+n2-1 (rows right of the block, columns above it, the block itself);
 * Ql (nq rows, may be NULL) <- Ql U and Zr (nz rows, may be NULL) <- Zr V on the same
 * columns.  Returns 0, or 1 if the swap is rejected (G3/G4; nothing modified). */
int or_gswap(int64_t nt, double* S, int64_t lds, double* T, int64_t ldt, int64_t j, int n1, int n2,
             double* Ql, int64_t ldq, int64_t nq, double* Zr, int64_t ldz, int64_t nz);

/* Diagnostics of the last or_gswap call (not thread-safe): 0 a 1x1|1x1 swap (G1), 1 the
 * Sylvester pair (U0, V0) kept, 2 the left re-triangularisation, 3 the right one (G2/G3),
 * -1 rejected (G3/G4). */
int or_gswap_last_variant(void);

/* Generalized reordering (S, T) = Q3 (Ŝ, T̂) Z3^T, Q <- Q Q3, Z <- Z Z3 (Q, Z may be
 * NULL), with the schedule of or_reorder (it depends only on the block map of S and
 * the selection).  mode 0 = swaps applied to the full matrices, 1 = per window
 * accumulated UL/VR and naive panel updates (G6).  Other arguments and the return
 * value as or_reorder; -5 if T has a nonzero below its diagonal. */
int or_greorder(int mode, int64_t n, double* S, int64_t lds, double* T, int64_t ldt,
                double* Q, int64_t ldq, double* Z, int64_t ldz, int32_t* select, int64_t* m,
                int64_t w, int64_t max_windows, int64_t force_reject_at, int8_t* bmap_out,
                or_stats* st);

/* ---- eigenvectors (Eq. (5)-(6); overflow protection P:104-105).
 * Readings E1-E6 in sn_oracle.c and DESIGN.md §3.2.
 *
 * Number of columns for a selection: one per selected 1x1 block, two per selected 2x2
 * block (a 2x2 block is selected if either of its rows is).  Returns 0 or -2 (S not
 * quasi-triangular). */
int or_eig_count(int64_t n, const double* S, int64_t lds, const int32_t* select, int64_t* ncols);

/* Right eigenvectors of the selected blocks of S (standardised quasi-triangular), columns
 * in block order (2x2: real part, imaginary part), back-transformed X = Q Y if Q != NULL,
 * each column (pair) normalised so that max_i(|re_i| + |im_i|) = 1.  X: n x ncols, ld ldx.
 * scale_exp (may be NULL): per column the e of the power-of-two scaling 2^-e the overflow
 * protection applied (E4).  Returns 0 or -i for argument i. */
int or_eigvec(int64_t n, const double* S, int64_t lds, const double* Q, int64_t ldq, const int32_t* select,
              double* X, int64_t ldx, int32_t* scale_exp);

/* ---- bulge-chasing sweep of multishift QR (Table 1).
 * Readings B1-B5 in sn_oracle.c and DESIGN.md §3.3.  One sweep with nshift (even) shifts
 * sr + i si in pairs (two real shifts or a conjugate pair) on the upper Hessenberg H:
 * H <- U^T H U (Hessenberg again), Q <- Q U (Q: nq <= n rows, may be NULL).  Bulges are
 * introduced and chased to the bottom one after another (B4).  Returns 0 or -i. */
int or_qr_sweep(int64_t n, double* H, int64_t ldh, double* Q, int64_t ldq, int64_t nq, int64_t nshift,
                const double* sr, const double* si);

#ifdef __cplusplus
}
#endif
#endif
