/*
 * sn_oracle.c -- CPU oracle for Schur-form eigenvalue reordering.
 *
 * TEST INFRASTRUCTURE ONLY (see sn_oracle.h).  Plain, slow, fp64, written to
 * be checked against the paper by eye:
 *   - PAPER.md P:84-88, Eq. (7)      the problem  S = Q3 Ŝ Q3^T
 *   - PAPER.md P:119                 swaps are built from Givens rotations and
 *                                    3x3 Householder reflectors
 *   - PAPER.md P:154-158, Fig. 1a/b  scalar vs accumulated (window) updates
 *   - PAPER.md P:167-184, Fig. 2     chains of windows, W/R/L tasks,
 *                                    sequentially consistent order
 * and the readings of SURVEY.md §8c-2..c4 (listed again in DESIGN.md §3),
 * which fill in what the paper leaves unstated: the swap primitive (the
 * Bai-Demmel direct swap, restated here in our own code), its sign
 * conventions, the window schedule, and the stability test.
 *
 * No blocking, no fusion, no vectorisation: every update is a scalar loop.
 */
#include "sn_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define IDX(a, ld, i, j) ((a)[(i) + (int64_t)(j) * (ld)])

static double dmax(double a, double b) { return a > b ? a : b; }
static double dmin(double a, double b) { return a < b ? a : b; }
/* Fortran SIGN(1, x): +1 for x >= +0, -1 for negative x (sign bit). */
static double sgn1(double x) { return copysign(1.0, x); }

/* sqrt(x^2 + y^2) without destructive underflow/overflow (LAPACK xLAPY2). */
static double lapy2(double x, double y) {
  double xa = fabs(x), ya = fabs(y);
  double w = dmax(xa, ya), z = dmin(xa, ya);
  if (isnan(x)) return x;
  if (isnan(y)) return y;
  if (z == 0.0 || w > DBL_MAX) return w;
  return w * sqrt(1.0 + (z / w) * (z / w));
}

/* ---------------------------------------------------------------------------
 * Givens rotation, SURVEY c4 #2 (LAPACK >= 3.10 xLARTG): c >= 0,
 * r = sign(f) * hypot(f, g), s = g / r.  g == 0 -> identity; f == 0 ->
 * (c, s) = (0, sign(g)).
 * Attribution: follows the algorithm and safe-scaling constants of the reference
 * LAPACK routine named above (LAPACK, Univ. of Tennessee / UC Berkeley / Univ. of
 * Colorado Denver / NAG Ltd., modified-BSD licence), restated in C here.
 * ------------------------------------------------------------------------- */
void or_lartg(double f, double g, double* c, double* s, double* r) {
  const double safmin = DBL_MIN, safmax = 1.0 / DBL_MIN;
  const double rtmin = sqrt(safmin), rtmax = sqrt(safmax / 2.0);
  double f1 = fabs(f), g1 = fabs(g);
  if (g == 0.0) {
    *c = 1.0; *s = 0.0; *r = f;
  } else if (f == 0.0) {
    *c = 0.0; *s = sgn1(g); *r = g1;
  } else if (f1 > rtmin && f1 < rtmax && g1 > rtmin && g1 < rtmax) {
    double d = sqrt(f * f + g * g);
    *c = f1 / d;
    *r = copysign(d, f);
    *s = g / *r;
  } else {
    double u = dmin(safmax, dmax(safmin, dmax(f1, g1)));
    double fs = f / u, gs = g / u;
    double d = sqrt(fs * fs + gs * gs);
    *c = fabs(fs) / d;
    *r = copysign(d, f);
    *s = gs / *r;
    *r *= u;
  }
}

/* ---------------------------------------------------------------------------
 * 3-element Householder reflector, SURVEY c4 #3 (LAPACK xLARFG convention):
 * beta = -sign(alpha) * ||(alpha, x)||, tau = (beta - alpha) / beta,
 * v = (1, x / (alpha - beta)).  tau = 0 (H = I) when x == 0.
 * Attribution: follows the algorithm and safe-scaling constants of the reference
 * LAPACK routine named above (LAPACK, Univ. of Tennessee / UC Berkeley / Univ. of
 * Colorado Denver / NAG Ltd., modified-BSD licence), restated in C here.
 * ------------------------------------------------------------------------- */
void or_larfg3(double* alpha, double x[2], double* tau) {
  const double safmin = DBL_MIN / (DBL_EPSILON * 0.5); /* dlamch('S')/dlamch('E') */
  double xnorm = lapy2(x[0], x[1]);
  if (xnorm == 0.0) { *tau = 0.0; return; }
  double beta = -copysign(lapy2(*alpha, xnorm), *alpha);
  int knt = 0;
  if (fabs(beta) < safmin) {
    const double rsafmn = 1.0 / safmin;
    do {
      knt++;
      x[0] *= rsafmn; x[1] *= rsafmn;
      beta *= rsafmn; *alpha *= rsafmn;
    } while (fabs(beta) < safmin && knt < 20);
    xnorm = lapy2(x[0], x[1]);
    beta = -copysign(lapy2(*alpha, xnorm), *alpha);
  }
  *tau = (beta - *alpha) / beta;
  double sc = 1.0 / (*alpha - beta);
  x[0] *= sc; x[1] *= sc;
  for (int i = 0; i < knt; ++i) beta *= safmin;
  *alpha = beta;
}

/* ---------------------------------------------------------------------------
 * Standardisation of a 2x2 block, SURVEY c4 #6 (xLANV2 semantics).
 * Attribution: follows the algorithm and safe-scaling constants of the reference
 * LAPACK routine named above (LAPACK, Univ. of Tennessee / UC Berkeley / Univ. of
 * Colorado Denver / NAG Ltd., modified-BSD licence), restated in C here.
 * ------------------------------------------------------------------------- */
void or_lanv2(double* pa, double* pb, double* pc, double* pd, double* pcs, double* psn) {
  const double eps = DBL_EPSILON;          /* dlamch('P') */
  const double multpl = 4.0;
  const double safmn2 = ldexp(1.0, -485);  /* base^(int(log(safmin/eps)/log(base)/2)) */
  const double safmx2 = 1.0 / safmn2;
  double a = *pa, b = *pb, c = *pc, d = *pd, cs, sn;
  if (c == 0.0) {
    cs = 1.0; sn = 0.0;
  } else if (b == 0.0) {
    /* swap rows and columns */
    cs = 0.0; sn = 1.0;
    double t = d; d = a; a = t;
    b = -c; c = 0.0;
  } else if ((a - d) == 0.0 && sgn1(b) != sgn1(c)) {
    cs = 1.0; sn = 0.0;   /* already standard, complex pair */
  } else {
    double temp = a - d;
    double p = 0.5 * temp;
    double bcmax = dmax(fabs(b), fabs(c));
    double bcmis = dmin(fabs(b), fabs(c)) * sgn1(b) * sgn1(c);
    double scale = dmax(fabs(p), bcmax);
    double z = (p / scale) * p + (bcmax / scale) * bcmis;
    if (z >= multpl * eps) {
      /* real eigenvalues: compute a and d */
      z = p + copysign(sqrt(scale) * sqrt(z), p);
      a = d + z;
      d = d - (bcmax / z) * bcmis;
      double tau = lapy2(c, z);
      cs = z / tau;
      sn = c / tau;
      b = b - c;
      c = 0.0;
    } else {
      /* complex, or real (almost) equal eigenvalues: make diagonal equal */
      int count = 0;
      double sigma = b + c;
      for (;;) {
        count++;
        scale = dmax(fabs(temp), fabs(sigma));
        if (scale >= safmx2) {
          sigma *= safmn2; temp *= safmn2;
          if (count <= 20) continue;
        }
        if (scale <= safmn2) {
          sigma *= safmx2; temp *= safmx2;
          if (count <= 20) continue;
        }
        break;
      }
      p = 0.5 * temp;
      double tau = lapy2(sigma, temp);
      cs = sqrt(0.5 * (1.0 + fabs(sigma) / tau));
      sn = -(p / (tau * cs)) * sgn1(sigma);
      /* [aa bb; cc dd] = [a b; c d] [cs -sn; sn cs] */
      double aa = a * cs + b * sn, bb = -a * sn + b * cs;
      double cc = c * cs + d * sn, dd = -c * sn + d * cs;
      /* [a b; c d] = [cs sn; -sn cs] [aa bb; cc dd] */
      a = aa * cs + cc * sn; b = bb * cs + dd * sn;
      c = -aa * sn + cc * cs; d = -bb * sn + dd * cs;
      temp = 0.5 * (a + d);
      a = temp; d = temp;
      if (c != 0.0) {
        if (b != 0.0) {
          if (sgn1(b) == sgn1(c)) {
            /* real eigenvalues: reduce to upper triangular form */
            double sab = sqrt(fabs(b)), sac = sqrt(fabs(c));
            p = copysign(sab * sac, c);
            tau = 1.0 / sqrt(fabs(b + c));
            a = temp + p;
            d = temp - p;
            b = b - c;
            c = 0.0;
            double cs1 = sab * tau, sn1 = sac * tau;
            temp = cs * cs1 - sn * sn1;
            sn = cs * sn1 + sn * cs1;
            cs = temp;
          }
        } else {
          b = -c; c = 0.0;
          temp = cs; cs = -sn; sn = temp;
        }
      }
    }
  }
  *pa = a; *pb = b; *pc = c; *pd = d; *pcs = cs; *psn = sn;
}

/* ---------------------------------------------------------------------------
 * Small Sylvester equation T11*X - X*T22 = scale*T12:
 * Kronecker system K x = scale*vec(T12), K = I (x) T11 - T22^T (x) I, solved by
 * Gaussian elimination with complete pivoting.  Pivot search scans the active
 * submatrix column by column (top to bottom) and takes the first strict max.
 * Pivots below smin = max(eps*max|T|, smlnum) are replaced by smin.
 * ------------------------------------------------------------------------- */
int or_sylv(int n1, int n2, const double* T11, const double* T22, const double* T12,
            double* X, double* scale) {
  const double eps = DBL_EPSILON, smlnum = DBL_MIN / DBL_EPSILON;
  const int N = n1 * n2;
  double K[4][4], rhs[4], y[4];
  int perm[4];
  double tmax = 0.0;
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1; ++j) tmax = dmax(tmax, fabs(T11[i + 2 * j]));
  for (int i = 0; i < n2; ++i)
    for (int j = 0; j < n2; ++j) tmax = dmax(tmax, fabs(T22[i + 2 * j]));
  const double smin = dmax(eps * tmax, smlnum);
  /* equation (p,q) <-> row p + n1*q ; unknown X(r,s) <-> column r + n1*s */
  for (int q = 0; q < n2; ++q)
    for (int p = 0; p < n1; ++p) {
      int row = p + n1 * q;
      rhs[row] = T12[p + 2 * q];
      for (int s = 0; s < n2; ++s)
        for (int r = 0; r < n1; ++r) {
          int col = r + n1 * s;
          double v = 0.0;
          if (q == s) v += T11[p + 2 * r];
          if (p == r) v -= T22[s + 2 * q];
          K[row][col] = v;
        }
    }
  for (int i = 0; i < N; ++i) perm[i] = i;
  int info = 0;
  for (int i = 0; i < N; ++i) {
    double xmax = -1.0;
    int ip = i, jp = i;
    for (int c = i; c < N; ++c)
      for (int r = i; r < N; ++r)
        if (fabs(K[r][c]) > xmax) { xmax = fabs(K[r][c]); ip = r; jp = c; }
    if (ip != i) {
      for (int c = 0; c < N; ++c) { double t = K[i][c]; K[i][c] = K[ip][c]; K[ip][c] = t; }
      double t = rhs[i]; rhs[i] = rhs[ip]; rhs[ip] = t;
    }
    if (jp != i) {
      for (int r = 0; r < N; ++r) { double t = K[r][i]; K[r][i] = K[r][jp]; K[r][jp] = t; }
      int t = perm[i]; perm[i] = perm[jp]; perm[jp] = t;
    }
    if (fabs(K[i][i]) < smin) { K[i][i] = smin; info = 1; }
    for (int r = i + 1; r < N; ++r) {
      double l = K[r][i] / K[i][i];
      K[r][i] = 0.0;
      for (int c = i + 1; c < N; ++c) K[r][c] -= l * K[i][c];
      rhs[r] -= l * rhs[i];
    }
  }
  /* overflow guard: scale the right-hand side down if a division could overflow */
  *scale = 1.0;
  double bmax = 0.0;
  for (int i = 0; i < N; ++i) bmax = dmax(bmax, fabs(rhs[i]));
  for (int i = 0; i < N; ++i) {
    if ((8.0 * smlnum) * fabs(rhs[i]) > fabs(K[i][i])) {
      *scale = 0.125 / bmax;
      for (int r = 0; r < N; ++r) rhs[r] *= *scale;
      break;
    }
  }
  for (int i = N - 1; i >= 0; --i) {
    double t = rhs[i];
    for (int c = i + 1; c < N; ++c) t -= K[i][c] * y[c];
    y[i] = t / K[i][i];
  }
  for (int i = 0; i < N; ++i) {
    int u = perm[i];
    int r = u % n1, s = u / n1;
    X[r + 2 * s] = y[i];
  }
  return info;
}

/* ---- plain application of a reflector / rotation to parts of a matrix ---- */

/* rows r0..r0+2, columns c0..c1-1:  A <- (I - tau v v^T) A */
static void refl_left(double* A, int64_t lda, int64_t r0, int64_t c0, int64_t c1,
                      const double v[3], double tau) {
  if (tau == 0.0) return;
  double t0 = tau * v[0], t1 = tau * v[1], t2 = tau * v[2];
  for (int64_t c = c0; c < c1; ++c) {
    double* a = &IDX(A, lda, r0, c);
    double sum = v[0] * a[0] + v[1] * a[1] + v[2] * a[2];
    a[0] -= sum * t0;
    a[1] -= sum * t1;
    a[2] -= sum * t2;
  }
}

/* columns c0..c0+2, rows r0..r1-1:  A <- A (I - tau v v^T) */
static void refl_right(double* A, int64_t lda, int64_t c0, int64_t r0, int64_t r1,
                       const double v[3], double tau) {
  if (tau == 0.0) return;
  double t0 = tau * v[0], t1 = tau * v[1], t2 = tau * v[2];
  double* a0 = &IDX(A, lda, 0, c0);
  double* a1 = &IDX(A, lda, 0, c0 + 1);
  double* a2 = &IDX(A, lda, 0, c0 + 2);
  for (int64_t r = r0; r < r1; ++r) {
    double sum = v[0] * a0[r] + v[1] * a1[r] + v[2] * a2[r];
    a0[r] -= sum * t0;
    a1[r] -= sum * t1;
    a2[r] -= sum * t2;
  }
}

/* rows r0, r0+1, columns c0..c1-1:  x' = c x + s y, y' = c y - s x */
static void rot_left(double* A, int64_t lda, int64_t r0, int64_t c0, int64_t c1, double c, double s) {
  for (int64_t k = c0; k < c1; ++k) {
    double x = IDX(A, lda, r0, k), y = IDX(A, lda, r0 + 1, k);
    IDX(A, lda, r0, k) = c * x + s * y;
    IDX(A, lda, r0 + 1, k) = c * y - s * x;
  }
}

/* columns c0, c0+1, rows r0..r1-1: same formulas on column pairs */
static void rot_right(double* A, int64_t lda, int64_t c0, int64_t r0, int64_t r1, double c, double s) {
  double* x = &IDX(A, lda, 0, c0);
  double* y = &IDX(A, lda, 0, c0 + 1);
  for (int64_t k = r0; k < r1; ++k) {
    double xv = x[k], yv = y[k];
    x[k] = c * xv + s * yv;
    y[k] = c * yv - s * xv;
  }
}

/* ---------------------------------------------------------------------------
 * Adjacent block swap.
 * ------------------------------------------------------------------------- */
static int g_last_reject = 0;   /* diagnostics: why the last or_swap call rejected */
int or_swap_last_reject(void) { return g_last_reject; }

int or_swap(int64_t nt, double* T, int64_t ldt, int64_t j, int n1, int n2,
            double* Qm, int64_t ldq, int64_t nq) {
  const int nd = n1 + n2;
  g_last_reject = 0;
  if (n1 == 1 && n2 == 1) {
    /* Givens rotation from (t12, t22 - t11); the diagonal entries are swapped
     * exactly and t12 is left untouched. */
    double t11 = IDX(T, ldt, j, j), t22 = IDX(T, ldt, j + 1, j + 1);
    double c, s, r;
    or_lartg(IDX(T, ldt, j, j + 1), t22 - t11, &c, &s, &r);
    rot_left(T, ldt, j, j + 2, nt, c, s);
    rot_right(T, ldt, j, 0, j, c, s);
    IDX(T, ldt, j, j) = t22;
    IDX(T, ldt, j + 1, j + 1) = t11;
    if (Qm) rot_right(Qm, ldq, j, 0, nq, c, s);
    return 0;
  }

  /* D = the (n1+n2)x(n1+n2) diagonal block, column-major, ld 4 */
  double D[16];
  memset(D, 0, sizeof(D));
  double dnorm = 0.0;
  for (int c = 0; c < nd; ++c)
    for (int r = 0; r < nd; ++r) {
      D[r + 4 * c] = IDX(T, ldt, j + r, j + c);
      dnorm = dmax(dnorm, fabs(D[r + 4 * c]));
    }
  const double eps = DBL_EPSILON, smlnum = DBL_MIN / DBL_EPSILON;
  const double thresh = dmax(10.0 * eps * dnorm, smlnum);

  /* T11 X - X T22 = scale T12 */
  double T11[4] = {0}, T22[4] = {0}, T12[4] = {0}, X[4] = {0}, scale;
  for (int c = 0; c < n1; ++c)
    for (int r = 0; r < n1; ++r) T11[r + 2 * c] = D[r + 4 * c];
  for (int c = 0; c < n2; ++c)
    for (int r = 0; r < n2; ++r) T22[r + 2 * c] = D[(n1 + r) + 4 * (n1 + c)];
  for (int c = 0; c < n2; ++c)
    for (int r = 0; r < n1; ++r) T12[r + 2 * c] = D[r + 4 * (n1 + c)];
  or_sylv(n1, n2, T11, T22, T12, X, &scale);

  /* reflector(s) mapping span[-X; scale*I] onto the leading n2 coordinates */
  double v1[3], v2[3] = {0, 0, 0}, tau1, tau2 = 0.0;
  int nrefl;
  if (n1 == 1) {
    /* n2 == 2: the complement (scale, X11, X12) goes to the last coordinate */
    double alpha = X[0 + 2 * 1], x[2] = {scale, X[0]};
    or_larfg3(&alpha, x, &tau1);
    v1[0] = x[0]; v1[1] = x[1]; v1[2] = 1.0;
    nrefl = 1;
  } else if (n2 == 1) {
    double alpha = -X[0], x[2] = {-X[1], scale};
    or_larfg3(&alpha, x, &tau1);
    v1[0] = 1.0; v1[1] = x[0]; v1[2] = x[1];
    nrefl = 1;
  } else {
    double alpha = -X[0], x[2] = {-X[1], scale};
    or_larfg3(&alpha, x, &tau1);
    v1[0] = 1.0; v1[1] = x[0]; v1[2] = x[1];
    /* image of the second column of [-X; scale*I] under H1, rows 2..4 */
    double temp = -tau1 * (X[0 + 2 * 1] + v1[1] * X[1 + 2 * 1]);
    double alpha2 = -temp * v1[1] - X[1 + 2 * 1];
    double x2[2] = {-temp * v1[2], scale};
    or_larfg3(&alpha2, x2, &tau2);
    v2[0] = 1.0; v2[1] = x2[0]; v2[2] = x2[1];
    nrefl = 2;
  }

  /* trial on D */
  double Dn[16];
  memcpy(Dn, D, sizeof(D));
  if (nrefl == 1) {
    refl_left(Dn, 4, 0, 0, nd, v1, tau1);
    refl_right(Dn, 4, 0, 0, nd, v1, tau1);
  } else {
    refl_left(Dn, 4, 0, 0, 4, v1, tau1);
    refl_right(Dn, 4, 0, 0, 4, v1, tau1);
    refl_left(Dn, 4, 1, 0, 4, v2, tau2);
    refl_right(Dn, 4, 1, 0, 4, v2, tau2);
  }

  /* weak stability test */
  double resid;
  if (n1 == 1) {        /* (1,2): old 1x1 now at position 2 */
    resid = dmax(dmax(fabs(Dn[2 + 4 * 0]), fabs(Dn[2 + 4 * 1])), fabs(Dn[2 + 4 * 2] - D[0]));
  } else if (n2 == 1) { /* (2,1): old 1x1 now at position 0 */
    resid = dmax(dmax(fabs(Dn[1 + 4 * 0]), fabs(Dn[2 + 4 * 0])), fabs(Dn[0] - D[2 + 4 * 2]));
  } else {
    resid = dmax(dmax(fabs(Dn[2 + 4 * 0]), fabs(Dn[2 + 4 * 1])),
                 dmax(fabs(Dn[3 + 4 * 0]), fabs(Dn[3 + 4 * 1])));
  }
  if (!(resid <= thresh)) { g_last_reject = 1; return 1; }

  /* exact zeros below the new blocks and the exact moved 1x1 eigenvalue (c4 #7) */
  if (n1 == 1) {
    Dn[2 + 4 * 0] = 0.0; Dn[2 + 4 * 1] = 0.0; Dn[2 + 4 * 2] = D[0];
  } else if (n2 == 1) {
    Dn[0] = D[2 + 4 * 2]; Dn[1 + 4 * 0] = 0.0; Dn[2 + 4 * 0] = 0.0;
  } else {
    Dn[2 + 4 * 0] = 0.0; Dn[2 + 4 * 1] = 0.0; Dn[3 + 4 * 0] = 0.0; Dn[3 + 4 * 1] = 0.0;
  }

  /* re-standardise each moved 2x2 block; a block that would split (real
   * eigenvalues) is a structure change and the swap is rejected. */
  double rc[2] = {1, 1}, rs[2] = {0, 0};
  int rpos[2] = {-1, -1};
  int nrot = 0;
  if (n2 == 2) rpos[nrot++] = 0;
  if (n1 == 2) rpos[nrot++] = n2;
  for (int q = 0; q < nrot; ++q) {
    int p = rpos[q];
    double a = Dn[p + 4 * p], b = Dn[p + 4 * (p + 1)], c = Dn[(p + 1) + 4 * p], d = Dn[(p + 1) + 4 * (p + 1)];
    double cs, sn;
    or_lanv2(&a, &b, &c, &d, &cs, &sn);
    if (c == 0.0) { g_last_reject = 2; return 1; }
    Dn[p + 4 * p] = a; Dn[p + 4 * (p + 1)] = b; Dn[(p + 1) + 4 * p] = c; Dn[(p + 1) + 4 * (p + 1)] = d;
    rot_left(Dn, 4, p, p + 2, nd, cs, sn);
    rot_right(Dn, 4, p, 0, p, cs, sn);
    rc[q] = cs; rs[q] = sn;
  }

  /* commit: rows j..j+nd-1 right of the block, columns j..j+nd-1 above it, Qm */
  if (nrefl == 1) {
    refl_left(T, ldt, j, j + nd, nt, v1, tau1);
    refl_right(T, ldt, j, 0, j, v1, tau1);
    if (Qm) refl_right(Qm, ldq, j, 0, nq, v1, tau1);
  } else {
    refl_left(T, ldt, j, j + nd, nt, v1, tau1);
    refl_left(T, ldt, j + 1, j + nd, nt, v2, tau2);
    refl_right(T, ldt, j, 0, j, v1, tau1);
    refl_right(T, ldt, j + 1, 0, j, v2, tau2);
    if (Qm) {
      refl_right(Qm, ldq, j, 0, nq, v1, tau1);
      refl_right(Qm, ldq, j + 1, 0, nq, v2, tau2);
    }
  }
  for (int q = 0; q < nrot; ++q) {
    int64_t p = j + rpos[q];
    rot_left(T, ldt, p, j + nd, nt, rc[q], rs[q]);
    rot_right(T, ldt, p, 0, j, rc[q], rs[q]);
    if (Qm) rot_right(Qm, ldq, p, 0, nq, rc[q], rs[q]);
  }
  for (int c = 0; c < nd; ++c)
    for (int r = 0; r < nd; ++r) IDX(T, ldt, j + r, j + c) = Dn[r + 4 * c];
  return 0;
}

/* ---------------------------------------------------------------------------
 * Structure ("upper quasi-triangular with 1x1 and 2x2 blocks").
 * ------------------------------------------------------------------------- */
int or_scan(int64_t n, const double* S, int64_t lds, int8_t* bmap) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = j + 2; i < n; ++i)
      if (IDX(S, lds, i, j) != 0.0) return -2;
  int64_t i = 0;
  while (i < n) {
    if (i + 1 < n && IDX(S, lds, i + 1, i) != 0.0) {
      if (i + 2 < n && IDX(S, lds, i + 2, i + 1) != 0.0) return -2;
      bmap[i] = 1; bmap[i + 1] = 2; i += 2;
    } else {
      bmap[i] = 0; i += 1;
    }
  }
  return 0;
}

void or_select(int64_t n, const int8_t* bmap, const int32_t* select, int8_t* selrow, int64_t* m) {
  int64_t cnt = 0;
  for (int64_t i = 0; i < n;) {
    if (bmap[i] == 1) {
      int8_t s = (select[i] != 0 || select[i + 1] != 0) ? 1 : 0;
      selrow[i] = s; selrow[i + 1] = s;
      cnt += 2 * s;
      i += 2;
    } else {
      selrow[i] = select[i] != 0 ? 1 : 0;
      cnt += selrow[i];
      i += 1;
    }
  }
  *m = cnt;
}

/* ---------------------------------------------------------------------------
 * Window schedule.  The block list evolves as windows are
 * executed; the schedule only depends on block sizes and selection flags.
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t B, w, ks, placed;
  int8_t* bsz;     /* block sizes, current order */
  int8_t* bsel;    /* selection flags, current order */
  int64_t* brow;   /* first row of each block */
  int in_chain;    /* 1 while following a chain upward */
  int64_t bottom;  /* block index one past the movers of the current chain */
  int64_t nmov;    /* movers of the current chain */
} sched_t;

static int sched_init(sched_t* st, int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w) {
  memset(st, 0, sizeof(*st));
  st->bsz = (int8_t*)malloc((size_t)(n + 1));
  st->bsel = (int8_t*)malloc((size_t)(n + 1));
  st->brow = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  if (!st->bsz || !st->bsel || !st->brow) return -1;
  int64_t B = 0;
  for (int64_t i = 0; i < n;) {
    int sz = bmap[i] == 1 ? 2 : 1;
    st->bsz[B] = (int8_t)sz;
    st->bsel[B] = selrow[i];
    st->brow[B] = i;
    B++;
    i += sz;
  }
  st->B = B; st->w = w; st->ks = w / 2; st->placed = 0; st->in_chain = 0;
  return 0;
}

static void sched_free(sched_t* st) {
  free(st->bsz); free(st->bsel); free(st->brow);
}

/* Next non-empty window.  Appends its swaps (global row j, n1, n2) to the
 * callback buffers via sw_* arrays of capacity cap (may be NULL) and returns
 * the number of swaps; returns -1 when the schedule is complete. */
static int64_t sched_next(sched_t* st, int64_t* j1, int64_t* j2,
                          int64_t* sw_j, int8_t* sw_n1, int8_t* sw_n2) {
  for (;;) {
    if (!st->in_chain) {
      /* (a) G = longest prefix of the unplaced selected blocks with <= ks rows */
      int64_t f = st->placed;
      while (f < st->B && !st->bsel[f]) f++;
      if (f >= st->B) return -1;
      int64_t rows = 0, cnt = 0, last = -1;
      for (int64_t b = f; b < st->B; ++b) {
        if (!st->bsel[b]) continue;
        if (cnt > 0 && rows + st->bsz[b] > st->ks) break;
        rows += st->bsz[b]; cnt++; last = b;
      }
      /* (b) already contiguous at `placed`: nothing to move */
      if (f == st->placed && last == st->placed + cnt - 1) {
        st->placed += cnt;
        continue;
      }
      /* (c) */
      st->bottom = last + 1;
      st->nmov = cnt;
      st->in_chain = 1;
    }
    /* (d) top = smallest block index >= placed with rows(top..bottom) <= w */
    int64_t top = st->bottom, rw = 0;
    while (top > st->placed && rw + st->bsz[top - 1] <= st->w) { top--; rw += st->bsz[top]; }
    int64_t wj1 = st->brow[top], wj2 = wj1 + rw;
    /* (e) movers in top-to-bottom order; mover i ends at block top+i */
    int64_t nsw = 0, im = 0;
    for (int64_t b = top; b < st->bottom; ++b) {
      if (!st->bsel[b]) continue;
      int64_t tgt = top + im;
      for (int64_t q = b; q > tgt; --q) {
        if (sw_j) { sw_j[nsw] = st->brow[q - 1]; sw_n1[nsw] = st->bsz[q - 1]; sw_n2[nsw] = st->bsz[q]; }
        nsw++;
        int8_t tsz = st->bsz[q - 1], tsel = st->bsel[q - 1];
        st->bsz[q - 1] = st->bsz[q]; st->bsel[q - 1] = st->bsel[q];
        st->bsz[q] = tsz; st->bsel[q] = tsel;
        st->brow[q] = st->brow[q - 1] + st->bsz[q - 1];
      }
      im++;
    }
    /* (f) */
    if (top == st->placed) {
      st->placed = top + im;
      st->in_chain = 0;
    } else {
      st->bottom = top + im;
    }
    if (nsw > 0) { *j1 = wj1; *j2 = wj2; return nsw; }
  }
}

/* Roll the block list back to the state reached in a window whose swap `done` was
 * rejected: undo the swaps done..k-1 that sched_next performed symbolically. */
static void sched_rollback(sched_t* st, const int64_t* tj, int64_t k, int64_t done) {
  sched_t sc = *st;
  for (int64_t i = k - 1; i >= done; --i) {
    /* the swap exchanged blocks at rows tj[i] (size t1) and tj[i]+t1 (size t2);
     * after it the block of size t2 is at row tj[i].  Find its index. */
    int64_t lo = 0, hi = sc.B - 1, b = -1;
    while (lo <= hi) {
      int64_t mid = (lo + hi) / 2;
      if (sc.brow[mid] == tj[i]) { b = mid; break; }
      if (sc.brow[mid] < tj[i]) lo = mid + 1; else hi = mid - 1;
    }
    int8_t tsz = sc.bsz[b], tsel = sc.bsel[b];
    sc.bsz[b] = sc.bsz[b + 1]; sc.bsel[b] = sc.bsel[b + 1];
    sc.bsz[b + 1] = tsz; sc.bsel[b + 1] = tsel;
    sc.brow[b + 1] = sc.brow[b] + sc.bsz[b];
  }
}

/* Upper bound on the swaps of one window: a mover passes each other block at most once. */
static int64_t max_swaps_per_window(int64_t w) { return (w * w) / 4 + w + 4; }

int or_schedule(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w,
                int64_t* nwin, int64_t* nswap,
                int64_t* win_j1, int64_t* win_j2, int64_t* swap_off,
                int64_t* swap_j, int8_t* swap_n1, int8_t* swap_n2) {
  if (w < 4) return -4;
  sched_t st;
  if (sched_init(&st, n, bmap, selrow, w)) return -100;
  int64_t cap = max_swaps_per_window(w);
  int64_t* tj = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  int8_t* t1 = (int8_t*)malloc((size_t)cap);
  int8_t* t2 = (int8_t*)malloc((size_t)cap);
  int64_t nw = 0, ns = 0, j1, j2, k;
  while ((k = sched_next(&st, &j1, &j2, tj, t1, t2)) >= 0) {
    if (win_j1) {
      win_j1[nw] = j1; win_j2[nw] = j2; swap_off[nw] = ns;
      for (int64_t i = 0; i < k; ++i) { swap_j[ns + i] = tj[i]; swap_n1[ns + i] = t1[i]; swap_n2[ns + i] = t2[i]; }
    }
    nw++; ns += k;
  }
  if (win_j1) swap_off[nw] = ns;
  *nwin = nw; *nswap = ns;
  free(tj); free(t1); free(t2);
  sched_free(&st);
  return 0;
}

/* ---------------------------------------------------------------------------
 * The reordering, Eq. (7).
 * ------------------------------------------------------------------------- */
static void window_updates_naive(int64_t n, double* S, int64_t lds, double* Q, int64_t ldq, int64_t nq,
                                 int64_t j1, int64_t j2, const double* Z) {
  /* Every column (left update) and every row (right / Q updates) is independent, so the loops
   * may run on several host threads (built with -fopenmp: the "CPU baseline, N cores" row of
   * SURVEY §8d-5); each keeps its own summation order, so the result does not depend on it. */
  const int64_t k = j2 - j1;
#ifdef _OPENMP
#pragma omp parallel
#endif
  {
    double* tmp = (double*)malloc(sizeof(double) * (size_t)k);
    /* left update: S[j1:j2, j2:n] <- Z^T S[j1:j2, j2:n] */
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t c = j2; c < n; ++c) {
      for (int64_t r = 0; r < k; ++r) {
        double acc = 0.0;
        for (int64_t l = 0; l < k; ++l) acc += Z[l + r * k] * IDX(S, lds, j1 + l, c);
        tmp[r] = acc;
      }
      for (int64_t r = 0; r < k; ++r) IDX(S, lds, j1 + r, c) = tmp[r];
    }
    /* right update: S[0:j1, j1:j2] <- S[0:j1, j1:j2] Z */
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t r = 0; r < j1; ++r) {
      for (int64_t c = 0; c < k; ++c) {
        double acc = 0.0;
        for (int64_t l = 0; l < k; ++l) acc += IDX(S, lds, r, j1 + l) * Z[l + c * k];
        tmp[c] = acc;
      }
      for (int64_t c = 0; c < k; ++c) IDX(S, lds, r, j1 + c) = tmp[c];
    }
    /* Q update (Q <- Q Q3): Q[:, j1:j2] <- Q[:, j1:j2] Z */
    if (Q) {
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
      for (int64_t r = 0; r < nq; ++r) {
        for (int64_t c = 0; c < k; ++c) {
          double acc = 0.0;
          for (int64_t l = 0; l < k; ++l) acc += IDX(Q, ldq, r, j1 + l) * Z[l + c * k];
          tmp[c] = acc;
        }
        for (int64_t c = 0; c < k; ++c) IDX(Q, ldq, r, j1 + c) = tmp[c];
      }
    }
    free(tmp);
  }
}

int or_reorder(int mode, int64_t n, double* S, int64_t lds, double* Q, int64_t ldq,
               int32_t* select, int64_t* m, int64_t w, int64_t max_windows,
               int64_t force_reject_at, int8_t* bmap_out, or_stats* st) {
  return or_reorder_q(mode, n, S, lds, Q, ldq, n, select, m, w, max_windows, force_reject_at, bmap_out, st);
}

int or_reorder_q(int mode, int64_t n, double* S, int64_t lds, double* Q, int64_t ldq, int64_t nq,
                 int32_t* select, int64_t* m, int64_t w, int64_t max_windows,
                 int64_t force_reject_at, int8_t* bmap_out, or_stats* st) {
  if (mode != 0 && mode != 1) return -1;
  if (n < 0) return -2;
  if (n > 0 && S == NULL) return -3;
  if (lds < (n > 1 ? n : 1)) return -4;
  if (Q && (nq < 0 || nq > n || ldq < (nq > 1 ? nq : 1))) return -6;
  if (n > 0 && select == NULL) return -7;
  if (m == NULL) return -8;
  if (w < 4) return -9;
  or_stats local;
  if (!st) st = &local;
  memset(st, 0, sizeof(*st));
  st->rejected_window = -1; st->rejected_swap = -1; st->rejected_row = -1;
  *m = 0;
  if (n == 0) return 0;

  int8_t* bmap = (int8_t*)malloc((size_t)n);
  int8_t* selrow = (int8_t*)malloc((size_t)n);
  if (or_scan(n, S, lds, bmap)) { free(bmap); free(selrow); return -3; }
  or_select(n, bmap, select, selrow, m);

  sched_t sc;
  sched_init(&sc, n, bmap, selrow, w);
  int64_t cap = max_swaps_per_window(w);
  int64_t* tj = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  int8_t* t1 = (int8_t*)malloc((size_t)cap);
  int8_t* t2 = (int8_t*)malloc((size_t)cap);
  double* D = (double*)malloc(sizeof(double) * (size_t)w * (size_t)w);
  double* Z = (double*)malloc(sizeof(double) * (size_t)w * (size_t)w);
  int rc = 0;
  int64_t j1, j2, k, gswap = 0;
  while ((max_windows < 0 || st->windows < max_windows) &&
         (k = sched_next(&sc, &j1, &j2, tj, t1, t2)) >= 0) {
    const int64_t kw = j2 - j1;
    int64_t done = 0;
    if (mode == 0) {
      for (; done < k; ++done) {
        if (gswap + done == force_reject_at ||
            or_swap(n, S, lds, tj[done], t1[done], t2[done], Q, ldq, Q ? nq : 0)) {
          rc = 1; break;
        }
        st->swaps_by_type[(t1[done] - 1) * 2 + (t2[done] - 1)]++;
      }
    } else {
      for (int64_t c = 0; c < kw; ++c)
        for (int64_t r = 0; r < kw; ++r) {
          D[r + c * kw] = IDX(S, lds, j1 + r, j1 + c);
          Z[r + c * kw] = (r == c) ? 1.0 : 0.0;
        }
      for (; done < k; ++done) {
        if (gswap + done == force_reject_at ||
            or_swap(kw, D, kw, tj[done] - j1, t1[done], t2[done], Z, kw, kw)) {
          rc = 1; break;
        }
        st->swaps_by_type[(t1[done] - 1) * 2 + (t2[done] - 1)]++;
      }
      for (int64_t c = 0; c < kw; ++c)
        for (int64_t r = 0; r < kw; ++r) IDX(S, lds, j1 + r, j1 + c) = D[r + c * kw];
      window_updates_naive(n, S, lds, Q, ldq, nq, j1, j2, Z);
    }
    st->swaps += done;
    st->windows++;
    st->eq_flops += 2.0 * kw * kw * ((double)(n - j2) + (double)j1 + (Q ? (double)nq : 0.0));
    if (rc) {
      st->rejected_window = st->windows - 1;
      st->rejected_swap = gswap + done;
      st->rejected_row = tj[done];
      st->rejected_n1 = t1[done];
      st->rejected_n2 = t2[done];
      sched_rollback(&sc, tj, k, done);
      break;
    }
    gswap += k;
  }
  /* achieved selection mask and block map */
  for (int64_t b = 0; b < sc.B; ++b) {
    int64_t r = sc.brow[b];
    for (int q = 0; q < sc.bsz[b]; ++q) {
      select[r + q] = sc.bsel[b];
      if (bmap_out) bmap_out[r + q] = (int8_t)(sc.bsz[b] == 1 ? 0 : 1 + q);
    }
  }
  free(tj); free(t1); free(t2); free(D); free(Z);
  free(bmap); free(selrow);
  sched_free(&sc);
  return rc;
}

/* ===========================================================================
 * Generalized reordering.  PAPER.md Eq. (7), right form
 * (P:84-88): (S, T) = Q3 (Ŝ, T̂) Z3^T with Q3, Z3 orthogonal, the selected
 * generalized eigenvalues moved to the leading diagonal blocks of (Ŝ, T̂);
 * Table 1 lists it beside the standard case, on the same windowed
 * machinery.  The paper gives no swap primitive for
 * a pencil; restated here is the direct swapping method for generalized
 * real Schur forms (Kågström 1993; Kågström & Poromaa 1996 -- the method of
 * LAPACK xTGEX2) with the readings G1-G6 of DESIGN.md §3:
 *   G1  1x1|1x1: a Givens pair from the eigenvector of the lower eigenvalue
 *       (right) and its image under S or T, whichever is relatively larger
 *       (left).
 *   G2  other cases: the generalized Sylvester equation
 *         S11 R - L S22 = S12,  T11 R - L T22 = T12   (scale 1)
 *       by Gaussian elimination with complete pivoting on its Kronecker
 *       form (order 2 n1 n2); orthogonal bases V0 of span[-R; I] (right) and
 *       U0 of span[-L; I] (left) by Householder QR.  Three candidate factor
 *       pairs: (U0, V0) itself, and the two re-triangularisations of T's
 *       block that xTGEX2 uses -- from the left (U from a QR of the first n2
 *       columns of T V0, V = V0) and from the right (V completing the row
 *       space of the last n1 rows of U0^T T, U = U0) -- which make T's block
 *       below the new leading block zero to working accuracy.
 *   G3  weak stability test: a candidate's residual is max(||S21||_F /
 *       threshA, ||T21||_F / threshB) over the blocks below the new leading
 *       block, thresh = max(100 eps ||block||_F, smlnum); the candidate with
 *       the smallest residual is kept (ties: the earlier one) and the swap is
 *       rejected (nothing changed) if that residual exceeds 1.  (1x1|1x1:
 *       the G1 pair, both blocks tested.)  Passed blocks become exact zeros.
 *       (The Sylvester pair's own residual governs (U0, V0): it passes where
 *       the re-triangularised variants lose accuracy to a large R, L, and
 *       vice versa; keeping the best of the three rejects fewer well-
 *       conditioned swaps than either rule alone -- DESIGN.md §3.1.)
 *   G4  standard form: every 2x2 diagonal block of T is diagonal with
 *       t11 >= t22 > 0 (a 2x2 SVD applied to both matrices); the paired
 *       2x2 block of S is left general; a moved 1x1 block has t >= 0.  A moved 2x2 block whose pencil has
 *       real eigenvalues, or a singular 2x2 block of T, rejects the swap.
 *   G5  accumulators: the left factor U (Q-side) and the right factor V
 *       (Z-side) of each swap; a window accumulates UL and VR from I.
 *   G6  updates of a window [j1, j2): (S, T)[j1:j2, j2:n] <- UL^T (.),
 *       (S, T)[0:j1, j1:j2] <- (.) VR, Q[:, j1:j2] <- Q UL, Z[:, j1:j2] <- Z VR.
 *   G7  basis signs: the swap's factors are fixed only up to a simultaneous
 *       sign flip of a column of U and the same column of V (G1-G4 leave it
 *       free; which variant G2 keeps can flip it).  Convention: the entry of
 *       largest magnitude of every column of V (the first such entry) is
 *       positive; U's column follows.  This makes the result a function of
 *       the data rather than of rounding-level choices.
 * ========================================================================= */

/* m x m matrices (m <= 4) column-major with ld 4 */
static void sm_eye(double* U, int m) {
  memset(U, 0, 16 * sizeof(double));
  for (int i = 0; i < m; ++i) U[i + 4 * i] = 1.0;
}

/* C = A^T B V (all m x m) */
static void sm_congruence(const double* U, const double* B, const double* V, double* C, int m) {
  double W[16];
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) {
      double acc = 0.0;
      for (int l = 0; l < m; ++l) acc += B[r + 4 * l] * V[l + 4 * c];
      W[r + 4 * c] = acc;
    }
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) {
      double acc = 0.0;
      for (int l = 0; l < m; ++l) acc += U[l + 4 * r] * W[l + 4 * c];
      C[r + 4 * c] = acc;
    }
}

/* A <- A P (m x m) */
static void sm_mul_right(double* A, const double* P, int m) {
  double W[16];
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) {
      double acc = 0.0;
      for (int l = 0; l < m; ++l) acc += A[r + 4 * l] * P[l + 4 * c];
      W[r + 4 * c] = acc;
    }
  memcpy(A, W, sizeof(W));
}

/* rows r0..r0+m-1, columns c0..c1-1 of A <- U^T (those rows) */
static void apply_left_small(double* A, int64_t lda, int64_t r0, int m, int64_t c0, int64_t c1,
                             const double* U) {
  double x[4], y[4];
  for (int64_t c = c0; c < c1; ++c) {
    for (int i = 0; i < m; ++i) x[i] = IDX(A, lda, r0 + i, c);
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int l = 0; l < m; ++l) acc += U[l + 4 * i] * x[l];
      y[i] = acc;
    }
    for (int i = 0; i < m; ++i) IDX(A, lda, r0 + i, c) = y[i];
  }
}

/* columns c0..c0+m-1, rows r0..r1-1 of A <- (those columns) V */
static void apply_right_small(double* A, int64_t lda, int64_t c0, int m, int64_t r0, int64_t r1,
                              const double* V) {
  double x[4], y[4];
  for (int64_t r = r0; r < r1; ++r) {
    for (int i = 0; i < m; ++i) x[i] = IDX(A, lda, r, c0 + i);
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int l = 0; l < m; ++l) acc += x[l] * V[l + 4 * i];
      y[i] = acc;
    }
    for (int i = 0; i < m; ++i) IDX(A, lda, r, c0 + i) = y[i];
  }
}

/* Householder QR of the m x p matrix M (ld 4): H = H_1 ... H_p explicitly (m x m),
 * H_c = I - 2 v v^T / (v^T v); the first p columns of H span range(M). */
static void sm_qr_basis(double* M, int m, int p, double* H) {
  sm_eye(H, m);
  for (int c = 0; c < p; ++c) {
    double nrm = 0.0;
    for (int i = c; i < m; ++i) nrm += M[i + 4 * c] * M[i + 4 * c];
    nrm = sqrt(nrm);
    if (nrm == 0.0) continue;
    double v[4] = {0, 0, 0, 0}, vtv = 0.0;
    for (int i = c; i < m; ++i) v[i] = M[i + 4 * c];
    v[c] += copysign(nrm, M[c + 4 * c]);
    for (int i = c; i < m; ++i) vtv += v[i] * v[i];
    for (int cc = c; cc < p; ++cc) {
      double s = 0.0;
      for (int i = c; i < m; ++i) s += v[i] * M[i + 4 * cc];
      const double f = 2.0 * s / vtv;
      for (int i = c; i < m; ++i) M[i + 4 * cc] -= f * v[i];
    }
    for (int r = 0; r < m; ++r) {
      double s = 0.0;
      for (int i = c; i < m; ++i) s += H[r + 4 * i] * v[i];
      const double f = 2.0 * s / vtv;
      for (int i = c; i < m; ++i) H[r + 4 * i] -= f * v[i];
    }
  }
}

int or_gsylv(int n1, int n2, const double* A11, const double* A22, const double* A12,
             const double* B11, const double* B22, const double* B12, double* R, double* L) {
  /* unknowns x = [vec R; vec L] (column-major vec, R(i,j) at i + n1*j) */
  const int N = n1 * n2, K = 2 * N;
  double M[8][8], rhs[8];
  memset(M, 0, sizeof(M));
  for (int jj = 0; jj < n2; ++jj)
    for (int i = 0; i < n1; ++i) {
      const int e = i + n1 * jj;
      /* (A11 R)(i,jj) = sum_l A11(i,l) R(l,jj);  (L A22)(i,jj) = sum_l L(i,l) A22(l,jj) */
      for (int l = 0; l < n1; ++l) {
        M[e][l + n1 * jj] += A11[i + 2 * l];
        M[N + e][l + n1 * jj] += B11[i + 2 * l];
      }
      for (int l = 0; l < n2; ++l) {
        M[e][N + i + n1 * l] -= A22[l + 2 * jj];
        M[N + e][N + i + n1 * l] -= B22[l + 2 * jj];
      }
      rhs[e] = A12[i + 2 * jj];
      rhs[N + e] = B12[i + 2 * jj];
    }
  /* Gaussian elimination with complete pivoting */
  int perm_c[8], perturbed = 0;
  for (int q = 0; q < K; ++q) perm_c[q] = q;
  double mx = 0.0;
  for (int r = 0; r < K; ++r)
    for (int c = 0; c < K; ++c) mx = dmax(mx, fabs(M[r][c]));
  const double smin = dmax(DBL_EPSILON * mx, DBL_MIN / DBL_EPSILON);
  for (int p = 0; p < K; ++p) {
    int pr = p, pc = p;
    double best = -1.0;
    for (int r = p; r < K; ++r)
      for (int c = p; c < K; ++c)
        if (fabs(M[r][c]) > best) { best = fabs(M[r][c]); pr = r; pc = c; }
    if (pr != p) {
      for (int c = 0; c < K; ++c) { double t = M[p][c]; M[p][c] = M[pr][c]; M[pr][c] = t; }
      double t = rhs[p]; rhs[p] = rhs[pr]; rhs[pr] = t;
    }
    if (pc != p) {
      for (int r = 0; r < K; ++r) { double t = M[r][p]; M[r][p] = M[r][pc]; M[r][pc] = t; }
      int t = perm_c[p]; perm_c[p] = perm_c[pc]; perm_c[pc] = t;
    }
    if (fabs(M[p][p]) < smin) { M[p][p] = smin; perturbed = 1; }
    for (int r = p + 1; r < K; ++r) {
      const double f = M[r][p] / M[p][p];
      for (int c = p; c < K; ++c) M[r][c] -= f * M[p][c];
      rhs[r] -= f * rhs[p];
    }
  }
  double y[8], x[8];
  for (int p = K - 1; p >= 0; --p) {
    double acc = rhs[p];
    for (int c = p + 1; c < K; ++c) acc -= M[p][c] * y[c];
    y[p] = acc / M[p][p];
  }
  for (int p = 0; p < K; ++p) x[perm_c[p]] = y[p];
  for (int jj = 0; jj < n2; ++jj)
    for (int i = 0; i < n1; ++i) {
      R[i + 2 * jj] = x[i + n1 * jj];
      L[i + 2 * jj] = x[N + i + n1 * jj];
    }
  return perturbed;
}

/* Frobenius norm of the n1 x n2 block below the leading n2 x n2 block (G3) */
static double lowblock_fro(const double* X, int n1, int n2) {
  double acc = 0.0;
  for (int c = 0; c < n2; ++c)
    for (int r = n2; r < n1 + n2; ++r) acc += X[r + 4 * c] * X[r + 4 * c];
  return sqrt(acc);
}

/* 2x2 standard form of a T block (G4): orthogonal P, W with P^T Tb W = diag(s1, s2),
 * s1 >= s2 > 0 (one-sided Jacobi on the columns of Tb).  Tb, P, W ld 2.  Returns 1 if Tb
 * is singular. */
static int std_t22(const double* Tb, double* P, double* W) {
  const double a = Tb[0] * Tb[0] + Tb[1] * Tb[1];          /* |col0|^2 */
  const double b = Tb[2] * Tb[2] + Tb[3] * Tb[3];          /* |col1|^2 */
  const double g = Tb[0] * Tb[2] + Tb[1] * Tb[3];          /* col0 . col1 */
  double c = 1.0, s = 0.0;
  if (g != 0.0) {
    const double zeta = (b - a) / (2.0 * g);
    const double t = sgn1(zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
    c = 1.0 / sqrt(1.0 + t * t);
    s = c * t;
  }
  /* W = [c s; -s c]: col0' = c col0 - s col1, col1' = s col0 + c col1 (orthogonal) */
  W[0] = c; W[1] = -s; W[2] = s; W[3] = c;
  double u0 = c * Tb[0] - s * Tb[2], u1 = c * Tb[1] - s * Tb[3];
  double w0 = s * Tb[0] + c * Tb[2], w1 = s * Tb[1] + c * Tb[3];
  if (lapy2(u0, u1) < lapy2(w0, w1)) {
    /* order the singular values, s1 >= s2: exchange the columns of W */
    double t;
    t = W[0]; W[0] = W[2]; W[2] = t;
    t = W[1]; W[1] = W[3]; W[3] = t;
    t = u0; u0 = w0; w0 = t;
    t = u1; u1 = w1; w1 = t;
  }
  const double s1 = lapy2(u0, u1);
  if (s1 == 0.0) return 1;
  P[0] = u0 / s1; P[1] = u1 / s1;
  /* second column orthogonal to the first, oriented so that P(:,1) . col1' > 0 */
  double p2r = -P[1], p2c = P[0];
  if (p2r * w0 + p2c * w1 < 0.0) { p2r = -p2r; p2c = -p2c; }
  P[2] = p2r; P[3] = p2c;
  if (!(p2r * w0 + p2c * w1 > 0.0)) return 1;
  return 0;
}

/* G3's constant: SPEC's 10^2 eps acceptance constant for a direct swap
 * (S:437); LAPACK xTGEX2 uses 20 */
#define OR_G3_C 100.0
static int g_gswap_variant = 0;   /* diagnostics: 0 G1, 1 (U0, V0), 2 left, 3 right variant kept, -1 rejected */
int or_gswap_last_variant(void) { return g_gswap_variant; }

int or_gswap(int64_t nt, double* S, int64_t lds, double* T, int64_t ldt, int64_t j, int n1, int n2,
             double* Ql, int64_t ldq, int64_t nq, double* Zr, int64_t ldz, int64_t nz) {
  const int m = n1 + n2;
  g_gswap_variant = 0;
  double A[16], B[16];
  memset(A, 0, sizeof(A));
  memset(B, 0, sizeof(B));
  double anorm = 0.0, bnorm = 0.0;      /* Frobenius norms of the blocks (G3) */
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) {
      A[r + 4 * c] = IDX(S, lds, j + r, j + c);
      B[r + 4 * c] = IDX(T, ldt, j + r, j + c);
      anorm += A[r + 4 * c] * A[r + 4 * c];
      bnorm += B[r + 4 * c] * B[r + 4 * c];
    }
  anorm = sqrt(anorm);
  bnorm = sqrt(bnorm);
  const double smlnum = DBL_MIN / DBL_EPSILON;
  const double threshA = dmax(OR_G3_C * DBL_EPSILON * anorm, smlnum);
  const double threshB = dmax(OR_G3_C * DBL_EPSILON * bnorm, smlnum);
  double U[16], V[16];
  sm_eye(U, m);
  sm_eye(V, m);
  if (n1 == 1 && n2 == 1) {
    /* G1: x spans the null space of b22 A - a22 B = [m11 m12; 0 0] */
    const double a11 = A[0], a12 = A[4], a22 = A[5], b11 = B[0], b12 = B[4], b22 = B[5];
    const double m11 = b22 * a11 - a22 * b11, m12 = b22 * a12 - a22 * b12;
    double c, s, r;
    or_lartg(m12, -m11, &c, &s, &r);
    V[0] = c; V[1] = s; V[4] = -s; V[5] = c;               /* V e1 = (c, s) ~ x */
    const double ax0 = a11 * c + a12 * s, ax1 = a22 * s;
    const double bx0 = b11 * c + b12 * s, bx1 = b22 * s;
    const double ra = anorm > 0.0 ? lapy2(ax0, ax1) / anorm : 0.0;
    const double rb = bnorm > 0.0 ? lapy2(bx0, bx1) / bnorm : 0.0;
    double c2, s2, r2;
    if (ra >= rb) or_lartg(ax0, ax1, &c2, &s2, &r2);
    else or_lartg(bx0, bx1, &c2, &s2, &r2);
    U[0] = c2; U[1] = s2; U[4] = -s2; U[5] = c2;
  } else {
    /* G2: Sylvester bases, then both re-triangularisations of T's block (xTGEX2) */
    double A11[4] = {0}, A22[4] = {0}, A12[4] = {0}, B11[4] = {0}, B22[4] = {0}, B12[4] = {0};
    double R[4] = {0}, L[4] = {0};
    for (int c = 0; c < n1; ++c)
      for (int r = 0; r < n1; ++r) { A11[r + 2 * c] = A[r + 4 * c]; B11[r + 2 * c] = B[r + 4 * c]; }
    for (int c = 0; c < n2; ++c)
      for (int r = 0; r < n2; ++r) {
        A22[r + 2 * c] = A[(n1 + r) + 4 * (n1 + c)];
        B22[r + 2 * c] = B[(n1 + r) + 4 * (n1 + c)];
      }
    for (int c = 0; c < n2; ++c)
      for (int r = 0; r < n1; ++r) { A12[r + 2 * c] = A[r + 4 * (n1 + c)]; B12[r + 2 * c] = B[r + 4 * (n1 + c)]; }
    or_gsylv(n1, n2, A11, A22, A12, B11, B22, B12, R, L);
    double Mr[16], Ml[16], U0[16], V0[16];
    memset(Mr, 0, sizeof(Mr));
    memset(Ml, 0, sizeof(Ml));
    for (int c = 0; c < n2; ++c) {
      for (int r = 0; r < n1; ++r) { Mr[r + 4 * c] = -R[r + 2 * c]; Ml[r + 4 * c] = -L[r + 2 * c]; }
      Mr[(n1 + c) + 4 * c] = 1.0;
      Ml[(n1 + c) + 4 * c] = 1.0;
    }
    sm_qr_basis(Mr, m, n2, V0);
    sm_qr_basis(Ml, m, n2, U0);
    /* from the left: Uq from a QR of the first n2 columns of T V0 */
    double I4[16], TV[16], UT[16], Uq[16], H[16], Vr[16], Mq[16], Mrr[16];
    sm_eye(I4, m);
    sm_congruence(I4, B, V0, TV, m);
    memset(Mq, 0, sizeof(Mq));
    for (int c = 0; c < n2; ++c)
      for (int r = 0; r < m; ++r) Mq[r + 4 * c] = TV[r + 4 * c];
    sm_qr_basis(Mq, m, n2, Uq);
    /* from the right: Vr = [complement of the row space of rows n2.. of U0^T T, that row space] */
    sm_congruence(U0, B, I4, UT, m);
    memset(Mrr, 0, sizeof(Mrr));
    for (int c = 0; c < n1; ++c)
      for (int r = 0; r < m; ++r) Mrr[r + 4 * c] = UT[(n2 + c) + 4 * r];
    sm_qr_basis(Mrr, m, n1, H);
    memset(Vr, 0, sizeof(Vr));
    for (int c = 0; c < n2; ++c)
      for (int r = 0; r < m; ++r) Vr[r + 4 * c] = H[r + 4 * (n1 + c)];
    for (int c = 0; c < n1; ++c)
      for (int r = 0; r < m; ++r) Vr[r + 4 * (n2 + c)] = H[r + 4 * c];
    /* G3: each candidate's residual, max(||S21|| / threshA, ||T21|| / threshB); keep the
     * smallest (ties: the earlier candidate) */
    const double* cu[3] = {U0, Uq, U0};
    const double* cv[3] = {V0, V0, Vr};
    double best = 0.0;
    int bi = -1;
    for (int q = 0; q < 3; ++q) {
      double Aq[16], Bq[16];
      sm_congruence(cu[q], A, cv[q], Aq, m);
      sm_congruence(cu[q], B, cv[q], Bq, m);
      const double r = dmax(lowblock_fro(Aq, n1, n2) / threshA, lowblock_fro(Bq, n1, n2) / threshB);
      if (bi < 0 || r < best) { best = r; bi = q; }
    }
    memcpy(U, cu[bi], sizeof(U0));
    memcpy(V, cv[bi], sizeof(V0));
    g_gswap_variant = bi + 1;
    if (!(best <= 1.0)) { g_gswap_variant = -1; return 1; }
  }
  double An[16], Bn[16];
  sm_congruence(U, A, V, An, m);
  sm_congruence(U, B, V, Bn, m);
  if (n1 == 1 && n2 == 1) {
    /* G3 (1x1|1x1): both blocks below the new leading block */
    const double resA = lowblock_fro(An, n1, n2), resB = lowblock_fro(Bn, n1, n2);
    if (!(resA <= threshA && resB <= threshB)) {
      g_gswap_variant = -1;
      return 1;
    }
  }
  for (int c = 0; c < n2; ++c)
    for (int r = n2; r < m; ++r) { An[r + 4 * c] = 0.0; Bn[r + 4 * c] = 0.0; }
  /* G4: standard form of each new 2x2 block */
  int pos[2], np = 0;
  if (n2 == 2) pos[np++] = 0;
  if (n1 == 2) pos[np++] = n2;
  for (int q = 0; q < np; ++q) {
    const int p = pos[q];
    double Tb[4] = {Bn[p + 4 * p], Bn[(p + 1) + 4 * p], Bn[p + 4 * (p + 1)], Bn[(p + 1) + 4 * (p + 1)]};
    double P2[4], W2[4];
    if (std_t22(Tb, P2, W2)) { g_gswap_variant = -1; return 1; }
    double Pm[16], Wm[16];
    sm_eye(Pm, m);
    sm_eye(Wm, m);
    Pm[p + 4 * p] = P2[0]; Pm[(p + 1) + 4 * p] = P2[1]; Pm[p + 4 * (p + 1)] = P2[2]; Pm[(p + 1) + 4 * (p + 1)] = P2[3];
    Wm[p + 4 * p] = W2[0]; Wm[(p + 1) + 4 * p] = W2[1]; Wm[p + 4 * (p + 1)] = W2[2]; Wm[(p + 1) + 4 * (p + 1)] = W2[3];
    double A2[16], B2[16];
    sm_congruence(Pm, An, Wm, A2, m);
    sm_congruence(Pm, Bn, Wm, B2, m);
    memcpy(An, A2, sizeof(A2));
    memcpy(Bn, B2, sizeof(B2));
    Bn[(p + 1) + 4 * p] = 0.0;
    Bn[p + 4 * (p + 1)] = 0.0;
    sm_mul_right(U, Pm, m);
    sm_mul_right(V, Wm, m);
    /* complex pair?  eigenvalues of diag(1/t11, 1/t22) * S block */
    const double t11 = Bn[p + 4 * p], t22 = Bn[(p + 1) + 4 * (p + 1)];
    const double e11 = An[p + 4 * p] / t11, e12 = An[p + 4 * (p + 1)] / t11;
    const double e21 = An[(p + 1) + 4 * p] / t22, e22 = An[(p + 1) + 4 * (p + 1)] / t22;
    const double h = 0.5 * (e11 - e22);
    if (!(h * h + e12 * e21 < 0.0)) { g_gswap_variant = -1; return 1; }
  }
  /* G4: a new 1x1 block has t >= 0 (negate its row of the pencil and its column of U) */
  int one[2], no = 0;
  if (n2 == 1) one[no++] = 0;
  if (n1 == 1) one[no++] = n2;
  for (int q = 0; q < no; ++q) {
    const int p = one[q];
    if (Bn[p + 4 * p] < 0.0) {
      for (int c = 0; c < m; ++c) { An[p + 4 * c] = -An[p + 4 * c]; Bn[p + 4 * c] = -Bn[p + 4 * c]; }
      for (int r = 0; r < m; ++r) U[r + 4 * p] = -U[r + 4 * p];
    }
  }
  /* G7: the largest-magnitude entry of every column of V is positive (U's column follows;
   * the block entries change as D An D, D Bn D with D = diag(+-1)) */
  double d[4] = {1.0, 1.0, 1.0, 1.0};
  for (int c = 0; c < m; ++c) {
    int im = 0;
    for (int r = 1; r < m; ++r)
      if (fabs(V[r + 4 * c]) > fabs(V[im + 4 * c])) im = r;
    if (V[im + 4 * c] < 0.0) d[c] = -1.0;
  }
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) {
      U[r + 4 * c] *= d[c];
      V[r + 4 * c] *= d[c];
      An[r + 4 * c] *= d[r] * d[c];
      Bn[r + 4 * c] *= d[r] * d[c];
    }
  /* commit */
  apply_left_small(S, lds, j, m, j + m, nt, U);
  apply_left_small(T, ldt, j, m, j + m, nt, U);
  apply_right_small(S, lds, j, m, 0, j, V);
  apply_right_small(T, ldt, j, m, 0, j, V);
  if (Ql) apply_right_small(Ql, ldq, j, m, 0, nq, U);
  if (Zr) apply_right_small(Zr, ldz, j, m, 0, nz, V);
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) {
      IDX(S, lds, j + r, j + c) = An[r + 4 * c];
      IDX(T, ldt, j + r, j + c) = Bn[r + 4 * c];
    }
  return 0;
}

/* G6: the updates of one window of the generalized reordering (naive loops) */
/* Every column (left) / row (right) is independent: with -fopenmp the loops run on several host
 * threads, each keeping its own summation order, so the result does not depend on it (as
 * window_updates_naive). */
static void gpanel_left(int64_t n, double* A, int64_t lda, int64_t j1, int64_t j2, const double* U,
                        double* tmp0) {
  const int64_t k = j2 - j1;
#ifdef _OPENMP
#pragma omp parallel
#endif
  {
#ifdef _OPENMP
    double* tmp = (double*)malloc(sizeof(double) * (size_t)k);
#pragma omp for schedule(static)
#else
    double* tmp = tmp0;
#endif
    for (int64_t c = j2; c < n; ++c) {
      for (int64_t r = 0; r < k; ++r) {
        double acc = 0.0;
        for (int64_t l = 0; l < k; ++l) acc += U[l + r * k] * IDX(A, lda, j1 + l, c);
        tmp[r] = acc;
      }
      for (int64_t r = 0; r < k; ++r) IDX(A, lda, j1 + r, c) = tmp[r];
    }
#ifdef _OPENMP
    free(tmp);
#endif
  }
  (void)tmp0;
}

static void gpanel_right(int64_t rows, double* A, int64_t lda, int64_t j1, int64_t j2, const double* V,
                         double* tmp0) {
  const int64_t k = j2 - j1;
#ifdef _OPENMP
#pragma omp parallel
#endif
  {
#ifdef _OPENMP
    double* tmp = (double*)malloc(sizeof(double) * (size_t)k);
#pragma omp for schedule(static)
#else
    double* tmp = tmp0;
#endif
    for (int64_t r = 0; r < rows; ++r) {
      for (int64_t c = 0; c < k; ++c) {
        double acc = 0.0;
        for (int64_t l = 0; l < k; ++l) acc += IDX(A, lda, r, j1 + l) * V[l + c * k];
        tmp[c] = acc;
      }
      for (int64_t c = 0; c < k; ++c) IDX(A, lda, r, j1 + c) = tmp[c];
    }
#ifdef _OPENMP
    free(tmp);
#endif
  }
  (void)tmp0;
}

int or_greorder(int mode, int64_t n, double* S, int64_t lds, double* T, int64_t ldt,
                double* Q, int64_t ldq, double* Z, int64_t ldz, int32_t* select, int64_t* m,
                int64_t w, int64_t max_windows, int64_t force_reject_at, int8_t* bmap_out,
                or_stats* st) {
  if (mode != 0 && mode != 1) return -1;
  if (n < 0) return -2;
  if (n > 0 && (S == NULL || T == NULL)) return -3;
  if (lds < (n > 1 ? n : 1)) return -4;
  if (ldt < (n > 1 ? n : 1)) return -6;
  if (Q && ldq < (n > 1 ? n : 1)) return -8;
  if (Z && ldz < (n > 1 ? n : 1)) return -10;
  if (n > 0 && select == NULL) return -11;
  if (m == NULL) return -12;
  if (w < 4) return -13;
  or_stats local;
  if (!st) st = &local;
  memset(st, 0, sizeof(*st));
  st->rejected_window = -1; st->rejected_swap = -1; st->rejected_row = -1;
  *m = 0;
  if (n == 0) return 0;
  /* T upper triangular (exact zeros below the diagonal) */
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = c + 1; r < n; ++r)
      if (IDX(T, ldt, r, c) != 0.0) return -5;

  int8_t* bmap = (int8_t*)malloc((size_t)n);
  int8_t* selrow = (int8_t*)malloc((size_t)n);
  if (or_scan(n, S, lds, bmap)) { free(bmap); free(selrow); return -3; }
  or_select(n, bmap, select, selrow, m);

  sched_t sc;
  sched_init(&sc, n, bmap, selrow, w);
  int64_t cap = max_swaps_per_window(w);
  int64_t* tj = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  int8_t* t1 = (int8_t*)malloc((size_t)cap);
  int8_t* t2 = (int8_t*)malloc((size_t)cap);
  double* DS = (double*)malloc(sizeof(double) * (size_t)w * (size_t)w);
  double* DT = (double*)malloc(sizeof(double) * (size_t)w * (size_t)w);
  double* UL = (double*)malloc(sizeof(double) * (size_t)w * (size_t)w);
  double* VR = (double*)malloc(sizeof(double) * (size_t)w * (size_t)w);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)w);
  int rc = 0;
  int64_t j1, j2, k, gswap = 0;
  while ((max_windows < 0 || st->windows < max_windows) &&
         (k = sched_next(&sc, &j1, &j2, tj, t1, t2)) >= 0) {
    const int64_t kw = j2 - j1;
    int64_t done = 0;
    if (mode == 0) {
      for (; done < k; ++done) {
        if (gswap + done == force_reject_at ||
            or_gswap(n, S, lds, T, ldt, tj[done], t1[done], t2[done], Q, ldq, Q ? n : 0, Z, ldz, Z ? n : 0)) {
          rc = 1; break;
        }
        st->swaps_by_type[(t1[done] - 1) * 2 + (t2[done] - 1)]++;
      }
    } else {
      for (int64_t c = 0; c < kw; ++c)
        for (int64_t r = 0; r < kw; ++r) {
          DS[r + c * kw] = IDX(S, lds, j1 + r, j1 + c);
          DT[r + c * kw] = IDX(T, ldt, j1 + r, j1 + c);
          UL[r + c * kw] = VR[r + c * kw] = (r == c) ? 1.0 : 0.0;
        }
      for (; done < k; ++done) {
        if (gswap + done == force_reject_at ||
            or_gswap(kw, DS, kw, DT, kw, tj[done] - j1, t1[done], t2[done], UL, kw, kw, VR, kw, kw)) {
          rc = 1; break;
        }
        st->swaps_by_type[(t1[done] - 1) * 2 + (t2[done] - 1)]++;
      }
      for (int64_t c = 0; c < kw; ++c)
        for (int64_t r = 0; r < kw; ++r) {
          IDX(S, lds, j1 + r, j1 + c) = DS[r + c * kw];
          IDX(T, ldt, j1 + r, j1 + c) = DT[r + c * kw];
        }
      gpanel_left(n, S, lds, j1, j2, UL, tmp);
      gpanel_left(n, T, ldt, j1, j2, UL, tmp);
      gpanel_right(j1, S, lds, j1, j2, VR, tmp);
      gpanel_right(j1, T, ldt, j1, j2, VR, tmp);
      if (Q) gpanel_right(n, Q, ldq, j1, j2, UL, tmp);
      if (Z) gpanel_right(n, Z, ldz, j1, j2, VR, tmp);
    }
    st->swaps += done;
    st->windows++;
    st->eq_flops += 2.0 * kw * kw * (2.0 * (double)(n - j2) + 2.0 * (double)j1 + (Q ? (double)n : 0.0) +
                                     (Z ? (double)n : 0.0));
    if (rc) {
      st->rejected_window = st->windows - 1;
      st->rejected_swap = gswap + done;
      st->rejected_row = tj[done];
      st->rejected_n1 = t1[done];
      st->rejected_n2 = t2[done];
      sched_rollback(&sc, tj, k, done);
      break;
    }
    gswap += k;
  }
  for (int64_t b = 0; b < sc.B; ++b) {
    int64_t r = sc.brow[b];
    for (int q = 0; q < sc.bsz[b]; ++q) {
      select[r + q] = sc.bsel[b];
      if (bmap_out) bmap_out[r + q] = (int8_t)(sc.bsz[b] == 1 ? 0 : 1 + q);
    }
  }
  free(tj); free(t1); free(t2); free(DS); free(DT); free(UL); free(VR); free(tmp);
  free(bmap); free(selrow);
  sched_free(&sc);
  return rc;
}

/* ===========================================================================
 * Eigenvectors.  PAPER.md Eq. (5): vectors y_i with
 * (S - lambda_i I) y_i = 0 for the quasi-triangular S, and Eq. (6):
 * the back-transform x_i = Q y_i; "the computations must be protected against
 * floating-point overflow".  Readings E1-E6:
 *   E1  columns: one per selected 1x1 block (real lambda = s_kk), two per
 *       selected 2x2 block [a b; c a] (bc < 0, lambda = a + i w, w =
 *       sqrt|b| sqrt|c|): the real and imaginary parts of the eigenvector of
 *       lambda, in the order of the blocks.
 *   E2  the eigenvector's own block (LAPACK xTREVC): real y_k = 1; complex
 *       (y_k, y_k+1) = (1, i w / b) if |b| >= |c|, else (-w / c, i).
 *       Entries below the block are 0.
 *   E3  rows above the block, bottom to top over S's block structure: a 1x1
 *       row i solves (s_ii - lambda) y_i = r_i, a 2x2 block the 2x2 (real or
 *       complex) system (S_blk - lambda I) y_blk = r_blk by Gaussian
 *       elimination with complete pivoting; a pivot below smin = max(eps
 *       (|Re lambda| + |Im lambda|), DBL_MIN / eps) is replaced by smin
 *       (xLALN2's perturbation); then r_l -= S[l, blk] y_blk for the rows l
 *       above.  Complex arithmetic on (re, im) pairs.
 *   E4  overflow protection (SPEC eigvec: Omega = 2^500, power-of-two
 *       scalings): the column (pair) carries a scale 2^-e; before a division
 *       whose result would exceed Omega, and before an update whose result
 *       could exceed Omega (max_l |r_l| + max_l |S[l, blk]| |y_blk| > Omega),
 *       the whole column is multiplied by the smallest power of two 2^-s that
 *       makes it safe; every stored value stays <= Omega.
 *   E5  normalisation (xTREVC): the column (pair) is divided by
 *       max_i (|re_i| + |im_i|) (multiplied by its reciprocal).
 *   E6  back-transform: X = Q Y (naive triple loop) before the normalisation.
 * ========================================================================= */
#define OR_OMEGA 3.273390607896142e+150   /* 2^500 */

/* smallest s >= 0 with v * 2^-s <= lim (v, lim > 0; v finite) */
static int pow2_steps(double v, double lim) {
  int s = 0;
  while (v > lim && s < 4000) { v *= 0.5; ++s; }
  return s;
}

/* complex helpers on (re, im) pairs */
static double cabs1(double re, double im) { return fabs(re) + fabs(im); }
static void cdiv(double ar, double ai, double br, double bi, double* cr, double* ci) {
  /* (ar + i ai) / (br + i bi), Smith's algorithm */
  if (fabs(br) >= fabs(bi)) {
    const double r = bi / br, d = br + bi * r;
    *cr = (ar + ai * r) / d;
    *ci = (ai - ar * r) / d;
  } else {
    const double r = br / bi, d = bi + br * r;
    *cr = (ar * r + ai) / d;
    *ci = (ai * r - ar) / d;
  }
}

/* Solve the nb x nb (nb = 1, 2) complex system (B - (wr + i wi) I) y = r, B real (ld 2),
 * by Gaussian elimination with complete pivoting; pivots below smin are replaced by smin.
 * Returns the largest |y| (cabs1). */
static double small_csolve(int nb, const double* B, double wr, double wi, double smin, const double* rr,
                           const double* ri, double* yr, double* yi) {
  if (nb == 1) {
    double dr = B[0] - wr, di = -wi;
    if (cabs1(dr, di) < smin) { dr = smin; di = 0.0; }
    cdiv(rr[0], ri[0], dr, di, &yr[0], &yi[0]);
    return cabs1(yr[0], yi[0]);
  }
  /* M = B - lambda I (2x2 complex), complete pivoting */
  double mr[2][2] = {{B[0] - wr, B[2]}, {B[1], B[3] - wr}};
  double mi[2][2] = {{-wi, 0.0}, {0.0, -wi}};
  double br[2] = {rr[0], rr[1]}, bi[2] = {ri[0], ri[1]};
  int pr = 0, pc = 0;
  double best = -1.0;
  for (int c = 0; c < 2; ++c)
    for (int r = 0; r < 2; ++r)
      if (cabs1(mr[r][c], mi[r][c]) > best) { best = cabs1(mr[r][c], mi[r][c]); pr = r; pc = c; }
  if (pr == 1) {
    for (int c = 0; c < 2; ++c) {
      double t = mr[0][c]; mr[0][c] = mr[1][c]; mr[1][c] = t;
      t = mi[0][c]; mi[0][c] = mi[1][c]; mi[1][c] = t;
    }
    double t = br[0]; br[0] = br[1]; br[1] = t;
    t = bi[0]; bi[0] = bi[1]; bi[1] = t;
  }
  if (pc == 1) {
    for (int r = 0; r < 2; ++r) {
      double t = mr[r][0]; mr[r][0] = mr[r][1]; mr[r][1] = t;
      t = mi[r][0]; mi[r][0] = mi[r][1]; mi[r][1] = t;
    }
  }
  if (cabs1(mr[0][0], mi[0][0]) < smin) { mr[0][0] = smin; mi[0][0] = 0.0; }
  double lr, li;                                   /* l = m10 / m00 */
  cdiv(mr[1][0], mi[1][0], mr[0][0], mi[0][0], &lr, &li);
  double ur = mr[1][1] - (lr * mr[0][1] - li * mi[0][1]);
  double ui = mi[1][1] - (lr * mi[0][1] + li * mr[0][1]);
  const double b1r = br[1] - (lr * br[0] - li * bi[0]);
  const double b1i = bi[1] - (lr * bi[0] + li * br[0]);
  if (cabs1(ur, ui) < smin) { ur = smin; ui = 0.0; }
  double x1r, x1i, x0r, x0i;
  cdiv(b1r, b1i, ur, ui, &x1r, &x1i);
  const double tr = br[0] - (mr[0][1] * x1r - mi[0][1] * x1i);
  const double ti = bi[0] - (mr[0][1] * x1i + mi[0][1] * x1r);
  cdiv(tr, ti, mr[0][0], mi[0][0], &x0r, &x0i);
  if (pc == 1) { yr[0] = x1r; yi[0] = x1i; yr[1] = x0r; yi[1] = x0i; }
  else { yr[0] = x0r; yi[0] = x0i; yr[1] = x1r; yi[1] = x1i; }
  return dmax(cabs1(yr[0], yi[0]), cabs1(yr[1], yi[1]));
}

int or_eig_count(int64_t n, const double* S, int64_t lds, const int32_t* select, int64_t* ncols) {
  if (n < 0) return -1;
  if (n > 0 && (S == NULL || select == NULL)) return -2;
  int8_t* bmap = (int8_t*)malloc((size_t)(n > 0 ? n : 1));
  if (n > 0 && or_scan(n, S, lds, bmap)) { free(bmap); return -2; }
  int64_t c = 0;
  for (int64_t i = 0; i < n;) {
    const int bs = bmap[i] == 1 ? 2 : 1;
    if (select[i] || (bs == 2 && select[i + 1])) c += bs;
    i += bs;
  }
  free(bmap);
  *ncols = c;
  return 0;
}

int or_eigvec(int64_t n, const double* S, int64_t lds, const double* Q, int64_t ldq, const int32_t* select,
              double* X, int64_t ldx, int32_t* scale_exp) {
  if (n < 0) return -1;
  if (n == 0) return 0;
  if (S == NULL || lds < n) return -2;
  if (Q != NULL && ldq < n) return -4;
  if (select == NULL) return -6;
  if (X == NULL || ldx < n) return -7;
  int8_t* bmap = (int8_t*)malloc((size_t)n);
  if (or_scan(n, S, lds, bmap)) { free(bmap); return -2; }
  const double eps = DBL_EPSILON, smlnum = DBL_MIN / DBL_EPSILON;
  double* yr = (double*)malloc(sizeof(double) * (size_t)n);
  double* yi = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t col = 0;
  for (int64_t k = 0; k < n;) {
    const int bs = bmap[k] == 1 ? 2 : 1;
    if (!(select[k] || (bs == 2 && select[k + 1]))) { k += bs; continue; }
    /* E1/E2: lambda and the block's own entries */
    double wr, wi = 0.0;
    for (int64_t i = 0; i < n; ++i) { yr[i] = 0.0; yi[i] = 0.0; }
    if (bs == 1) {
      wr = IDX(S, lds, k, k);
      yr[k] = 1.0;
    } else {
      const double b = IDX(S, lds, k, k + 1), c = IDX(S, lds, k + 1, k);
      wr = IDX(S, lds, k, k);
      wi = sqrt(fabs(b)) * sqrt(fabs(c));
      if (fabs(b) >= fabs(c)) { yr[k] = 1.0; yi[k + 1] = wi / b; }
      else { yr[k] = -wi / c; yi[k + 1] = 1.0; }
    }
    const double smin = dmax(eps * (fabs(wr) + fabs(wi)), smlnum);
    int e = 0;                                     /* the column holds (true vector) * 2^-e */
    /* right-hand side of the rows above: r_l = -S[l, k:k+bs] y_blk (protected as E4) */
    {
      double cmax = 0.0, ymax = 0.0;
      for (int64_t l = 0; l < k; ++l)
        for (int q = 0; q < bs; ++q) cmax = dmax(cmax, fabs(IDX(S, lds, l, k + q)));
      for (int q = 0; q < bs; ++q) ymax = dmax(ymax, cabs1(yr[k + q], yi[k + q]));
      const double g = ((double)bs * (ymax / OR_OMEGA)) * cmax;   /* (growth) / Omega */
      if (g > 1.0) {
        const int s = pow2_steps(g, 1.0);
        const double f = ldexp(1.0, -s);
        for (int q = 0; q < bs; ++q) { yr[k + q] *= f; yi[k + q] *= f; }
        e += s;
      }
    }
    for (int64_t l = 0; l < k; ++l)
      for (int q = 0; q < bs; ++q) {
        yr[l] -= IDX(S, lds, l, k + q) * yr[k + q];
        yi[l] -= IDX(S, lds, l, k + q) * yi[k + q];
      }
    /* E3/E4: blocks above, bottom to top */
    int64_t i = k;
    while (i > 0) {
      const int nb = (i >= 2 && bmap[i - 1] == 2) ? 2 : 1;
      i -= nb;
      double B[4] = {IDX(S, lds, i, i), 0.0, 0.0, 0.0};
      if (nb == 2) {
        B[1] = IDX(S, lds, i + 1, i); B[2] = IDX(S, lds, i, i + 1); B[3] = IDX(S, lds, i + 1, i + 1);
      }
      double rr[2] = {yr[i], nb == 2 ? yr[i + 1] : 0.0}, ri[2] = {yi[i], nb == 2 ? yi[i + 1] : 0.0};
      double sr[2], si[2];
      double ymax = small_csolve(nb, B, wr, wi, smin, rr, ri, sr, si);
      if (!(ymax <= OR_OMEGA)) {
        /* scale the column so that the solve stays below Omega (the right-hand side is
         * scaled and the small system solved again: exact powers of two) */
        double rmax = dmax(cabs1(rr[0], ri[0]), nb == 2 ? cabs1(rr[1], ri[1]) : 0.0);
        int s = 1;
        if (ymax < 1e308) s = pow2_steps(ymax, OR_OMEGA);
        else s = pow2_steps(rmax / smin, OR_OMEGA) + 1;   /* |y| <~ |r| / smin */
        for (;;) {
          const double f = ldexp(1.0, -s);
          double r2r[2] = {rr[0] * f, rr[1] * f}, r2i[2] = {ri[0] * f, ri[1] * f};
          ymax = small_csolve(nb, B, wr, wi, smin, r2r, r2i, sr, si);
          if (ymax <= OR_OMEGA || s > 4000) break;
          ++s;
        }
        const double f = ldexp(1.0, -s);
        for (int64_t l = 0; l < n; ++l) { yr[l] *= f; yi[l] *= f; }
        e += s;
      }
      for (int q = 0; q < nb; ++q) { yr[i + q] = sr[q]; yi[i + q] = si[q]; }
      if (i == 0) break;
      /* update of the rows above: protect against overflow of r_l - S[l, blk] y_blk */
      double rmax = 0.0, cmax = 0.0;
      for (int64_t l = 0; l < i; ++l) {
        rmax = dmax(rmax, cabs1(yr[l], yi[l]));
        for (int q = 0; q < nb; ++q) cmax = dmax(cmax, fabs(IDX(S, lds, l, i + q)));
      }
      const double g = rmax / OR_OMEGA + ((double)nb * (ymax / OR_OMEGA)) * cmax;   /* (growth) / Omega */
      if (g > 1.0) {
        const int s = pow2_steps(g, 1.0);
        const double f = ldexp(1.0, -s);
        for (int64_t l = 0; l < n; ++l) { yr[l] *= f; yi[l] *= f; }
        e += s;
      }
      for (int64_t l = 0; l < i; ++l)
        for (int q = 0; q < nb; ++q) {
          yr[l] -= IDX(S, lds, l, i + q) * yr[i + q];
          yi[l] -= IDX(S, lds, l, i + q) * yi[i + q];
        }
    }
    /* E6: back-transform (rows of Y below k + bs are zero) */
    double* xr = &IDX(X, ldx, 0, col);
    double* xi = bs == 2 ? &IDX(X, ldx, 0, col + 1) : NULL;
    if (Q) {
      for (int64_t r = 0; r < n; ++r) {
        double ar = 0.0, ai = 0.0;
        for (int64_t l = 0; l < k + bs; ++l) {
          ar += IDX(Q, ldq, r, l) * yr[l];
          ai += IDX(Q, ldq, r, l) * yi[l];
        }
        xr[r] = ar;
        if (xi) xi[r] = ai;
      }
    } else {
      for (int64_t r = 0; r < n; ++r) { xr[r] = yr[r]; if (xi) xi[r] = yi[r]; }
    }
    /* E5: normalisation */
    double emax = 0.0;
    for (int64_t r = 0; r < n; ++r) emax = dmax(emax, fabs(xr[r]) + (xi ? fabs(xi[r]) : 0.0));
    if (emax > 0.0) {
      const double rem = 1.0 / emax;
      for (int64_t r = 0; r < n; ++r) { xr[r] *= rem; if (xi) xi[r] *= rem; }
    }
    if (scale_exp) { scale_exp[col] = e; if (bs == 2) scale_exp[col + 1] = e; }
    col += bs;
    k += bs;
  }
  free(yr); free(yi); free(bmap);
  return 0;
}

/* ===========================================================================
 * Bulge-chasing sweep of the multishift QR algorithm.  PAPER.md
 * "The bulge chasing step creates a set of bulges which are chased
 * down the diagonal to complete one pipelined QR iteration.  This is
 * accomplished by applying sequences of overlapping 3 x 3 Householder
 * reflectors to H."  Readings B1-B5:
 *   B1  shifts come in pairs (s_2j, s_2j+1): two real shifts or a complex
 *       conjugate pair; pair j makes bulge j (a double-shift Francis step).
 *   B2  bulge j is introduced at the top by the reflector that maps
 *       p_j(H) e1 = (H^2 - sigma H + pi I) e1 (rows 0..2; sigma = s + s',
 *       pi = s s') onto e1 (Golub & Van Loan, Algorithm 7.5.1).
 *   B3  chase: for p = 1 .. n-3 the reflector from H[p:p+3, p-1] (3 entries)
 *       annihilates H[p+1, p-1], H[p+2, p-1]; for p = n-2 a 2-element
 *       reflector from H[n-2:n, n-3].  Each reflector is applied from the
 *       left to its rows (columns p-1 .. n-1), from the right to its columns
 *       (rows 0 .. min(p+3, n-1)) and to the columns of Q; the annihilated
 *       entries are set to exact zeros.  Reflectors follow xLARFG (R3).
 *   B4  one sweep = bulge 0 chased to the bottom, then bulge 1, ...: in exact
 *       arithmetic the same reflectors as the pipelined chain of bulges the
 *       paper describes (bulges spaced >= 4 rows apart; each reflector reads
 *       only entries every earlier bulge has finished with), so the windowed
 *       GPU chase agrees with it to rounding.
 *   B5  Q may hold nq <= n rows (row sample, as or_reorder_q).
 * ========================================================================= */
static void or_larfg2(double* alpha, double* x, double* tau) {
  /* 2-element xLARFG: H (alpha, x) = (beta, 0), v = (1, x'), beta = -sign(alpha) ||.|| */
  if (*x == 0.0) { *tau = 0.0; return; }
  const double beta = -copysign(lapy2(*alpha, *x), *alpha);
  *tau = (beta - *alpha) / beta;
  *x = *x / (*alpha - beta);
  *alpha = beta;
}

/* apply H = I - tau v v^T (v of length m, v[0] = 1) to rows r0..r0+m-1, columns c0..c1-1 */
static void refl_left_m(double* A, int64_t lda, int m, int64_t r0, int64_t c0, int64_t c1, const double* v,
                        double tau) {
  if (tau == 0.0) return;
  for (int64_t c = c0; c < c1; ++c) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += v[i] * IDX(A, lda, r0 + i, c);
    s *= tau;
    for (int i = 0; i < m; ++i) IDX(A, lda, r0 + i, c) -= s * v[i];
  }
}

/* apply H from the right to columns c0..c0+m-1, rows r0..r1-1 */
static void refl_right_m(double* A, int64_t lda, int m, int64_t c0, int64_t r0, int64_t r1, const double* v,
                         double tau) {
  if (tau == 0.0) return;
  for (int64_t r = r0; r < r1; ++r) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += IDX(A, lda, r, c0 + i) * v[i];
    s *= tau;
    for (int i = 0; i < m; ++i) IDX(A, lda, r, c0 + i) -= s * v[i];
  }
}

int or_qr_sweep(int64_t n, double* H, int64_t ldh, double* Q, int64_t ldq, int64_t nq, int64_t nshift,
                const double* sr, const double* si) {
  if (n < 0) return -1;
  if (n > 0 && (H == NULL || ldh < n)) return -2;
  if (Q && (nq < 0 || nq > n || ldq < (nq > 1 ? nq : 1))) return -4;
  if (nshift < 0 || (nshift & 1)) return -7;
  if (nshift > 0 && (sr == NULL || si == NULL)) return -8;
  for (int64_t j = 0; j < nshift; j += 2) {
    const int conj = si[j] != 0.0 || si[j + 1] != 0.0;
    if (conj && !(sr[j] == sr[j + 1] && si[j] == -si[j + 1])) return -9;   /* B1 */
  }
  if (n < 3) return 0;
  for (int64_t j = 0; j < nshift; j += 2) {
    /* B2: introduce bulge j */
    const double sigma = sr[j] + sr[j + 1];
    const double pi = sr[j] * sr[j + 1] - si[j] * si[j + 1];
    const double h00 = IDX(H, ldh, 0, 0), h01 = IDX(H, ldh, 0, 1), h10 = IDX(H, ldh, 1, 0);
    const double h11 = IDX(H, ldh, 1, 1), h21 = IDX(H, ldh, 2, 1);
    double alpha = h00 * h00 + h01 * h10 - sigma * h00 + pi;
    double x[2] = {h10 * (h00 + h11 - sigma), h10 * h21};
    double tau;
    or_larfg3(&alpha, x, &tau);
    double v[3] = {1.0, x[0], x[1]};
    refl_left_m(H, ldh, 3, 0, 0, n, v, tau);
    refl_right_m(H, ldh, 3, 0, 0, n < 4 ? n : 4, v, tau);
    if (Q) refl_right_m(Q, ldq, 3, 0, 0, nq, v, tau);
    /* B3: chase it to the bottom */
    for (int64_t p = 1; p <= n - 2; ++p) {
      const int m = p <= n - 3 ? 3 : 2;
      alpha = IDX(H, ldh, p, p - 1);
      if (m == 3) {
        x[0] = IDX(H, ldh, p + 1, p - 1);
        x[1] = IDX(H, ldh, p + 2, p - 1);
        or_larfg3(&alpha, x, &tau);
        v[0] = 1.0; v[1] = x[0]; v[2] = x[1];
      } else {
        x[0] = IDX(H, ldh, p + 1, p - 1);
        or_larfg2(&alpha, &x[0], &tau);
        v[0] = 1.0; v[1] = x[0]; v[2] = 0.0;
      }
      IDX(H, ldh, p, p - 1) = alpha;
      for (int i = 1; i < m; ++i) IDX(H, ldh, p + i, p - 1) = 0.0;
      refl_left_m(H, ldh, m, p, p, n, v, tau);
      const int64_t r1 = p + 4 < n ? p + 4 : n;
      refl_right_m(H, ldh, m, p, 0, r1, v, tau);
      if (Q) refl_right_m(Q, ldq, m, p, 0, nq, v, tau);
    }
  }
  return 0;
}
