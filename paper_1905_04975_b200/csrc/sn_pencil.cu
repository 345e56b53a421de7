// sn_pencil.cu -- generalized reordering of a matrix pencil (PAPER.md
// Eq. (7) right form: (S, T) = Q3 (Ŝ, T̂) Z3^T; Table 1).  Product code.
//
// Same schedule, levels and panel kernels as the standard path (sn_plan.cpp,
// sn_kernels_panel*.cu); what differs is the window task and that every window carries two
// accumulators: UL (left factors, applied as UL^T to the rows right of the window of S and
// T, and to the columns of Q) and VR (right factors, applied to the columns above the window
// of S and T, and to the columns of Z).  The swap transform is the direct swap of generalized
// real Schur forms with the readings G1-G6 of DESIGN.md §3.1 (1x1|1x1: a Givens pair from the
// eigenvector of the lower eigenvalue; otherwise the generalized Sylvester pair by complete
// pivoting on its Kronecker form, bases of span[-R; I] and span[-L; I] by Householder QR; the
// weak stability test; T's 2x2 blocks diagonal with t11 >= t22 > 0 by a 2x2 SVD; moved 1x1
// blocks with t >= 0).
//
// Window task: one CTA per window; the swaps run in steps of swaps on disjoint rows (one
// thread per swap computes its transform, 256 threads apply them to the window of S and T in
// place in global memory -- L2 resident -- and to UL / VR); the column nonzero intervals of the
// accumulators are tracked as in the standard window kernel so the panel kernels skip
// structural zeros.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "sn_device.cuh"
#include "sn_exec.h"
#include "sn_plan.h"
#include "sn_reorder.h"

namespace cg = cooperative_groups;

namespace sn {
namespace {

inline double __longlong_as_double_host(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof(d));
  return d;
}

// ---------------------------------------------------------------- the swap transform (device)
// G3's constant: residual <= kG3C eps ||block||_F (SPEC's 10^2 eps acceptance constant for a
// direct swap; LAPACK xTGEX2 uses 20 -- DESIGN.md §3.1)
constexpr double kG3C = 100.0;
// 4x4 matrices column-major with ld 4 in per-thread arrays.

__host__ __device__ __forceinline__ void pl_lartg(double f, double g, double& c, double& s, double& r) {
  // c >= 0, r = sign(f) hypot(f, g), [c s; -s c] [f; g] = [r; 0]
  if (g == 0.0) { c = 1.0; s = 0.0; r = f; return; }
  if (f == 0.0) { c = 0.0; s = copysign(1.0, g); r = fabs(g); return; }
  const double d = hypot(f, g);
  c = fabs(f) / d;
  r = copysign(d, f);
  s = g / r;
}

__host__ __device__ __forceinline__ void pl_eye(double* U, int m) {
#pragma unroll
  for (int i = 0; i < 16; ++i) U[i] = 0.0;
#pragma unroll
  for (int i = 0; i < m; ++i) U[i * 5] = 1.0;
}

// C = U^T X V
__host__ __device__ __forceinline__ void pl_congr(const double* U, const double* X, const double* V, double* C, int m) {
  double W[16];
#pragma unroll
  for (int c = 0; c < m; ++c)
#pragma unroll
    for (int r = 0; r < m; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < m; ++l) acc = fma(X[r + 4 * l], V[l + 4 * c], acc);
      W[r + 4 * c] = acc;
    }
#pragma unroll
  for (int c = 0; c < m; ++c)
#pragma unroll
    for (int r = 0; r < m; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < m; ++l) acc = fma(U[l + 4 * r], W[l + 4 * c], acc);
      C[r + 4 * c] = acc;
    }
}

// X <- X P
__host__ __device__ __forceinline__ void pl_mulr(double* X, const double* P, int m) {
  double W[16];
#pragma unroll
  for (int c = 0; c < m; ++c)
#pragma unroll
    for (int r = 0; r < m; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < m; ++l) acc = fma(X[r + 4 * l], P[l + 4 * c], acc);
      W[r + 4 * c] = acc;
    }
#pragma unroll
  for (int c = 0; c < m; ++c)
#pragma unroll
    for (int r = 0; r < m; ++r) X[r + 4 * c] = W[r + 4 * c];   // entries outside m x m stay 0
}

// orthogonal H (m x m) whose first p columns span range(M) (M: m x p, destroyed)
__host__ __device__ __forceinline__ void pl_qr_basis(double* M, int m, int p, double* H) {
  pl_eye(H, m);
#pragma unroll
  for (int c = 0; c < p; ++c) {
    double nrm = 0.0;
#pragma unroll
    for (int i = c; i < m; ++i) nrm = fma(M[i + 4 * c], M[i + 4 * c], nrm);
    nrm = sqrt(nrm);
    if (nrm == 0.0) continue;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = c; i < m; ++i) v[i] = M[i + 4 * c];
    v[c] += copysign(nrm, M[c + 4 * c]);
    double vtv = 0.0;
#pragma unroll
    for (int i = c; i < m; ++i) vtv = fma(v[i], v[i], vtv);
    const double f2 = 2.0 / vtv;
#pragma unroll
    for (int cc = c; cc < p; ++cc) {
      double s = 0.0;
#pragma unroll
      for (int i = c; i < m; ++i) s = fma(v[i], M[i + 4 * cc], s);
#pragma unroll
      for (int i = c; i < m; ++i) M[i + 4 * cc] -= (f2 * s) * v[i];
    }
#pragma unroll
    for (int r = 0; r < m; ++r) {
      double s = 0.0;
#pragma unroll
      for (int i = c; i < m; ++i) s = fma(H[r + 4 * i], v[i], s);
#pragma unroll
      for (int i = c; i < m; ++i) H[r + 4 * i] -= (f2 * s) * v[i];
    }
  }
}

// Generalized Sylvester pair S11 R - L S22 = S12, T11 R - L T22 = T12 (G2): Kronecker system
// x = [vec R; vec L] (column-major vec) by Gaussian elimination with complete pivoting.
// A = the m x m block of S, B = of T (ld 4).  R, L: n1 x n2 with ld 2.  Compile-time sizes and
// predicated row / column exchanges keep the system in registers.
template <int N1, int N2>
__host__ __device__ __forceinline__ void pl_gsylv(const double* A, const double* B, double* R, double* L) {
  constexpr int N = N1 * N2, K = 2 * N;
  double M[K][K], y[K];
  int cp[K];
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c) M[r][c] = 0.0;
#pragma unroll
  for (int jj = 0; jj < N2; ++jj)
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      const int e = i + N1 * jj;
#pragma unroll
      for (int l = 0; l < N1; ++l) {
        M[e][l + N1 * jj] += A[i + 4 * l];
        M[N + e][l + N1 * jj] += B[i + 4 * l];
      }
#pragma unroll
      for (int l = 0; l < N2; ++l) {
        M[e][N + i + N1 * l] -= A[(N1 + l) + 4 * (N1 + jj)];
        M[N + e][N + i + N1 * l] -= B[(N1 + l) + 4 * (N1 + jj)];
      }
      y[e] = A[i + 4 * (N1 + jj)];
      y[N + e] = B[i + 4 * (N1 + jj)];
    }
  double mx = 0.0;
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c) mx = fmax(mx, fabs(M[r][c]));
  const double smin = fmax(2.220446049250313e-16 * mx, 2.2250738585072014e-308 / 2.220446049250313e-16);
#pragma unroll
  for (int q = 0; q < K; ++q) cp[q] = q;
#pragma unroll
  for (int p = 0; p < K; ++p) {
    int pr = p, pc = p;
    double best = -1.0;
#pragma unroll
    for (int r = p; r < K; ++r)
#pragma unroll
      for (int c = p; c < K; ++c)
        if (fabs(M[r][c]) > best) { best = fabs(M[r][c]); pr = r; pc = c; }
#pragma unroll
    for (int r = p + 1; r < K; ++r)
      if (r == pr) {
#pragma unroll
        for (int c = 0; c < K; ++c) { const double t = M[p][c]; M[p][c] = M[r][c]; M[r][c] = t; }
        const double t = y[p]; y[p] = y[r]; y[r] = t;
      }
#pragma unroll
    for (int c = p + 1; c < K; ++c)
      if (c == pc) {
#pragma unroll
        for (int r = 0; r < K; ++r) { const double t = M[r][p]; M[r][p] = M[r][c]; M[r][c] = t; }
        const int t = cp[p]; cp[p] = cp[c]; cp[c] = t;
      }
    if (fabs(M[p][p]) < smin) M[p][p] = smin;
    const double ip = 1.0 / M[p][p];
#pragma unroll
    for (int r = p + 1; r < K; ++r) {
      const double f = M[r][p] * ip;
#pragma unroll
      for (int c = p; c < K; ++c) M[r][c] -= f * M[p][c];
      y[r] -= f * y[p];
    }
  }
  double z[K], x[K];
#pragma unroll
  for (int p = K - 1; p >= 0; --p) {
    double acc = y[p];
#pragma unroll
    for (int c = p + 1; c < K; ++c) acc -= M[p][c] * z[c];
    z[p] = acc / M[p][p];
  }
#pragma unroll
  for (int q = 0; q < K; ++q) {
    double v = 0.0;
#pragma unroll
    for (int p = 0; p < K; ++p)
      if (cp[p] == q) v = z[p];
    x[q] = v;
  }
#pragma unroll
  for (int jj = 0; jj < N2; ++jj)
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      R[i + 2 * jj] = x[i + N1 * jj];
      L[i + 2 * jj] = x[N + i + N1 * jj];
    }
}

// pl_gsylv by a group of 4 lanes (all 32 lanes of the warp call it; lane & 3 = role): the same
// Kronecker system, pivots, eliminations and back substitution, so the same R and L.  Role q
// holds K/4 rows of the system (physical rows q K/4 ..); row exchanges are tracked as logical
// positions instead of moving rows, column exchanges are made in every row as in pl_gsylv.  The
// complete-pivoting search is a per-lane scan plus a two-step shuffle reduction with
// pl_gsylv's tie rule (the first maximum in row-major order of the active submatrix); the
// pivot row and every back-substituted unknown are broadcast by the lane that holds them.
template <int N1, int N2>
__device__ __forceinline__ void pl_gsylv_lanes(const double* A, const double* B, double* R, double* L, int lane) {
  constexpr int N = N1 * N2, K = 2 * N, RPL = K / 4;
  const int q = lane & 3, gbase = lane & ~3;
  double M[RPL][K], y[RPL];
  int lpos[RPL];
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    lpos[k] = q * RPL + k;
#pragma unroll
    for (int c = 0; c < K; ++c) M[k][c] = 0.0;
    y[k] = 0.0;
  }
  // rows of the system (pl_gsylv's construction: every entry is set once)
#pragma unroll
  for (int jj = 0; jj < N2; ++jj)
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      const int e = i + N1 * jj;
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int rho = q * RPL + k;
        if (rho == e || rho == N + e) {
          const double* X = rho == e ? A : B;
#pragma unroll
          for (int l = 0; l < N1; ++l) M[k][l + N1 * jj] = 0.0 + X[i + 4 * l];
#pragma unroll
          for (int l = 0; l < N2; ++l) M[k][N + i + N1 * l] = 0.0 - X[(N1 + l) + 4 * (N1 + jj)];
          y[k] = X[i + 4 * (N1 + jj)];
        }
      }
    }
  double mx = 0.0;
#pragma unroll
  for (int k = 0; k < RPL; ++k)
#pragma unroll
    for (int c = 0; c < K; ++c) mx = fmax(mx, fabs(M[k][c]));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
  const double smin = fmax(2.220446049250313e-16 * mx, 2.2250738585072014e-308 / 2.220446049250313e-16);
  int cp[K];
#pragma unroll
  for (int c = 0; c < K; ++c) cp[c] = c;
#pragma unroll
  for (int p = 0; p < K; ++p) {
    // this lane's candidate, then the group's: larger |v|, ties to the smaller (row, column)
    double bv = -1.0;
    int br = K, bc = K;
#pragma unroll
    for (int k = 0; k < RPL; ++k)
#pragma unroll
      for (int c = p; c < K; ++c) {
        const double v = fabs(M[k][c]);
        const bool ok = lpos[k] >= p && (v > bv || (v == bv && (lpos[k] < br || (lpos[k] == br && c < bc))));
        if (ok) { bv = v; br = lpos[k]; bc = c; }
      }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int orr = __shfl_xor_sync(0xffffffffu, br, o), oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ov > bv || (ov == bv && (orr < br || (orr == br && oc < bc)))) { bv = ov; br = orr; bc = oc; }
    }
    const int pr = br < K ? br : p, pc = br < K ? bc : p;
    // row exchange p <-> pr (logical positions)
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      if (pr != p) {
        if (lpos[k] == p) lpos[k] = pr;
        else if (lpos[k] == pr) lpos[k] = p;
      }
    }
    // column exchange p <-> pc in every row
#pragma unroll
    for (int c = p + 1; c < K; ++c)
      if (c == pc) {
#pragma unroll
        for (int k = 0; k < RPL; ++k) { const double t = M[k][p]; M[k][p] = M[k][c]; M[k][c] = t; }
        const int t = cp[p]; cp[p] = cp[c]; cp[c] = t;
      }
    // the pivot row (clamped pivot) from the lane that holds logical row p
    double prow[K], py = 0.0;
#pragma unroll
    for (int c = 0; c < K; ++c) prow[c] = 0.0;
    bool has = false;
#pragma unroll
    for (int k = 0; k < RPL; ++k)
      if (lpos[k] == p) {
        has = true;
        if (fabs(M[k][p]) < smin) M[k][p] = smin;
#pragma unroll
        for (int c = p; c < K; ++c) prow[c] = M[k][c];
        py = y[k];
      }
    const unsigned own = (__ballot_sync(0xffffffffu, has) >> gbase) & 0xFu;
    const int src = gbase + __ffs(own) - 1;
#pragma unroll
    for (int c = p; c < K; ++c) prow[c] = __shfl_sync(0xffffffffu, prow[c], src);
    py = __shfl_sync(0xffffffffu, py, src);
    const double ip = 1.0 / prow[p];
#pragma unroll
    for (int k = 0; k < RPL; ++k)
      if (lpos[k] > p) {
        const double f = M[k][p] * ip;
#pragma unroll
        for (int c = p; c < K; ++c) M[k][c] -= f * prow[c];
        y[k] -= f * py;
      }
  }
  double z[K], x[K];
#pragma unroll
  for (int p = K - 1; p >= 0; --p) {
    double zp = 0.0;
    bool has = false;
#pragma unroll
    for (int k = 0; k < RPL; ++k)
      if (lpos[k] == p) {
        has = true;
        double acc = y[k];
#pragma unroll
        for (int c = p + 1; c < K; ++c) acc -= M[k][c] * z[c];
        zp = acc / M[k][p];
      }
    const unsigned own = (__ballot_sync(0xffffffffu, has) >> gbase) & 0xFu;
    z[p] = __shfl_sync(0xffffffffu, zp, gbase + __ffs(own) - 1);
  }
#pragma unroll
  for (int qq = 0; qq < K; ++qq) {
    double v = 0.0;
#pragma unroll
    for (int p = 0; p < K; ++p)
      if (cp[p] == qq) v = z[p];
    x[qq] = v;
  }
#pragma unroll
  for (int jj = 0; jj < N2; ++jj)
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      R[i + 2 * jj] = x[i + N1 * jj];
      L[i + 2 * jj] = x[N + i + N1 * jj];
    }
}

// Frobenius norm of the n1 x n2 block below the leading n2 x n2 block (G3)
__host__ __device__ __forceinline__ double pl_lowfro(const double* X, int n1, int n2) {
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < n2; ++c)
#pragma unroll
    for (int r = n2; r < n1 + n2; ++r) acc = fma(X[r + 4 * c], X[r + 4 * c], acc);
  return sqrt(acc);
}

// 2x2 SVD of a T block (G4): P^T Tb W = diag(s1, s2), s1 >= s2 > 0.  Tb, P, W ld 2.
// Returns false if Tb is singular.
__host__ __device__ __forceinline__ bool pl_std_t22(const double* Tb, double* P, double* W) {
  const double a = Tb[0] * Tb[0] + Tb[1] * Tb[1];
  const double b = Tb[2] * Tb[2] + Tb[3] * Tb[3];
  const double g = Tb[0] * Tb[2] + Tb[1] * Tb[3];
  double c = 1.0, s = 0.0;
  if (g != 0.0) {
    const double zeta = (b - a) / (2.0 * g);
    const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
    c = 1.0 / sqrt(1.0 + t * t);
    s = c * t;
  }
  W[0] = c; W[1] = -s; W[2] = s; W[3] = c;
  double u0 = c * Tb[0] - s * Tb[2], u1 = c * Tb[1] - s * Tb[3];
  double w0 = s * Tb[0] + c * Tb[2], w1 = s * Tb[1] + c * Tb[3];
  if (hypot(u0, u1) < hypot(w0, w1)) {
    double t;
    t = W[0]; W[0] = W[2]; W[2] = t;
    t = W[1]; W[1] = W[3]; W[3] = t;
    t = u0; u0 = w0; w0 = t;
    t = u1; u1 = w1; w1 = t;
  }
  const double s1 = hypot(u0, u1);
  if (s1 == 0.0) return false;
  P[0] = u0 / s1; P[1] = u1 / s1;
  double p2r = -P[1], p2c = P[0];
  if (p2r * w0 + p2c * w1 < 0.0) { p2r = -p2r; p2c = -p2c; }
  P[2] = p2r; P[3] = p2c;
  return p2r * w0 + p2c * w1 > 0.0;
}

// G4 and G7 on a swap's accepted transform: the new blocks below the leading one set to zero,
// T's 2x2 blocks diagonal (2x2 SVD), moved 1x1 blocks with t >= 0, the sign convention.
template <int N1, int N2>
__host__ __device__ __forceinline__ bool pl_swap_tail(double* U, double* V, double* An, double* Bn, double* why) {
  constexpr int n1 = N1, n2 = N2, m = N1 + N2;
#pragma unroll
  for (int c = 0; c < n2; ++c)
#pragma unroll
    for (int r = n2; r < m; ++r) { An[r + 4 * c] = 0.0; Bn[r + 4 * c] = 0.0; }
  // G4: 2x2 blocks
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    int p = -1;
    if (q == 0 && n2 == 2) p = 0;
    if (q == 1 && n1 == 2) p = n2;
    if (p < 0) continue;
    const double Tb[4] = {Bn[p + 4 * p], Bn[(p + 1) + 4 * p], Bn[p + 4 * (p + 1)], Bn[(p + 1) + 4 * (p + 1)]};
    double P2[4], W2[4];
    if (!pl_std_t22(Tb, P2, W2)) {
      if (why) { why[0] = 2.0; why[1] = 0.0; }
      return false;
    }
    double Pm[16], Wm[16];
    pl_eye(Pm, m);
    pl_eye(Wm, m);
    Pm[p + 4 * p] = P2[0]; Pm[(p + 1) + 4 * p] = P2[1]; Pm[p + 4 * (p + 1)] = P2[2]; Pm[(p + 1) + 4 * (p + 1)] = P2[3];
    Wm[p + 4 * p] = W2[0]; Wm[(p + 1) + 4 * p] = W2[1]; Wm[p + 4 * (p + 1)] = W2[2]; Wm[(p + 1) + 4 * (p + 1)] = W2[3];
    double A2[16], B2[16];
    pl_congr(Pm, An, Wm, A2, m);
    pl_congr(Pm, Bn, Wm, B2, m);
#pragma unroll
    for (int i = 0; i < 16; ++i) { An[i] = A2[i]; Bn[i] = B2[i]; }
    Bn[(p + 1) + 4 * p] = 0.0;
    Bn[p + 4 * (p + 1)] = 0.0;
    pl_mulr(U, Pm, m);
    pl_mulr(V, Wm, m);
    const double t11 = Bn[p + 4 * p], t22 = Bn[(p + 1) + 4 * (p + 1)];
    const double e11 = An[p + 4 * p] / t11, e12 = An[p + 4 * (p + 1)] / t11;
    const double e21 = An[(p + 1) + 4 * p] / t22, e22 = An[(p + 1) + 4 * (p + 1)] / t22;
    const double h = 0.5 * (e11 - e22);
    if (!(h * h + e12 * e21 < 0.0)) {
      if (why) { why[0] = 3.0; why[1] = h * h + e12 * e21; }
      return false;
    }
  }
  // G4: moved 1x1 blocks with t >= 0
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    int p = -1;
    if (q == 0 && n2 == 1) p = 0;
    if (q == 1 && n1 == 1) p = n2;
    if (p < 0 || !(Bn[p + 4 * p] < 0.0)) continue;
#pragma unroll
    for (int c = 0; c < m; ++c) { An[p + 4 * c] = -An[p + 4 * c]; Bn[p + 4 * c] = -Bn[p + 4 * c]; }
#pragma unroll
    for (int r = 0; r < m; ++r) U[r + 4 * p] = -U[r + 4 * p];
  }
  // G7: the largest-magnitude entry (the first such) of every column of V is positive; U's
  // column follows, the blocks change as D An D, D Bn D
  double d[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    int im = 0;
#pragma unroll
    for (int r = 1; r < m; ++r)
      if (fabs(V[r + 4 * c]) > fabs(V[im + 4 * c])) im = r;
    double vm = V[4 * c];
#pragma unroll
    for (int r = 1; r < m; ++r)
      if (r == im) vm = V[r + 4 * c];
    d[c] = (c < m && vm < 0.0) ? -1.0 : 1.0;
  }
#pragma unroll
  for (int c = 0; c < m; ++c)
#pragma unroll
    for (int r = 0; r < m; ++r) {
      U[r + 4 * c] *= d[c];
      V[r + 4 * c] *= d[c];
      An[r + 4 * c] *= d[r] * d[c];
      Bn[r + 4 * c] *= d[r] * d[c];
    }
  return true;
}

// The transform of one swap (G1-G4, G7).  A, B: the m x m blocks of S and T (ld 4, m = n1 + n2).
// Out: U, V (m x m), An = U^T A V, Bn = U^T B V in standard form.  Returns false = rejected.
template <int N1, int N2>
__host__ __device__ __forceinline__ bool pl_swap_t(const double* A, const double* B, double* U, double* V, double* An,
                                                   double* Bn, double* why) {
  constexpr int n1 = N1, n2 = N2, m = N1 + N2;
  double anorm = 0.0, bnorm = 0.0;   // Frobenius norms of the blocks (G3)
#pragma unroll
  for (int c = 0; c < m; ++c)
#pragma unroll
    for (int r = 0; r < m; ++r) {
      anorm = fma(A[r + 4 * c], A[r + 4 * c], anorm);
      bnorm = fma(B[r + 4 * c], B[r + 4 * c], bnorm);
    }
  anorm = sqrt(anorm);
  bnorm = sqrt(bnorm);
  const double eps = 2.220446049250313e-16, sml = 2.2250738585072014e-308 / 2.220446049250313e-16;
  const double thA = fmax(kG3C * eps * anorm, sml), thB = fmax(kG3C * eps * bnorm, sml);
  pl_eye(U, m);
  pl_eye(V, m);
  if (n1 == 1 && n2 == 1) {
    // G1: V e1 along the null vector of t22 S - s22 T; U e1 along S x or T x
    const double m11 = B[5] * A[0] - A[5] * B[0], m12 = B[5] * A[4] - A[5] * B[4];
    double c, s, r;
    pl_lartg(m12, -m11, c, s, r);
    V[0] = c; V[1] = s; V[4] = -s; V[5] = c;
    const double ax0 = A[0] * c + A[4] * s, ax1 = A[5] * s;
    const double bx0 = B[0] * c + B[4] * s, bx1 = B[5] * s;
    const double ra = anorm > 0.0 ? hypot(ax0, ax1) / anorm : 0.0;
    const double rb = bnorm > 0.0 ? hypot(bx0, bx1) / bnorm : 0.0;
    double c2, s2, r2;
    if (ra >= rb) pl_lartg(ax0, ax1, c2, s2, r2);
    else pl_lartg(bx0, bx1, c2, s2, r2);
    U[0] = c2; U[1] = s2; U[4] = -s2; U[5] = c2;
  } else {
    // G2: Sylvester bases V0, U0, and the two re-triangularisations of T's block (xTGEX2): from
    // the left (U from the QR of (T V0)(:, 1:n2), V = V0) and from the right (V completing the
    // row space of (U0^T T)(n2+1:m, :), U = U0)
    double R[4] = {0.0, 0.0, 0.0, 0.0}, L[4] = {0.0, 0.0, 0.0, 0.0};
    pl_gsylv<N1, N2>(A, B, R, L);
    double Mr[16], Ml[16], U0[16], V0[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { Mr[i] = 0.0; Ml[i] = 0.0; }
#pragma unroll
    for (int c = 0; c < n2; ++c) {
#pragma unroll
      for (int r = 0; r < n1; ++r) { Mr[r + 4 * c] = -R[r + 2 * c]; Ml[r + 4 * c] = -L[r + 2 * c]; }
      Mr[(n1 + c) + 4 * c] = 1.0;
      Ml[(n1 + c) + 4 * c] = 1.0;
    }
    pl_qr_basis(Mr, m, n2, V0);
    pl_qr_basis(Ml, m, n2, U0);
    double I4[16], TV[16], UT[16], Uq[16], H[16], Vr[16], Aq[16], Ar[16];
    pl_eye(I4, m);
    pl_congr(I4, B, V0, TV, m);
#pragma unroll
    for (int i = 0; i < 16; ++i) { Mr[i] = 0.0; Ml[i] = 0.0; }
#pragma unroll
    for (int c = 0; c < n2; ++c)
#pragma unroll
      for (int r = 0; r < m; ++r) Ml[r + 4 * c] = TV[r + 4 * c];
    pl_qr_basis(Ml, m, n2, Uq);
    pl_congr(U0, B, I4, UT, m);
#pragma unroll
    for (int c = 0; c < n1; ++c)
#pragma unroll
      for (int r = 0; r < m; ++r) Mr[r + 4 * c] = UT[(n2 + c) + 4 * r];
    pl_qr_basis(Mr, m, n1, H);
#pragma unroll
    for (int i = 0; i < 16; ++i) Vr[i] = 0.0;
#pragma unroll
    for (int c = 0; c < n2; ++c)
#pragma unroll
      for (int r = 0; r < m; ++r) Vr[r + 4 * c] = H[r + 4 * (n1 + c)];
#pragma unroll
    for (int c = 0; c < n1; ++c)
#pragma unroll
      for (int r = 0; r < m; ++r) Vr[r + 4 * (n2 + c)] = H[r + 4 * c];
    // G3: each candidate's residual max(||S21|| / thA, ||T21|| / thB); keep the smallest (ties:
    // the earlier) -- the Sylvester pair (U0, V0), the left and the right re-triangularisation
    double best = 0.0;
    int bi = 0;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double* cu = q == 1 ? Uq : U0;
      const double* cv = q == 2 ? Vr : V0;
      pl_congr(cu, A, cv, Aq, m);
      pl_congr(cu, B, cv, Ar, m);
      const double r = fmax(pl_lowfro(Aq, n1, n2) / thA, pl_lowfro(Ar, n1, n2) / thB);
      if (q == 0 || r < best) { best = r; bi = q; }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      U[i] = bi == 1 ? Uq[i] : U0[i];
      V[i] = bi == 2 ? Vr[i] : V0[i];
    }
    if (!(best <= 1.0)) {
      if (why) { why[0] = 1.0; why[1] = best; }
      return false;
    }
    if (why) { why[0] = 0.0; why[1] = best; }
  }
  pl_congr(U, A, V, An, m);
  pl_congr(U, B, V, Bn, m);
  if (n1 == 1 && n2 == 1) {
    // G3 (1x1|1x1): both blocks below the new leading block
    const double resA = pl_lowfro(An, n1, n2), resB = pl_lowfro(Bn, n1, n2);
    if (!(resA <= thA && resB <= thB)) {
      if (why) { why[0] = 1.0; why[1] = fmax(resA / thA, resB / thB); }
      return false;
    }
    if (why) { why[0] = 0.0; why[1] = fmax(resA / thA, resB / thB); }
  }
  return pl_swap_tail<N1, N2>(U, V, An, Bn, why);
}


// The same transform for N1 + N2 >= 3 by a group of 4 lanes (all 32 lanes of the warp call it;
// role = lane & 3), with the same arithmetic on every value it produces (so the same record as
// pl_swap_t): the Sylvester pair on every lane; the two Sylvester bases V0 (even lanes) and U0
// (odd lanes), exchanged; the two re-triangularisations Uq (even) and Vr (odd) -- each one
// congruence and one QR -- exchanged; the three G3 candidates on roles 0, 1, 2; the winner's
// blocks by shuffle; then G4 / G7 on every lane.  Critical path: one Sylvester solve, two QRs,
// three congruences instead of one Sylvester solve, four QRs and nine congruences.
__device__ __forceinline__ void pl_xchg16(const double* mine, double* other, int lane) {
#pragma unroll
  for (int i = 0; i < 16; ++i) other[i] = __shfl_sync(0xffffffffu, mine[i], lane ^ 1);
}

template <int N1, int N2>
__device__ bool pl_swap_lanes(const double* A, const double* B, double* U, double* V, double* An, double* Bn,
                              double* why, int lane, unsigned long long* prof = nullptr) {
  constexpr int n1 = N1, n2 = N2, m = N1 + N2;
  // debug (SN_PPROF): cycles to the end of the Sylvester solve, the bases, the candidates, all
  const long long k0 = prof ? clock64() : 0;
  auto mark = [&](int q) { if (prof && lane == 0) atomicAdd(&prof[q], (unsigned long long)(clock64() - k0)); };
  const int role = lane & 3, odd = lane & 1, gbase = lane & ~3;
  double anorm = 0.0, bnorm = 0.0;
#pragma unroll
  for (int c = 0; c < m; ++c)
#pragma unroll
    for (int r = 0; r < m; ++r) {
      anorm = fma(A[r + 4 * c], A[r + 4 * c], anorm);
      bnorm = fma(B[r + 4 * c], B[r + 4 * c], bnorm);
    }
  anorm = sqrt(anorm);
  bnorm = sqrt(bnorm);
  const double eps = 2.220446049250313e-16, sml = 2.2250738585072014e-308 / 2.220446049250313e-16;
  const double thA = fmax(kG3C * eps * anorm, sml), thB = fmax(kG3C * eps * bnorm, sml);
  double R[4] = {0.0, 0.0, 0.0, 0.0}, L[4] = {0.0, 0.0, 0.0, 0.0};
  pl_gsylv_lanes<N1, N2>(A, B, R, L, lane);
  mark(0);
  // Sylvester bases: even lanes V0 = basis of span[-R; I], odd lanes U0 = basis of span[-L; I]
  double M[16], X[16], Y[16], U0[16], V0[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) M[i] = 0.0;
#pragma unroll
  for (int c = 0; c < n2; ++c) {
#pragma unroll
    for (int r = 0; r < n1; ++r) M[r + 4 * c] = -(odd ? L[r + 2 * c] : R[r + 2 * c]);
    M[(n1 + c) + 4 * c] = 1.0;
  }
  pl_qr_basis(M, m, n2, X);
  pl_xchg16(X, Y, lane);
#pragma unroll
  for (int i = 0; i < 16; ++i) { V0[i] = odd ? Y[i] : X[i]; U0[i] = odd ? X[i] : Y[i]; }
  // re-triangularisations: even lanes Uq from the QR of (T V0)(:, 1:n2); odd lanes Vr completing
  // the row space of (U0^T T)(n2+1:m, :)
  double I4[16], Ua[16], Va[16], W[16];
  pl_eye(I4, m);
#pragma unroll
  for (int i = 0; i < 16; ++i) { Ua[i] = odd ? U0[i] : I4[i]; Va[i] = odd ? I4[i] : V0[i]; }
  pl_congr(Ua, B, Va, W, m);
#pragma unroll
  for (int i = 0; i < 16; ++i) M[i] = 0.0;
  if (odd) {
#pragma unroll
    for (int c = 0; c < n1; ++c)
#pragma unroll
      for (int r = 0; r < m; ++r) M[r + 4 * c] = W[(n2 + c) + 4 * r];
    pl_qr_basis(M, m, n1, X);
  } else {
#pragma unroll
    for (int c = 0; c < n2; ++c)
#pragma unroll
      for (int r = 0; r < m; ++r) M[r + 4 * c] = W[r + 4 * c];
    pl_qr_basis(M, m, n2, X);
  }
  if (odd) {   // Vr: H's last n2 columns, then its first n1
#pragma unroll
    for (int i = 0; i < 16; ++i) Y[i] = 0.0;
#pragma unroll
    for (int c = 0; c < n2; ++c)
#pragma unroll
      for (int r = 0; r < m; ++r) Y[r + 4 * c] = X[r + 4 * (n1 + c)];
#pragma unroll
    for (int c = 0; c < n1; ++c)
#pragma unroll
      for (int r = 0; r < m; ++r) Y[r + 4 * (n2 + c)] = X[r + 4 * c];
#pragma unroll
    for (int i = 0; i < 16; ++i) X[i] = Y[i];
  }
  double Uq[16], Vr[16];
  pl_xchg16(X, Y, lane);
#pragma unroll
  for (int i = 0; i < 16; ++i) { Uq[i] = odd ? Y[i] : X[i]; Vr[i] = odd ? X[i] : Y[i]; }
  mark(1);
  // G3 candidates: role 0 (U0, V0), 1 (Uq, V0), 2 (U0, Vr) (role 3 repeats role 0)
  double Aq[16], Ar[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { Ua[i] = role == 1 ? Uq[i] : U0[i]; Va[i] = role == 2 ? Vr[i] : V0[i]; }
  pl_congr(Ua, A, Va, Aq, m);
  pl_congr(Ua, B, Va, Ar, m);
  const double rq = fmax(pl_lowfro(Aq, n1, n2) / thA, pl_lowfro(Ar, n1, n2) / thB);
  const double r0 = __shfl_sync(0xffffffffu, rq, gbase), r1 = __shfl_sync(0xffffffffu, rq, gbase + 1),
               r2 = __shfl_sync(0xffffffffu, rq, gbase + 2);
  double best = r0;
  int bi = 0;
  if (r1 < best) { best = r1; bi = 1; }
  if (r2 < best) { best = r2; bi = 2; }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    U[i] = bi == 1 ? Uq[i] : U0[i];
    V[i] = bi == 2 ? Vr[i] : V0[i];
    An[i] = __shfl_sync(0xffffffffu, Aq[i], gbase + bi);   // = U^T A V, bitwise (same congruence)
    Bn[i] = __shfl_sync(0xffffffffu, Ar[i], gbase + bi);
  }
  if (!(best <= 1.0)) {
    if (why) { why[0] = 1.0; why[1] = best; }
    return false;
  }
  if (why) { why[0] = 0.0; why[1] = best; }
  mark(2);
  const bool ok = pl_swap_tail<N1, N2>(U, V, An, Bn, why);
  mark(3);
  if (prof && lane == 0) atomicAdd(&prof[4], 1ull);   // marks taken
  return ok;
}

__host__ __device__ inline bool pl_swap(const double* A, const double* B, int n1, int n2, double* U, double* V,
                                        double* An, double* Bn, double* why = nullptr) {
  if (n1 == 1 && n2 == 1) return pl_swap_t<1, 1>(A, B, U, V, An, Bn, why);
  if (n1 == 1) return pl_swap_t<1, 2>(A, B, U, V, An, Bn, why);
  if (n2 == 1) return pl_swap_t<2, 1>(A, B, U, V, An, Bn, why);
  return pl_swap_t<2, 2>(A, B, U, V, An, Bn, why);
}

// One thread's transform of a swap of type (N1, N2) at window row j into the record R.
template <int N1, int N2>
__device__ __forceinline__ bool pl_transform(const double* Sw, int64_t ldS, const double* Tw, int64_t ldT, int j,
                                             double* R, double* why) {
  constexpr int m = N1 + N2;
  double A[16], B[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { A[i] = 0.0; B[i] = 0.0; }
#pragma unroll
  for (int c = 0; c < m; ++c)
#pragma unroll
    for (int r = 0; r < m; ++r) {
      A[r + 4 * c] = __ldcg(Sw + (j + r) + (int64_t)(j + c) * ldS);
      B[r + 4 * c] = __ldcg(Tw + (j + r) + (int64_t)(j + c) * ldT);
    }
  double U[16], V[16], An[16], Bn[16];
  const bool ok = pl_swap_t<N1, N2>(A, B, U, V, An, Bn, why);
#pragma unroll
  for (int i = 0; i < 16; ++i) { R[i] = U[i]; R[16 + i] = V[i]; R[32 + i] = An[i]; R[48 + i] = Bn[i]; }
  return ok;
}

// A group of 4 lanes' transform of a swap of type (N1, N2), N1 + N2 >= 3 (pl_swap_lanes); the
// lane with `write` stores the record.
template <int N1, int N2>
__device__ __forceinline__ bool pl_transform_lanes(const double* Sw, int64_t ldS, const double* Tw, int64_t ldT, int j,
                                                   double* R, double* why, int lane, bool write,
                                                   unsigned long long* prof) {
  constexpr int m = N1 + N2;
  double A[16], B[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { A[i] = 0.0; B[i] = 0.0; }
#pragma unroll
  for (int c = 0; c < m; ++c)
#pragma unroll
    for (int r = 0; r < m; ++r) {
      A[r + 4 * c] = __ldcg(Sw + (j + r) + (int64_t)(j + c) * ldS);
      B[r + 4 * c] = __ldcg(Tw + (j + r) + (int64_t)(j + c) * ldT);
    }
  double U[16], V[16], An[16], Bn[16];
  const bool ok = pl_swap_lanes<N1, N2>(A, B, U, V, An, Bn, why, lane, prof);
  if (write) {
#pragma unroll
    for (int i = 0; i < 16; ++i) { R[i] = U[i]; R[16 + i] = V[i]; R[32 + i] = An[i]; R[48 + i] = Bn[i]; }
  }
  return ok;
}

// ---------------------------------------------------------------- the window task (device)
// The swaps of a window run in steps: the host assigns each swap (in the order of the standard
// kernel's swap list) the step after the last earlier swap whose rows it overlaps, so the
// swaps of one step act on pairwise disjoint row ranges.  Such swaps commute exactly (their
// left and right transforms touch disjoint rows / columns, and none touches another's
// diagonal block), so one step is: every swap's transform from the current blocks (one thread
// each), then all row applications, then all column applications.  A step with a rejected swap
// is not applied (the window stops after the previous step, a closed set of swaps).
constexpr int kRecD = 64;   // doubles per swap record in shared memory: U, V, An, Bn (4x4 each)

struct PencilWinArgs {
  const WinDev* wins;       // this level's windows
  int32_t nwin;
  int32_t base;
  const int64_t* swap_off;  // per sorted window: first swap (nw + 1 entries), step-sorted
  const int32_t* step_off;  // per sorted window: steps at step_base[sidx] .. (+ nsteps + 1)
  const int64_t* step_base;
  const int16_t* sj;        // window-local first row of each swap
  const int8_t* s12;        // (n1 << 4) | n2
  const int32_t* sidx;      // index of each swap in the window's list order
  double* S;
  int64_t ldS;
  double* T;
  int64_t ldT;
  double* UL;               // slot arrays (kZslot doubles per slot)
  double* VR;
  int16_t* zrange;          // per slot (shared by UL and VR: same column structure)
  int32_t* status;
  int32_t* done;            // per sorted window: swaps completed (a prefix of the step-sorted list)
  Control* ctl;
  int64_t force_order;
  int32_t force_swap;
  unsigned long long* pprof;   // debug (SN_PPROF): cycles per phase summed over windows, or NULL
};

// pre[0] = 0, pre[i + 1] = pre[i] + val(i) for i < cnt, by one warp (lane: 0..31)
template <class F>
__device__ __forceinline__ void pl_warp_prefix(int* pre, int cnt, int lane, F val) {
  const int per = (cnt + 31) >> 5, b = lane * per, e = min(b + per, cnt);
  int local = 0;
  for (int i = b; i < e; ++i) local += val(i);
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  int run = incl - local;
  if (lane == 0) pre[0] = 0;
  for (int i = b; i < e; ++i) { run += val(i); pre[i + 1] = run; }
}

// index i with pre[i] <= q < pre[i + 1]
__device__ __forceinline__ int pl_find(const int* pre, int cnt, int q) {
  int lo = 0, hi = cnt - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= q) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ unsigned pl_cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned pl_cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

// Window task on a thread-block cluster of C CTAs (C = 1: a plain CTA).  The transforms of a
// step are split over the CTAs (swap i on CTA i % C), each CTA gathers the others' records
// from distributed shared memory (the same values: the applications do not depend on which CTA
// evaluated a transform), the block-size bookkeeping runs in every CTA's own shared memory,
// and the row and column applications -- the bulk of the work -- are split over the C x 256
// threads.  Phases that
// read what another CTA wrote are separated by cluster barriers (release / acquire), and every
// global read of the window, T, UL and VR bypasses L1 (ld.global.cg), so no CTA sees a stale
// line of another SM's writes.
__global__ void __launch_bounds__(256) pencil_window_kernel(PencilWinArgs a) {
  extern __shared__ double rec[];            // kRecD doubles per swap of the current step
  const unsigned C = pl_cluster_size(), rank = pl_cluster_rank();
  const WinDev wd = a.wins[blockIdx.x / C];
  const int tid = threadIdx.x;
  const int gt = (int)rank * (int)blockDim.x + tid, GC = (int)(C * blockDim.x);   // cluster thread id / count
  auto csync = [&]() {
    if (C > 1)
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else
      __syncthreads();
  };
  const int k = wd.k;
  double* Sw = a.S + wd.j1 + wd.j1 * a.ldS;
  double* Tw = a.T + wd.j1 + wd.j1 * a.ldT;
  double* UL = a.UL + (int64_t)wd.slot * kZslot;
  double* VR = a.VR + (int64_t)wd.slot * kZslot;
  const int64_t ldS = a.ldS, ldT = a.ldT;
  __shared__ int16_t zlo[kZld], zhi[kZld];
  __shared__ int s_pre[kZld + 1];
  __shared__ int16_t s_j[kZld];      // per swap of the current step: window row, size m
  __shared__ int8_t s_m[kZld];
  __shared__ int16_t s_lo[kZld], s_hi[kZld];   // merged nonzero row interval of its UL/VR columns
  __shared__ int s_tstart[4];                  // first swap of each type in the current step
  __shared__ int8_t s_owner[kZld];             // CTA of the cluster that evaluates each swap
  __shared__ int s_rej, s_rejall;   // first rejected swap (list index): this CTA's, the cluster's
  __shared__ double s_why[2];
  cg::cluster_group cl = cg::this_cluster();
  for (int64_t i = gt; i < kZslot; i += GC) {
    const int r = (int)(i % kZld), c = (int)(i / kZld);
    const double v = (r == c && c < k) ? 1.0 : 0.0;
    UL[i] = v;
    VR[i] = v;
  }
  if (tid < kZld) {
    zlo[tid] = (int16_t)(tid < k ? tid : kZld - 1);
    zhi[tid] = (int16_t)(tid < k ? tid : 0);
  }
  if (tid == 0) s_rej = s_rejall = 0x7fffffff;
  csync();
  const int64_t s0 = a.swap_off[wd.sidx];
  const int32_t* soff = a.step_off + a.step_base[wd.sidx];
  const int nsteps = (int)(a.step_base[wd.sidx + 1] - a.step_base[wd.sidx]) - 1;
  int done_steps = 0;
  unsigned long long pc[6] = {0, 0, 0, 0, 0, 0};   // transforms, intervals, rows, columns, tid 0's own row /
                                                  // column tasks (tid 0, SN_PPROF)
  long long pk = a.pprof && tid == 0 ? clock64() : 0;
  auto ptick = [&](int q) {
    if (a.pprof && tid == 0) { const long long c = clock64(); pc[q] += (unsigned long long)(c - pk); pk = c; }
  };
  for (int st = 0; st < nsteps; ++st) {
    const int b0 = soff[st], cnt = soff[st + 1] - b0;
    // (1) transforms, one thread per swap.  The step's swaps are sorted by type (host); a warp
    // takes up to 32 swaps of ONE type (a warp running several specialisations of the
    // transform would run them one after the other), and the warp tasks are spread over the
    // cluster's CTAs first (task g on CTA g % C, warp g / C).
    if (tid < 4) s_tstart[tid] = cnt;
    __syncthreads();
    for (int i = tid; i < cnt; i += blockDim.x) {
      const int64_t s = s0 + b0 + i;
      const int8_t v = a.s12[s];
      s_j[i] = (int16_t)a.sj[s];
      s_m[i] = (int8_t)((v >> 4) + (v & 15));
      const int ty = ((v >> 4) - 1) * 2 + ((v & 15) - 1);
      int tp = -1;
      if (i > 0) { const int8_t u = a.s12[s - 1]; tp = ((u >> 4) - 1) * 2 + ((u & 15) - 1); }
      for (int t = tp + 1; t <= ty; ++t) s_tstart[t] = i;   // first swap of type >= t
    }
    __syncthreads();
    // a warp task: 32 swaps of type (1,1) (one per lane), or 8 of another type (a group of 4
    // lanes per swap, pl_swap_lanes)
    int tbase[5];                                      // first warp task of each type
    tbase[0] = 0;
    for (int t = 0; t < 4; ++t) {
      const int lg = t == 0 ? 5 : 3;
      tbase[t + 1] = tbase[t] + (((t < 3 ? s_tstart[t + 1] : cnt) - s_tstart[t] + (1 << lg) - 1) >> lg);
    }
    for (int i = tid; i < cnt; i += blockDim.x) {
      int t = 0;
      while (t < 3 && s_tstart[t + 1] <= i) ++t;
      s_owner[i] = (int8_t)((tbase[t] + ((i - s_tstart[t]) >> (t == 0 ? 5 : 3))) % (int)C);
    }
    const int lane = tid & 31;
    for (int g = (tid >> 5) * (int)C + (int)rank; g < tbase[4]; g += (int)(C * (blockDim.x >> 5))) {
      int t = 0;
      while (t < 3 && tbase[t + 1] <= g) ++t;
      const int tend = t < 3 ? s_tstart[t + 1] : cnt;
      const int i0 = s_tstart[t] + (t == 0 ? ((g - tbase[t]) << 5) + lane : ((g - tbase[t]) << 3) + (lane >> 2));
      const bool mine = i0 < tend && (t == 0 || (lane & 3) == 0);   // writes the record
      const int i = min(i0, tend - 1);               // idle groups repeat a valid swap (no writes)
      if (t == 0 && i0 >= tend) continue;
      {
        const int64_t s = s0 + b0 + i;
        const int j = a.sj[s];
        double* R = rec + i * kRecD;
        double why[2] = {0.0, 0.0};
        bool ok;
        const long long tq0 = a.pprof ? clock64() : 0;
        if (t == 0) ok = pl_transform<1, 1>(Sw, ldS, Tw, ldT, j, R, why);
        else if (t == 1) ok = pl_transform_lanes<1, 2>(Sw, ldS, Tw, ldT, j, R, why, lane, mine, nullptr);
        else if (t == 2) ok = pl_transform_lanes<2, 1>(Sw, ldS, Tw, ldT, j, R, why, lane, mine, nullptr);
        else ok = pl_transform_lanes<2, 2>(Sw, ldS, Tw, ldT, j, R, why, lane, mine, a.pprof ? a.pprof + 18 : nullptr);
        if (mine) {
          if (a.pprof) {   // per-type transform latency (sum, count)
            atomicAdd(&a.pprof[8 + t], (unsigned long long)(clock64() - tq0));
            atomicAdd(&a.pprof[12 + t], 1ull);
          }
          if (wd.order == a.force_order && a.sidx[s] == a.force_swap) { ok = false; why[0] = 0.0; }
          if (ok) atomicMax(&a.ctl->ratio_bits, (unsigned long long)__double_as_longlong(why[1]));
          if (!ok) {
            const int key = a.sidx[s];
            if (atomicMin(&s_rej, key) > key) { s_why[0] = why[0]; s_why[1] = why[1]; }
          }
        }
      }
    }
    csync();   // every transform is done (and every diagonal block read) before any is overwritten
    if (C > 1) {
      // gather the records the other CTAs computed (distributed shared memory) and the
      // cluster-wide first rejection
      for (int q = tid; q < cnt * kRecD; q += blockDim.x) {
        const unsigned owner = (unsigned)s_owner[q / kRecD];
        if (owner != rank) rec[q] = cl.map_shared_rank(rec, owner)[q];
      }
      if (tid == 0) {
        int best = s_rej;
        for (unsigned r = 0; r < C; ++r) best = min(best, *cl.map_shared_rank(&s_rej, r));
        if (best != 0x7fffffff && rank == 0 && s_rej != best)
          for (unsigned r = 1; r < C; ++r)
            if (*cl.map_shared_rank(&s_rej, r) == best) {
              s_why[0] = cl.map_shared_rank(s_why, r)[0];
              s_why[1] = cl.map_shared_rank(s_why, r)[1];
            }
        s_rejall = best;
      }
      __syncthreads();
    } else if (tid == 0) {
      s_rejall = s_rej;
    }
    __syncthreads();
    ptick(0);
    if (s_rejall != 0x7fffffff) break;
    // (2) column intervals of the accumulators; row-application task counts
    if (tid < cnt) {
      const int j = s_j[tid], m = s_m[tid];
      int lo = zlo[j], hi = zhi[j];
      for (int c = 1; c < m; ++c) { lo = min(lo, (int)zlo[j + c]); hi = max(hi, (int)zhi[j + c]); }
      for (int c = 0; c < m; ++c) { zlo[j + c] = (int16_t)lo; zhi[j + c] = (int16_t)hi; }
      s_lo[tid] = (int16_t)lo;
      s_hi[tid] = (int16_t)hi;
    }
    if (tid < 32) pl_warp_prefix(s_pre, cnt, tid, [&](int i) { return 2 * (k - s_j[i] - s_m[i]); });
    __syncthreads();
    ptick(1);
    // (3) rows j..j+m-1 right of each block (S, T); the new diagonal blocks
    for (int q = gt; q < cnt * 16; q += GC) {
      const int i = q >> 4, d = q & 15, m = s_m[i];
      if (d >= m * m) continue;
      const int j = s_j[i], r = d % m, c = d / m;
      const double* R = rec + i * kRecD;
      Sw[(j + r) + (int64_t)(j + c) * ldS] = R[32 + r + 4 * c];
      Tw[(j + r) + (int64_t)(j + c) * ldT] = R[48 + r + 4 * c];
    }
    // a task = one m-vector of S, T, UL or VR times an m x m factor G: y[t] = sum_l G[l + 4t] x[l]
    // (rows: x along a column, G = U; columns: x along a row, G = V or U); two tasks per
    // thread and round, loads first, so their memory latencies overlap (tasks are disjoint)
    auto row_task = [&](int q, double*& X, int64_t& base, int64_t& stride, const double*& G, int& m) {
      const int i = pl_find(s_pre, cnt, q);
      const int j = s_j[i];
      m = s_m[i];
      G = rec + i * kRecD;
      const int nl = k - j - m, e = q - s_pre[i];
      const bool isT = e >= nl;
      X = isT ? Tw : Sw;
      const int64_t ld = isT ? ldT : ldS;
      base = j + (int64_t)(j + m + (isT ? e - nl : e)) * ld;
      stride = 1;
    };
    auto col_task = [&](int q, double*& X, int64_t& base, int64_t& stride, const double*& G, int& m) {
      const int i = pl_find(s_pre, cnt, q);
      const int j = s_j[i];
      m = s_m[i];
      const double* R = rec + i * kRecD;
      const int e = q - s_pre[i];
      int64_t r;
      if (e < 2 * j) {
        const bool isT = e >= j;
        X = isT ? Tw : Sw; stride = isT ? ldT : ldS; r = isT ? e - j : e; G = R + 16;
      } else {
        // UL / VR columns j..j+m-1 are exact zeros outside the merged interval [lo, hi]
        const int e3 = e - 2 * j, len = s_hi[i] - s_lo[i] + 1;
        const bool isV = e3 >= len;
        X = isV ? VR : UL; stride = kZld; r = s_lo[i] + (isV ? e3 - len : e3); G = isV ? R + 16 : R;
      }
      base = r + (int64_t)j * stride;
    };
    for (int phase = 0; phase < 2; ++phase) {
      if (phase == 1) {
        csync();   // row applications (all CTAs) before column applications (corner order)
        ptick(2);
        if (tid < 32) pl_warp_prefix(s_pre, cnt, tid, [&](int i) { return 2 * s_j[i] + 2 * (s_hi[i] - s_lo[i] + 1); });
        __syncthreads();
      }
      const int total = s_pre[cnt];
      constexpr int NU = 4;   // tasks per thread and round: their loads are all in flight at once
      const long long lq0 = a.pprof && tid == 0 ? clock64() : 0;
      for (int q0 = gt; q0 < total; q0 += NU * GC) {
        double* X[NU];
        int64_t base[NU], stride[NU];
        const double* G[NU];
        int m[NU];
        double x[NU][4];
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          const int q = q0 + u * GC;
          m[u] = 0;
          if (q < total) {
            if (phase == 0) row_task(q, X[u], base[u], stride[u], G[u], m[u]);
            else col_task(q, X[u], base[u], stride[u], G[u], m[u]);
          }
#pragma unroll
          for (int t = 0; t < 4; ++t) x[u][t] = t < m[u] ? __ldcg(X[u] + base[u] + t * stride[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          double y[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            double acc = 0.0;
#pragma unroll
            for (int l = 0; l < 4; ++l) acc = (l < m[u]) ? fma(G[u][l + 4 * t], x[u][l], acc) : acc;
            y[t] = acc;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (t < m[u]) X[u][base[u] + t * stride[u]] = y[t];
        }
      }
      if (a.pprof && tid == 0) pc[4 + phase] += (unsigned long long)(clock64() - lq0);   // tid 0's own tasks
    }
    done_steps = st + 1;
    csync();
    ptick(3);
  }
  if (a.pprof && tid == 0 && rank == 0) {
    for (int q = 0; q < 4; ++q) atomicAdd(&a.pprof[q], pc[q]);
    atomicAdd(&a.pprof[16], pc[4]);
    atomicAdd(&a.pprof[17], pc[5]);
    atomicAdd(&a.pprof[4], (unsigned long long)nsteps);
    atomicAdd(&a.pprof[5], 1ull);
    atomicAdd(&a.pprof[6], (unsigned long long)(soff[nsteps] - soff[0]));
  }
  const int done = soff[done_steps] - soff[0];
  const int total = soff[nsteps] - soff[0];
  csync();   // no CTA leaves while another may still read its shared memory
  if (rank != 0) return;
  if (tid < kZld) {
    int16_t* zr = a.zrange + (int64_t)wd.slot * kZrange;
    zr[tid] = zlo[tid];
    zr[kZld + tid] = zhi[tid];
  }
  if (tid == 0) {
    const bool partial = done < total;
    a.status[wd.sidx] = partial ? kWinPartial : kWinDone;
    a.done[wd.sidx] = done;
    if (partial && atomicCAS(&a.ctl->abort, 0, 1) == 0) {
      // the rejecting swap with the smallest list index in the failed step
      int64_t s = s0 + done;
      for (int64_t q = s0 + soff[done_steps]; q < s0 + soff[done_steps + 1]; ++q)
        if (a.sidx[q] == s_rej) s = q;
      a.ctl->rej_window = wd.sidx;
      a.ctl->rej_swaps_done = done;
      a.ctl->rej_row = (int32_t)(wd.j1 + a.sj[s]);
      a.ctl->rej_n1 = a.s12[s] >> 4;
      a.ctl->rej_n2 = a.s12[s] & 15;
      a.ctl->pad[0] = (int32_t)s_why[0];                       // failed test: 1 G3, 2/3 G4, 0 forced
      a.ctl->pad[1] = (int32_t)fmin(s_why[1] * 1000.0, 2e9);   // G3: residual / threshold x 1000
    }
  }
}

#define PK(x)                                                          \
  do {                                                                 \
    cudaError_t e_ = (x);                                              \
    if (e_ != cudaSuccess) {                                           \
      if (std::getenv("SN_DEBUG"))                                     \
        std::fprintf(stderr, "sn: %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      rc = SN_ERR_CUDA;                                                \
      goto done;                                                       \
    }                                                                  \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 8); }
};

int run_pencil(const sn_opts& o, int64_t n, double* S, int64_t ldS, double* T, int64_t ldT, double* Q, int64_t ldQ,
               double* Zm, int64_t ldZ, int32_t* select, int64_t* m, int8_t* bmap_out, sn_stats* st,
               cudaStream_t sA) {
  const double t0 = now_ms();
  int rc = 0;
  DevBuf dpprof;
  DevBuf dsub, dbad, dwins, doff, dsj, ds12, dpref, dstatus, ddone, dctl, dUL, dVR, dzr, dstep, dstepb, didx;
  std::vector<uint8_t> sub((size_t)n);
  int32_t bad = 0;
  std::vector<int8_t> bmap((size_t)n), selrow((size_t)n);
  Plan P;
  std::vector<int64_t> sorted, lstart;
  std::vector<WinDev> wd;
  std::vector<int64_t> off;
  std::vector<int16_t> hsj;
  std::vector<int8_t> hs12;
  std::vector<int32_t> hidx, hstep;
  std::vector<int64_t> hstep_base;
  int max_step_cnt = 1;
  std::vector<int32_t> pref;
  std::vector<int64_t> pref_off;
  std::vector<int32_t> nstr;
  std::vector<int32_t> hstatus, hdone;
  int64_t maxper = 0, nw = 0, levels_run = 0;
  Control hctl{};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const int NT = 64;
  PanelMaps mSL{}, mTL{}, mSR{}, mTR{}, mQ{}, mZ{};
  std::memset(st, 0, sizeof(*st));
  st->rejected_window = -1;
  st->rejected_row = -1;

  PK(dsub.alloc((size_t)n + 8));
  PK(dbad.alloc(8));
  PK(cudaMemsetAsync(dbad.p, 0, 4, sA));
  launch_scan(S, ldS, n, o.validate_lower, (uint8_t*)dsub.p, (int32_t*)dbad.p, sA);
  PK(cudaGetLastError());
  PK(cudaMemcpyAsync(sub.data(), dsub.p, (size_t)n, cudaMemcpyDeviceToHost, sA));
  PK(cudaMemcpyAsync(&bad, dbad.p, 4, cudaMemcpyDeviceToHost, sA));
  PK(cudaStreamSynchronize(sA));
  if (bad) return -2;
  if ((rc = structure_from_sub(n, sub.data(), select, bmap.data(), selrow.data(), m))) return rc;
  if (build_plan(n, bmap.data(), selrow.data(), o.window, o.inner_window, o.max_windows, &P)) return SN_ERR_UNSUPPORTED;
  nw = (int64_t)P.wins.size();
  sorted.resize(nw);
  for (int64_t i = 0; i < nw; ++i) sorted[i] = i;
  std::stable_sort(sorted.begin(), sorted.end(), [&](int64_t x, int64_t y) { return P.wins[x].level < P.wins[y].level; });
  lstart.assign(P.nlevels + 1, 0);
  for (int64_t i = 0; i < nw; ++i) lstart[P.wins[sorted[i]].level + 1]++;
  for (int64_t l = 0; l < P.nlevels; ++l) lstart[l + 1] += lstart[l];
  for (int64_t l = 0; l < P.nlevels; ++l) maxper = std::max(maxper, lstart[l + 1] - lstart[l]);
  // per window: swap list (kernel execution order), descriptors; per level and kind: strips
  wd.resize(nw);
  off.assign(nw + 1, 0);
  {
    const int64_t cap = o.window * o.window / 4 + o.window + 4;
    std::vector<int64_t> sj((size_t)cap);
    std::vector<int8_t> a1((size_t)cap), a2((size_t)cap);
    for (int64_t i = 0; i < nw; ++i) {
      const WindowPlan& w = P.wins[sorted[i]];
      const int64_t cnt = window_swaps(P, sorted[i], cap, sj.data(), a1.data(), a2.data());
      if (cnt < 0) return SN_ERR_UNSUPPORTED;
      // steps: each swap goes one step after the last earlier swap overlapping its rows
      std::vector<int32_t> last((size_t)w.k + 4, -1), stp((size_t)cnt);
      int32_t ns = 0;
      for (int64_t q = 0; q < cnt; ++q) {
        const int64_t j = sj[q] - w.j1;
        const int mm = a1[q] + a2[q];
        int32_t t = 0;
        for (int r = 0; r < mm; ++r) t = std::max(t, last[j + r] + 1);
        for (int r = 0; r < mm; ++r) last[j + r] = t;
        stp[q] = t;
        ns = std::max(ns, t + 1);
      }
      std::vector<int32_t> per((size_t)ns + 1, 0);
      for (int64_t q = 0; q < cnt; ++q) per[stp[q] + 1]++;
      for (int32_t t = 0; t < ns; ++t) {
        max_step_cnt = std::max(max_step_cnt, per[t + 1]);
        per[t + 1] += per[t];
      }
      hstep_base.push_back((int64_t)hstep.size());
      for (int32_t t = 0; t <= ns; ++t) hstep.push_back(per[t]);
      // within a step, group the swaps by type (consecutive threads, so most warps run one
      // specialisation of the transform), in list order within a type
      std::vector<int64_t> ord((size_t)cnt);
      {
        std::vector<int32_t> fill((size_t)ns * 4 + 1, 0);   // counting sort by (step, type)
        for (int64_t q = 0; q < cnt; ++q) fill[(size_t)stp[q] * 4 + (a1[q] - 1) * 2 + (a2[q] - 1) + 1]++;
        for (size_t t = 1; t < fill.size(); ++t) fill[t] += fill[t - 1];
        for (int64_t q = 0; q < cnt; ++q) ord[fill[(size_t)stp[q] * 4 + (a1[q] - 1) * 2 + (a2[q] - 1)]++] = q;
      }
      for (int64_t q = 0; q < cnt; ++q) {
        const int64_t o = ord[q];
        hsj.push_back((int16_t)(sj[o] - w.j1));
        hs12.push_back((int8_t)((a1[o] << 4) | a2[o]));
        hidx.push_back((int32_t)o);
      }
      off[i + 1] = off[i] + cnt;
    }
  }
  pref_off.assign(P.nlevels * 3, 0);
  nstr.assign(P.nlevels * 3, 0);
  for (int64_t l = 0; l < P.nlevels; ++l) {
    const int64_t a = lstart[l], b = lstart[l + 1];
    for (int kind = 0; kind < 3; ++kind) {
      pref_off[l * 3 + kind] = (int64_t)pref.size();
      int32_t acc = 0;
      pref.push_back(0);
      for (int64_t i = a; i < b; ++i) {
        const WindowPlan& w = P.wins[sorted[i]];
        const int64_t cnt = kind == 0 ? (n - (w.j1 + w.k) + NT - 1) / NT : kind == 1 ? (w.j1 + NT - 1) / NT
                                                                          : (n + NT - 1) / NT;
        acc += (int32_t)cnt;
        pref.push_back(acc);
      }
      nstr[l * 3 + kind] = acc;
    }
    for (int64_t i = a; i < b; ++i) {
      const WindowPlan& w = P.wins[sorted[i]];
      WinDev& d = wd[i];
      std::memset(&d, 0, sizeof(d));
      d.j1 = w.j1; d.k = w.k; d.nblk = w.nblk; d.ninner = w.ninner;
      d.slot = (int32_t)(i - a);
      d.pool = w.pool; d.order = w.order;
      d.sidx = (int32_t)i;
    }
  }
  st->ms_schedule = now_ms() - t0;
  if (nw > 0) {
    PK(dwins.alloc(sizeof(WinDev) * nw));
    PK(doff.alloc(sizeof(int64_t) * (nw + 1)));
    hstep_base.push_back((int64_t)hstep.size());
    PK(dstep.alloc(sizeof(int32_t) * hstep.size()));
    PK(dstepb.alloc(sizeof(int64_t) * hstep_base.size()));
    PK(didx.alloc(sizeof(int32_t) * (hidx.size() + 1)));
    PK(cudaMemcpyAsync(dstep.p, hstep.data(), sizeof(int32_t) * hstep.size(), cudaMemcpyHostToDevice, sA));
    PK(cudaMemcpyAsync(dstepb.p, hstep_base.data(), sizeof(int64_t) * hstep_base.size(), cudaMemcpyHostToDevice, sA));
    if (!hidx.empty())
      PK(cudaMemcpyAsync(didx.p, hidx.data(), sizeof(int32_t) * hidx.size(), cudaMemcpyHostToDevice, sA));
    PK(dsj.alloc(sizeof(int16_t) * hsj.size()));
    PK(ds12.alloc(hs12.size()));
    PK(dpref.alloc(sizeof(int32_t) * pref.size()));
    PK(dstatus.alloc(sizeof(int32_t) * nw));
    PK(ddone.alloc(sizeof(int32_t) * nw));
    PK(dctl.alloc(sizeof(Control)));
    PK(dUL.alloc(sizeof(double) * kZslot * maxper));
    PK(dVR.alloc(sizeof(double) * kZslot * maxper));
    PK(dzr.alloc(sizeof(int16_t) * kZrange * maxper));
    PK(cudaMemcpyAsync(dwins.p, wd.data(), sizeof(WinDev) * nw, cudaMemcpyHostToDevice, sA));
    PK(cudaMemcpyAsync(doff.p, off.data(), sizeof(int64_t) * (nw + 1), cudaMemcpyHostToDevice, sA));
    if (!hsj.empty()) {
      PK(cudaMemcpyAsync(dsj.p, hsj.data(), sizeof(int16_t) * hsj.size(), cudaMemcpyHostToDevice, sA));
      PK(cudaMemcpyAsync(ds12.p, hs12.data(), hs12.size(), cudaMemcpyHostToDevice, sA));
    }
    PK(cudaMemcpyAsync(dpref.p, pref.data(), sizeof(int32_t) * pref.size(), cudaMemcpyHostToDevice, sA));
    PK(cudaMemsetAsync(dstatus.p, 0, sizeof(int32_t) * nw, sA));
    PK(cudaMemsetAsync(ddone.p, 0, sizeof(int32_t) * nw, sA));
    PK(cudaMemsetAsync(dctl.p, 0, sizeof(Control), sA));
    // TMA descriptors: S and T against UL (left) and VR (right), Q against UL, Z against VR
    panel_maps_init(&mSL, (double*)dUL.p, maxper, S, n, n, ldS);
    panel_maps_init(&mTL, (double*)dUL.p, maxper, T, n, n, ldT);
    panel_maps_init(&mSR, (double*)dVR.p, maxper, S, n, n, ldS);
    panel_maps_init(&mTR, (double*)dVR.p, maxper, T, n, n, ldT);
    if (Q) panel_maps_init(&mQ, (double*)dUL.p, maxper, Q, n, n, ldQ);
    if (Zm) panel_maps_init(&mZ, (double*)dVR.p, maxper, Zm, n, n, ldZ);
    if (std::getenv("SN_PPROF")) {
      PK(dpprof.alloc(24 * sizeof(unsigned long long)));
      PK(cudaMemsetAsync(dpprof.p, 0, 24 * sizeof(unsigned long long), sA));
    }
    PK(cudaEventCreate(&e0));
    PK(cudaEventCreate(&e1));
    PK(cudaEventRecord(e0, sA));
    const int mt = o.window <= 64 ? 64 : (o.window <= 128 ? 128 : 256);
    const size_t smem_rec = sizeof(double) * kRecD * (size_t)max_step_cnt;
    int num_sms = 148;
    {
      int dev = 0;
      PK(cudaGetDevice(&dev));
      PK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (max_step_cnt > 256) { rc = SN_ERR_UNSUPPORTED; goto done; }
    PK(cudaFuncSetAttribute(pencil_window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_rec));
    for (int64_t l = 0; l < P.nlevels; ++l) {
      const int64_t a = lstart[l], b = lstart[l + 1];
      PencilWinArgs wa{};
      wa.wins = (const WinDev*)dwins.p + a; wa.nwin = (int32_t)(b - a); wa.base = (int32_t)a;
      wa.swap_off = (const int64_t*)doff.p; wa.sj = (const int16_t*)dsj.p; wa.s12 = (const int8_t*)ds12.p;
      wa.step_off = (const int32_t*)dstep.p; wa.step_base = (const int64_t*)dstepb.p;
      wa.sidx = (const int32_t*)didx.p;
      wa.S = S; wa.ldS = ldS; wa.T = T; wa.ldT = ldT;
      wa.UL = (double*)dUL.p; wa.VR = (double*)dVR.p; wa.zrange = (int16_t*)dzr.p;
      wa.status = (int32_t*)dstatus.p; wa.done = (int32_t*)ddone.p; wa.ctl = (Control*)dctl.p;
      wa.force_order = o.force_reject_window; wa.force_swap = (int32_t)o.force_reject_swap;
      wa.pprof = (unsigned long long*)dpprof.p;
      {
        // CTAs per window: as many as the level's windows leave SMs for (a cluster of <= 8)
        int C = o.pencil_cluster;
        if (C <= 0) C = (int)std::min<int64_t>(8, std::max<int64_t>(1, num_sms / (b - a)));
        C = std::min(C, 8);
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute at[1];
        cfg.gridDim = dim3((unsigned)((b - a) * C));
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem_rec;
        cfg.stream = sA;
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        PK(cudaLaunchKernelEx(&cfg, pencil_window_kernel, wa));
      }
      PK(cudaGetLastError());
      st->launches[0]++;
      auto panel = [&](int kind, double* M, int64_t ld, const double* Zs, const PanelMaps* pm) {
        const int32_t ns = nstr[l * 3 + kind];
        if (ns <= 0 || M == nullptr) return;
        PanelArgs pa{};
        pa.wins = (const WinDev*)dwins.p + a; pa.nwin = (int32_t)(b - a); pa.base = (int32_t)a;
        pa.prefix = (const int32_t*)dpref.p + pref_off[l * 3 + kind];
        pa.strips = nullptr; pa.nseg = 0; pa.part = 0;
        pa.vec16 = (((uintptr_t)M & 15) == 0 && (ld % 2) == 0) ? 1 : 0;
        pa.status = (const int32_t*)dstatus.p;
        pa.M = M; pa.ld = ld; pa.n = n; pa.Z = Zs; pa.zrange = (const int16_t*)dzr.p;
        pa.maps = pm;
        launch_panel(kind, mt, pa, ns, sA);
        st->launches[kind + 1]++;
      };
      panel(0, S, ldS, (double*)dUL.p, &mSL);
      panel(0, T, ldT, (double*)dUL.p, &mTL);
      panel(1, S, ldS, (double*)dVR.p, &mSR);
      panel(1, T, ldT, (double*)dVR.p, &mTR);
      panel(2, Q, ldQ, (double*)dUL.p, &mQ);
      panel(2, Zm, ldZ, (double*)dVR.p, &mZ);
      PK(cudaGetLastError());
      levels_run = l + 1;
      // a rejection stops the run after this level (its panels apply the partial factors)
      int32_t abort_flag = 0;
      PK(cudaMemcpyAsync(&abort_flag, dctl.p, sizeof(int32_t), cudaMemcpyDeviceToHost, sA));
      PK(cudaStreamSynchronize(sA));
      if (abort_flag) break;
    }
    PK(cudaEventRecord(e1, sA));
    PK(cudaEventSynchronize(e1));
    float ms = 0.0f;
    PK(cudaEventElapsedTime(&ms, e0, e1));
    st->ms_device = ms;
    hstatus.resize(nw);
    hdone.resize(nw);
    PK(cudaMemcpy(hstatus.data(), dstatus.p, sizeof(int32_t) * nw, cudaMemcpyDeviceToHost));
    PK(cudaMemcpy(hdone.data(), ddone.p, sizeof(int32_t) * nw, cudaMemcpyDeviceToHost));
    PK(cudaMemcpy(&hctl, dctl.p, sizeof(Control), cudaMemcpyDeviceToHost));
    if (dpprof.p) {
      unsigned long long h[24];
      PK(cudaMemcpy(h, dpprof.p, sizeof(h), cudaMemcpyDeviceToHost));
      const double w = h[5] ? (double)h[5] : 1.0;
      double lat[4];
      for (int q = 0; q < 4; ++q) lat[q] = h[12 + q] ? (double)h[8 + q] / (double)h[12 + q] : 0.0;
      const double c22 = h[22] ? (double)h[22] : 1.0;   // warps that marked (lane 0)
      std::fprintf(stderr,
                   "{\"probe\": \"pencil_window_phases\", \"windows\": %llu, \"steps_per_window\": %.1f, "
                   "\"swaps_per_window\": %.1f, \"cycles_per_window\": {\"transform\": %.0f, \"intervals\": %.0f, "
                   "\"rows\": %.0f, \"cols\": %.0f}, \"transform_cycles_by_type\": [%.0f, %.0f, %.0f, %.0f], "
                   "\"swaps_by_type\": [%llu, %llu, %llu, %llu], \"own_task_cycles\": {\"rows\": %.0f, \"cols\": %.0f}, "
                   "\"swap22_cumulative_cycles\": {\"sylvester\": %.0f, \"bases\": %.0f, \"candidates\": %.0f, \"all\": %.0f}}\n",
                   h[5], h[4] / w, h[6] / w, h[0] / w, h[1] / w, h[2] / w, h[3] / w, lat[0], lat[1], lat[2], lat[3],
                   h[12], h[13], h[14], h[15], h[16] / w, h[17] / w, h[18] / c22, h[19] / c22, h[20] / c22, h[21] / c22);
    }
  }
  {
    // final block list: replay the executed swaps on the initial list (block at each first row)
    std::vector<int8_t> bsz((size_t)n + 2, 0), bsel((size_t)n + 2, 0);   // indexed by first row
    for (int64_t i = 0; i < n;) {
      const int sz = bmap[i] == 1 ? 2 : 1;
      bsz[i] = (int8_t)sz;
      bsel[i] = selrow[i];
      i += sz;
    }
    int64_t executed = 0, swaps = 0;
    for (int64_t i = 0; i < lstart[levels_run]; ++i) {
      if (hstatus.empty() || hstatus[i] == kWinSkipped) continue;
      const WindowPlan& w = P.wins[sorted[i]];
      ++executed;
      const int64_t cnt = hstatus[i] == kWinDone ? off[i + 1] - off[i] : hdone[i];
      for (int64_t q = 0; q < cnt; ++q) {
        const int64_t j = w.j1 + hsj[off[i] + q];
        const int n1 = hs12[off[i] + q] >> 4, n2 = hs12[off[i] + q] & 15;
        const int8_t sel1 = bsel[j], sel2 = bsel[j + n1];
        bsz[j] = 0; bsz[j + n1] = 0;
        bsz[j] = (int8_t)n2; bsel[j] = sel2;
        bsz[j + n2] = (int8_t)n1; bsel[j + n2] = sel1;
        st->swaps_by_type[(n1 - 1) * 2 + (n2 - 1)]++;
      }
      swaps += cnt;
      const double k = w.k;
      st->eq_flops += 2.0 * k * k * (2.0 * (double)(n - w.j1 - w.k) + 2.0 * (double)w.j1 + (Q ? (double)n : 0.0) +
                                     (Zm ? (double)n : 0.0));
    }
    for (int64_t i = 0; i < n;) {
      const int sz = bsz[i];
      for (int q = 0; q < sz; ++q) {
        select[i + q] = bsel[i];
        if (bmap_out) bmap_out[i + q] = (int8_t)(sz == 1 ? 0 : 1 + q);
      }
      i += sz;
    }
    st->windows = executed;
    st->swaps = swaps;
    st->levels = P.nlevels;
    st->g3_max_ratio = __longlong_as_double_host(hctl.ratio_bits);
    if (hctl.abort) {
      rc = SN_ERR_REJECTED;
      if (std::getenv("SN_DEBUG"))
        std::fprintf(stderr, "sn pencil: rejected window %d (order %lld) swap %d row %d (%d|%d): test %d ratio %.3f\n",
                     hctl.rej_window, (long long)P.wins[sorted[hctl.rej_window]].order, hctl.rej_swaps_done,
                     hctl.rej_row, hctl.rej_n1, hctl.rej_n2, hctl.pad[0], hctl.pad[1] / 1000.0);
      st->rejected_window = P.wins[sorted[hctl.rej_window]].order;
      st->rejected_row = hctl.rej_row;
      st->rejected_n1 = hctl.rej_n1;
      st->rejected_n2 = hctl.rej_n2;
    }
  }
  st->ms_total = now_ms() - t0;
done:
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  return rc;
}

}  // namespace
}  // namespace sn

extern "C" int sn_reorder_pencil_ex(const sn_opts* opts, int64_t n, double* S, int64_t ldS, double* T, int64_t ldT,
                                    double* Q, int64_t ldQ, double* Z, int64_t ldZ, int32_t* select, int64_t* m,
                                    int8_t* bmap_out, sn_stats* stats, void* stream) {
  using namespace sn;
  sn_opts o;
  if (opts) o = *opts;
  else sn_default_opts(&o);
  if (n < 0) return -2;
  if (m == nullptr) return -12;
  *m = 0;
  if (n == 0) return 0;
  if (!S) return -3;
  if (ldS < n) return -4;
  if (!T) return -5;
  if (ldT < n) return -6;
  if (Q && ldQ < n) return -8;
  if (Z && ldZ < n) return -10;
  if (!select) return -11;
  if (o.window < 4 || o.window > 256 || o.inner_window < 4 || o.inner_window > kInner) return SN_ERR_UNSUPPORTED;
  std::lock_guard<std::mutex> lock(g_mu);
  sn_stats local;
  sn_stats* st = stats ? stats : &local;
  cudaStream_t sA = (cudaStream_t)stream;
  // Host buffers: each host matrix is staged through a compact (ld = n) device copy, copied
  // in before the call and back after it (also after SN_ERR_REJECTED: a valid partial form).
  double* user[4] = {S, T, Q, Z};
  const int64_t uld[4] = {ldS, ldT, ldQ, ldZ};
  double* dev[4] = {S, T, Q, Z};
  int64_t dld[4] = {ldS, ldT, ldQ, ldZ};
  DevBuf stage[4];
  bool staged = false;
  double h2d = 0.0;
  for (int i = 0; i < 4; ++i) {
    if (!user[i] || is_device_ptr(user[i])) continue;
    const double t = now_ms();
    if (stage[i].alloc(sizeof(double) * (size_t)n * (size_t)n) != cudaSuccess) return SN_ERR_CUDA;
    if (cudaMemcpy2DAsync(stage[i].p, sizeof(double) * n, user[i], sizeof(double) * uld[i], sizeof(double) * n, n,
                          cudaMemcpyHostToDevice, sA) != cudaSuccess)
      return SN_ERR_CUDA;
    dev[i] = (double*)stage[i].p;
    dld[i] = n;
    staged = true;
    if (cudaStreamSynchronize(sA) != cudaSuccess) return SN_ERR_CUDA;
    h2d += now_ms() - t;
  }
  int rc = run_pencil(o, n, dev[0], dld[0], dev[1], dld[1], dev[2], dld[2], dev[3], dld[3], select, m, bmap_out, st,
                      sA);
  if (staged) {
    st->ms_h2d = h2d;
    if (rc == SN_OK || rc == SN_ERR_REJECTED) {
      const double t = now_ms();
      for (int i = 0; i < 4; ++i) {
        if (!stage[i].p) continue;
        if (cudaMemcpy2DAsync(user[i], sizeof(double) * uld[i], stage[i].p, sizeof(double) * n, sizeof(double) * n, n,
                              cudaMemcpyDeviceToHost, sA) != cudaSuccess)
          return SN_ERR_CUDA;
      }
      if (cudaStreamSynchronize(sA) != cudaSuccess) return SN_ERR_CUDA;
      st->ms_d2h = now_ms() - t;
    }
  }
  return rc;
}
