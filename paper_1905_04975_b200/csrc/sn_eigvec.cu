// sn_eigvec.cu -- eigenvectors of a real Schur form with overflow protection and the
// back-transform (Eq. (5) P:72-76 "(S - lambda_i I) y_i = 0",
// Eq. (6) P:77-79 "x_i = Q y_i", "the computations must be protected against
// floating-point overflow").  Product code; readings E1-E6 in DESIGN.md §3.2.
//
// Blocked right-looking back substitution over row tiles of S (about 128 rows, never splitting
// a 2x2 block), bottom tile first.  Per tile:
//   * eig_solve_kernel -- one warp per eigenvector (a real column, or a complex pair as two
//     real columns): the tile's diagonal block of S is staged in shared memory, the tile rows
//     of the right-hand side sit in registers (lane l holds rows l, l+32, ...), and the rows
//     are solved bottom to top over S's block structure (1x1: a complex division, 2x2: a 2x2
//     complex system by complete pivoting, pivots below smin perturbed as xLALN2), each solved
//     block updating the tile rows above it.  Overflow protection (E4): the eigenvector
//     carries a power-of-two scale 2^-e; a division or an update that could exceed
//     Omega = 2^500 first rescales the whole eigenvector (rare: a warp loop over its rows);
//     the update of the rows above the tile is bounded by bound + ||S[0:i0, tile]||_inf *
//     max|y_tile| (a per-eigenvector running bound), so the GEMM below cannot overflow.
//   * eig_gemm_kernel -- Y[0:i0, cols] -= S[0:i0, tile] * Y[tile, cols] for every eigenvector
//     whose block lies at or below the tile: an FP64 DMMA (mma.sync m16n8k4) GEMM, 128 x 64
//     output tiles, K chunks of 16 staged by cp.async in a 4-stage ring.
// Then X = Q Y with the same GEMM kernel (per 64-column tile the K extent stops at the last
// nonzero row of its eigenvectors) and a per-eigenvector normalisation max(|re|+|im|) = 1 (E5).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sn_device.cuh"
#include "sn_exec.h"
#include "sn_reorder.h"

namespace sn {
namespace {

constexpr double kOmega = 3.273390607896142e+150;   // 2^500 (E4)
// a protective rescale brings the eigenvector down to 2^-900 of the bound (not just below it),
// so that an exponentially growing vector rescales once per 2^900 of growth; the normalised
// result is the same (power-of-two scalings) up to entries below 2^-674 of the vector's
// largest one, which may underflow to zero -- far below any comparison bar
constexpr double kHeadroom = 1.18575755001e-271;   // 2^-900
// Row tiles of 128 rows (64-row tiles were measured slower: 0.62 s of solves instead of 0.46 s
// at config 3 -- twice the launches, the same serial chain length per eigenvector)
constexpr int kTileRows = 128;                        // nominal row tile (<= 129 with a 2x2 shift)
constexpr int kTileMax = 130;
constexpr int kLdT = kTileMax + 1;                    // odd stride of the staged diagonal tile
constexpr int kRegs = 5;                              // rows per lane: 5 x 32 >= kTileMax
constexpr int kSolveWarps = 16;
constexpr int kSolveCtasPerSm = 1;
constexpr int kSuper = 4;                             // row tiles per update super-tile

struct EigUnit {
  int64_t k;      // first row of the eigenvalue's block
  int32_t bs;     // block size (1 real, 2 complex pair)
  int32_t col;    // first column of X / Y
  double wr, wi;  // lambda = wr + i wi (wi > 0 for a pair)
};

struct EigState {
  int32_t e;      // the columns hold (eigenvector) * 2^-e
  int32_t pad;
  double bound;   // upper bound of |Y[0:i0, col]| (rows above the current tile)
};

struct SolveArgs {
  const double* S;
  int64_t ldS;
  double* Y;
  int64_t ldY;
  const int8_t* bmap;
  const EigUnit* units;
  EigState* state;
  int32_t u0, nu;      // active units [u0, u0 + nu)
  int64_t i0, i1;      // tile rows
  double snorm;        // ||S[0:i0, i0:i1]||_inf
  int32_t* rescales;   // count of protective rescalings (statistics)
};

// ---- complex helpers ((re, im) pairs)
__device__ __forceinline__ double cabs1(double r, double i) { return fabs(r) + fabs(i); }
__device__ __forceinline__ void cdiv(double ar, double ai, double br, double bi, double& cr, double& ci) {
  if (fabs(br) >= fabs(bi)) {
    const double r = bi / br, d = br + bi * r;
    cr = (ar + ai * r) / d;
    ci = (ai - ar * r) / d;
  } else {
    const double r = br / bi, d = bi + br * r;
    cr = (ar * r + ai) / d;
    ci = (ai * r - ar) / d;
  }
}

// (B - (wr + i wi) I) y = r for nb = 1, 2 (B: b00 b10 b01 b11), complete pivoting, pivots below
// smin replaced by smin (xLALN2).  Returns max |y| (cabs1).
__device__ __forceinline__ double small_csolve(int nb, double b00, double b10, double b01, double b11, double wr,
                                               double wi, double smin, double r0r, double r0i, double r1r,
                                               double r1i, double& y0r, double& y0i, double& y1r, double& y1i) {
  if (nb == 1) {
    double dr = b00 - wr, di = -wi;
    if (cabs1(dr, di) < smin) { dr = smin; di = 0.0; }
    cdiv(r0r, r0i, dr, di, y0r, y0i);
    y1r = 0.0; y1i = 0.0;
    return cabs1(y0r, y0i);
  }
  double m00r = b00 - wr, m00i = -wi, m01r = b01, m01i = 0.0;
  double m10r = b10, m10i = 0.0, m11r = b11 - wr, m11i = -wi;
  double c0r = r0r, c0i = r0i, c1r = r1r, c1i = r1i;
  // pivot: largest of the four entries (column-major scan, first maximum)
  const double a00 = cabs1(m00r, m00i), a10 = cabs1(m10r, m10i), a01 = cabs1(m01r, m01i), a11 = cabs1(m11r, m11i);
  int pr = 0, pc = 0;
  double best = a00;
  if (a10 > best) { best = a10; pr = 1; pc = 0; }
  if (a01 > best) { best = a01; pr = 0; pc = 1; }
  if (a11 > best) { best = a11; pr = 1; pc = 1; }
  if (pr == 1) {
    double t;
    t = m00r; m00r = m10r; m10r = t; t = m00i; m00i = m10i; m10i = t;
    t = m01r; m01r = m11r; m11r = t; t = m01i; m01i = m11i; m11i = t;
    t = c0r; c0r = c1r; c1r = t; t = c0i; c0i = c1i; c1i = t;
  }
  if (pc == 1) {
    double t;
    t = m00r; m00r = m01r; m01r = t; t = m00i; m00i = m01i; m01i = t;
    t = m10r; m10r = m11r; m11r = t; t = m10i; m10i = m11i; m11i = t;
  }
  if (cabs1(m00r, m00i) < smin) { m00r = smin; m00i = 0.0; }
  double lr, li;
  cdiv(m10r, m10i, m00r, m00i, lr, li);
  double ur = m11r - (lr * m01r - li * m01i);
  double ui = m11i - (lr * m01i + li * m01r);
  const double b1r = c1r - (lr * c0r - li * c0i);
  const double b1i = c1i - (lr * c0i + li * c0r);
  if (cabs1(ur, ui) < smin) { ur = smin; ui = 0.0; }
  double x1r, x1i, x0r, x0i;
  cdiv(b1r, b1i, ur, ui, x1r, x1i);
  const double tr = c0r - (m01r * x1r - m01i * x1i);
  const double ti = c0i - (m01r * x1i + m01i * x1r);
  cdiv(tr, ti, m00r, m00i, x0r, x0i);
  if (pc == 1) { y0r = x1r; y0i = x1i; y1r = x0r; y1i = x0i; }
  else { y0r = x0r; y0i = x0i; y1r = x1r; y1i = x1i; }
  return fmax(cabs1(y0r, y0i), cabs1(y1r, y1i));
}

// the real case of small_csolve (wi = 0 and real right-hand sides): the same pivots and the
// same operation sequence on the real parts
__device__ __forceinline__ double small_rsolve(int nb, double b00, double b10, double b01, double b11, double wr,
                                               double smin, double r0, double r1, double& y0, double& y1) {
  if (nb == 1) {
    double d = b00 - wr;
    if (fabs(d) < smin) d = smin;
    y0 = r0 / d;
    y1 = 0.0;
    return fabs(y0);
  }
  double m00 = b00 - wr, m01 = b01, m10 = b10, m11 = b11 - wr, c0 = r0, c1 = r1;
  const double a00 = fabs(m00), a10 = fabs(m10), a01 = fabs(m01), a11 = fabs(m11);
  int pr = 0, pc = 0;
  double best = a00;
  if (a10 > best) { best = a10; pr = 1; pc = 0; }
  if (a01 > best) { best = a01; pr = 0; pc = 1; }
  if (a11 > best) { best = a11; pr = 1; pc = 1; }
  if (pr == 1) {
    double t;
    t = m00; m00 = m10; m10 = t;
    t = m01; m01 = m11; m11 = t;
    t = c0; c0 = c1; c1 = t;
  }
  if (pc == 1) {
    double t;
    t = m00; m00 = m01; m01 = t;
    t = m10; m10 = m11; m11 = t;
  }
  if (fabs(m00) < smin) m00 = smin;
  const double l = m10 / m00;
  double uu = m11 - l * m01;
  const double b1 = c1 - l * c0;
  if (fabs(uu) < smin) uu = smin;
  const double x1 = b1 / uu;
  const double x0 = (c0 - m01 * x1) / m00;
  if (pc == 1) { y0 = x1; y1 = x0; }
  else { y0 = x0; y1 = x1; }
  return fmax(fabs(y0), fabs(y1));
}

template <bool CPLX>
__device__ __forceinline__ double small_solve(int nb, double b00, double b10, double b01, double b11, double wr,
                                              double wi, double smin, double r0r, double r0i, double r1r,
                                              double r1i, double& y0r, double& y0i, double& y1r, double& y1i) {
  if (CPLX) return small_csolve(nb, b00, b10, b01, b11, wr, wi, smin, r0r, r0i, r1r, r1i, y0r, y0i, y1r, y1i);
  y0i = 0.0;
  y1i = 0.0;
  return small_rsolve(nb, b00, b10, b01, b11, wr, smin, r0r, r1r, y0r, y1r);
}

__device__ __forceinline__ int pow2_steps(double v, double lim) {
  int s = 0;
  while (v > lim && s < 4000) { v *= 0.5; ++s; }
  return s;
}

// steps of a protective rescale for a growth bound g (in units of Omega, > 1): at least enough
// to bring it to 1, as many as the headroom asks, but never below 2^-400 for the vector's
// current magnitude ymag (a bound scaled by a huge matrix entry must not push the vector
// itself into underflow)
__device__ __forceinline__ int rescale_steps(double g, double ymag) {
  const int smin = pow2_steps(g, 1.0);
  int s = pow2_steps(g, kHeadroom);
  if (ymag > 0.0) s = min(s, ilogb(ymag) + 400);
  return max(s, smin);
}

// register j of the lane owning local row r: select without dynamic indexing
__device__ __forceinline__ double reg_get(const double (&v)[kRegs], int j) {
  double x = v[0];
#pragma unroll
  for (int q = 1; q < kRegs; ++q)
    if (j == q) x = v[q];
  return x;
}
__device__ __forceinline__ void reg_set(double (&v)[kRegs], int j, double x) {
#pragma unroll
  for (int q = 0; q < kRegs; ++q)
    if (j == q) v[q] = x;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// multiply global rows [r0, r1) of the unit's columns by f (warp-cooperative)
__device__ void scale_rows(double* Y, int64_t ldY, int col, int ncol, int64_t r0, int64_t r1, double f, int lane) {
  for (int q = 0; q < ncol; ++q) {
    double* c = Y + (int64_t)(col + q) * ldY;
    for (int64_t r = r0 + lane; r < r1; r += 32) c[r] *= f;
  }
}

// one eigenvector (a warp): CPLX = a complex pair (two columns, complex arithmetic), else a
// real eigenvalue (real arithmetic: the same operations with the imaginary parts dropped, so
// the values are those of the complex routine with zero imaginary parts)
template <bool CPLX>
__device__ __forceinline__ void solve_unit(const SolveArgs& a, const double* Ts, const double* cmx, const int8_t* bm,
                                           int tb, int u, int lane) {
  const EigUnit U = a.units[u];
  constexpr bool cplx = CPLX;
  const int ncol = U.bs;
  double* Yr = a.Y + (int64_t)U.col * a.ldY;
  double* Yi = cplx ? Yr + a.ldY : nullptr;
  const double wr = U.wr, wi = U.wi;
  const double smin = fmax(2.220446049250313e-16 * (fabs(wr) + fabs(wi)), 2.2250738585072014e-308 / 2.220446049250313e-16);
  EigState stt = a.state[u];
  int e = stt.e;
  const int rend = (int)(min(a.i1, U.k) - a.i0);   // local rows [0, rend) are solved here
  double vr[kRegs], vi[kRegs];
  double ynorm = 0.0;                               // max |y| over the tile rows of Y
  if (U.k < a.i1) {
    // E2: the block's own entries (rows k, k+1), then the in-tile right-hand side
    double y0r = 1.0, y0i = 0.0, y1r = 0.0, y1i = 0.0;
    const int kl = (int)(U.k - a.i0);
    if (cplx) {
      const double b = Ts[kl + (kl + 1) * kLdT], c = Ts[(kl + 1) + kl * kLdT];
      if (fabs(b) >= fabs(c)) { y0r = 1.0; y0i = 0.0; y1r = 0.0; y1i = wi / b; }
      else { y0r = -wi / c; y0i = 0.0; y1r = 0.0; y1i = 1.0; }
    }
    // protect the initial update of the rows above (every row above, through this tile's
    // in-register update and the GEMM: bounded by the tile's own column max and snorm)
    {
      double cm = cmx[kl];
      if (cplx) cm = fmax(cm, cmx[kl + 1]);
      const double ym = fmax(cabs1(y0r, y0i), cabs1(y1r, y1i));
      const double g = fmax(((double)U.bs * (ym / kOmega)) * cm, (ym / kOmega) * a.snorm);
      if (g > 1.0) {
        const int s = rescale_steps(g, ym);
        const double f = ldexp(1.0, -s);
        y0r *= f; y0i *= f; y1r *= f; y1i *= f;
        e += s;
        if (lane == 0) atomicAdd(a.rescales, 1);
      }
    }
    if (lane == 0) {
      Yr[U.k] = y0r;
      if (cplx) { Yr[U.k + 1] = y1r; Yi[U.k] = y0i; Yi[U.k + 1] = y1i; }
    }
    __syncwarp();   // a rescale below may read these rows on other lanes
    ynorm = fmax(cabs1(y0r, y0i), cabs1(y1r, y1i));
#pragma unroll
    for (int j = 0; j < kRegs; ++j) {
      const int r = lane + 32 * j;
      double xr = 0.0, xi = 0.0;
      if (r < rend) {
        const double s0 = Ts[r + kl * kLdT];
        xr = -s0 * y0r;
        xi = -s0 * y0i;
        if (cplx) {
          const double s1 = Ts[r + (kl + 1) * kLdT];
          xr -= s1 * y1r;
          xi -= s1 * y1i;
        }
      }
      vr[j] = xr;
      vi[j] = xi;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kRegs; ++j) {
      const int r = lane + 32 * j;
      vr[j] = r < rend ? Yr[a.i0 + r] : 0.0;
      vi[j] = (cplx && r < rend) ? Yi[a.i0 + r] : 0.0;
    }
  }
  // exact bound of the tile's right-hand side, then a running bound through the updates
  double B = 0.0;
#pragma unroll
  for (int j = 0; j < kRegs; ++j) B = fmax(B, cabs1(vr[j], vi[j]));
  B = warp_max(B);
  // rows of the unit below the tile part solved here (global): [i0 + rend, k + bs)
  const int64_t below0 = a.i0 + rend, below1 = U.k + U.bs;
  // Rows solved bottom to top, in phases J = kRegs-1 .. 0 of 32 rows: register J of lane l
  // holds row 32J + l, so inside a phase the register index is a compile-time constant (no
  // runtime register selection), and a solved block updates register J (lanes above it) and
  // the lower registers.  A 2x2 block whose rows straddle two phases belongs to the lower
  // phase (its first row), its second row read from / written to register J+1, lane 0.
  int i = rend;
#pragma unroll
  for (int J = kRegs - 1; J >= 0; --J) {
    while (i > 32 * J) {
      const int nb = (i >= 2 && bm[i - 1] == 2) ? 2 : 1;
      if (i - nb < 32 * J) break;            // a straddling 2x2 block: the next phase's
      i -= nb;
      const int l0 = i - 32 * J;             // lane of the block's first row
      const bool up = (nb == 2 && l0 == 31); // its second row in register J+1, lane 0
      double r0r = __shfl_sync(0xffffffffu, vr[J], l0);
      double r0i = CPLX ? __shfl_sync(0xffffffffu, vi[J], l0) : 0.0;
      double r1r = 0.0, r1i = 0.0;
      if (nb == 2) {
        const double nr = (J + 1 < kRegs) ? vr[J + 1 < kRegs ? J + 1 : J] : 0.0;
        const double ni = (J + 1 < kRegs) ? vi[J + 1 < kRegs ? J + 1 : J] : 0.0;
        const double sr = up ? nr : vr[J];
        const double si2 = up ? ni : vi[J];
        r1r = __shfl_sync(0xffffffffu, sr, up ? 0 : l0 + 1);
        r1i = CPLX ? __shfl_sync(0xffffffffu, si2, up ? 0 : l0 + 1) : 0.0;
      }
      const double b00 = Ts[i + i * kLdT];
      const double b10 = nb == 2 ? Ts[(i + 1) + i * kLdT] : 0.0;
      const double b01 = nb == 2 ? Ts[i + (i + 1) * kLdT] : 0.0;
      const double b11 = nb == 2 ? Ts[(i + 1) + (i + 1) * kLdT] : 0.0;
      double y0r, y0i, y1r, y1i;
      double ym = small_solve<CPLX>(nb, b00, b10, b01, b11, wr, wi, smin, r0r, r0i, r1r, r1i, y0r, y0i, y1r, y1i);
      if (!(ym <= kOmega)) {
        // E4: rescale the whole eigenvector so that this solve stays below Omega
        const double rmax = fmax(cabs1(r0r, r0i), cabs1(r1r, r1i));
        int s = (ym < 1e308) ? pow2_steps(ym, kOmega * kHeadroom) : pow2_steps(rmax / smin, kOmega * kHeadroom) + 1;
        for (;;) {
          const double f = ldexp(1.0, -s);
          ym = small_solve<CPLX>(nb, b00, b10, b01, b11, wr, wi, smin, r0r * f, r0i * f, r1r * f, r1i * f, y0r, y0i,
                                 y1r, y1i);
          if (ym <= kOmega || s > 4000) break;
          ++s;
        }
        const double f = ldexp(1.0, -s);
#pragma unroll
        for (int j = 0; j < kRegs; ++j) { vr[j] *= f; vi[j] *= f; }
        scale_rows(a.Y, a.ldY, U.col, ncol, 0, a.i0, f, lane);
        scale_rows(a.Y, a.ldY, U.col, ncol, below0, below1, f, lane);
        stt.bound *= f;
        ynorm *= f;
        B *= f;
        e += s;
        if (lane == 0) atomicAdd(a.rescales, 1);
      }
      // the solved rows replace their right-hand side
      if (lane == l0) { vr[J] = y0r; if (CPLX) vi[J] = y0i; }
      if (nb == 2) {
        if (up) {
          if (J + 1 < kRegs && lane == 0) {
            vr[J + 1 < kRegs ? J + 1 : J] = y1r;
            if (CPLX) vi[J + 1 < kRegs ? J + 1 : J] = y1i;
          }
        } else if (lane == l0 + 1) {
          vr[J] = y1r;
          if (CPLX) vi[J] = y1i;
        }
      }
      ynorm = fmax(ynorm, ym);
      if (i == 0) break;
      // update of the tile rows above: protect with the running bound
      double cm = cmx[i];
      if (nb == 2) cm = fmax(cm, cmx[i + 1]);
      const double g = B / kOmega + ((double)nb * (ym / kOmega)) * cm;
      if (g > 1.0) {
        const int s = rescale_steps(g, fmax(fmax(B, ym), ynorm));
        const double f = ldexp(1.0, -s);
#pragma unroll
        for (int j = 0; j < kRegs; ++j) { vr[j] *= f; vi[j] *= f; }
        y0r *= f; y0i *= f; y1r *= f; y1i *= f;
        scale_rows(a.Y, a.ldY, U.col, ncol, 0, a.i0, f, lane);
        scale_rows(a.Y, a.ldY, U.col, ncol, below0, below1, f, lane);
        stt.bound *= f;
        ynorm *= f;
        B *= f;
        ym *= f;
        e += s;
        if (lane == 0) atomicAdd(a.rescales, 1);
      }
      B += (double)nb * cm * ym;
      // register J: the lanes above the block; registers below J: every lane
      {
        const int r = lane + 32 * J;
        if (lane < l0) {
          const double s0 = Ts[r + i * kLdT];
          double xr = vr[J] - s0 * y0r, xi = CPLX ? vi[J] - s0 * y0i : 0.0;
          if (nb == 2) {
            const double s1 = Ts[r + (i + 1) * kLdT];
            xr -= s1 * y1r;
            if (CPLX) xi -= s1 * y1i;
          }
          vr[J] = xr;
          if (CPLX) vi[J] = xi;
        }
      }
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int r = lane + 32 * j;
        const double s0 = Ts[r + i * kLdT];
        double xr = vr[j] - s0 * y0r, xi = CPLX ? vi[j] - s0 * y0i : 0.0;
        if (nb == 2) {
          const double s1 = Ts[r + (i + 1) * kLdT];
          xr -= s1 * y1r;
          if (CPLX) xi -= s1 * y1i;
        }
        vr[j] = xr;
        if (CPLX) vi[j] = xi;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kRegs; ++j) {
    const int r = lane + 32 * j;
    if (r < rend) {
      Yr[a.i0 + r] = vr[j];
      if (cplx) Yi[a.i0 + r] = vi[j];
    }
  }
  // protection of the GEMM update of rows [0, i0): bound + snorm * max|y_tile| <= Omega
  if (a.i0 > 0) {
    const double g = stt.bound / kOmega + (ynorm / kOmega) * a.snorm;
    if (g > 1.0) {
      const int s = rescale_steps(g, ynorm);
      const double f = ldexp(1.0, -s);
      __syncwarp();
      scale_rows(a.Y, a.ldY, U.col, ncol, 0, below1, f, lane);
      stt.bound *= f;
      ynorm *= f;
      e += s;
      if (lane == 0) atomicAdd(a.rescales, 1);
    }
    stt.bound += ynorm * a.snorm;
  }
  if (lane == 0) {
    stt.e = e;
    a.state[u] = stt;
  }
}

__global__ void __launch_bounds__(kSolveWarps * 32, kSolveCtasPerSm) eig_solve_kernel(SolveArgs a) {
  extern __shared__ __align__(16) double sm[];
  double* Ts = sm;                                   // tile x tile, column-major, ld kLdT
  double* cmx = Ts + kLdT * kTileMax;                // per tile column: max |Ts[0:c, c]|
  int8_t* bm = reinterpret_cast<int8_t*>(cmx + kTileMax);
  const int tb = (int)(a.i1 - a.i0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int idx = tid; idx < tb * tb; idx += blockDim.x) {
    const int r = idx % tb, c = idx / tb;
    Ts[r + c * kLdT] = r <= c + 1 ? a.S[(a.i0 + r) + (a.i0 + c) * a.ldS] : 0.0;
  }
  for (int r = tid; r < tb; r += blockDim.x) bm[r] = a.bmap[a.i0 + r];
  __syncthreads();
  for (int c = warp; c < tb; c += kSolveWarps) {
    double m = 0.0;
    for (int r = lane; r < c; r += 32) m = fmax(m, fabs(Ts[r + c * kLdT]));
    m = warp_max(m);
    if (lane == 0) cmx[c] = m;
  }
  __syncthreads();
  const int u = a.u0 + blockIdx.x * kSolveWarps + warp;
  if (u >= a.u0 + a.nu) return;
  const EigUnit U = a.units[u];
  if (U.bs == 2) solve_unit<true>(a, Ts, cmx, bm, tb, u, lane);
  else solve_unit<false>(a, Ts, cmx, bm, tb, u, lane);
}

// ---- ||S[0:i0, i0:i1]||_inf per tile (one CTA per tile)
__global__ void eig_snorm_kernel(const double* S, int64_t ldS, const int64_t* tb, int ntiles, double* snorm) {
  const int t = blockIdx.x;
  if (t >= ntiles) return;
  const int64_t i0 = tb[t], i1 = tb[t + 1];
  double m = 0.0;
  for (int64_t r = threadIdx.x; r < i0; r += blockDim.x) {
    double s = 0.0;
    for (int64_t c = i0; c < i1; ++c) s += fabs(S[r + c * ldS]);
    m = fmax(m, s);
  }
  __shared__ double red[32];
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_max(v);
    if (threadIdx.x == 0) snorm[t] = v;
  }
}

// ---- FP64 DMMA GEMM:  C[0:M, n0:n0+N) (-)= A[0:M, k0:k0+K) * B[k0:k0+K, n0:n0+N)
constexpr int GBM = 128, GBN = 64, GBK = 16, GST = 4;
constexpr int GLDA = GBM + 4;   // As[k][m]: stride == 4 mod 16 doubles (conflict-free fragments)
constexpr int GLDB = GBK + 4;   // Bs[n][k]
constexpr int GTHREADS = 128;   // 4 warps, each 32 x 64
constexpr size_t GSMEM = sizeof(double) * (size_t)GST * (GBK * GLDA + GBN * GLDB);

struct GemmArgs {
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  int64_t M;
  int32_t N;            // columns of C from n0
  int64_t k0;           // first K index (row of B, column of A)
  int64_t K;            // K extent (if kend == NULL)
  const int32_t* kend;  // optional: per 64-column tile, K extent from k0
  int32_t minus;        // 1: C -= A B, 0: C = A B
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool pred) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__global__ void __launch_bounds__(GTHREADS, 2) eig_gemm_kernel(GemmArgs g) {
  extern __shared__ __align__(16) double gs[];
  double* As = gs;                                 // GST x [GBK][GLDA]
  double* Bs = gs + GST * GBK * GLDA;              // GST x [GBN][GLDB]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * GBM;
  const int n0 = blockIdx.y * GBN;
  const int64_t K = g.kend ? (int64_t)g.kend[blockIdx.y] : g.K;
  const int nk = (int)((K + GBK - 1) / GBK);
  auto load = [&](int kc, int st) {
    const int64_t kb = (int64_t)kc * GBK;
    double* as = As + st * GBK * GLDA;
    double* bs = Bs + st * GBN * GLDB;
#pragma unroll 4
    for (int idx = tid; idx < GBK * GBM; idx += GTHREADS) {
      const int m = idx & (GBM - 1), kk = idx >> 7;
      const bool p = (m0 + m < g.M) && (kb + kk < K);
      const double* src = p ? g.A + (m0 + m) + (g.k0 + kb + kk) * g.lda : g.A;
      cp_async8(as + kk * GLDA + m, src, p);
    }
#pragma unroll 4
    for (int idx = tid; idx < GBK * GBN; idx += GTHREADS) {
      const int kk = idx & (GBK - 1), c = idx >> 4;
      const bool p = (n0 + c < g.N) && (kb + kk < K);
      const double* src = p ? g.B + (g.k0 + kb + kk) + (int64_t)(n0 + c) * g.ldb : g.B;
      cp_async8(bs + c * GLDB + kk, src, p);
    }
  };
  double acc[2][8][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;
#pragma unroll
  for (int s = 0; s < GST - 1; ++s) {
    if (s < nk) load(s, s);
    cp_commit();
  }
  const int gq = lane >> 2, t = lane & 3, wm0 = warp * 32;
  for (int kc = 0; kc < nk; ++kc) {
    cp_wait<GST - 2>();
    __syncthreads();
    {
      const int nx = kc + GST - 1;
      if (nx < nk) load(nx, nx % GST);
      cp_commit();
    }
    const double* as = As + (kc % GST) * GBK * GLDA;
    const double* bs = Bs + (kc % GST) * GBN * GLDB;
#pragma unroll
    for (int ks = 0; ks < GBK; ks += 4) {
      double a0[2], a1[2], bf[8];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        a0[i] = as[(ks + t) * GLDA + wm0 + i * 16 + gq];
        a1[i] = as[(ks + t) * GLDA + wm0 + i * 16 + gq + 8];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) bf[j] = bs[(j * 8 + gq) * GLDB + ks + t];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma_16x8x4(acc[i][j], a0[i], a1[i], bf[j]);
    }
  }
  cp_wait<0>();
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t m = m0 + wm0 + i * 16 + gq + 8 * h;
        if (m >= g.M) continue;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int c = n0 + j * 8 + 2 * t + q;
          if (c >= g.N) continue;
          double* p = g.C + m + (int64_t)c * g.ldc;
          const double v = acc[i][j][2 * h + q];
          *p = g.minus ? *p - v : v;
        }
      }
}

// ---- E5: per eigenvector, divide by max_r (|re_r| + |im_r|) (multiply by the reciprocal)
__global__ void eig_normalize_kernel(double* X, int64_t ldX, int64_t rows, const EigUnit* units, int nunits) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nunits) return;
  const EigUnit U = units[warp];
  double* xr = X + (int64_t)U.col * ldX;
  double* xi = U.bs == 2 ? xr + ldX : nullptr;
  double m = 0.0;
  for (int64_t r = lane; r < rows; r += 32) m = fmax(m, fabs(xr[r]) + (xi ? fabs(xi[r]) : 0.0));
  m = warp_max(m);
  if (m > 0.0) {
    const double f = 1.0 / m;
    for (int64_t r = lane; r < rows; r += 32) {
      xr[r] *= f;
      if (xi) xi[r] *= f;
    }
  }
}

// lambda of every unit: S[k, k] and, for a pair, S[k, k+1] and S[k+1, k]
__global__ void eig_gather_kernel(const double* S, int64_t ldS, const int64_t* ks, const int8_t* bs, int nk,
                                  double* out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nk) return;
  const int64_t k = ks[q];
  out[3 * q] = S[k + k * ldS];
  out[3 * q + 1] = bs[q] == 2 ? S[k + (k + 1) * ldS] : 0.0;
  out[3 * q + 2] = bs[q] == 2 ? S[(k + 1) + k * ldS] : 0.0;
}

__global__ void eig_exp_kernel(const EigUnit* units, const EigState* st, int nunits, int32_t* out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nunits) return;
  const EigUnit U = units[u];
  out[U.col] = st[u].e;
  if (U.bs == 2) out[U.col + 1] = st[u].e;
}

struct EigBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
};

struct EigWorkspace {
  EigBuf sub, bad, bmap, units, state, tiles, snorm, kend, Y, expo, cnt;
  cudaEvent_t ev[6] = {};
  int device = -1;
};
EigWorkspace g_ews;

#define EK(x)                                                                                    \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      if (std::getenv("SN_DEBUG")) std::fprintf(stderr, "sn_eig: %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return SN_ERR_CUDA;                                                                       \
    }                                                                                           \
  } while (0)

void launch_gemm(const GemmArgs& g, int64_t ntiles_n, cudaStream_t st) {
  static bool attr[kMaxDevices] = {};
  const int d = device_slot();
  if (!attr[d]) {
    cudaFuncSetAttribute(eig_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GSMEM);
    attr[d] = true;
  }
  const dim3 grid((unsigned)((g.M + GBM - 1) / GBM), (unsigned)ntiles_n);
  if (g.M > 0 && ntiles_n > 0) eig_gemm_kernel<<<grid, GTHREADS, GSMEM, st>>>(g);
}

}  // namespace

int eigvec_run(int64_t n, const double* S, int64_t ldS, const double* Q, int64_t ldQ, const int32_t* select,
               double* X, int64_t ldX, int64_t* ncols, int32_t* scale_exp, sn_eig_stats* st, cudaStream_t sA) {
  EigWorkspace& ws = g_ews;
  const double t0 = now_ms();
  int dev = 0;
  EK(cudaGetDevice(&dev));
  if (ws.device != dev) {
    if (ws.device >= 0) {
      EK(cudaSetDevice(ws.device));
      for (EigBuf* b : {&ws.sub, &ws.bad, &ws.bmap, &ws.units, &ws.state, &ws.tiles, &ws.snorm, &ws.kend, &ws.Y,
                        &ws.expo, &ws.cnt}) {
        if (b->p) cudaFree(b->p);
        b->p = nullptr;
        b->cap = 0;
      }
      for (auto& e : ws.ev) cudaEventDestroy(e);
      EK(cudaSetDevice(dev));
    }
    for (auto& e : ws.ev) EK(cudaEventCreate(&e));
    ws.device = dev;
  }
  // a1: block structure from the subdiagonal (the scan kernel of the reordering)
  EK(ws.sub.ensure((size_t)n + 8));
  EK(ws.bad.ensure(8));
  EK(cudaMemsetAsync(ws.bad.p, 0, 4, sA));
  // (the lower part is validated too: the kernels read only the quasi-triangular part)
  launch_scan(S, ldS, n, 1, (uint8_t*)ws.sub.p, (int32_t*)ws.bad.p, sA);
  EK(cudaGetLastError());
  std::vector<uint8_t> sub((size_t)n);
  int32_t bad = 0;
  EK(cudaMemcpyAsync(sub.data(), ws.sub.p, (size_t)n, cudaMemcpyDeviceToHost, sA));
  EK(cudaMemcpyAsync(&bad, ws.bad.p, 4, cudaMemcpyDeviceToHost, sA));
  EK(cudaStreamSynchronize(sA));
  if (bad) return -2;
  std::vector<int8_t> bmap((size_t)n), selrow((size_t)n);
  int64_t m = 0;
  if (structure_from_sub(n, sub.data(), select, bmap.data(), selrow.data(), &m)) return -2;
  // E1: units (selected blocks in row order) and their columns; lambda from S's block
  std::vector<EigUnit> units;
  std::vector<double> diag;
  {
    std::vector<int64_t> ks;
    for (int64_t i = 0; i < n;) {
      const int bs = bmap[i] == 1 ? 2 : 1;
      if (selrow[i]) ks.push_back(i);
      i += bs;
    }
    // the block entries (diagonal and, for pairs, b and c), gathered on the device
    std::vector<double> blk(ks.size() * 3 + 3);
    std::vector<int8_t> kb(ks.size() + 1);
    for (size_t q = 0; q < ks.size(); ++q) kb[q] = bmap[ks[q]] == 1 ? 2 : 1;
    if (!ks.empty()) {
      EK(ws.units.ensure(ks.size() * (sizeof(int64_t) + 1 + 3 * sizeof(double)) + 64));
      int64_t* dks = (int64_t*)ws.units.p;
      double* dout = (double*)(dks + ks.size());
      int8_t* dbs = (int8_t*)(dout + 3 * ks.size());
      EK(cudaMemcpyAsync(dks, ks.data(), sizeof(int64_t) * ks.size(), cudaMemcpyHostToDevice, sA));
      EK(cudaMemcpyAsync(dbs, kb.data(), ks.size(), cudaMemcpyHostToDevice, sA));
      eig_gather_kernel<<<(unsigned)((ks.size() + 255) / 256), 256, 0, sA>>>(S, ldS, dks, dbs, (int)ks.size(), dout);
      EK(cudaGetLastError());
      EK(cudaMemcpyAsync(blk.data(), dout, sizeof(double) * 3 * ks.size(), cudaMemcpyDeviceToHost, sA));
    }
    EK(cudaStreamSynchronize(sA));
    int32_t col = 0;
    for (size_t q = 0; q < ks.size(); ++q) {
      EigUnit U;
      U.k = ks[q];
      U.bs = bmap[ks[q]] == 1 ? 2 : 1;
      U.col = col;
      U.wr = blk[3 * q];
      U.wi = U.bs == 2 ? std::sqrt(std::fabs(blk[3 * q + 1])) * std::sqrt(std::fabs(blk[3 * q + 2])) : 0.0;
      col += U.bs;
      units.push_back(U);
    }
    *ncols = col;
  }
  const int64_t nc = *ncols;
  const int nu = (int)units.size();
  if (X == nullptr || nc == 0) {
    if (st) st->columns = nc;
    return 0;
  }
  // tiles: boundaries near multiples of kTileRows, never inside a 2x2 block
  std::vector<int64_t> tb;
  tb.push_back(0);
  for (int64_t b = kTileRows; b < n; b += kTileRows) {
    int64_t bb = b;
    if (bmap[bb] == 2) bb += 1;
    if (bb > tb.back() && bb < n) tb.push_back(bb);
  }
  tb.push_back(n);
  const int ntiles = (int)tb.size() - 1;
  // Y: the Schur-basis eigenvectors (X itself without a back-transform)
  double* Y = X;
  int64_t ldY = ldX;
  if (Q) {
    ldY = (n + 1) & ~(int64_t)1;
    EK(ws.Y.ensure(sizeof(double) * (size_t)ldY * (size_t)nc));
    Y = (double*)ws.Y.p;
  }
  EK(ws.bmap.ensure((size_t)n));
  EK(ws.units.ensure(sizeof(EigUnit) * (size_t)nu));
  EK(ws.state.ensure(sizeof(EigState) * (size_t)nu));
  EK(ws.tiles.ensure(sizeof(int64_t) * tb.size()));
  EK(ws.snorm.ensure(sizeof(double) * (size_t)ntiles));
  EK(ws.cnt.ensure(sizeof(int32_t) * 4));
  EK(cudaMemcpyAsync(ws.bmap.p, bmap.data(), (size_t)n, cudaMemcpyHostToDevice, sA));
  EK(cudaMemcpyAsync(ws.units.p, units.data(), sizeof(EigUnit) * nu, cudaMemcpyHostToDevice, sA));
  EK(cudaMemsetAsync(ws.state.p, 0, sizeof(EigState) * nu, sA));
  EK(cudaMemcpyAsync(ws.tiles.p, tb.data(), sizeof(int64_t) * tb.size(), cudaMemcpyHostToDevice, sA));
  EK(cudaMemsetAsync(ws.cnt.p, 0, sizeof(int32_t) * 4, sA));
  EK(cudaMemset2DAsync(Y, sizeof(double) * ldY, 0, sizeof(double) * n, nc, sA));
  EK(cudaEventRecord(ws.ev[0], sA));
  int64_t launches = 0;
  eig_snorm_kernel<<<ntiles, 256, 0, sA>>>(S, ldS, (const int64_t*)ws.tiles.p, ntiles, (double*)ws.snorm.p);
  ++launches;
  std::vector<double> snorm(ntiles);
  EK(cudaMemcpyAsync(snorm.data(), ws.snorm.p, sizeof(double) * ntiles, cudaMemcpyDeviceToHost, sA));
  EK(cudaStreamSynchronize(sA));
  const size_t smem_solve = sizeof(double) * (size_t)(kLdT * kTileMax + kTileMax) + kTileMax + 16;
  {
    static bool attr[kMaxDevices] = {};
    const int d = device_slot();
    if (!attr[d]) {
      EK(cudaFuncSetAttribute(eig_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_solve));
      attr[d] = true;
    }
  }
  // back substitution, bottom tile first
  double fl_solve = 0.0, fl_update = 0.0, fl_bt = 0.0;
  // SN_EIG_PROFILE: events around every solve / GEMM launch (split of ms_backsubstitution)
  const bool prof = std::getenv("SN_EIG_PROFILE") != nullptr;
  std::vector<cudaEvent_t> pev;
  std::vector<int> pkind;
  auto mark = [&](int kind) {
    if (!prof) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, sA);
    pev.push_back(e);
    pkind.push_back(kind);
  };
  const int64_t kmax = units.back().k;
  int uA = nu;   // active units: k >= i0 (a suffix: units are sorted by k)
  for (int t = ntiles - 1; t >= 0; --t) {
    const int64_t i0 = tb[t], i1 = tb[t + 1];
    if (i0 > kmax) continue;
    while (uA > 0 && units[uA - 1].k >= i0) --uA;
    const int na = nu - uA;
    if (na <= 0) continue;
    SolveArgs sa{};
    sa.S = S; sa.ldS = ldS; sa.Y = Y; sa.ldY = ldY; sa.bmap = (const int8_t*)ws.bmap.p;
    sa.units = (const EigUnit*)ws.units.p; sa.state = (EigState*)ws.state.p;
    sa.u0 = uA; sa.nu = na; sa.i0 = i0; sa.i1 = i1; sa.snorm = snorm[t];
    sa.rescales = (int32_t*)ws.cnt.p;
    mark(0);
    eig_solve_kernel<<<(na + kSolveWarps - 1) / kSolveWarps, kSolveWarps * 32, smem_solve, sA>>>(sa);
    mark(-1);
    ++launches;
    EK(cudaGetLastError());
    const int64_t colA = units[uA].col;
    for (int q = uA; q < nu; ++q) {
      const double rows = (double)(std::min(i1, units[q].k) - i0);
      fl_solve += 4.0 * units[q].bs * rows * rows;     // 2 flops per entry, complex = 2 real columns
    }
    // updates: within the super-tile (kSuper row tiles) the rows above this tile at once; the
    // rows above the super-tile once its top tile is solved, with K = the super-tile's rows
    // (a 4x longer K loop and a quarter of the passes over Y)
    const int t0 = (t / kSuper) * kSuper;
    const int64_t r0 = tb[t0];
    auto gemm = [&](int64_t rlo, int64_t rhi, int64_t klo, int64_t khi) -> int {
      if (rhi <= rlo) return 0;
      GemmArgs g{};
      // A = S[rlo:rhi, klo:khi] (columns from k0), B = Y[klo:khi, colA:], C = Y[rlo:rhi, colA:]
      g.A = S + rlo; g.lda = ldS;
      g.B = Y + colA * ldY; g.ldb = ldY;
      g.C = Y + colA * ldY + rlo; g.ldc = ldY;
      g.M = rhi - rlo; g.N = (int32_t)(nc - colA); g.k0 = klo; g.K = khi - klo; g.kend = nullptr; g.minus = 1;
      mark(1);
      launch_gemm(g, (g.N + GBN - 1) / GBN, sA);
      mark(-1);
      ++launches;
      EK(cudaGetLastError());
      fl_update += 2.0 * (double)(rhi - rlo) * (double)(khi - klo) * (double)g.N;
      return 0;
    };
    if (int rc = gemm(r0, i0, i0, i1)) return rc;
    if (t == t0) {
      const int64_t s1 = tb[std::min(t0 + kSuper, ntiles)];
      if (int rc = gemm(0, r0, r0, s1)) return rc;
    }
  }
  EK(cudaEventRecord(ws.ev[1], sA));
  // E6: back-transform X = Q Y (per 64-column tile, K up to its last nonzero row)
  if (Q) {
    const int64_t ntn = (nc + GBN - 1) / GBN;
    std::vector<int32_t> kend((size_t)ntn, 0);
    for (const EigUnit& U : units)
      for (int q = 0; q < U.bs; ++q) {
        int32_t& ke = kend[(size_t)((U.col + q) / GBN)];
        ke = std::max<int32_t>(ke, (int32_t)(U.k + U.bs));
      }
    for (size_t q = 0; q < kend.size(); ++q) fl_bt += 2.0 * (double)n * (double)kend[q] * (double)std::min<int64_t>(GBN, nc - (int64_t)q * GBN);
    EK(ws.kend.ensure(sizeof(int32_t) * kend.size()));
    EK(cudaMemcpyAsync(ws.kend.p, kend.data(), sizeof(int32_t) * kend.size(), cudaMemcpyHostToDevice, sA));
    GemmArgs g{};
    g.A = Q; g.lda = ldQ; g.B = Y; g.ldb = ldY; g.C = X; g.ldc = ldX;
    g.M = n; g.N = (int32_t)nc; g.k0 = 0; g.K = n; g.kend = (const int32_t*)ws.kend.p; g.minus = 0;
    launch_gemm(g, ntn, sA);
    ++launches;
    EK(cudaGetLastError());
  }
  EK(cudaEventRecord(ws.ev[2], sA));
  eig_normalize_kernel<<<(nu * 32 + 255) / 256, 256, 0, sA>>>(X, ldX, n, (const EigUnit*)ws.units.p, nu);
  ++launches;
  if (scale_exp) {
    EK(ws.expo.ensure(sizeof(int32_t) * (size_t)nc));
    eig_exp_kernel<<<(nu + 255) / 256, 256, 0, sA>>>((const EigUnit*)ws.units.p, (const EigState*)ws.state.p, nu,
                                                     (int32_t*)ws.expo.p);
    ++launches;
    EK(cudaMemcpyAsync(scale_exp, ws.expo.p, sizeof(int32_t) * (size_t)nc, cudaMemcpyDeviceToHost, sA));
  }
  EK(cudaGetLastError());
  EK(cudaEventRecord(ws.ev[3], sA));
  int32_t cnt[4] = {0, 0, 0, 0};
  EK(cudaMemcpyAsync(cnt, ws.cnt.p, sizeof(cnt), cudaMemcpyDeviceToHost, sA));
  EK(cudaStreamSynchronize(sA));
  if (prof) {
    double acc[2] = {0.0, 0.0};
    for (size_t q = 0; q + 1 < pev.size(); q += 2) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, pev[q], pev[q + 1]);
      acc[pkind[q]] += ms;
    }
    for (auto e : pev) cudaEventDestroy(e);
    std::fprintf(stderr, "{\"probe\":\"eigvec_phases\",\"ms_solve\":%.2f,\"ms_update_gemm\":%.2f,\"flops_update\":%.4g}\n",
                 acc[0], acc[1], fl_update);
  }
  if (st) {
    float a = 0.f, b = 0.f, c = 0.f;
    cudaEventElapsedTime(&a, ws.ev[0], ws.ev[1]);
    cudaEventElapsedTime(&b, ws.ev[1], ws.ev[2]);
    cudaEventElapsedTime(&c, ws.ev[2], ws.ev[3]);
    st->columns = nc;
    st->vectors = nu;
    st->tiles = ntiles;
    st->rescales = cnt[0];
    st->launches = launches;
    st->flops_solve = fl_solve;
    st->flops_update = fl_update;
    st->flops_backtransform = fl_bt;
    st->ms_backsubstitution = a;
    st->ms_backtransform = b;
    st->ms_normalize = c;
    st->ms_device = a + b + c;
    st->ms_total = now_ms() - t0;
  }
  return 0;
}

}  // namespace sn

extern "C" int sn_eigenvectors(int64_t n, const double* S, int64_t ldS, const double* Q, int64_t ldQ,
                               const int32_t* select, double* X, int64_t ldX, int64_t* ncols, int32_t* scale_exp,
                               sn_eig_stats* stats, void* stream) {
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (ncols == nullptr) return -9;
  *ncols = 0;
  if (n < 0) return -1;
  if (n == 0) return 0;
  if (S == nullptr) return -2;
  if (ldS < n) return -3;
  if (Q != nullptr && ldQ < n) return -5;
  if (select == nullptr) return -6;
  if (X != nullptr && ldX < n) return -8;
  std::lock_guard<std::mutex> lock(sn::g_mu);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return SN_ERR_CUDA;
  }
  if (!sn::is_device_ptr(S)) return -2;
  if (Q && !sn::is_device_ptr(Q)) return -4;
  if (X && !sn::is_device_ptr(X)) return -7;
  return sn::eigvec_run(n, S, ldS, Q, ldQ, select, X, ldX, ncols, scale_exp, stats, (cudaStream_t)stream);
}
