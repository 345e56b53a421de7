// sn_kernels_window.cu -- the window task ("applies a set of local
// transformations inside the diagonal window ... produces updated tiles and an accumulator
// matrix as output").
//
// One CTA per window of a DAG level.  The window (k <= 256 rows) is processed as a chain of
// inner windows of <= 64 rows (the plan's inner schedule): each inner window
// is staged in shared memory, its block swaps run as a wavefront of movers (all 8 warps,
// sn_swap.cuh) into an inner accumulator Zin, and Zin is then applied with FP64 DMMA (mma.sync m16n8k8 f64) to
// the rest of the outer window and to the outer accumulator Z -- the paper's accumulated
// level-3 update, one level down.  The outer Z is left in a 256x256 slot for
// the panel kernels.
#include <cstdint>
#include <cstdlib>

#include "sn_device.cuh"
#include "sn_swap.cuh"

namespace sn {
namespace {

#ifndef SN_WIN_THREADS
#define SN_WIN_THREADS 256
#endif
// 4 transform warps + (kThreads/32 - 4) apply warps (the DMMA tiles use warps 0-7)
constexpr int kThreads = SN_WIN_THREADS;
static_assert(kThreads % 32 == 0 && kThreads >= 256, "window kernel needs >= 8 warps");
constexpr int LDD = 65;   // inner window (odd stride: conflict-free row walks)
constexpr int LDZ = 68;   // inner accumulator (== 4 mod 16: conflict-free DMMA fragments)
constexpr int LDT = 68;   // staging tile

__device__ int g_tprof_on;   // debug timing switch (set with WindowArgs::tprof)

// block list of the window being processed (one CTA per window)
__shared__ uint8_t g_bsz[256], g_bsel[256];
__shared__ int16_t g_brow[257];
// nonzero row interval of every column of the outer accumulator Z (sn_device.cuh kZrange)
__shared__ int16_t g_zlo[256], g_zhi[256];

__device__ __forceinline__ void mma_16x8x8(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// 64x64 tile product with K = kin (<= 64, zero padded to a multiple of 8).
//   LEFT : out[m][c] = sum_l Zin[l][m] * Tb[l][c]   (Tb stored l + c*LDT)
//   RIGHT: out[r][c] = sum_l Tb[r][l] * Zin[l][c]   (Tb stored l*LDT + r)
// Warps: 4 (M, 16 rows each) x 2 (N, 32 cols each).
template <bool LEFT>
__device__ __forceinline__ void tile_mma(const double* Tb, const double* Zin, int kin, double (&acc)[4][4],
                                         int warp, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (warp & 3) * 16, n0 = (warp >> 2) * 32;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = 0.0;
  for (int ks = 0; ks < kin; ks += 8) {
    double a[4], b[2];
    if (LEFT) {
      a[0] = Zin[(ks + t) + (m0 + g) * LDZ];
      a[1] = Zin[(ks + t) + (m0 + g + 8) * LDZ];
      a[2] = Zin[(ks + t + 4) + (m0 + g) * LDZ];
      a[3] = Zin[(ks + t + 4) + (m0 + g + 8) * LDZ];
    } else {
      a[0] = Tb[(ks + t) * LDT + m0 + g];
      a[1] = Tb[(ks + t) * LDT + m0 + g + 8];
      a[2] = Tb[(ks + t + 4) * LDT + m0 + g];
      a[3] = Tb[(ks + t + 4) * LDT + m0 + g + 8];
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int nn = n0 + ni * 8 + g;
      if (LEFT) {
        b[0] = Tb[(ks + t) + nn * LDT];
        b[1] = Tb[(ks + t + 4) + nn * LDT];
      } else {
        b[0] = Zin[(ks + t) + nn * LDZ];
        b[1] = Zin[(ks + t + 4) + nn * LDZ];
      }
      mma_16x8x8(acc[ni], a, b);
    }
  }
}

// P[rows r0.., cols c0..c0+kin) <- P * Zin for R rows starting at r0 (RIGHT), or
// P[rows r0..r0+kin, cols c0..c0+C) <- Zin^T * P (LEFT); processed in 64-wide tiles.
template <bool LEFT>
__device__ void inner_update(double* P, int64_t ld, int64_t r0, int64_t c0, int extent, int kin,
                             const double* Zin, double* Tb, int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (warp & 3) * 16, n0 = (warp >> 2) * 32;
  const int kpad = (kin + 7) & ~7;
  for (int e0 = 0; e0 < extent; e0 += 64) {
    const int ne = min(64, extent - e0);
    __syncthreads();
    for (int idx = tid; idx < 64 * 64; idx += kThreads) {
      const int u = idx & 63, v = idx >> 6;
      if (LEFT) {
        // Tb[l + c*LDT] = P[r0 + l, c0 + e0 + c]
        const int l = u, c = v;
        Tb[l + c * LDT] = (l < kin && c < ne) ? P[(r0 + l) + (c0 + e0 + c) * ld] : 0.0;
      } else {
        // Tb[l*LDT + r] = P[r0 + e0 + r, c0 + l]
        const int r = u, l = v;
        Tb[l * LDT + r] = (r < ne && l < kin) ? P[(r0 + e0 + r) + (c0 + l) * ld] : 0.0;
      }
    }
    __syncthreads();
    if (warp >= 8) continue;   // 4 (M) x 2 (N) warps per 64 x 64 tile
    double acc[4][4];
    tile_mma<LEFT>(Tb, Zin, kpad, acc, warp, lane);
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int mm = m0 + g + 8 * h, nn = n0 + ni * 8 + 2 * t + q;
          const double v = acc[ni][2 * h + q];
          if (LEFT) {
            if (mm < kin && nn < ne) P[(r0 + mm) + (c0 + e0 + nn) * ld] = v;
          } else {
            if (mm < ne && nn < kin) P[(r0 + e0 + mm) + (c0 + nn) * ld] = v;
          }
        }
  }
}

// ---- wavefront of movers inside one inner window ---------------------------------------
// Mover i (i-th selected block of [top, bottom), top to bottom) starts at block P_i, passes
// the u_i unselected blocks above it and ends at block top+i.  It performs its s-th swap at
// step 2i + s, so concurrent swaps are at least two blocks apart: their index sets are
// disjoint and their orthogonal factors commute.
//
// Software pipeline: while the apply warps perform step t -- (B) the row applications, then,
// after a barrier among themselves, (C) the column applications to the window and to Zin --
// the transform warps already evaluate the transforms of step t+1, one thread per swap
// grouped by type (a lane pair per 2x2|2x2 swap).  This is legal because the transform of
// mover i's step-(t+1) swap reads only (a) the diagonal block of the unselected block u it
// passes next, last written two or more steps earlier by mover i-1, (b) mover i's new
// diagonal block, which is part of its step-t record, and (c) the coupling rows of u in the
// columns of mover i's step-t pair, which only mover i's step-t column application changes:
// the transform thread applies that column transform to those rows itself (and writes them
// back), and the apply warps skip them.  One CTA barrier per step.
#ifndef SN_WIN_QUAD
#define SN_WIN_QUAD 0
#endif
constexpr int kG22 = SN_WIN_QUAD ? 4 : 2;  // lanes per 2x2|2x2 transform (quad: lane-parallel Sylvester)
constexpr int kWT = 4;                     // transform warps: w < 3 swap type w, w = 3 2x2|2x2
constexpr int kWA = kThreads / 32 - kWT;   // apply warps
constexpr int kRecBuf = 4 * 32 * dev::kRec;   // doubles per record buffer (type x slot)

struct WaveShared {
  int M, U, T;                        // movers, unselected blocks, steps
  uint8_t msz[64], usz[64];           // sizes of movers / unselected blocks (top to bottom)
  int16_t mpos[64], mu[64];           // initial block position, unselected blocks above
  int16_t mrows[65], urows[65];       // row prefixes of movers / unselected blocks
  // step lists, triple-buffered by t % 3 (step t applied, t+1 transformed, t+2 prepared)
  int16_t lj[3][4][32];               // per type, slot: local row j
  int8_t lflat[3][4][32];             // ... flat index (mover order among active swaps)
  int8_t ftype[3][64], fslot[3][64], fmover[3][64];
  int8_t mflat[3][32];                // mover -> flat index of its swap in the step, or -1
  int16_t lprev[3][4][32];            // per type, slot: the mover's previous record (type*32 +
                                      // slot, in the other record buffer), or -1 (first swap)
  int cnt[3][4], nflat[3];
  int8_t frej[3][64];
  int anyrej[3];
  int done, laststep, rejected;
  int8_t zlo[64], zhi[64];            // nonzero row interval of every column of Zin
  int rej_row, rej_n1, rej_n2;
  unsigned long long tmax[4], tsum[4];  // debug timing (tprof): per-step maxima
};

__device__ void wave_prepare(WaveShared& W, int t, int lane) {
  // one warp: lists of the active swaps of step t, grouped by type and in mover order
  const int buf = t % 3;
  const int i = lane;
  bool act = false;
  int ty = 0, j = 0;
  if (i < W.M) {
    const int s = t - 2 * i;
    if (s >= 0 && s < W.mu[i]) {
      act = true;
      const int q = W.mu[i] - 1 - s;           // unselected block being passed
      ty = (W.usz[q] - 1) * 2 + (W.msz[i] - 1);
      j = W.mrows[i] + W.urows[q];
    }
  }
  const unsigned amask = __ballot_sync(0xffffffffu, act);
  const unsigned lt = (1u << lane) - 1u;
  const int flat = __popc(amask & lt);
  W.mflat[buf][lane] = act ? (int8_t)flat : (int8_t)-1;
  for (int q = 0; q < 4; ++q) {
    const unsigned tm = __ballot_sync(0xffffffffu, act && ty == q);
    if (act && ty == q) {
      const int slot = __popc(tm & lt);
      int pv = -1;
      if (t > 0) {
        const int pb = (t - 1) % 3, pf = W.mflat[pb][i];   // lists of t-1 are already prepared
        if (pf >= 0) pv = W.ftype[pb][pf] * 32 + W.fslot[pb][pf];
      }
      W.lprev[buf][q][slot] = (int16_t)pv;
      W.lj[buf][q][slot] = (int16_t)j;
      W.lflat[buf][q][slot] = (int8_t)flat;
      W.ftype[buf][flat] = (int8_t)q;
      W.fslot[buf][flat] = (int8_t)slot;
      W.fmover[buf][flat] = (int8_t)i;
    }
    if (lane == 0) W.cnt[buf][q] = __popc(tm);
  }
  if (lane == 0) W.nflat[buf] = __popc(amask);
}

// The (n1+n2)^2 block of a step-t swap (type ty at local row j, flat index `flat`): from the
// window directly for a mover's first swap, else assembled from the window (the unselected
// block), the mover's step t-1 record (its new diagonal block) and the coupling rows, to which
// the step t-1 column transform is applied here (returned in cpl for the write-back).
template <int N1, int N2>
__device__ __forceinline__ int wave_assemble(int t, int j, int pv, const double* Din, const double* recs,
                                             double (&Db)[4][4], double (&cpl)[2][4], int& jp, int& pnd) {
  constexpr int nd = N1 + N2;
  if (pv < 0) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) Db[r][c] = (r < nd && c < nd) ? Din[(j + r) + (j + c) * LDD] : 0.0;
    return 0;
  }
  const int pt = pv >> 5;
  const double* prec = recs + ((t - 1) & 1) * kRecBuf + pv * dev::kRec;
  jp = j + N1;                                 // mover i's previous pair
  pnd = (pt >> 1) + (pt & 1) + 2;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) Db[r][c] = 0.0;
#pragma unroll
  for (int r = 0; r < N1; ++r) {
#pragma unroll
    for (int c = 0; c < N1; ++c) Db[r][c] = Din[(j + r) + (j + c) * LDD];
    double x[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = c < pnd ? Din[(j + r) + (jp + c) * LDD] : 0.0;
    dev::rec_apply_generic(x, prec);
#pragma unroll
    for (int c = 0; c < 4; ++c) cpl[r][c] = x[c];
#pragma unroll
    for (int c = 0; c < N2; ++c) Db[r][N1 + c] = x[c];
  }
  if (pt == 0) {
    Db[N1][N1] = prec[3];                      // a moved 1x1 keeps its exact value (R7)
  } else {
#pragma unroll
    for (int a2 = 0; a2 < N2; ++a2)
#pragma unroll
      for (int b2 = 0; b2 < N2; ++b2) Db[N1 + a2][N1 + b2] = prec[10 + a2 + 4 * b2];
  }
  return N1;
}

template <int N1>
__device__ __forceinline__ void wave_writeback(int jp, int pnd, int j, double* Din, const double (&cpl)[2][4]) {
#pragma unroll
  for (int r = 0; r < N1; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < pnd) Din[(j + r) + (jp + c) * LDD] = cpl[r][c];
}

// one swap of type (N1, N2) by one thread (warps 0-2)
template <int N1, int N2>
__device__ __forceinline__ void wave_transform_one(int t, int base, int lane, double* Din, double* recs,
                                                   WaveShared& W, bool force_here, int force_swap) {
  constexpr int ty = (N1 - 1) * 2 + (N2 - 1);
  const int sb = t % 3;
  double* rec_t = recs + (t & 1) * kRecBuf;
  const int j = W.lj[sb][ty][lane];
  const int flat = W.lflat[sb][ty][lane];
  double Db[4][4], cpl[2][4];
  int jp = 0, pnd = 0;
  const long long q0 = g_tprof_on ? clock64() : 0;
  if (wave_assemble<N1, N2>(t, j, W.lprev[sb][ty][lane], Din, recs, Db, cpl, jp, pnd))
    wave_writeback<N1>(jp, pnd, j, Din, cpl);
  const long long q1 = g_tprof_on ? clock64() : 0;
  bool rj = force_here && (base + flat == force_swap);
  if (!rj) {
    double* rec = rec_t + (ty * 32 + lane) * dev::kRec;
    rj = dev::swap_compute_blk<N1, N2>(Db, rec);
    dev::rec_generic(ty, rec);
  }
  if (g_tprof_on) {
    atomicMax(&W.tmax[2], (unsigned long long)(q1 - q0));
    atomicMax(&W.tmax[3], (unsigned long long)(clock64() - q1));
  }
  W.frej[sb][flat] = rj ? 1 : 0;
  if (rj) atomicOr(&W.anyrej[sb], 1);
}

// transforms of step t by the transform warps
__device__ void wave_transform(int t, int base, double* Din, double* recs, WaveShared& W, int warp, int lane,
                               bool force_here, int force_swap) {
  const int sb = t % 3;
  double* rec_t = recs + (t & 1) * kRecBuf;
  if (warp < 3) {
    if (lane < W.cnt[sb][warp]) {
      if (warp == 0) wave_transform_one<1, 1>(t, base, lane, Din, recs, W, force_here, force_swap);
      else if (warp == 1) wave_transform_one<1, 2>(t, base, lane, Din, recs, W, force_here, force_swap);
      else wave_transform_one<2, 1>(t, base, lane, Din, recs, W, force_here, force_swap);
    }
  } else if (warp == 3) {
    const int c3 = W.cnt[sb][3];
    for (int b0 = 0; b0 < c3; b0 += 32 / kG22) {
      const int slot = b0 + lane / kG22, role = lane % kG22;
      const bool act = slot < c3;
      const int sl = act ? slot : b0;
      const int j = W.lj[sb][3][sl];
      const int flat = W.lflat[sb][3][sl];
      double Db[4][4], cpl[2][4];
      int jp = 0, pnd = 0;
      const int nw = wave_assemble<2, 2>(t, j, W.lprev[sb][3][sl], Din, recs, Db, cpl, jp, pnd);
      __syncwarp();   // every lane has read the coupling rows before they are written back
      if (act && role == 0 && nw) wave_writeback<2>(jp, pnd, j, Din, cpl);
      double tmp[dev::kGen];
      const long long q1 = g_tprof_on ? clock64() : 0;
      bool rj = kG22 == 4 ? dev::swap_compute_22_quad_blk(Db, tmp, role) : dev::swap_compute_22_paired_blk(Db, tmp, role);
      if (g_tprof_on) atomicMax(&W.tmax[3], (unsigned long long)(clock64() - q1));
      if (act && role == 0) {
        rj = rj || (force_here && (base + flat == force_swap));
        double* dst = rec_t + (3 * 32 + slot) * dev::kRec;
#pragma unroll
        for (int q = 0; q < dev::kGen; ++q) dst[q] = tmp[q];
        dev::rec_generic(3, dst);
        W.frej[sb][flat] = rj ? 1 : 0;
        if (rj) atomicOr(&W.anyrej[sb], 1);
      }
    }
  }
}

__device__ void wavefront_swaps(int top, int bottom, int i1, int kin, double* Din, double* Zin, double* recs,
                                WaveShared& W, int tid, int warp, int lane, bool force_here, int force_swap,
                                int done_before, unsigned long long* tp) {
  const long long c0 = tp && tid == 0 ? clock64() : 0;
  if (tid == 0) {
    // movers / unselected lists of the inner window (block list in s_bsz/s_bsel)
    int M = 0, U = 0, T = 0;
    W.mrows[0] = 0; W.urows[0] = 0;
    for (int b = top; b < bottom; ++b) {
      if (g_bsel[b]) {
        W.msz[M] = g_bsz[b];
        W.mpos[M] = (int16_t)b;
        W.mu[M] = (int16_t)(b - top - M);
        W.mrows[M + 1] = (int16_t)(W.mrows[M] + g_bsz[b]);
        T = max(T, 2 * M + (b - top - M));
        ++M;
      } else {
        W.usz[U] = g_bsz[b];
        W.urows[U + 1] = (int16_t)(W.urows[U] + g_bsz[b]);
        ++U;
      }
    }
    W.M = M; W.U = U; W.T = T;
    W.anyrej[0] = W.anyrej[1] = W.anyrej[2] = 0;
    W.rejected = 0;
    for (int q = 0; q < 4; ++q) { W.tmax[q] = 0; W.tsum[q] = 0; }
  }
  if (tid < kInner) { W.zlo[tid] = (int8_t)tid; W.zhi[tid] = (int8_t)tid; }
  __syncthreads();
  const int T = W.T;
  if (warp == 0) {
    wave_prepare(W, 0, lane);
    __syncwarp();
    if (T > 1) wave_prepare(W, 1, lane);   // reads step 0's lists
  }
  __syncthreads();
  int base = done_before;
  if (warp < kWT) wave_transform(0, base, Din, recs, W, warp, lane, force_here, force_swap);
  __syncthreads();
  int t = 0;
  bool stop_now = false;
  for (; t < T; ++t) {
    const int sb = t % 3;
    stop_now = W.anyrej[sb] != 0;          // a swap of step t was rejected: apply the rest, stop
    const bool last = stop_now || t + 1 == T;
    const int nf = W.nflat[sb];
    if (tid == 0) W.anyrej[(t + 2) % 3] = 0;
    const long long cs = tp ? clock64() : 0;
    if (warp < kWT) {
      if (!last) wave_transform(t + 1, base + nf, Din, recs, W, warp, lane, force_here, force_swap);
    } else {
      const double* rec_t = recs + (t & 1) * kRecBuf;
      const int aw = warp - kWT;
      // B: rows
      for (int f = aw; f < nf; f += kWA) {
        if (W.frej[sb][f]) continue;
        const int ty = W.ftype[sb][f], sl = W.fslot[sb][f];
        dev::swap_apply_rows_t(ty, Din, LDD, kin, W.lj[sb][ty][sl], rec_t + (ty * 32 + sl) * dev::kRec, lane);
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kWA * 32) : "memory");
      // C: columns of the window (less the coupling rows the next transform applies) and of Zin
      for (int f = aw; f < nf; f += kWA) {
        if (W.frej[sb][f]) continue;
        const int ty = W.ftype[sb][f], sl = W.fslot[sb][f];
        const int j = W.lj[sb][ty][sl];
        const double* rec = rec_t + (ty * 32 + sl) * dev::kRec;
        int rows = j;
        if (!last) {
          const int nf1 = W.mflat[(t + 1) % 3][W.fmover[sb][f]];
          if (nf1 >= 0) rows = j - ((W.ftype[(t + 1) % 3][nf1] >> 1) + 1);
        }
        dev::swap_apply_cols_t(ty, Din, LDD, rows, j, rec, lane);
        {
          // Zin columns j..j+nd-1 are zero outside the union of their row intervals (Zin starts
          // as I and every swap mixes adjacent columns): apply the transform there only
          const int nd = (ty >> 1) + (ty & 1) + 2;
          int lo = W.zlo[j], hi = W.zhi[j];
          for (int c = 1; c < nd; ++c) { lo = min(lo, (int)W.zlo[j + c]); hi = max(hi, (int)W.zhi[j + c]); }
          dev::swap_apply_cols_t(ty, Zin + lo, LDZ, hi - lo + 1, j, rec, lane);
          __syncwarp();
          if (lane < nd) { W.zlo[j + lane] = (int8_t)lo; W.zhi[j + lane] = (int8_t)hi; }
        }
        {
          // the swap mixes outer Z columns i1+j .. i1+j+n1+n2-1 (concurrent swaps: disjoint);
          // lanes 0..3 hold one column each, reduced over groups of 4 lanes
          const int c = i1 + j + (lane & 3), nc = (ty >> 1) + (ty & 1) + 2;
          const bool mine = (lane & 3) < nc;
          int lo = mine ? g_zlo[c] : kZld, hi = mine ? g_zhi[c] : -1;
          lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, 1));
          hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, 1));
          lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, 2));
          hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, 2));
          if (lane < 4 && mine) { g_zlo[c] = (int16_t)lo; g_zhi[c] = (int16_t)hi; }
        }
      }
      // the last apply warp prepares the lists of step t+2 (buffer (t+2) % 3 is idle)
      if (warp == kThreads / 32 - 1 && t + 2 < T) wave_prepare(W, t + 2, lane);
    }
    if (tp && lane == 0) atomicMax(&W.tmax[warp < kWT ? 0 : 1], (unsigned long long)(clock64() - cs));
    __syncthreads();
    if (tp && tid == 0) {
      for (int q = 0; q < 4; ++q) { W.tsum[q] += W.tmax[q]; W.tmax[q] = 0; }
    }
    if (stop_now) break;
    base += nf;
  }
  if (tid == 0) {
    const int tl = min(t, T - 1);
    W.laststep = tl;
    if (stop_now) {
      const int sb = tl % 3;
      int nrej = 0, first = -1;
      for (int f = 0; f < W.nflat[sb]; ++f)
        if (W.frej[sb][f]) { ++nrej; if (first < 0) first = f; }
      W.done = base + W.nflat[sb] - nrej;
      const int ty = W.ftype[sb][first], sl = W.fslot[sb][first];
      W.rej_row = i1 + W.lj[sb][ty][sl];   // window-local row
      W.rej_n1 = (ty >> 1) + 1;
      W.rej_n2 = (ty & 1) + 1;
      W.rejected = 1;
    } else {
      W.done = base;
    }
    if (tp) {
      atomicAdd(&tp[1], (unsigned long long)(clock64() - c0));
      atomicAdd(&tp[4], (unsigned long long)T);
      atomicAdd(&tp[0], W.tsum[0]);   // transform side, per-step max summed
      atomicAdd(&tp[2], W.tsum[1]);   // apply side
      atomicAdd(&tp[13], W.tsum[2]);   // assembly (max per step)
      atomicAdd(&tp[14], W.tsum[3]);   // transform proper (max per step)
    }
  }
  __syncthreads();
  // new block arrangement of [top, bottom)
  if (tid == 0) {
    uint8_t nsz[64], nsel[64];
    int8_t occ[64];
    const int nb = bottom - top;
    for (int b = 0; b < nb; ++b) occ[b] = 0;
    const int tl = W.laststep;
    for (int i = 0; i < W.M; ++i) {
      int applied = W.mu[i];
      if (W.rejected) {
        applied = min(max(tl + 1 - 2 * i, 0), (int)W.mu[i]);
        // a rejected swap of this mover at the last step was not applied
        const int s = tl - 2 * i;
        if (s >= 0 && s < W.mu[i]) {
          const int buf = tl % 3;
          for (int f = 0; f < W.nflat[buf]; ++f)
            if (W.fmover[buf][f] == i && W.frej[buf][f]) { applied -= 1; break; }
        }
      }
      const int pos = W.mpos[i] - top - applied;
      nsz[pos] = W.msz[i]; nsel[pos] = 1; occ[pos] = 1;
    }
    int q = 0;
    for (int b = 0; b < nb; ++b)
      if (!occ[b]) { nsz[b] = W.usz[q++]; nsel[b] = 0; }
    for (int b = 0; b < nb; ++b) { g_bsz[top + b] = nsz[b]; g_bsel[top + b] = nsel[b]; }
    for (int b = top; b < bottom; ++b) g_brow[b + 1] = (int16_t)(g_brow[b] + g_bsz[b]);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 1) window_kernel(WindowArgs a) {
  extern __shared__ __align__(16) double smem[];
  double* Din = smem;                       // kInner x LDD
  double* Zin = Din + kInner * LDD;         // kInner x LDZ
  double* Tb = Zin + kInner * LDZ;          // 64 x LDT
  double* recs = Tb + 64 * LDT;             // transform records, 2 step buffers x 4 types x 32
  __shared__ WaveShared W;
  uint8_t* bsz = g_bsz;
  uint8_t* bsel = g_bsel;
  int16_t* brow = g_brow;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int widx = blockIdx.x;
  const WinDev wd = a.wins[widx];
  const int sidx = wd.sidx;
  {
    // a rejection in an earlier level stops the run; windows of the rejecting level all run
    const int32_t al = *(volatile int32_t*)&a.ctl->abort_level;
    if (al != 0 && al - 1 < a.level) {
      if (tid == 0) a.status[sidx] = kWinSkipped;
      return;
    }
  }
  const int k = wd.k, nb = wd.nblk;
  const uint8_t* pool = a.pool + wd.pool;
  for (int b = tid; b < nb; b += kThreads) { bsz[b] = pool[b]; bsel[b] = pool[nb + b]; }
  for (int c = tid; c < kZld; c += kThreads) {
    g_zlo[c] = (int16_t)(c < wd.k ? c : kZld - 1);
    g_zhi[c] = (int16_t)(c < wd.k ? c : 0);
  }
  int64_t ioff = wd.pool + 2 * nb;
  ioff += ioff & 1;
  const uint16_t* inner = reinterpret_cast<const uint16_t*>(a.pool + ioff);
  const int64_t ld = a.ldS;
  double* S = a.S + wd.coff * ld;   // column j of S at column j + coff of the array
  const int64_t j1 = wd.j1;
  double* Z = a.Z + (int64_t)wd.slot * kZslot;
  // Z <- I (k x k, zero padded to 256 x 256)
  for (int idx = tid; idx < kZld * kZld; idx += kThreads) {
    const int r = idx & (kZld - 1), c = idx >> 8;
    Z[idx] = (r == c && r < k) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    W.rejected = 0;
    int r = 0;
    for (int b = 0; b < nb; ++b) { brow[b] = (int16_t)r; r += bsz[b]; }
    brow[nb] = (int16_t)r;
  }
  __syncthreads();

  int swaps_done = 0;
  long long ck = clock64();
  const long long ck0 = ck;
  for (int q = 0; q < wd.ninner; ++q) {
    const int top = inner[2 * q], bottom = inner[2 * q + 1];
    const int i1 = brow[top], i2 = brow[bottom];
    const int kin = i2 - i1;
    // stage the inner window and Zin = I
    for (int idx = tid; idx < kInner * kInner; idx += kThreads) {
      const int r = idx & (kInner - 1), c = idx >> 6;
      if (r < kin && c < kin) Din[r + c * LDD] = S[(j1 + i1 + r) + (j1 + i1 + c) * ld];
      Zin[r + c * LDZ] = (r == c && r < kin) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (a.tprof && tid == 0) { const long long c = clock64(); atomicAdd(&a.tprof[6], (unsigned long long)(c - ck)); ck = c; }
    // debug knob: reject in the window of schedule order force_order, or (force_order <= -2)
    // in every window of DAG level -2 - force_order
    const bool force_here = wd.order == a.force_order || (a.force_order <= -2 && a.level == -2 - a.force_order);
    wavefront_swaps(top, bottom, i1, kin, Din, Zin, recs, W, tid, warp, lane, force_here, a.force_swap, swaps_done,
                    a.tprof);
    if (a.tprof && tid == 0) ck = clock64();
    swaps_done = W.done;
    // write the inner window back
    for (int idx = tid; idx < kInner * kInner; idx += kThreads) {
      const int r = idx & (kInner - 1), c = idx >> 6;
      if (r < kin && c < kin) S[(j1 + i1 + r) + (j1 + i1 + c) * ld] = Din[r + c * LDD];
    }
    // inner accumulated updates restricted to the outer window
    inner_update<false>(S, ld, j1, j1 + i1, i1, kin, Zin, Tb, tid);              // rows above
    inner_update<true>(S, ld, j1 + i1, j1 + i2, k - i2, kin, Zin, Tb, tid);      // cols right
    inner_update<false>(Z, kZld, 0, i1, k, kin, Zin, Tb, tid);                   // Z columns
    __syncthreads();
    if (a.tprof && tid == 0) { const long long c = clock64(); atomicAdd(&a.tprof[7], (unsigned long long)(c - ck)); ck = c; }
    if (W.rejected) break;
  }
  {
    int16_t* zr = a.zrange + (int64_t)wd.slot * kZrange;
    for (int c = tid; c < kZld; c += kThreads) { zr[c] = g_zlo[c]; zr[kZld + c] = g_zhi[c]; }
    // executed work of the panel kernels for this Z: per 32-row group of Z^T rows (a warp's M
    // rows), the k4 steps of [0, 16*ceil(k/16)) that meet the group's K interval
    if (warp == 0 && a.kwork) {
      int total = 0;
      const int kpad = 16 * ((k + 15) / 16);
      for (int g0 = 0; g0 < kZld; g0 += 32) {
        int lo = g_zlo[g0 + lane], hi = g_zhi[g0 + lane];
        for (int o = 16; o > 0; o >>= 1) {
          lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
          hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (g0 < k && hi >= lo) {
          int cnt = 0;
          for (int kg = 0; kg < kpad; kg += 4) cnt += (kg + 3 >= lo && kg <= hi) ? 1 : 0;
          total += cnt;
        }
      }
      if (lane == 0) a.kwork[sidx] = total;
    }
  }
  if (a.tprof && tid == 0) {
    atomicAdd(&a.tprof[8], (unsigned long long)(clock64() - ck0));
    atomicAdd(&a.tprof[9], 1ull);
  }
  if (tid == 0) {
    if (W.rejected) {
      WinRec* rc = a.recs + sidx;
      rc->done = swaps_done;
      rc->row = (int)(j1 + W.rej_row);
      rc->n1 = W.rej_n1;
      rc->n2 = W.rej_n2;
      for (int b = 0; b < nb; ++b) { rc->sz[b] = bsz[b]; rc->sel[b] = bsel[b]; }
      atomicCAS(&a.ctl->abort_level, 0, a.level + 1);
      atomicExch(&a.ctl->abort, 1);
      a.status[sidx] = kWinPartial;
    } else {
      a.status[sidx] = kWinDone;
    }
  }
}

}  // namespace

size_t window_smem_bytes() {
  return sizeof(double) * (size_t)(kInner * LDD + kInner * LDZ + 64 * LDT + 2 * kRecBuf);
}

void launch_window(const WindowArgs& a, cudaStream_t st) {
  // per device: the opt-in shared-memory attribute and the debug switch are device state
  static bool attr[kMaxDevices] = {};
  static int tprof_state[kMaxDevices];
  static bool init = false;
  if (!init) { for (int d = 0; d < kMaxDevices; ++d) tprof_state[d] = -1; init = true; }
  const int dev = device_slot();
  const int want = a.tprof ? 1 : 0;
  if (tprof_state[dev] != want) { cudaMemcpyToSymbol(g_tprof_on, &want, sizeof(int)); tprof_state[dev] = want; }
  const size_t smem = window_smem_bytes();
  if (!attr[dev]) {
    cudaFuncSetAttribute(window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[dev] = true;
  }
  if (a.nwin > 0) window_kernel<<<a.nwin, kThreads, smem, st>>>(a);
}

}  // namespace sn
