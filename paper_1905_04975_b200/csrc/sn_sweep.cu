// sn_sweep.cu -- one bulge-chasing sweep of the multishift QR algorithm (
// "The bulge chasing step creates a set of bulges which are chased down
// the diagonal to complete one pipelined QR iteration.  This is accomplished by applying
// sequences of overlapping 3 x 3 Householder reflectors to H"; Table 1).  Product code;
// readings B1-B5 in DESIGN.md §3.3.
//
// The reflectors run on the same window / accumulator / panel machinery as the reordering
// (Fig. 1b): bulges travel in chains of up to `bulges_per_chain` bulges spaced 4
// rows apart (so the reflectors of one chain step act on disjoint rows and columns); a chain
// is chased through overlapping diagonal windows of <= 256 rows.  The window task applies the
// chain's reflectors to the window only and accumulates them into a 256 x 256 Z slot; the
// left update (row panel right of the window), the right update (column panel above it) and
// the Q update are the reordering's TMA + DMMA panel kernels.  Windows are levelled like the
// reordering's (a window depends on every earlier window whose row range meets its own; the
// remaining left/right corner conflicts commute), chain c+1 following chain c.
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

constexpr int kSweepThreads = 256;
constexpr int kMaxChainBulges = 60;   // 4 (m - 1) + 8 <= 256 rows
constexpr int kZgenS = 4;             // Z slot generations in flight (Q stream)

struct BulgeDev {
  int32_t tau0, tau1;   // chain steps executed by this window
  int32_t m;            // bulges of the chain
  int32_t b0;           // first global bulge index of the chain (shift pair index)
};

struct SweepArgs {
  const WinDev* wins;   // this level's windows
  const BulgeDev* bw;
  int32_t nwin;
  double* H;
  int64_t ldH;
  int64_t n;
  double* Z;
  int16_t* zrange;
  int32_t* status;
  const double* sr;     // shifts (device), 2 per bulge
  const double* si;
};

// 3- or 2-element reflector (xLARFG, reading R3): (alpha, x) -> (beta, 0); v = (1, x')
__device__ __forceinline__ void larfg(int m, double& alpha, double& x0, double& x1, double& tau) {
  const double xn = m == 3 ? hypot(x0, x1) : fabs(x0);
  if (xn == 0.0) { tau = 0.0; return; }
  const double beta = -copysign(hypot(alpha, xn), alpha);
  tau = (beta - alpha) / beta;
  const double sc = 1.0 / (alpha - beta);
  x0 *= sc;
  if (m == 3) x1 *= sc;
  alpha = beta;
}

// STAGED: the window (k <= kStageMax) is copied to shared memory, worked on there and written
// back (the per-step left/right updates then cost shared-memory latency, not L2 round trips);
// otherwise it is updated in place in global memory (L2 resident).
constexpr int kStageMax = 160;
constexpr int kStageLd = kStageMax + 1;   // odd stride: conflict-free row walks

template <bool STAGED>
__global__ void __launch_bounds__(kSweepThreads, 1) bulge_window_kernel(SweepArgs a) {
  extern __shared__ __align__(16) double hs[];
  __shared__ double rv[kMaxChainBulges][3];
  __shared__ double rt[kMaxChainBulges];
  __shared__ int rp[kMaxChainBulges];    // local first row of the reflector, -1 inactive
  __shared__ int rm[kMaxChainBulges];    // 3 or 2 elements
  __shared__ int16_t zlo[kZld], zhi[kZld];
  const int tid = threadIdx.x;
  const WinDev wd = a.wins[blockIdx.x];
  const BulgeDev bd = a.bw[blockIdx.x];
  const int k = wd.k;
  const int64_t w0 = wd.j1, n = a.n;
  double* Hg = a.H + w0 + w0 * a.ldH;                 // the window in global memory
  double* Hw = STAGED ? hs : Hg;                      // local (r, c) at Hw[r + c * ld]
  const int64_t ld = STAGED ? kStageLd : a.ldH;
  if (STAGED) {
    for (int idx = tid; idx < k * k; idx += kSweepThreads) {
      const int r = idx % k, c = idx / k;
      hs[r + c * kStageLd] = Hg[r + (int64_t)c * a.ldH];
    }
  }
  double* Z = a.Z + (int64_t)wd.slot * kZslot;
  for (int idx = tid; idx < kZld * kZld; idx += kSweepThreads) {
    const int r = idx & (kZld - 1), c = idx >> 8;
    Z[idx] = (r == c && r < k) ? 1.0 : 0.0;
  }
  for (int c = tid; c < kZld; c += kSweepThreads) {
    zlo[c] = (int16_t)(c < k ? c : kZld - 1);
    zhi[c] = (int16_t)(c < k ? c : 0);
  }
  __syncthreads();
  for (int tau = bd.tau0; tau < bd.tau1; ++tau) {
    // phase 1: the reflectors of this chain step (one thread per bulge)
    for (int b = tid; b < bd.m; b += kSweepThreads) {
      const int64_t p = (int64_t)tau - 4 * b;                 // global first row (B3)
      int pl = -1;
      if (p >= 0 && p <= n - 2) {
        pl = (int)(p - w0);
        const int m = p <= n - 3 ? 3 : 2;
        double alpha, x0, x1 = 0.0, t;
        if (p == 0) {
          // B2: introduce the bulge from its shift pair: p(H) e1 = (H^2 - sigma H + pi I) e1
          const int j = 2 * (bd.b0 + b);
          const double sigma = a.sr[j] + a.sr[j + 1];
          const double pi = a.sr[j] * a.sr[j + 1] - a.si[j] * a.si[j + 1];
          const double h00 = Hw[0], h10 = Hw[1], h01 = Hw[ld], h11 = Hw[1 + ld], h21 = Hw[2 + ld];
          alpha = h00 * h00 + h01 * h10 - sigma * h00 + pi;
          x0 = h10 * (h00 + h11 - sigma);
          x1 = h10 * h21;
          larfg(3, alpha, x0, x1, t);
        } else {
          double* col = Hw + (int64_t)(pl - 1) * ld;
          alpha = col[pl];
          x0 = col[pl + 1];
          if (m == 3) x1 = col[pl + 2];
          larfg(m, alpha, x0, x1, t);
          col[pl] = alpha;
          col[pl + 1] = 0.0;
          if (m == 3) col[pl + 2] = 0.0;
        }
        rv[b][0] = 1.0; rv[b][1] = x0; rv[b][2] = m == 3 ? x1 : 0.0;
        rt[b] = t;
        rm[b] = m;
        // Z structure: the reflector mixes columns pl .. pl+m-1
        int lo = zlo[pl], hi = zhi[pl];
        for (int q = 1; q < m; ++q) { lo = min(lo, (int)zlo[pl + q]); hi = max(hi, (int)zhi[pl + q]); }
        for (int q = 0; q < m; ++q) { zlo[pl + q] = (int16_t)lo; zhi[pl + q] = (int16_t)hi; }
      }
      rp[b] = pl;
    }
    __syncthreads();
    // phase 2: left updates, rows pl.. of columns pl .. k-1 (one thread per column)
    for (int c = tid; c < k; c += kSweepThreads) {
      double* col = Hw + (int64_t)c * ld;
      for (int b = 0; b < bd.m; ++b) {
        const int pl = rp[b];
        if (pl < 0 || c < pl) continue;
        const double t = rt[b];
        if (t == 0.0) continue;
        const int m = rm[b];
        const double v1 = rv[b][1], v2 = rv[b][2];
        const double y0 = col[pl], y1 = col[pl + 1], y2 = m == 3 ? col[pl + 2] : 0.0;
        const double s = t * (y0 + v1 * y1 + v2 * y2);
        col[pl] = y0 - s;
        col[pl + 1] = y1 - s * v1;
        if (m == 3) col[pl + 2] = y2 - s * v2;
      }
    }
    __syncthreads();
    // phase 3: right updates, columns pl.. of rows 0 .. pl+3 of the window, and of Z
    for (int r = tid; r < k; r += kSweepThreads) {
      for (int b = 0; b < bd.m; ++b) {
        const int pl = rp[b];
        if (pl < 0) continue;
        const double t = rt[b];
        if (t == 0.0) continue;
        const int m = rm[b];
        const double v1 = rv[b][1], v2 = rv[b][2];
        if (r <= pl + 3) {
          double* h = Hw + r + (int64_t)pl * ld;
          const double y0 = h[0], y1 = h[ld], y2 = m == 3 ? h[2 * ld] : 0.0;
          const double s = t * (y0 + v1 * y1 + v2 * y2);
          h[0] = y0 - s;
          h[ld] = y1 - s * v1;
          if (m == 3) h[2 * ld] = y2 - s * v2;
        }
        double* z = Z + r + pl * kZld;
        const double y0 = z[0], y1 = z[kZld], y2 = m == 3 ? z[2 * kZld] : 0.0;
        const double s = t * (y0 + v1 * y1 + v2 * y2);
        z[0] = y0 - s;
        z[kZld] = y1 - s * v1;
        if (m == 3) z[2 * kZld] = y2 - s * v2;
      }
    }
    __syncthreads();
  }
  if (STAGED) {
    for (int idx = tid; idx < k * k; idx += kSweepThreads) {
      const int r = idx % k, c = idx / k;
      Hg[r + (int64_t)c * a.ldH] = hs[r + c * kStageLd];
    }
  }
  int16_t* zr = a.zrange + (int64_t)wd.slot * kZrange;
  for (int c = tid; c < kZld; c += kSweepThreads) { zr[c] = zlo[c]; zr[kZld + c] = zhi[c]; }
  if (tid == 0) a.status[wd.sidx] = kWinDone;
}

struct SBuf {
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

struct SweepWorkspace {
  SBuf wins, bw, pref, status, Z, zr, shifts, sub, bad;
  cudaStream_t sB = nullptr, sC = nullptr;   // Q updates / remaining (non-critical) strips
  cudaEvent_t evW[kZgenS] = {}, evQ[kZgenS] = {}, evCrit[kZgenS] = {}, evRest[kZgenS] = {};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evIn = nullptr, evJoin = nullptr;
  int device = -1;
};
SweepWorkspace g_sws;

#define SK(x)                                                                                   \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      if (std::getenv("SN_DEBUG")) std::fprintf(stderr, "sn_sweep: %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return SN_ERR_CUDA;                                                                      \
    }                                                                                          \
  } while (0)

struct HostWin {
  int64_t w0;
  int32_t k, chain, tau0, tau1, m, b0;
  int64_t level;
};

}  // namespace

// The window schedule of one sweep (host, a pure function of n, the shift count, w, m_max).
int sweep_plan(int64_t n, int64_t nshift, int64_t w, int64_t mmax, std::vector<HostWin>* out, int64_t* nlevels) {
  out->clear();
  const int64_t nb = nshift / 2;
  if (n < 3 || nb == 0) { *nlevels = 0; return 0; }
  for (int64_t c0 = 0; c0 < nb; c0 += mmax) {
    const int m = (int)std::min(mmax, nb - c0);
    const int64_t T = (n - 2) + 4 * (int64_t)(m - 1) + 1;    // chain steps: the last bulge leaves
    int64_t tau = 0, w0 = 0;
    while (tau < T) {
      const int64_t k = std::min(w, n - w0);
      int64_t tau1;
      if (w0 + k == n) tau1 = T;
      else tau1 = w0 + k - 3;                                 // lowest bulge: p = tau <= w0 + k - 4
      if (tau1 <= tau) return SN_ERR_UNSUPPORTED;
      HostWin hw;
      hw.w0 = w0; hw.k = (int32_t)k; hw.chain = (int32_t)(c0 / mmax);
      hw.tau0 = (int32_t)tau; hw.tau1 = (int32_t)tau1; hw.m = m; hw.b0 = (int32_t)c0; hw.level = 0;
      out->push_back(hw);
      tau = tau1;
      if (tau >= T) break;
      // the next window starts one column left of the highest bulge's next reflector
      const int64_t ptop = tau - 4 * (int64_t)(m - 1);
      if (ptop < 1) return SN_ERR_UNSUPPORTED;                // the chain does not fit the window
      w0 = ptop - 1;
    }
  }
  // levels: 1 + the highest level of earlier windows whose row range meets this one
  std::vector<int64_t> rowlev((size_t)n, -1);
  int64_t nl = 0;
  for (HostWin& hw : *out) {
    int64_t lv = 0;
    for (int64_t r = hw.w0; r < hw.w0 + hw.k; ++r) lv = std::max(lv, rowlev[(size_t)r] + 1);
    hw.level = lv;
    for (int64_t r = hw.w0; r < hw.w0 + hw.k; ++r) rowlev[(size_t)r] = lv;
    nl = std::max(nl, lv + 1);
  }
  *nlevels = nl;
  return 0;
}

int sweep_run(int64_t n, double* H, int64_t ldH, double* Q, int64_t ldQ, int64_t nshift, const double* sr,
              const double* si, const sn_sweep_opts& o, sn_sweep_stats* st, cudaStream_t sUser) {
  SweepWorkspace& ws = g_sws;
  const double t0 = now_ms();
  int dev = 0;
  SK(cudaGetDevice(&dev));
  if (ws.device != dev) {
    if (ws.device >= 0) {
      SK(cudaSetDevice(ws.device));
      for (SBuf* b : {&ws.wins, &ws.bw, &ws.pref, &ws.status, &ws.Z, &ws.zr, &ws.shifts, &ws.sub, &ws.bad}) {
        if (b->p) cudaFree(b->p);
        b->p = nullptr;
        b->cap = 0;
      }
      cudaStreamDestroy(ws.sB);
      cudaStreamDestroy(ws.sC);
      for (int i = 0; i < kZgenS; ++i) {
        cudaEventDestroy(ws.evW[i]); cudaEventDestroy(ws.evQ[i]);
        cudaEventDestroy(ws.evCrit[i]); cudaEventDestroy(ws.evRest[i]);
      }
      for (cudaEvent_t e : {ws.ev0, ws.ev1, ws.evIn, ws.evJoin}) cudaEventDestroy(e);
      SK(cudaSetDevice(dev));
    }
    int least = 0, greatest = 0;
    SK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    SK(cudaStreamCreateWithPriority(&ws.sB, cudaStreamNonBlocking, least));
    SK(cudaStreamCreateWithPriority(&ws.sC, cudaStreamNonBlocking, least));
    for (int i = 0; i < kZgenS; ++i) {
      SK(cudaEventCreateWithFlags(&ws.evW[i], cudaEventDisableTiming));
      SK(cudaEventCreateWithFlags(&ws.evQ[i], cudaEventDisableTiming));
      SK(cudaEventCreateWithFlags(&ws.evCrit[i], cudaEventDisableTiming));
      SK(cudaEventCreateWithFlags(&ws.evRest[i], cudaEventDisableTiming));
    }
    SK(cudaEventCreate(&ws.ev0));
    SK(cudaEventCreate(&ws.ev1));
    SK(cudaEventCreateWithFlags(&ws.evIn, cudaEventDisableTiming));
    SK(cudaEventCreateWithFlags(&ws.evJoin, cudaEventDisableTiming));
    ws.device = dev;
  }
  cudaStream_t sA = sUser;
  // H must be upper Hessenberg (exact zeros below the subdiagonal)
  SK(ws.sub.ensure((size_t)n + 8));
  SK(ws.bad.ensure(8));
  SK(cudaMemsetAsync(ws.bad.p, 0, 4, sA));
  launch_scan(H, ldH, n, 1, (uint8_t*)ws.sub.p, (int32_t*)ws.bad.p, sA);
  SK(cudaGetLastError());
  int32_t bad = 0;
  SK(cudaMemcpyAsync(&bad, ws.bad.p, 4, cudaMemcpyDeviceToHost, sA));
  SK(cudaStreamSynchronize(sA));
  if (bad) return -2;
  // plan
  std::vector<HostWin> hw;
  int64_t nlev = 0;
  const int64_t W = o.window, mmax = o.bulges_per_chain;
  if (int rc = sweep_plan(n, nshift, W, mmax, &hw, &nlev)) return rc;
  const int64_t nw = (int64_t)hw.size();
  if (st) {
    st->windows = nw;
    st->levels = nlev;
    st->chains = nshift / 2 > 0 ? (nshift / 2 + mmax - 1) / mmax : 0;
    st->bulges = nshift / 2;
  }
  if (nw == 0) return 0;
  std::vector<int64_t> sorted((size_t)nw);
  for (int64_t i = 0; i < nw; ++i) sorted[(size_t)i] = i;
  std::stable_sort(sorted.begin(), sorted.end(), [&](int64_t x, int64_t y) { return hw[x].level < hw[y].level; });
  std::vector<int64_t> lstart((size_t)nlev + 1, 0);
  for (int64_t i = 0; i < nw; ++i) lstart[(size_t)hw[sorted[i]].level + 1]++;
  for (int64_t l = 0; l < nlev; ++l) lstart[l + 1] += lstart[l];
  int64_t maxper = 0;
  for (int64_t l = 0; l < nlev; ++l) maxper = std::max(maxper, lstart[l + 1] - lstart[l]);
  constexpr int NT = 64;
  std::vector<WinDev> wd((size_t)nw);
  std::vector<BulgeDev> bd((size_t)nw);
  // lookahead (as the reordering): a left strip (rows of the window, 64 columns
  // right of it) or a right strip (64 rows above it, its columns) is critical if a window of
  // the next level covers both its rows and its columns -- a prefix of the left strips, a
  // suffix of the right strips.  The critical strips run on the critical stream before the
  // next level's window kernel, the others on stream C concurrently with it.
  const bool look = o.lookahead != 0;
  const bool allcrit = std::getenv("SN_SWEEP_ALLCRIT") != nullptr;   // debug: every strip critical
  constexpr int NK = 5;   // 0 L crit, 1 L rest, 2 R crit, 3 R rest, 4 Q
  std::vector<int32_t> pref;
  std::vector<int64_t> poff((size_t)nlev * NK);
  std::vector<int32_t> nstr((size_t)nlev * NK);
  double eqf = 0.0, fk[3] = {0, 0, 0};
  for (int64_t l = 0; l < nlev; ++l) {
    const int64_t a = lstart[l], b = lstart[l + 1];
    std::vector<int32_t> cl((size_t)(b - a), 0), cr((size_t)(b - a), 0);
    for (int64_t i = a; i < b; ++i) {
      const HostWin& h = hw[sorted[i]];
      const int64_t nL = (n - (h.w0 + h.k) + NT - 1) / NT, nR = (h.w0 + NT - 1) / NT;
      if (!look || allcrit) { cl[i - a] = (int32_t)nL; cr[i - a] = (int32_t)nR; continue; }
      if (l + 1 >= nlev) continue;
      for (int64_t j = lstart[l + 1]; j < lstart[l + 2]; ++j) {
        const HostWin& g = hw[sorted[j]];
        const int64_t ga = g.w0, gb = g.w0 + g.k;
        // left strips: rows [w0, w0+k) meet [ga, gb), columns >= w0+k up to gb
        if (ga < h.w0 + h.k && gb > h.w0 && gb > h.w0 + h.k)
          cl[i - a] = (int32_t)std::max<int64_t>(cl[i - a], std::min(nL, (gb - (h.w0 + h.k) + NT - 1) / NT));
        // right strips: columns [w0, w0+k) meet [ga, gb), rows from ga (64-strips) below w0
        if (ga < h.w0 + h.k && gb > h.w0 && ga < h.w0)
          cr[i - a] = (int32_t)std::max<int64_t>(cr[i - a], nR - ga / NT);
      }
    }
    // corner order: a right update over rows of an upper window's left strips needs those
    // strips done on its whole column range first (it mixes the columns of the lower window;
    // left-updating some of them before and some after would not commute).  So when a lower
    // window's critical right strips reach an upper window's rows, the upper window's left
    // strips over the lower window's columns become critical too (run before it on the
    // critical stream), as in the reordering's lookahead (sn_plan.cpp).
    if (look && !allcrit) {
      for (int64_t ib = a; ib < b; ++ib) {
        const HostWin& B = hw[sorted[ib]];
        if (cr[ib - a] <= 0) continue;
        const int64_t nRB = (B.w0 + NT - 1) / NT;
        const int64_t crow0 = (nRB - cr[ib - a]) * NT;         // first row of B's critical right strips
        for (int64_t ia = a; ia < b; ++ia) {
          const HostWin& A = hw[sorted[ia]];
          if (A.w0 + A.k > B.w0 || A.w0 + A.k <= crow0) continue;   // A above B, rows meet
          const int64_t nLA = (n - (A.w0 + A.k) + NT - 1) / NT;
          const int64_t need = std::min(nLA, (B.w0 + B.k - (A.w0 + A.k) + NT - 1) / NT);
          cl[ia - a] = (int32_t)std::max<int64_t>(cl[ia - a], need);
        }
      }
    }
    for (int kind = 0; kind < NK; ++kind) {
      poff[l * NK + kind] = (int64_t)pref.size();
      int32_t acc = 0;
      pref.push_back(0);
      for (int64_t i = a; i < b; ++i) {
        const HostWin& h = hw[sorted[i]];
        const int64_t nL = (n - (h.w0 + h.k) + NT - 1) / NT, nR = (h.w0 + NT - 1) / NT;
        int64_t cnt = 0;
        switch (kind) {
          case 0: cnt = cl[i - a]; break;
          case 1: cnt = nL - cl[i - a]; break;
          case 2: cnt = cr[i - a]; break;
          case 3: cnt = nR - cr[i - a]; break;
          default: cnt = Q ? (n + NT - 1) / NT : 0; break;
        }
        acc += (int32_t)cnt;
        pref.push_back(acc);
      }
      nstr[l * NK + kind] = acc;
    }
    for (int64_t i = a; i < b; ++i) {
      const HostWin& h = hw[sorted[i]];
      WinDev& d = wd[i];
      std::memset(&d, 0, sizeof(d));
      d.j1 = h.w0; d.k = h.k; d.slot = (int32_t)((l % kZgenS) * maxper + (i - a));
      d.order = sorted[i]; d.sidx = (int32_t)i;
      d.crit_l = cl[i - a]; d.crit_r = cr[i - a];
      BulgeDev& e = bd[i];
      e.tau0 = h.tau0; e.tau1 = h.tau1; e.m = h.m; e.b0 = h.b0;
      const double k2 = 2.0 * (double)h.k * (double)h.k;
      const double eL = (double)(n - h.w0 - h.k), eR = (double)h.w0, eQ = Q ? (double)n : 0.0;
      eqf += k2 * (eL + eR + eQ);
      fk[0] += k2 * eL; fk[1] += k2 * eR; fk[2] += k2 * eQ;
    }
  }
  SK(ws.wins.ensure(sizeof(WinDev) * nw));
  SK(ws.bw.ensure(sizeof(BulgeDev) * nw));
  SK(ws.pref.ensure(sizeof(int32_t) * pref.size()));
  SK(ws.status.ensure(sizeof(int32_t) * nw));
  SK(ws.Z.ensure(sizeof(double) * (size_t)kZslot * (size_t)(kZgenS * maxper)));
  SK(ws.zr.ensure(sizeof(int16_t) * (size_t)kZrange * (size_t)(kZgenS * maxper)));
  SK(ws.shifts.ensure(sizeof(double) * 2 * (size_t)std::max<int64_t>(nshift, 1)));
  SK(cudaMemcpyAsync(ws.wins.p, wd.data(), sizeof(WinDev) * nw, cudaMemcpyHostToDevice, sA));
  SK(cudaMemcpyAsync(ws.bw.p, bd.data(), sizeof(BulgeDev) * nw, cudaMemcpyHostToDevice, sA));
  SK(cudaMemcpyAsync(ws.pref.p, pref.data(), sizeof(int32_t) * pref.size(), cudaMemcpyHostToDevice, sA));
  SK(cudaMemsetAsync(ws.status.p, 0, sizeof(int32_t) * nw, sA));
  double* dsr = (double*)ws.shifts.p;
  double* dsi = dsr + nshift;
  SK(cudaMemcpyAsync(dsr, sr, sizeof(double) * nshift, cudaMemcpyHostToDevice, sA));
  SK(cudaMemcpyAsync(dsi, si, sizeof(double) * nshift, cudaMemcpyHostToDevice, sA));
  const int mt = W <= 64 ? 64 : (W <= 128 ? 128 : 256);
  double* dZ = (double*)ws.Z.p;
  PanelMaps mapH{}, mapQ{};
  panel_maps_init(&mapH, dZ, (int64_t)kZgenS * maxper, H, n, n, ldH);
  if (Q) panel_maps_init(&mapQ, dZ, (int64_t)kZgenS * maxper, Q, n, n, ldQ);
  const bool overlapQ = o.q_stream_overlap != 0 && Q != nullptr;
  cudaStream_t sQ = overlapQ ? ws.sB : sA;
  cudaStream_t sC = look ? ws.sC : sA;
  SK(cudaEventRecord(ws.ev0, sA));
  if (overlapQ) SK(cudaStreamWaitEvent(ws.sB, ws.ev0, 0));
  if (look) SK(cudaStreamWaitEvent(ws.sC, ws.ev0, 0));
  int64_t launches = 0;
  int rc = SN_OK;
  for (int64_t l = 0; l < nlev && rc == SN_OK; ++l) {
    const int64_t a = lstart[l], cnt = lstart[l + 1] - a;
    const int gen = (int)(l % kZgenS);
    // the Z slots of this generation are free once the level kZgenS earlier has finished with
    // them (its Q update and its remaining strips)
    if (overlapQ && l >= kZgenS) SK(cudaStreamWaitEvent(sA, ws.evQ[gen], 0));
    if (look && l >= kZgenS) SK(cudaStreamWaitEvent(sA, ws.evRest[gen], 0));
    if (look && l > 0 && std::getenv("SN_SWEEP_DBG_WAITW"))   // debug: no overlap of W(l) with rest(l-1)
      SK(cudaStreamWaitEvent(sA, ws.evRest[(l - 1) % kZgenS], 0));
    SweepArgs sa{};
    sa.wins = (const WinDev*)ws.wins.p + a; sa.bw = (const BulgeDev*)ws.bw.p + a; sa.nwin = (int32_t)cnt;
    sa.H = H; sa.ldH = ldH; sa.n = n; sa.Z = dZ; sa.zrange = (int16_t*)ws.zr.p; sa.status = (int32_t*)ws.status.p;
    sa.sr = dsr; sa.si = dsi;
    if (W <= kStageMax) {
      static bool attr[kMaxDevices] = {};
      const int d = device_slot();
      const size_t smem = sizeof(double) * (size_t)kStageLd * kStageMax;
      if (!attr[d]) {
        SK(cudaFuncSetAttribute(bulge_window_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[d] = true;
      }
      bulge_window_kernel<true><<<(unsigned)cnt, kSweepThreads, smem, sA>>>(sa);
    } else {
      bulge_window_kernel<false><<<(unsigned)cnt, kSweepThreads, 0, sA>>>(sa);
    }
    ++launches;
    SK(cudaGetLastError());
    if (overlapQ) SK(cudaEventRecord(ws.evW[gen], sA));
    PanelArgs pa{};
    pa.wins = (const WinDev*)ws.wins.p + a; pa.nwin = (int32_t)cnt; pa.base = (int32_t)a;
    pa.status = (const int32_t*)ws.status.p; pa.n = n; pa.Z = dZ; pa.zrange = (const int16_t*)ws.zr.p;
    pa.M = H; pa.ld = ldH; pa.maps = &mapH;
    pa.vec16 = (ldH % 2 == 0 && ((uintptr_t)H % 16) == 0) ? 1 : 0;
    // the previous level's remaining strips may overlap this level's strips
    if (look && l > 0) SK(cudaStreamWaitEvent(sA, ws.evRest[(l - 1) % kZgenS], 0));
    auto part = [&](int kind, int prt, int slot_kind, cudaStream_t s) {
      if (nstr[l * NK + slot_kind] <= 0) return;
      pa.prefix = (const int32_t*)ws.pref.p + poff[l * NK + slot_kind];
      pa.part = look ? prt : 0;
      launch_panel(kind, mt, pa, nstr[l * NK + slot_kind], s);
      ++launches;
    };
    part(0, 1, 0, sA);             // left, critical strips (all strips without lookahead)
    part(1, 1, 2, sA);             // right, critical strips
    SK(cudaGetLastError());
    if (look) {
      SK(cudaEventRecord(ws.evCrit[gen], sA));
      SK(cudaStreamWaitEvent(sC, ws.evCrit[gen], 0));
      part(0, 2, 1, sC);           // the remaining strips overlap the next window kernel
      part(1, 2, 3, sC);
      SK(cudaEventRecord(ws.evRest[gen], sC));
      SK(cudaGetLastError());
    }
    if (Q && nstr[l * NK + 4] > 0) {
      if (overlapQ) SK(cudaStreamWaitEvent(sQ, ws.evW[gen], 0));
      pa.M = Q; pa.ld = ldQ; pa.maps = &mapQ;
      pa.vec16 = (ldQ % 2 == 0 && ((uintptr_t)Q % 16) == 0) ? 1 : 0;
      pa.prefix = (const int32_t*)ws.pref.p + poff[l * NK + 4];
      pa.part = 0;
      launch_panel(2, mt, pa, nstr[l * NK + 4], sQ);
      ++launches;
      SK(cudaGetLastError());
      if (overlapQ) SK(cudaEventRecord(ws.evQ[gen], sQ));
    }
  }
  if (overlapQ) {
    SK(cudaEventRecord(ws.evJoin, sQ));
    SK(cudaStreamWaitEvent(sA, ws.evJoin, 0));
  }
  if (look) {
    SK(cudaEventRecord(ws.evJoin, sC));
    SK(cudaStreamWaitEvent(sA, ws.evJoin, 0));
  }
  SK(cudaEventRecord(ws.ev1, sA));
  SK(cudaStreamSynchronize(sA));
  if (st) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ws.ev0, ws.ev1);
    st->eq_flops = eqf;
    st->flops_left = fk[0];
    st->flops_right = fk[1];
    st->flops_q = fk[2];
    st->launches = launches;
    st->ms_device = ms;
    st->ms_total = now_ms() - t0;
  }
  return rc;
}

}  // namespace sn

extern "C" {

void sn_sweep_default_opts(sn_sweep_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->window = 160;            // staged in shared memory (measured: 0.80 s vs 2.07 s at w = 256, n = 40000)
  o->bulges_per_chain = 16;
  o->q_stream_overlap = 1;
  o->lookahead = 1;
}

int sn_qr_sweep(int64_t n, double* H, int64_t ldH, double* Q, int64_t ldQ, int64_t nshift, const double* sr,
                const double* si, const sn_sweep_opts* opts, sn_sweep_stats* stats, void* stream) {
  sn_sweep_opts o;
  if (opts) o = *opts; else sn_sweep_default_opts(&o);
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (n < 0) return -1;
  if (n > 0 && H == nullptr) return -2;
  if (n > 0 && ldH < n) return -3;
  if (Q != nullptr && ldQ < n) return -5;
  if (nshift < 0 || (nshift & 1)) return -6;
  if (nshift > 0 && (sr == nullptr || si == nullptr)) return -7;
  for (int64_t j = 0; j < nshift; j += 2) {
    const bool conj = si[j] != 0.0 || si[j + 1] != 0.0;
    if (conj && !(sr[j] == sr[j + 1] && si[j] == -si[j + 1])) return -8;   // reading B1
  }
  if (o.window < 16 || o.window > 256 || o.bulges_per_chain < 1 || o.bulges_per_chain > sn::kMaxChainBulges ||
      4 * (o.bulges_per_chain - 1) + 8 > o.window)
    return SN_ERR_UNSUPPORTED;
  if (n < 3 || nshift == 0) return 0;
  std::lock_guard<std::mutex> lock(sn::g_mu);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return SN_ERR_CUDA;
  }
  if (!sn::is_device_ptr(H)) return -2;
  if (Q && !sn::is_device_ptr(Q)) return -4;
  return sn::sweep_run(n, H, ldH, Q, ldQ, nshift, sr, si, o, stats, (cudaStream_t)stream);
}

int sn_sweep_schedule(int64_t n, int64_t nshift, int64_t window, int64_t bulges_per_chain, int64_t* nwin,
                      int64_t* nlevels, int64_t* w0, int64_t* k, int64_t* level, int64_t* chain, int64_t* tau0,
                      int64_t* tau1) {
  if (n < 0 || nshift < 0 || (nshift & 1)) return -1;
  if (!nwin || !nlevels) return -5;
  std::vector<sn::HostWin> hw;
  if (int rc = sn::sweep_plan(n, nshift, window, bulges_per_chain, &hw, nlevels)) return rc;
  *nwin = (int64_t)hw.size();
  if (w0)
    for (size_t t = 0; t < hw.size(); ++t) {
      w0[t] = hw[t].w0;
      if (k) k[t] = hw[t].k;
      if (level) level[t] = hw[t].level;
      if (chain) chain[t] = hw[t].chain;
      if (tau0) tau0[t] = hw[t].tau0;
      if (tau1) tau1[t] = hw[t].tau1;
    }
  return 0;
}

}  // extern "C"
