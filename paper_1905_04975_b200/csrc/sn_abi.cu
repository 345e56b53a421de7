// sn_abi.cu -- C ABI entry points and the level executor (product code).
//
// Execution: the plan's windows are grouped by DAG level.  For each level:
//   stream A:  window kernel (all windows of the level, one CTA each)  -> event W(s)
//              left-update kernel (row panels right of every window)
//              right-update kernel (column panels above every window)
//   stream B:  waits W(s); Q-update kernel (columns of Q of every window)  -> event Q(s)
// Windows of one level have disjoint diagonal ranges; the only conflicts inside a
// level are between a left update of an upper window and a right update of a lower window
// on the same off-diagonal rectangle; they commute mathematically and are serialised by
// stream order (left, then right).  The next level's window kernel follows the right update
// on stream A; the Q update of level s overlaps it on stream B.  Z slots are reused every
// kZgen levels after the Q update that read them has finished.  This replaces the paper's
// StarPU runtime with a static schedule known before the first launch.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing without a tool attached

#include "sn_device.cuh"
#include "sn_exec.h"
#include "sn_plan.h"
#include "sn_reorder.h"

namespace sn {
namespace {

constexpr int kZgen = 4;   // Z slot generations (levels in flight on stream B)

struct DevBuf {
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

struct Workspace {
  DevBuf wins, pool, prefix, status, kwork, ctl, recs, Z, zr, sub, bad;
  DevBuf hS, hQ;                   // device staging of host-buffer calls (kept between calls)
  std::vector<cudaEvent_t> prof;   // event pool for opts.profile
  cudaStream_t sB = nullptr, sC = nullptr, sU = nullptr;   // sU: host->device upload of Q
  cudaStream_t sH = nullptr;      // high priority: window tasks and the strips they wait for
  cudaStream_t sD = nullptr;      // device -> host copies of final columns (host-buffer calls)
  std::vector<cudaEvent_t> evPool;
  cudaEvent_t evIn = nullptr, evOut = nullptr;
  cudaEvent_t evQup = nullptr;
  cudaEvent_t evW[kZgen] = {}, evQ[kZgen] = {}, evCrit[kZgen] = {}, evRest[kZgen] = {};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evJoin = nullptr, evJoinC = nullptr;
  int device = -1;
};

Workspace g_ws;

}  // namespace

std::mutex g_mu;

double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

#define CK(x)                                                          \
  do {                                                                 \
    cudaError_t e_ = (x);                                              \
    if (e_ != cudaSuccess) {                                           \
      if (std::getenv("SN_DEBUG"))                                     \
        std::fprintf(stderr, "sn: %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return SN_ERR_CUDA;                                              \
    }                                                                  \
  } while (0)

int ensure_runtime(Workspace& ws) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (ws.device != dev) {
    if (ws.device >= 0) {
      // the buffers, streams and events belong to the previous device: release them there
      cudaSetDevice(ws.device);
      for (DevBuf* b : {&ws.wins, &ws.pool, &ws.prefix, &ws.status, &ws.kwork, &ws.ctl, &ws.recs, &ws.Z, &ws.zr,
                        &ws.sub, &ws.bad, &ws.hS, &ws.hQ}) {
        if (b->p) cudaFree(b->p);
        b->p = nullptr;
        b->cap = 0;
      }
      for (auto e : ws.prof) cudaEventDestroy(e);
      ws.prof.clear();
    }
    if (ws.sB) {
      cudaStreamDestroy(ws.sB);
      cudaStreamDestroy(ws.sC);
      cudaStreamDestroy(ws.sH);
      cudaStreamDestroy(ws.sU);
      cudaStreamDestroy(ws.sD);
      for (auto e : ws.evPool) cudaEventDestroy(e);
      ws.evPool.clear();
      cudaEventDestroy(ws.evIn); cudaEventDestroy(ws.evOut); cudaEventDestroy(ws.evQup);
      for (int i = 0; i < kZgen; ++i) {
        cudaEventDestroy(ws.evW[i]); cudaEventDestroy(ws.evQ[i]);
        cudaEventDestroy(ws.evCrit[i]); cudaEventDestroy(ws.evRest[i]);
      }
      cudaEventDestroy(ws.ev0); cudaEventDestroy(ws.ev1);
      cudaEventDestroy(ws.evJoin); cudaEventDestroy(ws.evJoinC);
    }
    if (ws.device >= 0) CK(cudaSetDevice(dev));
    // Priorities: the critical path (window kernel -> critical strips -> next window kernel)
    // runs on the highest-priority stream so that its CTAs are dispatched ahead of the queued
    // update strips of the other streams (lowest priority).
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CK(cudaStreamCreateWithPriority(&ws.sH, cudaStreamNonBlocking, greatest));
    CK(cudaStreamCreateWithPriority(&ws.sB, cudaStreamNonBlocking, least));
    CK(cudaStreamCreateWithPriority(&ws.sC, cudaStreamNonBlocking, least));
    CK(cudaEventCreateWithFlags(&ws.evIn, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ws.evOut, cudaEventDisableTiming));
    CK(cudaStreamCreateWithPriority(&ws.sD, cudaStreamNonBlocking, least));
    CK(cudaStreamCreateWithFlags(&ws.sU, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ws.evQup, cudaEventDisableTiming));
    for (int i = 0; i < kZgen; ++i) {
      CK(cudaEventCreateWithFlags(&ws.evW[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ws.evQ[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ws.evCrit[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ws.evRest[i], cudaEventDisableTiming));
    }
    CK(cudaEventCreate(&ws.ev0));
    CK(cudaEventCreate(&ws.ev1));
    CK(cudaEventCreateWithFlags(&ws.evJoin, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ws.evJoinC, cudaEventDisableTiming));
    ws.device = dev;
  }
  return 0;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// movers-first stable partition of a block range
static void partition(std::vector<uint8_t>& sz, std::vector<uint8_t>& sel, int64_t top, int64_t nb,
               const uint8_t* psz, const uint8_t* psel) {
  int64_t o = top;
  for (int64_t b = 0; b < nb; ++b)
    if (psel[b]) { sz[o] = psz[b]; sel[o] = 1; ++o; }
  for (int64_t b = 0; b < nb; ++b)
    if (!psel[b]) { sz[o] = psz[b]; sel[o] = 0; ++o; }
}


int structure_from_sub(int64_t n, const uint8_t* sub, const int32_t* select, int8_t* bmap, int8_t* selrow,
                       int64_t* m) {
  int64_t msel = 0;
  for (int64_t i = 0; i < n;) {
    if (sub[i]) {
      if (i + 2 < n && sub[i + 1]) return -2;   // two consecutive nonzero subdiagonal entries
      bmap[i] = 1; bmap[i + 1] = 2;
      const int8_t s = (select[i] != 0 || select[i + 1] != 0) ? 1 : 0;
      selrow[i] = selrow[i + 1] = s;
      msel += 2 * s;
      i += 2;
    } else {
      bmap[i] = 0;
      selrow[i] = select[i] != 0 ? 1 : 0;
      msel += selrow[i];
      i += 1;
    }
  }
  *m = msel;
  return 0;
}

void final_blocks(const Plan& P, const std::vector<int64_t>& sorted, bool aborted, const int32_t* status,
                  const WinRec* recs, int64_t n, const int8_t* bmap, const int8_t* selrow, std::vector<uint8_t>& fsz,
                  std::vector<uint8_t>& fsel, int64_t* executed_out, int64_t* swaps_out, int64_t sbt[4],
                  int64_t* rej_sorted) {
  const int64_t nw = (int64_t)P.wins.size();
  int64_t executed = nw, swaps = 0;
  if (rej_sorted) *rej_sorted = -1;
  if (!aborted) {
    fsz = P.final_sz; fsel = P.final_sel;
    for (const auto& w : P.wins) {
      swaps += w.nswap;
      for (int q = 0; q < 4; ++q) sbt[q] += w.swaps_by_type[q];
    }
  } else {
    fsz.clear(); fsel.clear();
    for (int64_t i = 0; i < n;) {
      const int s = bmap[i] == 1 ? 2 : 1;
      fsz.push_back((uint8_t)s); fsel.push_back((uint8_t)selrow[i]);
      i += s;
    }
    std::vector<int64_t> pos_of(nw);
    for (int64_t i = 0; i < nw; ++i) pos_of[sorted[i]] = i;
    executed = 0;
    for (int64_t t = 0; t < nw; ++t) {   // schedule order: windows of one level are disjoint
      const WindowPlan& w = P.wins[t];
      const int64_t si = pos_of[t];
      const int32_t stt = status[si];
      if (stt == kWinDone) {
        partition(fsz, fsel, w.top, w.nblk, P.pool.data() + w.pool, P.pool.data() + w.pool + w.nblk);
        swaps += w.nswap;
        for (int q = 0; q < 4; ++q) sbt[q] += w.swaps_by_type[q];
        ++executed;
      } else if (stt == kWinPartial) {
        // this window's own record: several windows of the rejecting level may be partial
        std::memcpy(fsz.data() + w.top, recs[si].sz, (size_t)w.nblk);
        std::memcpy(fsel.data() + w.top, recs[si].sel, (size_t)w.nblk);
        swaps += recs[si].done;
        ++executed;
        if (rej_sorted && *rej_sorted < 0) *rej_sorted = si;   // first in schedule order
      }
    }
  }
  *executed_out = executed;
  *swaps_out = swaps;
}

void write_blocks(const std::vector<uint8_t>& fsz, const std::vector<uint8_t>& fsel, int32_t* select,
                  int8_t* bmap_out) {
  int64_t r = 0;
  for (size_t b = 0; b < fsz.size(); ++b) {
    for (int q = 0; q < fsz[b]; ++q) {
      select[r + q] = fsel[b];
      if (bmap_out) bmap_out[r + q] = (int8_t)(fsz[b] == 1 ? 0 : 1 + q);
    }
    r += fsz[b];
  }
}

namespace {

// Host-buffer calls: the host copies of S and Q, filled column block by column block as the
// columns become final (columns left of every later window's first row are never touched
// again: later windows, their panels and their Q columns all lie at or right of their j1).
struct HostOut {
  double* S;
  int64_t ldS;
  double* Q;
  int64_t ldQ;
  int64_t copied;   // columns [0, copied) are on their way to the host
};

// q_ready (optional): an event after which Q holds its input (a host upload still in flight
// while the structure scan, the plan and the first levels' S updates run)
int run_on(const sn_opts& o, int64_t n, double* S, int64_t ldS, double* Q, int64_t ldQ, int32_t* select,
           int64_t* m, int8_t* bmap_out, sn_stats* st, cudaStream_t sA, cudaEvent_t q_ready, HostOut* ho);

// The call is ordered on the caller's stream: the work runs on the library's streams between
// an event recorded on it and a wait it gets at the end.
int run(const sn_opts& o, int64_t n, double* S, int64_t ldS, double* Q, int64_t ldQ, int32_t* select,
        int64_t* m, int8_t* bmap_out, sn_stats* st, cudaStream_t sUser, cudaEvent_t q_ready = nullptr,
        HostOut* ho = nullptr) {
  Workspace& ws = g_ws;
  if (int rc = ensure_runtime(ws)) return rc;
  CK(cudaEventRecord(ws.evIn, sUser));
  CK(cudaStreamWaitEvent(ws.sH, ws.evIn, 0));
  const int rc = run_on(o, n, S, ldS, Q, ldQ, select, m, bmap_out, st, ws.sH, q_ready, ho);
  // join the library's other streams on every exit path (an error return may leave Q updates
  // or remaining strips queued on them): the caller's stream then waits for all of it
  cudaEventRecord(ws.evJoin, ws.sB);
  cudaStreamWaitEvent(ws.sH, ws.evJoin, 0);
  cudaEventRecord(ws.evJoinC, ws.sC);
  cudaStreamWaitEvent(ws.sH, ws.evJoinC, 0);
  cudaEventRecord(ws.evOut, ws.sH);
  cudaStreamWaitEvent(sUser, ws.evOut, 0);
  return rc;
}

int run_on(const sn_opts& o, int64_t n, double* S, int64_t ldS, double* Q, int64_t ldQ, int32_t* select,
           int64_t* m, int8_t* bmap_out, sn_stats* st, cudaStream_t sA, cudaEvent_t q_ready, HostOut* ho) {
  Workspace& ws = g_ws;
  const double t_start = now_ms();
  int64_t launches[5] = {0, 0, 0, 0, 0};
  std::vector<std::pair<int, int>> prof_marks;   // (kind, first event index)
  std::vector<std::pair<int64_t, int>> prof_lev;   // per mark: (level, stream: 0 critical, 1 rest, 2 Q)
  int64_t cur_level = -1;
  size_t prof_used = 0;
  auto prof_begin = [&](int kind, cudaStream_t s) -> int {
    if (!o.profile) return -1;
    while (ws.prof.size() < prof_used + 2) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return -1;
      ws.prof.push_back(e);
    }
    const int idx = (int)prof_used;
    prof_used += 2;
    cudaEventRecord(ws.prof[idx], s);
    prof_marks.push_back({kind, idx});
    prof_lev.push_back({cur_level, s == ws.sC ? 1 : (s == ws.sB ? 2 : 0)});
    return idx;
  };
  auto prof_end = [&](int idx, cudaStream_t s) {
    if (idx >= 0) cudaEventRecord(ws.prof[idx + 1], s);
  };

  // ---- a1: structure scan on the device, block map and selection on the host
  CK(ws.sub.ensure((size_t)n + 8));
  CK(ws.bad.ensure(8));
  CK(cudaMemsetAsync(ws.bad.p, 0, 4, sA));
  {
    const int pe = prof_begin(4, sA);
    launch_scan(S, ldS, n, o.validate_lower, (uint8_t*)ws.sub.p, (int32_t*)ws.bad.p, sA);
    prof_end(pe, sA);
    launches[4] += (o.validate_lower && n > 2) ? 2 : 1;
  }
  CK(cudaGetLastError());
  std::vector<uint8_t> sub((size_t)n);
  int32_t bad = 0;
  CK(cudaMemcpyAsync(sub.data(), ws.sub.p, (size_t)n, cudaMemcpyDeviceToHost, sA));
  CK(cudaMemcpyAsync(&bad, ws.bad.p, 4, cudaMemcpyDeviceToHost, sA));
  CK(cudaStreamSynchronize(sA));
  if (bad) return -2;
  std::vector<int8_t> bmap((size_t)n), selrow((size_t)n);
  if (int rc = structure_from_sub(n, sub.data(), select, bmap.data(), selrow.data(), m)) return rc;

  // ---- a2: plan (window schedule, inner schedules, DAG levels)
  Plan P;
  int prc = build_plan(n, bmap.data(), selrow.data(), o.window, o.inner_window, o.max_windows, &P);
  if (prc) return SN_ERR_UNSUPPORTED;
  const int64_t nw = (int64_t)P.wins.size();
  std::vector<int64_t> sorted(nw);
  for (int64_t i = 0; i < nw; ++i) sorted[i] = i;
  std::stable_sort(sorted.begin(), sorted.end(),
                   [&](int64_t x, int64_t y) { return P.wins[x].level < P.wins[y].level; });
  std::vector<int64_t> lstart(P.nlevels + 1, 0);
  for (int64_t i = 0; i < nw; ++i) lstart[P.wins[sorted[i]].level + 1]++;
  for (int64_t l = 0; l < P.nlevels; ++l) lstart[l + 1] += lstart[l];
  int64_t maxper = 0;
  for (int64_t l = 0; l < P.nlevels; ++l) maxper = std::max(maxper, lstart[l + 1] - lstart[l]);
  const int NT = 64;
  constexpr int NK = 5;                // per level: 0 L-crit, 1 L-rest, 2 R-crit, 3 R-rest, 4 Q
  std::vector<WinDev> wd(nw);
  std::vector<int32_t> pref;           // per level and kind: prefix over the level's windows
  std::vector<int64_t> pref_off(P.nlevels * NK);
  std::vector<int32_t> nstrips(P.nlevels * NK);
  const bool look = o.lookahead != 0;
  std::vector<int32_t> critL(nw, 0), critR(nw, 0);
  if (look) {
    std::vector<int32_t> cl, cr;
    lookahead_strips(P, NT, cl, cr);          // schedule order -> level-sorted order
    for (int64_t i = 0; i < nw; ++i) { critL[i] = cl[sorted[i]]; critR[i] = cr[sorted[i]]; }
  }
  // Row f1, fused chain updates (opts.fuse_chain): the Q update of a window x moves to the
  // level of its chain successor y (next in schedule order, one level later, above x and
  // overlapping it), whose Q launch applies Zx then Zy to each Q strip in one CTA pass.  No
  // other window of y's level may touch x's columns; pairs are disjoint (a y is never an x).
  std::vector<int32_t> qprev(nw, 0);    // level-sorted: 1 + level-sorted index of the predecessor
  std::vector<uint8_t> qdefer(nw, 0);   // level-sorted: Q update applied by the successor's launch
  const bool fuseQ = o.fuse_chain != 0 && Q != nullptr && ((uintptr_t)Q % 16) == 0 && (ldQ % 2) == 0;
  int64_t fused_pairs = 0;
  if (fuseQ) {
    std::vector<int64_t> pos_of(nw);
    for (int64_t i = 0; i < nw; ++i) pos_of[sorted[i]] = i;
    std::vector<uint8_t> isy(nw, 0);   // schedule order
    for (int64_t t = 0; t + 1 < nw; ++t) {
      if (isy[t]) continue;
      const WindowPlan& x = P.wins[t];
      const WindowPlan& y = P.wins[t + 1];
      if (y.level != x.level + 1 || y.j1 >= x.j1 || y.j1 + y.k <= x.j1) continue;
      bool ok = true;
      for (int64_t i = lstart[y.level]; i < lstart[y.level + 1] && ok; ++i) {
        const WindowPlan& w = P.wins[sorted[i]];
        if (sorted[i] != t + 1 && w.j1 < x.j1 + x.k && w.j1 + w.k > x.j1) ok = false;
      }
      if (!ok) continue;
      isy[t + 1] = 1;
      qprev[pos_of[t + 1]] = (int32_t)(pos_of[t] + 1);
      qdefer[pos_of[t]] = 1;
      ++fused_pairs;
    }
  }
  for (int64_t l = 0; l < P.nlevels; ++l) {
    const int64_t a = lstart[l], b = lstart[l + 1];
    for (int kind = 0; kind < NK; ++kind) {
      pref_off[l * NK + kind] = (int64_t)pref.size();
      int32_t acc = 0;
      pref.push_back(0);
      for (int64_t i = a; i < b; ++i) {
        const WindowPlan& w = P.wins[sorted[i]];
        const int64_t nL = (n - (w.j1 + w.k) + NT - 1) / NT, nR = (w.j1 + NT - 1) / NT;
        int64_t cnt = 0;
        switch (kind) {
          case 0: cnt = look ? critL[i] : nL; break;
          case 1: cnt = look ? nL - critL[i] : 0; break;
          case 2: cnt = look ? critR[i] : nR; break;
          case 3: cnt = look ? nR - critR[i] : 0; break;
          default: cnt = (Q && !qdefer[i]) ? (n + NT - 1) / NT : 0; break;
        }
        acc += (int32_t)cnt;
        pref.push_back(acc);
      }
      nstrips[l * NK + kind] = acc;
    }
    for (int64_t i = a; i < b; ++i) {
      const WindowPlan& w = P.wins[sorted[i]];
      WinDev& d = wd[i];
      d.j1 = w.j1; d.k = w.k; d.nblk = w.nblk; d.ninner = w.ninner;
      d.slot = (int32_t)((l % kZgen) * maxper + (i - a));
      d.pool = w.pool; d.order = w.order;
      d.crit_l = critL[i]; d.crit_r = critR[i];
      d.coff = 0; d.sidx = (int32_t)i; d.qprev = qprev[i];
    }
  }
  const double t_plan = now_ms();

  if (nw == 0) {
    if (q_ready) CK(cudaStreamWaitEvent(sA, q_ready, 0));
    if (bmap_out) std::memcpy(bmap_out, bmap.data(), (size_t)n);
    if (st) {
      std::memset(st, 0, sizeof(*st));
      st->rejected_window = -1; st->rejected_row = -1;
      st->ms_schedule = t_plan - t_start;
      st->ms_total = now_ms() - t_start;
      st->launches[4] = launches[4];
    }
    // selection output: achieved mask = input mask normalised per block
    for (int64_t i = 0; i < n; ++i) select[i] = selrow[i];
    return 0;
  }

  // ---- uploads
  CK(ws.wins.ensure(sizeof(WinDev) * nw));
  CK(ws.pool.ensure(P.pool.size() + 8));
  CK(ws.prefix.ensure(sizeof(int32_t) * pref.size()));
  CK(ws.status.ensure(sizeof(int32_t) * nw));
  CK(ws.kwork.ensure(sizeof(int32_t) * nw));
  CK(ws.ctl.ensure(sizeof(Control)));
  CK(ws.recs.ensure(sizeof(WinRec) * nw));
  CK(ws.Z.ensure(sizeof(double) * (size_t)kZslot * (size_t)(kZgen * maxper)));
  CK(ws.zr.ensure(sizeof(int16_t) * (size_t)kZrange * (size_t)(kZgen * maxper)));
  CK(cudaMemcpyAsync(ws.wins.p, wd.data(), sizeof(WinDev) * nw, cudaMemcpyHostToDevice, sA));
  CK(cudaMemcpyAsync(ws.pool.p, P.pool.data(), P.pool.size(), cudaMemcpyHostToDevice, sA));
  CK(cudaMemcpyAsync(ws.prefix.p, pref.data(), sizeof(int32_t) * pref.size(), cudaMemcpyHostToDevice, sA));
  CK(cudaMemsetAsync(ws.status.p, 0, sizeof(int32_t) * nw, sA));
  CK(cudaMemsetAsync(ws.ctl.p, 0, sizeof(Control), sA));
  CK(cudaMemsetAsync(ws.recs.p, 0, sizeof(WinRec) * nw, sA));

  const int mt = o.window <= 64 ? 64 : (o.window <= 128 ? 128 : 256);
  WinDev* dw = (WinDev*)ws.wins.p;
  int32_t* dstatus = (int32_t*)ws.status.p;
  int32_t* dpref = (int32_t*)ws.prefix.p;
  Control* dctl = (Control*)ws.ctl.p;
  double* dZ = (double*)ws.Z.p;
  const bool overlapQ = o.q_stream_overlap != 0 && Q != nullptr;
  cudaStream_t sQ = overlapQ ? ws.sB : sA;

  // TMA descriptors of S and Q (the cp.async kernels are used if TMA cannot describe them)
  PanelMaps mapS{}, mapQ{};
  panel_maps_init(&mapS, dZ, (int64_t)kZgen * maxper, S, n, n, ldS);
  if (Q) panel_maps_init(&mapQ, dZ, (int64_t)kZgen * maxper, Q, n, n, ldQ);
  if (fuseQ && !mapQ.valid) return SN_ERR_UNSUPPORTED;   // fused passes: TMA kernel only
  unsigned long long* dtp = nullptr;   // SN_WPROF: window-kernel phase cycles (debug)
  if (std::getenv("SN_WPROF")) {
    CK(cudaMalloc(&dtp, 16 * sizeof(unsigned long long)));
    CK(cudaMemsetAsync(dtp, 0, 16 * sizeof(unsigned long long), sA));
  }
  // final-column frontier after each level: the smallest first row of any later window
  std::vector<int64_t> frontier(P.nlevels, n);
  for (int64_t l = P.nlevels - 2; l >= 0; --l) {
    int64_t mn = frontier[l + 1];
    for (int64_t i = lstart[l + 1]; i < lstart[l + 2]; ++i) mn = std::min(mn, P.wins[sorted[i]].j1);
    frontier[l] = mn;
  }
  size_t evUsed = 0;
  auto next_event = [&]() -> cudaEvent_t {
    if (evUsed == ws.evPool.size()) {
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
      ws.evPool.push_back(e);
    }
    return ws.evPool[evUsed++];
  };
  CK(cudaEventRecord(ws.ev0, sA));
  if (overlapQ) {
    CK(cudaStreamWaitEvent(ws.sB, ws.ev0, 0));
  }
  cudaStream_t sC = look ? ws.sC : sA;
  if (look) CK(cudaStreamWaitEvent(ws.sC, ws.ev0, 0));
  for (int64_t l = 0; l < P.nlevels; ++l) {
    const int64_t a = lstart[l], cnt = lstart[l + 1] - a;
    const int gen = (int)(l % kZgen);
    cur_level = l;
    nvtxRangePushA("sn level");
    // Z slots of generation gen are rewritten: the Q launch that last read them must be done
    // (with fused Q updates that is the launch of the level after their own)
    if (overlapQ && !fuseQ && l >= kZgen) CK(cudaStreamWaitEvent(sA, ws.evQ[gen], 0));
    if (overlapQ && fuseQ && l >= kZgen) CK(cudaStreamWaitEvent(sA, ws.evQ[(l + 1) % kZgen], 0));
    WindowArgs wa{};
    wa.wins = dw + a; wa.nwin = (int32_t)cnt; wa.base = (int32_t)a;
    wa.pool = (const uint8_t*)ws.pool.p; wa.S = S; wa.ldS = ldS; wa.Z = dZ;
    wa.status = dstatus; wa.ctl = dctl; wa.zrange = (int16_t*)ws.zr.p; wa.kwork = (int32_t*)ws.kwork.p;
    wa.recs = (WinRec*)ws.recs.p; wa.level = (int32_t)l;
    wa.tprof = dtp;
    wa.force_order = o.force_reject_window; wa.force_swap = (int32_t)o.force_reject_swap;
    int pe = prof_begin(0, sA);
    launch_window(wa, sA);
    prof_end(pe, sA);
    launches[0]++;
    CK(cudaGetLastError());
    if (overlapQ) CK(cudaEventRecord(ws.evW[gen], sA));
    PanelArgs pa{};
    pa.strips = nullptr;
    pa.wins = dw + a; pa.nwin = (int32_t)cnt; pa.base = (int32_t)a; pa.status = dstatus;
    pa.n = n; pa.Z = dZ; pa.zrange = (const int16_t*)ws.zr.p;
    pa.M = S; pa.ld = ldS; pa.maps = &mapS;
    pa.vec16 = (ldS % 2 == 0 && ((uintptr_t)S % 16) == 0) ? 1 : 0;
    // the strips of the previous level's rest may overlap this level's strips
    if (look && l > 0) CK(cudaStreamWaitEvent(sA, ws.evRest[(l - 1) % kZgen], 0));
    auto launch_part = [&](int kind, int part, int slot_kind, cudaStream_t s) -> int {
      if (nstrips[l * NK + slot_kind] <= 0) return 0;
      pa.prefix = dpref + pref_off[l * NK + slot_kind];
      pa.part = look ? part : 0;
      const int p2 = prof_begin(1 + kind, s);
      launch_panel(kind, mt, pa, nstrips[l * NK + slot_kind], s);
      prof_end(p2, s);
      launches[1 + kind]++;
      return 0;
    };
    launch_part(0, 1, 0, sA);      // left, critical strips (all strips without lookahead)
    launch_part(1, 1, 2, sA);      // right, critical strips
    CK(cudaGetLastError());
    if (look) {
      CK(cudaEventRecord(ws.evCrit[gen], sA));
      CK(cudaStreamWaitEvent(sC, ws.evCrit[gen], 0));
      launch_part(0, 2, 1, sC);    // left, remaining strips: overlap the next window kernel
      launch_part(1, 2, 3, sC);
      CK(cudaEventRecord(ws.evRest[gen], sC));
      CK(cudaGetLastError());
    }
    if (Q) {
      if (l == 0 && q_ready) CK(cudaStreamWaitEvent(sQ, q_ready, 0));
      if (overlapQ) CK(cudaStreamWaitEvent(sQ, ws.evW[gen], 0));
      pa.M = Q; pa.ld = ldQ; pa.maps = &mapQ;
      pa.vec16 = (ldQ % 2 == 0 && ((uintptr_t)Q % 16) == 0) ? 1 : 0;
      pa.prefix = dpref + pref_off[l * NK + 4];
      pa.part = 0;
      pa.fuse = fuseQ ? 1 : 0;
      pe = prof_begin(3, sQ);
      launch_panel(2, mt, pa, nstrips[l * NK + 4], sQ);
      prof_end(pe, sQ);
      launches[3]++;
      CK(cudaGetLastError());
      if (overlapQ) CK(cudaEventRecord(ws.evQ[gen], sQ));
    }
    if (o.serialize) {
      CK(cudaStreamSynchronize(sA));
      if (overlapQ) CK(cudaStreamSynchronize(sQ));
      if (look) CK(cudaStreamSynchronize(sC));
    }
    // host-buffer call: columns [copied, frontier) are final once this level's work is done
    if (ho && frontier[l] - ho->copied >= 2048 && l + 1 < P.nlevels) {
      cudaEvent_t ea = next_event();
      if (!ea) return SN_ERR_CUDA;
      CK(cudaEventRecord(ea, sA));
      CK(cudaStreamWaitEvent(ws.sD, ea, 0));
      if (overlapQ) CK(cudaStreamWaitEvent(ws.sD, ws.evQ[gen], 0));
      if (look) CK(cudaStreamWaitEvent(ws.sD, ws.evRest[gen], 0));
      const int64_t c0 = ho->copied, nc = frontier[l] - c0;
      CK(cudaMemcpy2DAsync(ho->S + c0 * ho->ldS, ho->ldS * 8, S + c0 * ldS, ldS * 8, n * 8, nc,
                           cudaMemcpyDeviceToHost, ws.sD));
      if (Q && ho->Q)
        CK(cudaMemcpy2DAsync(ho->Q + c0 * ho->ldQ, ho->ldQ * 8, Q + c0 * ldQ, ldQ * 8, n * 8, nc,
                             cudaMemcpyDeviceToHost, ws.sD));
      ho->copied = frontier[l];
    }
    nvtxRangePop();
  }
  if (overlapQ) {
    CK(cudaEventRecord(ws.evJoin, sQ));
    CK(cudaStreamWaitEvent(sA, ws.evJoin, 0));
  }
  if (look) {
    CK(cudaEventRecord(ws.evJoinC, sC));
    CK(cudaStreamWaitEvent(sA, ws.evJoinC, 0));
  }
  CK(cudaEventRecord(ws.ev1, sA));
  Control ctl;
  CK(cudaMemcpyAsync(&ctl, dctl, sizeof(Control), cudaMemcpyDeviceToHost, sA));
  CK(cudaStreamSynchronize(sA));
  float dev_ms = 0.f;
  CK(cudaEventElapsedTime(&dev_ms, ws.ev0, ws.ev1));
  if (dtp) {
    unsigned long long h[16];
    CK(cudaMemcpy(h, dtp, sizeof(h), cudaMemcpyDeviceToHost));
    cudaFree(dtp);
    const double nwin = (double)(h[9] ? h[9] : 1);
    std::fprintf(stderr,
                 "{\"probe\":\"window_phases\",\"assembly_max\":%.0f,\"transform_max\":%.0f,\"windows\":%llu,\"steps_per_window\":%.1f,\"cycles_per_window\":"
                 "{\"A\":%.0f,\"B\":%.0f,\"C\":%.0f,\"wave_setup\":%.0f,\"staging\":%.0f,\"inner_updates\":%.0f,"
                 "\"total\":%.0f,\"B_work_avg_warp\":%.0f,\"B_work_max_warp\":%.0f,\"A_transform_max\":%.0f}}\n",
                 h[13] / nwin, h[14] / nwin, h[9], h[4] / nwin, h[0] / nwin, h[1] / nwin, h[2] / nwin, h[5] / nwin, h[6] / nwin, h[7] / nwin,
                 h[8] / nwin, h[10] / nwin / 8.0, h[11] / nwin, h[12] / nwin);
  }

  // ---- outputs: final block list
  std::vector<uint8_t> fsz, fsel;
  std::vector<int32_t> status;
  std::vector<WinRec> recs;
  int64_t executed = nw, swaps = 0, rej = -1;
  double eqf = 0.0;
  int64_t sbt[4] = {0, 0, 0, 0};
  if (ctl.abort) {
    status.resize(nw);
    recs.resize(nw);
    CK(cudaMemcpy(status.data(), dstatus, sizeof(int32_t) * nw, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(recs.data(), ws.recs.p, sizeof(WinRec) * nw, cudaMemcpyDeviceToHost));
  }
  final_blocks(P, sorted, ctl.abort != 0, ctl.abort ? status.data() : nullptr, recs.data(), n, bmap.data(),
               selrow.data(), fsz, fsel, &executed, &swaps, sbt, &rej);
  double fk[5] = {0, 0, 0, 0, 0}, bk[5] = {0, 0, 0, 0, 0}, fx[5] = {0, 0, 0, 0, 0};
  std::vector<int32_t> kwork(nw, 0);
  CK(cudaMemcpy(kwork.data(), ws.kwork.p, sizeof(int32_t) * nw, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < nw; ++i) {
    const WindowPlan& w = P.wins[sorted[i]];
    if (ctl.abort && status[i] == kWinSkipped) continue;
    const double kd = (double)w.k, k2 = 2.0 * kd * kd;
    const double eL = (double)(n - w.j1 - w.k), eR = (double)w.j1, eQ = Q ? (double)n : 0.0;
    eqf += k2 * (eL + eR + eQ);
    fk[1] += k2 * eL; fk[2] += k2 * eR; fk[3] += k2 * eQ;
    const double kx = 256.0 * (double)kwork[i];   // executed flops per panel column / row
    fx[1] += kx * eL; fx[2] += kx * eR; fx[3] += kx * eQ;
    bk[1] += 16.0 * kd * eL; bk[2] += 16.0 * kd * eR; bk[3] += 16.0 * kd * eQ;
    bk[0] += 16.0 * kd * kd + 8.0 * kZslot;
  }
  bk[4] = 8.0 * (double)n + (o.validate_lower ? 4.0 * (double)n * (double)n : 0.0);
  double mk[5] = {0, 0, 0, 0, 0};
  for (auto& pm : prof_marks) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ws.prof[pm.second], ws.prof[pm.second + 1]) == cudaSuccess) mk[pm.first] += ms;
  }
  // SN_TIMELINE=path (with opts.profile): every launch's start and end on its stream, from the
  // CUDA events around it, relative to the start of the run -- the overlap evidence of the
  // level executor (no nsys in this image)
  if (const char* tl = std::getenv("SN_TIMELINE")) {
    if (FILE* f = std::fopen(tl, "w")) {
      std::fprintf(f, "kind,level,stream,start_ms,end_ms\n");
      for (size_t q = 0; q < prof_marks.size(); ++q) {
        float a0 = 0.f, a1 = 0.f;
        cudaEventElapsedTime(&a0, ws.ev0, ws.prof[prof_marks[q].second]);
        cudaEventElapsedTime(&a1, ws.ev0, ws.prof[prof_marks[q].second + 1]);
        std::fprintf(f, "%d,%lld,%d,%.4f,%.4f\n", prof_marks[q].first, (long long)prof_lev[q].first, prof_lev[q].second, a0, a1);
      }
      std::fclose(f);
    }
  }
  write_blocks(fsz, fsel, select, bmap_out);
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->windows = executed;
    st->levels = P.nlevels;
    st->swaps = swaps;
    for (int q = 0; q < 4; ++q) st->swaps_by_type[q] = sbt[q];
    st->inner_windows = P.ninner;
    st->rejected_window = -1;
    st->rejected_row = -1;
    if (ctl.abort && rej >= 0) {
      st->rejected_window = P.wins[sorted[rej]].order;
      st->rejected_row = recs[rej].row;
      st->rejected_n1 = recs[rej].n1;
      st->rejected_n2 = recs[rej].n2;
    }
    st->eq_flops = eqf;
    st->ms_schedule = t_plan - t_start;
    st->ms_device = dev_ms;
    st->ms_total = now_ms() - t_start;
    for (int q = 0; q < 5; ++q) {
      st->launches[q] = launches[q];
      st->ms_kernel[q] = mk[q];
      st->flops_kernel[q] = fk[q];
      st->bytes_kernel[q] = bk[q];
      st->flops_exec_kernel[q] = fx[q];
    }
    st->fused_q_pairs = fused_pairs;
  }
  return ctl.abort ? SN_ERR_REJECTED : SN_OK;
}

}  // namespace
}  // namespace sn

extern "C" {

void sn_default_opts(sn_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->window = 256;
  o->inner_window = 64;
  o->max_windows = -1;
  o->force_reject_window = -1;
  o->force_reject_swap = -1;
  o->validate_lower = 0;
  o->serialize = 0;
  o->q_stream_overlap = 1;
  o->profile = 0;
  o->lookahead = 1;
}

const char* sn_strerror(int code) {
  switch (code) {
    case SN_OK: return "success";
    case SN_ERR_REJECTED: return "a block swap was rejected by the stability test; S and Q hold a valid, partially reordered Schur form";
    case SN_ERR_CUDA: return "CUDA error (no usable device, out of memory, or a kernel failure)";
    case SN_ERR_UNSUPPORTED: return "unsupported option value";
    default: break;
  }
  if (code < 0) return "invalid argument (-i: argument i of sn_reorder_schur)";
  return "unknown error";
}

const char* sn_version(void) { return "sn_b200 0.1 (sm_100a)"; }

void sn_release_workspace(void) {
  std::lock_guard<std::mutex> lock(sn::g_mu);
  sn::Workspace& ws = sn::g_ws;
  for (sn::DevBuf* b : {&ws.wins, &ws.pool, &ws.prefix, &ws.status, &ws.kwork, &ws.ctl, &ws.recs, &ws.Z, &ws.zr, &ws.sub,
                        &ws.bad, &ws.hS, &ws.hQ}) {
    if (b->p) cudaFree(b->p);
    b->p = nullptr;
    b->cap = 0;
  }
}

int sn_reorder_schur_ex(const sn_opts* opts, int64_t n, double* S, int64_t ldS, double* Q, int64_t ldQ,
                        int32_t* select, int64_t* m, int8_t* bmap_out, sn_stats* stats, void* stream) {
  sn_opts o;
  if (opts) o = *opts; else sn_default_opts(&o);
  if (m == nullptr) return -7;
  *m = 0;
  if (n < 0) return -1;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->rejected_window = -1;
    stats->rejected_row = -1;
  }
  if (n == 0) return 0;
  if (S == nullptr) return -2;
  if (ldS < n) return -3;
  if (Q != nullptr && ldQ < n) return -5;
  if (select == nullptr) return -6;
  if (o.window < 4 || o.window > 256 || o.inner_window < 4 || o.inner_window > 64) return SN_ERR_UNSUPPORTED;
  std::lock_guard<std::mutex> lock(sn::g_mu);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return SN_ERR_CUDA;
  }
  cudaStream_t sA = (cudaStream_t)stream;
  const bool devS = sn::is_device_ptr(S);
  const bool devQ = Q == nullptr || sn::is_device_ptr(Q);
  if (devS != devQ) return -4;
  if (devS) return sn::run(o, n, S, ldS, Q, ldQ, select, m, bmap_out, stats, sA);
  // host buffers: stage through device memory (the copies are part of the call).  S goes up
  // first (the scan and the plan need it); Q goes up on its own stream while the structure
  // scan, the plan and the first levels' S work run -- the Q updates wait for it.
  const double t0 = sn::now_ms();
  if (int rc = sn::ensure_runtime(sn::g_ws)) return rc;
  const size_t bytes = sizeof(double) * (size_t)n * (size_t)n;
  if (sn::g_ws.hS.ensure(bytes) != cudaSuccess) return SN_ERR_CUDA;
  if (Q && sn::g_ws.hQ.ensure(bytes) != cudaSuccess) return SN_ERR_CUDA;
  double* dS = (double*)sn::g_ws.hS.p;
  double* dQ = Q ? (double*)sn::g_ws.hQ.p : nullptr;
  auto copy = [&](double* dst, int64_t ldd, const double* src, int64_t lds, cudaMemcpyKind kind, cudaStream_t s) {
    if (ldd == n && lds == n) return cudaMemcpyAsync(dst, src, bytes, kind, s);   // one contiguous copy
    return cudaMemcpy2DAsync(dst, ldd * 8, src, lds * 8, n * 8, n, kind, s);
  };
  cudaStream_t sU = sn::g_ws.sU;
  int rc = SN_OK;
  if (copy(dS, n, S, ldS, cudaMemcpyHostToDevice, sA) != cudaSuccess) rc = SN_ERR_CUDA;
  if (rc == SN_OK && Q &&
      (copy(dQ, n, Q, ldQ, cudaMemcpyHostToDevice, sU) != cudaSuccess ||
       cudaEventRecord(sn::g_ws.evQup, sU) != cudaSuccess))
    rc = SN_ERR_CUDA;
  const double t1 = sn::now_ms();
  sn::HostOut ho{S, ldS, Q, ldQ, 0};
  if (rc == SN_OK)
    rc = sn::run(o, n, dS, n, dQ, n, select, m, bmap_out, stats, sA, Q ? sn::g_ws.evQup : nullptr, &ho);
  if (Q) cudaStreamSynchronize(sU);
  const double t2 = sn::now_ms();
  if (rc == SN_OK || rc == SN_ERR_REJECTED) {
    // the columns not streamed out during the run
    const int64_t c0 = ho.copied, nc = n - c0;
    if (nc > 0 &&
        (cudaMemcpy2DAsync(S + c0 * ldS, ldS * 8, dS + c0 * n, n * 8, n * 8, nc, cudaMemcpyDeviceToHost, sA) != cudaSuccess ||
         (Q && cudaMemcpy2DAsync(Q + c0 * ldQ, ldQ * 8, dQ + c0 * n, n * 8, n * 8, nc, cudaMemcpyDeviceToHost, sA) != cudaSuccess)))
      rc = SN_ERR_CUDA;
    if (cudaStreamSynchronize(sA) != cudaSuccess) rc = SN_ERR_CUDA;
  }
  if (cudaStreamSynchronize(sn::g_ws.sD) != cudaSuccess) rc = SN_ERR_CUDA;
  const double t3 = sn::now_ms();
  if (stats) {
    stats->ms_h2d = t1 - t0;     // issue time of the uploads (they overlap the run)
    stats->ms_d2h = t3 - t2;
    stats->ms_total = t3 - t0;
  }
  return rc;
}

int sn_reorder_schur(int64_t n, double* S, int64_t ldS, double* Q, int64_t ldQ, int32_t* select, int64_t* m) {
  return sn_reorder_schur_ex(nullptr, n, S, ldS, Q, ldQ, select, m, nullptr, nullptr, nullptr);
}

int sn_schedule_build(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w, int64_t* nwin,
                      int64_t* nswap, int64_t* nlevels, int64_t* win_j1, int64_t* win_k, int64_t* win_level,
                      int64_t* win_nswap) {
  if (n < 0) return -1;
  if (n > 0 && (!bmap || !selrow)) return -2;
  if (!nwin || !nswap || !nlevels) return -5;
  sn::Plan P;
  int rc = sn::build_plan(n, bmap, selrow, w, 64, -1, &P);
  if (rc) return rc;
  *nwin = (int64_t)P.wins.size();
  *nswap = P.nswap;
  *nlevels = P.nlevels;
  if (win_j1) {
    for (size_t t = 0; t < P.wins.size(); ++t) {
      win_j1[t] = P.wins[t].j1;
      if (win_k) win_k[t] = P.wins[t].k;
      if (win_level) win_level[t] = P.wins[t].level;
      if (win_nswap) win_nswap[t] = P.wins[t].nswap;
    }
  }
  return 0;
}

int sn_schedule_lookahead(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w, int64_t strip,
                          int32_t* crit_l, int32_t* crit_r) {
  if (n < 0) return -1;
  if (n > 0 && (!bmap || !selrow)) return -2;
  if (strip < 1) return -5;
  sn::Plan P;
  int rc = sn::build_plan(n, bmap, selrow, w, 64, -1, &P);
  if (rc) return rc;
  std::vector<int32_t> cl, cr;
  sn::lookahead_strips(P, strip, cl, cr);
  for (size_t t = 0; t < cl.size(); ++t) { crit_l[t] = cl[t]; crit_r[t] = cr[t]; }
  return 0;
}

int64_t sn_schedule_window_swaps(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w,
                                 int64_t inner_window, int64_t t, int64_t cap, int64_t* swap_j, int8_t* swap_n1,
                                 int8_t* swap_n2) {
  sn::Plan P;
  int rc = sn::build_plan(n, bmap, selrow, w, inner_window, t + 1, &P);
  if (rc) return rc;
  return sn::window_swaps(P, t, cap, swap_j, swap_n1, swap_n2);
}

}  // extern "C"
