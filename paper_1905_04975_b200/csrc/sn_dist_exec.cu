// sn_dist_exec.cu -- the sharded (multi-GPU) executor and its C ABI.
//
// One process per GPU.  S is sharded over column blocks (block-cyclic, width bc), Q over row
// blocks; every rank runs the program of sn_dist.h level by level on one stream (plus the Q
// updates on a second stream), so the order of every rank's kernels and collectives is fixed
// before the first launch and identical on all ranks (a sequentially consistent
// order needs no global synchronisation beyond the data each task reads).
//
// Communication per level (NCCL, over NVLink/NVSwitch, issued on the compute stream):
//   * pull / push of the straddled columns of windows that cross a block boundary
//     (ncclSend/ncclRecv of a packed S[0:j2, c:j2], one group per phase);
//   * one ncclBroadcast of every window's Z (k columns of its 256 x 256 slot) from the
//     window's owner, plus a max all-reduce of the level's window status words and of the
//     abort flag, in one group.
// Z is the only data every rank needs from a window task, so this is the whole exchange
// (P:158).  NCCL is loaded with dlopen on the first sn_dist_init; the one-GPU entry
// points never touch it.
//
// "Local ranks" (sn_reorder_schur_dist_local): P ranks' shards on the current device in one
// process, executed phase by phase in rank order on one stream, with device copies in place
// of the messages and shared Z / status buffers in place of the broadcast and reductions.
// Nothing waits on another rank's kernel; it runs the same program and kernels as the NCCL
// path and is how the sharded data path is checked on one GPU.
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "sn_device.cuh"
#include "sn_dist.h"
#include "sn_exec.h"
#include "sn_plan.h"
#include "sn_reorder.h"

namespace sn {
namespace {

constexpr int kZgenD = 4;   // Z slot generations in flight (Q stream)
constexpr int kStrip = 64;  // panel CTA width

#define DCK(x)                                                                                   \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) {                                                                     \
      if (std::getenv("SN_DEBUG"))                                                               \
        std::fprintf(stderr, "sn_dist: %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return SN_ERR_CUDA;                                                                        \
    }                                                                                            \
  } while (0)

// ---------------------------------------------------------------------------------------
// NCCL, loaded at run time
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;

int load_nccl() {
  if (g_nccl.h) return 0;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* nm : names)
    if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
  if (!h) return SN_ERR_NCCL;
#define SYM(f)                                                         \
  g_nccl.f = reinterpret_cast<decltype(g_nccl.f)>(dlsym(h, "nccl" #f)); \
  if (!g_nccl.f) return SN_ERR_NCCL;
  SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(Broadcast) SYM(AllReduce) SYM(Send) SYM(Recv)
  SYM(GroupStart) SYM(GroupEnd) SYM(GetErrorString)
#undef SYM
  g_nccl.h = h;
  return 0;
}

#define NCK(x)                                                                                  \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess) {                                                                    \
      if (std::getenv("SN_DEBUG"))                                                              \
        std::fprintf(stderr, "sn_dist: nccl %s at %s:%d\n", sn::g_nccl.GetErrorString(r_), __FILE__, __LINE__); \
      return SN_ERR_NCCL;                                                                       \
    }                                                                                           \
  } while (0)

struct DistComm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = -1;
  bool ready = false;
};
DistComm g_comm;

// ---------------------------------------------------------------------------------------
struct DBuf {
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
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct DistWorkspace {
  DBuf wins, pool, status, ctl, recs, Z, zr, sub, bad;
  std::vector<DBuf> Sx, own, strips, spref, stage;   // per local rank
  cudaStream_t sB = nullptr, sC = nullptr, sH = nullptr;   // Q / remaining strips / critical path
  cudaEvent_t evW[kZgenD] = {}, evQ[kZgenD] = {}, evCrit[kZgenD] = {}, evRest[kZgenD] = {};
  cudaEvent_t evIn = nullptr, evOut = nullptr, evJoinC = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evJoin = nullptr;
  int device = -1;
};
DistWorkspace g_dws;

int ensure_dist_runtime(DistWorkspace& ws, int64_t nlocal) {
  int dev = 0;
  DCK(cudaGetDevice(&dev));
  if (ws.device != dev) {
    if (ws.device >= 0) {
      // everything below belongs to the previous device: release it there
      DCK(cudaSetDevice(ws.device));
      for (DBuf* b : {&ws.wins, &ws.pool, &ws.status, &ws.ctl, &ws.recs, &ws.Z, &ws.zr, &ws.sub, &ws.bad}) b->release();
      for (auto* v : {&ws.Sx, &ws.own, &ws.strips, &ws.spref, &ws.stage})
        for (DBuf& b : *v) b.release();
      cudaStreamDestroy(ws.sH);
      cudaStreamDestroy(ws.sB);
      cudaStreamDestroy(ws.sC);
      for (int i = 0; i < kZgenD; ++i) {
        cudaEventDestroy(ws.evW[i]); cudaEventDestroy(ws.evQ[i]);
        cudaEventDestroy(ws.evCrit[i]); cudaEventDestroy(ws.evRest[i]);
      }
      for (cudaEvent_t e : {ws.evIn, ws.evOut, ws.evJoinC, ws.ev0, ws.ev1, ws.evJoin}) cudaEventDestroy(e);
      DCK(cudaSetDevice(dev));
    }
    int least = 0, greatest = 0;
    DCK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    DCK(cudaStreamCreateWithPriority(&ws.sH, cudaStreamNonBlocking, greatest));
    DCK(cudaStreamCreateWithPriority(&ws.sB, cudaStreamNonBlocking, least));
    DCK(cudaStreamCreateWithPriority(&ws.sC, cudaStreamNonBlocking, least));
    for (int i = 0; i < kZgenD; ++i) {
      DCK(cudaEventCreateWithFlags(&ws.evW[i], cudaEventDisableTiming));
      DCK(cudaEventCreateWithFlags(&ws.evQ[i], cudaEventDisableTiming));
      DCK(cudaEventCreateWithFlags(&ws.evCrit[i], cudaEventDisableTiming));
      DCK(cudaEventCreateWithFlags(&ws.evRest[i], cudaEventDisableTiming));
    }
    DCK(cudaEventCreateWithFlags(&ws.evIn, cudaEventDisableTiming));
    DCK(cudaEventCreateWithFlags(&ws.evOut, cudaEventDisableTiming));
    DCK(cudaEventCreateWithFlags(&ws.evJoinC, cudaEventDisableTiming));
    DCK(cudaEventCreate(&ws.ev0));
    DCK(cudaEventCreate(&ws.ev1));
    DCK(cudaEventCreateWithFlags(&ws.evJoin, cudaEventDisableTiming));
    ws.device = dev;
  }
  if ((int64_t)ws.Sx.size() < nlocal) {
    ws.Sx.resize(nlocal);
    ws.own.resize(nlocal);
    ws.strips.resize(nlocal);
    ws.spref.resize(nlocal);
    ws.stage.resize(nlocal);
  }
  return 0;
}

struct RankIO {
  double* Su;     // compact user layout (device), n rows x user_cols, ld ldu
  double* Q;      // Q rows [q0, q1) (device) or NULL
};

struct RankRun {
  int64_t rank = 0;
  DistProgram prog;
  double* Sx = nullptr;
  std::vector<WinDev> own;            // owned windows, level by level
  std::vector<int64_t> own_off;       // per level, offset into own
  WinDev* d_own = nullptr;
  StripDev* d_strips = nullptr;
  int32_t* d_spref = nullptr;
  char* stage = nullptr;
};

// copy the owned blocks between the compact user layout and the extended layout
cudaError_t copy_blocks(const DistLayout& lay, int64_t rank, double* Sx, int64_t ldx, double* Su, int64_t ldu,
                        bool to_ext, cudaStream_t s) {
  for (int64_t b = rank; b < lay.nblocks(); b += lay.P) {
    const int64_t j0 = b * lay.bc, nc = std::min(lay.bc, lay.n - j0);
    double* x = Sx + lay.ext_lcol(j0) * ldx;
    double* u = Su + lay.user_lcol(j0) * ldu;
    cudaError_t e = to_ext ? cudaMemcpy2DAsync(x, ldx * 8, u, ldu * 8, lay.n * 8, nc, cudaMemcpyDeviceToDevice, s)
                           : cudaMemcpy2DAsync(u, ldu * 8, x, ldx * 8, lay.n * 8, nc, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// pull / push messages of one level.  nccl: this process is local rank 0 == global rank.
int exchange(const std::vector<RankRun>& rr, const DistProgram& prog0, const std::vector<int64_t>& msgs,
             int64_t ldx, bool nccl, cudaStream_t s) {
  if (msgs.empty()) return 0;
  if (!nccl) {
    for (int64_t mi : msgs) {
      const DistMsg& m = prog0.msgs[mi];
      double* src = rr[m.src].Sx + m.src_lcol * ldx;
      double* dst = rr[m.dst].Sx + m.dst_lcol * ldx;
      DCK(cudaMemcpy2DAsync(dst, ldx * 8, src, ldx * 8, m.nrows * 8, m.ncols, cudaMemcpyDeviceToDevice, s));
    }
    return 0;
  }
  const RankRun& me = rr[0];
  const int r = (int)me.rank;
  // pack the sends, then one group of sends/receives, then unpack
  size_t off = 0;
  std::vector<size_t> where(msgs.size(), 0);
  for (size_t q = 0; q < msgs.size(); ++q) {
    const DistMsg& m = prog0.msgs[msgs[q]];
    if (m.src == m.dst) {
      if (m.src == r)
        DCK(cudaMemcpy2DAsync(me.Sx + m.dst_lcol * ldx, ldx * 8, me.Sx + m.src_lcol * ldx, ldx * 8, m.nrows * 8,
                              m.ncols, cudaMemcpyDeviceToDevice, s));
      continue;
    }
    if (m.src != r && m.dst != r) continue;
    where[q] = off;
    if (m.src == r)
      DCK(cudaMemcpy2DAsync(me.stage + off, m.nrows * 8, me.Sx + m.src_lcol * ldx, ldx * 8, m.nrows * 8, m.ncols,
                            cudaMemcpyDeviceToDevice, s));
    off += (size_t)(8 * m.nrows * m.ncols);
  }
  NCK(g_nccl.GroupStart());
  for (size_t q = 0; q < msgs.size(); ++q) {
    const DistMsg& m = prog0.msgs[msgs[q]];
    if (m.src == m.dst) continue;
    const size_t cnt = (size_t)(m.nrows * m.ncols);
    if (m.src == r) NCK(g_nccl.Send(me.stage + where[q], cnt, ncclFloat64, m.dst, g_comm.comm, s));
    if (m.dst == r) NCK(g_nccl.Recv(me.stage + where[q], cnt, ncclFloat64, m.src, g_comm.comm, s));
  }
  NCK(g_nccl.GroupEnd());
  for (size_t q = 0; q < msgs.size(); ++q) {
    const DistMsg& m = prog0.msgs[msgs[q]];
    if (m.src == m.dst || m.dst != r) continue;
    DCK(cudaMemcpy2DAsync(me.Sx + m.dst_lcol * ldx, ldx * 8, me.stage + where[q], m.nrows * 8, m.nrows * 8, m.ncols,
                          cudaMemcpyDeviceToDevice, s));
  }
  return 0;
}

// The sharded reordering.  io has one entry per local rank (NCCL: exactly one, rank =
// g_comm.rank; local: P entries, rank = index).
int run_dist_on(const sn_opts& o, int64_t n, int64_t bc, int64_t P, bool nccl, const std::vector<RankIO>& io,
                int64_t ldu, int64_t ldq, int32_t* select, int64_t* m, int8_t* bmap_out, sn_stats* st,
                cudaStream_t sA);

// ordered on the caller's stream; the work runs on the library's high-priority stream
int run_dist(const sn_opts& o, int64_t n, int64_t bc, int64_t P, bool nccl, const std::vector<RankIO>& io,
             int64_t ldu, int64_t ldq, int32_t* select, int64_t* m, int8_t* bmap_out, sn_stats* st,
             cudaStream_t sUser) {
  DistWorkspace& ws = g_dws;
  if (int rc = ensure_dist_runtime(ws, (int64_t)io.size())) return rc;
  DCK(cudaEventRecord(ws.evIn, sUser));
  DCK(cudaStreamWaitEvent(ws.sH, ws.evIn, 0));
  const int rc = run_dist_on(o, n, bc, P, nccl, io, ldu, ldq, select, m, bmap_out, st, ws.sH);
  // join the Q and remaining-strip streams on every exit path (see sn_abi.cu run())
  cudaEventRecord(ws.evJoin, ws.sB);
  cudaStreamWaitEvent(ws.sH, ws.evJoin, 0);
  cudaEventRecord(ws.evJoinC, ws.sC);
  cudaStreamWaitEvent(ws.sH, ws.evJoinC, 0);
  cudaEventRecord(ws.evOut, ws.sH);
  cudaStreamWaitEvent(sUser, ws.evOut, 0);
  return rc;
}

int run_dist_on(const sn_opts& o, int64_t n, int64_t bc, int64_t P, bool nccl, const std::vector<RankIO>& io,
                int64_t ldu, int64_t ldq, int32_t* select, int64_t* m, int8_t* bmap_out, sn_stats* st,
                cudaStream_t sA) {
  DistWorkspace& ws = g_dws;
  const double t_start = now_ms();
  const int64_t nloc = (int64_t)io.size();
  if (int rc = ensure_dist_runtime(ws, nloc)) return rc;
  const bool hasQ = io[0].Q != nullptr;
  DistLayout lay;
  lay.n = n; lay.P = P; lay.bc = bc; lay.hc = o.window;
  const int64_t ldx = (n + 1) & ~(int64_t)1;   // even: 16-byte row-strip copies
  int64_t launches[5] = {0, 0, 0, 0, 0};

  std::vector<RankRun> rr(nloc);
  for (int64_t q = 0; q < nloc; ++q) {
    rr[q].rank = nccl ? g_comm.rank : q;
    const size_t bytes = sizeof(double) * (size_t)ldx * (size_t)std::max<int64_t>(1, lay.ext_cols(rr[q].rank));
    DCK(ws.Sx[q].ensure(bytes));
    rr[q].Sx = (double*)ws.Sx[q].p;
    DCK(copy_blocks(lay, rr[q].rank, rr[q].Sx, ldx, io[q].Su, ldu, true, sA));
  }

  // ---- a1: structure scan of every rank's columns, combined
  DCK(ws.sub.ensure((size_t)n + 8));
  DCK(ws.bad.ensure(8));
  DCK(cudaMemsetAsync(ws.sub.p, 0, (size_t)n, sA));
  DCK(cudaMemsetAsync(ws.bad.p, 0, 4, sA));
  for (int64_t q = 0; q < nloc; ++q) {
    launch_scan_dist(rr[q].Sx, ldx, n, P, bc, lay.hc, rr[q].rank, o.validate_lower, (uint8_t*)ws.sub.p,
                     (int32_t*)ws.bad.p, sA);
    launches[4] += (o.validate_lower && n > 2) ? 2 : 1;
  }
  DCK(cudaGetLastError());
  if (nccl) {
    NCK(g_nccl.GroupStart());
    NCK(g_nccl.AllReduce(ws.sub.p, ws.sub.p, (size_t)n, ncclUint8, ncclMax, g_comm.comm, sA));
    NCK(g_nccl.AllReduce(ws.bad.p, ws.bad.p, 1, ncclInt32, ncclMax, g_comm.comm, sA));
    NCK(g_nccl.GroupEnd());
  }
  std::vector<uint8_t> sub((size_t)n);
  int32_t bad = 0;
  DCK(cudaMemcpyAsync(sub.data(), ws.sub.p, (size_t)n, cudaMemcpyDeviceToHost, sA));
  DCK(cudaMemcpyAsync(&bad, ws.bad.p, 4, cudaMemcpyDeviceToHost, sA));
  DCK(cudaStreamSynchronize(sA));
  if (bad) return -2;
  std::vector<int8_t> bmap((size_t)n), selrow((size_t)n);
  if (int rc = structure_from_sub(n, sub.data(), select, bmap.data(), selrow.data(), m)) return rc;

  // ---- a2: plan and the per-rank programs
  Plan plan;
  if (build_plan(n, bmap.data(), selrow.data(), o.window, o.inner_window, o.max_windows, &plan))
    return SN_ERR_UNSUPPORTED;
  for (int64_t q = 0; q < nloc; ++q)
    if (build_dist_program(plan, lay, rr[q].rank, kStrip, &rr[q].prog)) return SN_ERR_UNSUPPORTED;
  const DistProgram& G = rr[0].prog;   // windows, levels, messages: identical on every rank
  const int64_t nw = (int64_t)G.wins.size();
  const int64_t nlev = (int64_t)G.levels.size();
  const int64_t maxper = std::max<int64_t>(1, G.max_level_wins);
  std::vector<WinDev> wd(nw);
  for (int64_t i = 0; i < nw; ++i) {
    const DistWin& d = G.wins[i];
    const WindowPlan& w = plan.wins[d.t];
    WinDev& x = wd[i];
    std::memset(&x, 0, sizeof(x));
    x.j1 = d.j1; x.k = d.k; x.nblk = w.nblk; x.ninner = w.ninner;
    x.slot = (int32_t)((d.level % kZgenD) * maxper + (i - G.levels[d.level].w0));
    x.pool = w.pool; x.order = w.order;
    x.coff = d.coff; x.sidx = (int32_t)i;
  }
  for (int64_t q = 0; q < nloc; ++q) {
    RankRun& R = rr[q];
    R.own_off.assign(nlev + 1, 0);
    for (int64_t l = 0; l < nlev; ++l) {
      R.own_off[l] = (int64_t)R.own.size();
      for (int64_t i : R.prog.levels[l].own) R.own.push_back(wd[i]);
    }
    R.own_off[nlev] = (int64_t)R.own.size();
  }
  const double t_plan = now_ms();

  if (nw == 0) {
    for (int64_t q = 0; q < nloc; ++q) DCK(copy_blocks(lay, rr[q].rank, rr[q].Sx, ldx, io[q].Su, ldu, false, sA));
    DCK(cudaStreamSynchronize(sA));
    if (bmap_out) std::memcpy(bmap_out, bmap.data(), (size_t)n);
    for (int64_t i = 0; i < n; ++i) select[i] = selrow[i];
    if (st) {
      st->ms_schedule = t_plan - t_start;
      st->ms_total = now_ms() - t_start;
      st->launches[4] = launches[4];
    }
    return 0;
  }

  // ---- uploads
  DCK(ws.wins.ensure(sizeof(WinDev) * nw));
  DCK(ws.pool.ensure(plan.pool.size() + 8));
  DCK(ws.status.ensure(sizeof(int32_t) * nw));
  DCK(ws.ctl.ensure(sizeof(Control)));
  DCK(ws.recs.ensure(sizeof(WinRec) * nw));
  const size_t zbytes = sizeof(double) * (size_t)kZslot * (size_t)(kZgenD * maxper);
  if (ws.Z.cap < zbytes) {
    DCK(ws.Z.ensure(zbytes));
    DCK(cudaMemsetAsync(ws.Z.p, 0, zbytes, sA));
  }
  DCK(ws.zr.ensure(sizeof(int16_t) * (size_t)kZrange * (size_t)(kZgenD * maxper)));
  int16_t* dzr = (int16_t*)ws.zr.p;
  DCK(cudaMemcpyAsync(ws.wins.p, wd.data(), sizeof(WinDev) * nw, cudaMemcpyHostToDevice, sA));
  DCK(cudaMemcpyAsync(ws.pool.p, plan.pool.data(), plan.pool.size(), cudaMemcpyHostToDevice, sA));
  DCK(cudaMemsetAsync(ws.status.p, 0, sizeof(int32_t) * nw, sA));
  DCK(cudaMemsetAsync(ws.ctl.p, 0, sizeof(Control), sA));
  DCK(cudaMemsetAsync(ws.recs.p, 0, sizeof(WinRec) * nw, sA));
  for (int64_t q = 0; q < nloc; ++q) {
    RankRun& R = rr[q];
    DCK(ws.own[q].ensure(sizeof(WinDev) * std::max<size_t>(1, R.own.size())));
    DCK(ws.strips[q].ensure(sizeof(StripDev) * std::max<size_t>(1, R.prog.strips.size())));
    R.d_own = (WinDev*)ws.own[q].p;
    R.d_strips = (StripDev*)ws.strips[q].p;
    DCK(ws.spref[q].ensure(sizeof(int32_t) * std::max<size_t>(1, R.prog.sprefix.size())));
    R.d_spref = (int32_t*)ws.spref[q].p;
    if (!R.prog.sprefix.empty())
      DCK(cudaMemcpyAsync(R.d_spref, R.prog.sprefix.data(), sizeof(int32_t) * R.prog.sprefix.size(),
                          cudaMemcpyHostToDevice, sA));
    if (!R.own.empty())
      DCK(cudaMemcpyAsync(R.d_own, R.own.data(), sizeof(WinDev) * R.own.size(), cudaMemcpyHostToDevice, sA));
    if (!R.prog.strips.empty())
      DCK(cudaMemcpyAsync(R.d_strips, R.prog.strips.data(), sizeof(StripDev) * R.prog.strips.size(),
                          cudaMemcpyHostToDevice, sA));
    if (nccl && R.prog.max_msg_bytes > 0) {
      DCK(ws.stage[q].ensure((size_t)R.prog.max_msg_bytes));
      R.stage = (char*)ws.stage[q].p;
    }
  }

  const int mt = o.window <= 64 ? 64 : (o.window <= 128 ? 128 : 256);
  WinDev* dw = (WinDev*)ws.wins.p;
  int32_t* dstatus = (int32_t*)ws.status.p;
  Control* dctl = (Control*)ws.ctl.p;
  double* dZ = (double*)ws.Z.p;
  const bool overlapQ = o.q_stream_overlap != 0 && hasQ;
  cudaStream_t sQ = overlapQ ? ws.sB : sA;
  const bool look = o.lookahead != 0;
  cudaStream_t sC = ws.sC;
  std::vector<PanelMaps> mapS(nloc), mapQ(nloc);
  for (int64_t q = 0; q < nloc; ++q) {
    const int64_t r = rr[q].rank;
    std::memset(&mapS[q], 0, sizeof(PanelMaps));
    std::memset(&mapQ[q], 0, sizeof(PanelMaps));
    if (lay.ext_cols(r) > 0) panel_maps_init(&mapS[q], dZ, (int64_t)kZgenD * maxper, rr[q].Sx, n, lay.ext_cols(r), ldx);
    if (hasQ && lay.q1(r) > lay.q0(r))
      panel_maps_init(&mapQ[q], dZ, (int64_t)kZgenD * maxper, io[q].Q, lay.q1(r) - lay.q0(r), n, ldq);
  }
  DCK(cudaEventRecord(ws.ev0, sA));
  if (overlapQ) DCK(cudaStreamWaitEvent(ws.sB, ws.ev0, 0));
  if (look) DCK(cudaStreamWaitEvent(sC, ws.ev0, 0));

  for (int64_t l = 0; l < nlev; ++l) {
    const DistLevel& LG = G.levels[l];
    const int64_t w0 = LG.w0, cnt = LG.w1 - LG.w0;
    const int gen = (int)(l % kZgenD);
    if (overlapQ && l >= kZgenD) DCK(cudaStreamWaitEvent(sA, ws.evQ[gen], 0));
    // 1 PULL
    if (int rc = exchange(rr, G, LG.pulls, ldx, nccl, sA)) return rc;
    // 2 W
    for (int64_t q = 0; q < nloc; ++q) {
      RankRun& R = rr[q];
      const int64_t a = R.own_off[l], c = R.own_off[l + 1] - a;
      if (c == 0) continue;
      WindowArgs wa{};
      wa.wins = R.d_own + a; wa.nwin = (int32_t)c; wa.base = 0;
      wa.pool = (const uint8_t*)ws.pool.p; wa.S = R.Sx; wa.ldS = ldx; wa.Z = dZ;
      wa.status = dstatus; wa.ctl = dctl; wa.zrange = dzr;
      wa.recs = (WinRec*)ws.recs.p; wa.level = (int32_t)l;
      wa.force_order = o.force_reject_window; wa.force_swap = (int32_t)o.force_reject_swap;
      launch_window(wa, sA);
      launches[0]++;
    }
    DCK(cudaGetLastError());
    // 3 SYNC: Z from each owner, status words, abort flag
    if (nccl) {
      NCK(g_nccl.GroupStart());
      for (int64_t i = w0; i < w0 + cnt; ++i) {
        double* z = dZ + (int64_t)wd[i].slot * kZslot;
        NCK(g_nccl.Broadcast(z, z, (size_t)wd[i].k * kZld, ncclFloat64, G.wins[i].owner, g_comm.comm, sA));
        int16_t* zr = dzr + (int64_t)wd[i].slot * kZrange;
        NCK(g_nccl.Broadcast(zr, zr, (size_t)kZrange * 2, ncclUint8, G.wins[i].owner, g_comm.comm, sA));
      }
      NCK(g_nccl.AllReduce(dstatus + w0, dstatus + w0, (size_t)cnt, ncclInt32, ncclMax, g_comm.comm, sA));
      // abort and abort_level (adjacent): every rank skips the levels after a rejection
      NCK(g_nccl.AllReduce(&dctl->abort, &dctl->abort, 2, ncclInt32, ncclMax, g_comm.comm, sA));
      NCK(g_nccl.GroupEnd());
    }
    if (overlapQ) DCK(cudaEventRecord(ws.evW[gen], sA));
    // 4 L, 5 R: the critical strips on the critical path (after the previous level's
    // remaining strips), the remaining strips on stream C after the push
    if (look && l > 0) DCK(cudaStreamWaitEvent(sA, ws.evRest[(l - 1) % kZgenD], 0));
    auto panels = [&](int kind, bool crit, cudaStream_t s) {
      for (int64_t q = 0; q < nloc; ++q) {
        RankRun& R = rr[q];
        const DistLevel& LR = R.prog.levels[l];
        const int64_t s0 = kind == 0 ? (crit ? LR.L0 : LR.Lr0) : (crit ? LR.R0 : LR.Rr0);
        const int64_t s1 = kind == 0 ? (crit ? LR.L1 : LR.Lr1) : (crit ? LR.R1 : LR.Rr1);
        const int g = kind == 0 ? (crit ? 0 : 2) : (crit ? 1 : 3);
        if (s1 <= s0 || LR.nstr[g] <= 0) continue;
        PanelArgs pa{};
        pa.wins = dw + w0; pa.nwin = (int32_t)cnt; pa.base = (int32_t)w0; pa.status = dstatus;
        pa.strips = R.d_strips + s0; pa.nseg = (int32_t)(s1 - s0); pa.prefix = R.d_spref + LR.poff[g];
        pa.part = 0;
        pa.n = n; pa.Z = dZ; pa.zrange = dzr; pa.M = R.Sx; pa.ld = ldx; pa.maps = &mapS[q];
        pa.vec16 = ((uintptr_t)R.Sx % 16) == 0 ? 1 : 0;
        launch_panel(kind, mt, pa, LR.nstr[g], s);
        launches[1 + kind]++;
      }
    };
    panels(0, true, sA);
    panels(1, true, sA);
    if (!look) {
      // one-stream order: the remaining strips of this level right after its critical ones
      // (left before right on every corner, as in the one-GPU executor)
      panels(0, false, sA);
      panels(1, false, sA);
    }
    DCK(cudaGetLastError());
    // 6 PUSH
    if (int rc = exchange(rr, G, LG.pushes, ldx, nccl, sA)) return rc;
    if (look) {
      DCK(cudaEventRecord(ws.evCrit[gen], sA));
      DCK(cudaStreamWaitEvent(sC, ws.evCrit[gen], 0));
      panels(0, false, sC);
      panels(1, false, sC);
      DCK(cudaEventRecord(ws.evRest[gen], sC));
      DCK(cudaGetLastError());
    }
    // 7 Q
    if (hasQ) {
      if (overlapQ) DCK(cudaStreamWaitEvent(sQ, ws.evW[gen], 0));
      for (int64_t q = 0; q < nloc; ++q) {
        RankRun& R = rr[q];
        const DistLevel& LR = R.prog.levels[l];
        if (LR.Q1 <= LR.Q0 || LR.nstr[4] <= 0) continue;
        PanelArgs pa{};
        pa.wins = dw + w0; pa.nwin = (int32_t)cnt; pa.base = (int32_t)w0; pa.status = dstatus;
        pa.strips = R.d_strips + LR.Q0; pa.nseg = (int32_t)(LR.Q1 - LR.Q0); pa.prefix = R.d_spref + LR.poff[4];
        pa.part = 0;
        pa.n = lay.q1(R.rank) - lay.q0(R.rank); pa.Z = dZ; pa.zrange = dzr; pa.M = io[q].Q; pa.ld = ldq;
        pa.maps = &mapQ[q];
        pa.vec16 = (ldq % 2 == 0 && ((uintptr_t)io[q].Q % 16) == 0) ? 1 : 0;
        launch_panel(2, mt, pa, LR.nstr[4], sQ);
        launches[3]++;
      }
      DCK(cudaGetLastError());
      if (overlapQ) DCK(cudaEventRecord(ws.evQ[gen], sQ));
    }
    if (o.serialize) {
      DCK(cudaStreamSynchronize(sA));
      if (overlapQ) DCK(cudaStreamSynchronize(sQ));
    }
  }
  if (overlapQ) {
    DCK(cudaEventRecord(ws.evJoin, sQ));
    DCK(cudaStreamWaitEvent(sA, ws.evJoin, 0));
  }
  if (look) {
    DCK(cudaEventRecord(ws.evJoinC, sC));
    DCK(cudaStreamWaitEvent(sA, ws.evJoinC, 0));
  }
  DCK(cudaEventRecord(ws.ev1, sA));
  Control ctl;
  DCK(cudaMemcpyAsync(&ctl, dctl, sizeof(Control), cudaMemcpyDeviceToHost, sA));
  DCK(cudaStreamSynchronize(sA));
  float dev_ms = 0.f;
  DCK(cudaEventElapsedTime(&dev_ms, ws.ev0, ws.ev1));

  std::vector<int32_t> status;
  std::vector<WinRec> recs;
  if (ctl.abort) {
    status.resize(nw);
    recs.resize(nw);
    if (nccl) {
      // each partial window's record lives on its owner (the others hold zeros)
      NCK(g_nccl.AllReduce(ws.recs.p, ws.recs.p, sizeof(WinRec) * nw, ncclUint8, ncclMax, g_comm.comm, sA));
    }
    DCK(cudaMemcpyAsync(status.data(), dstatus, sizeof(int32_t) * nw, cudaMemcpyDeviceToHost, sA));
    DCK(cudaMemcpyAsync(recs.data(), ws.recs.p, sizeof(WinRec) * nw, cudaMemcpyDeviceToHost, sA));
    DCK(cudaStreamSynchronize(sA));
  }
  for (int64_t q = 0; q < nloc; ++q) DCK(copy_blocks(lay, rr[q].rank, rr[q].Sx, ldx, io[q].Su, ldu, false, sA));
  DCK(cudaStreamSynchronize(sA));

  // ---- outputs
  std::vector<uint8_t> fsz, fsel;
  int64_t executed = nw, swaps = 0, sbt[4] = {0, 0, 0, 0}, rej = -1;
  final_blocks(plan, G.sorted, ctl.abort != 0, ctl.abort ? status.data() : nullptr, recs.data(), n, bmap.data(),
               selrow.data(), fsz, fsel, &executed, &swaps, sbt, &rej);
  write_blocks(fsz, fsel, select, bmap_out);
  if (st) {
    double eqf = 0.0, fk[5] = {0, 0, 0, 0, 0};
    for (int64_t i = 0; i < nw; ++i) {
      if (ctl.abort && status[i] == kWinSkipped) continue;
      const DistWin& d = G.wins[i];
      const double kd = (double)d.k, k2 = 2.0 * kd * kd;
      const double eL = (double)(n - d.j1 - d.k), eR = (double)d.j1, eQ = hasQ ? (double)n : 0.0;
      eqf += k2 * (eL + eR + eQ);
      fk[1] += k2 * eL; fk[2] += k2 * eR; fk[3] += k2 * eQ;
    }
    st->windows = executed;
    st->levels = nlev;
    st->swaps = swaps;
    for (int q = 0; q < 4; ++q) st->swaps_by_type[q] = sbt[q];
    st->inner_windows = plan.ninner;
    st->rejected_window = -1;
    st->rejected_row = -1;
    if (ctl.abort && rej >= 0) {
      st->rejected_window = plan.wins[G.sorted[rej]].order;
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
      st->flops_kernel[q] = fk[q];
    }
  }
  return ctl.abort ? SN_ERR_REJECTED : SN_OK;
}

int check_common(const sn_opts& o, int64_t n, int64_t bc, int64_t ldu, int64_t ldq, bool hasQ, int32_t* select,
                 int64_t* m) {
  if (m == nullptr) return -9;
  *m = 0;
  if (n < 0) return -2;
  if (select == nullptr) return -8;
  if (ldu < n) return -5;
  if (hasQ && ldq < 1) return -7;
  if (o.window < 4 || o.window > 256 || o.inner_window < 4 || o.inner_window > 64) return SN_ERR_UNSUPPORTED;
  if (bc < o.window) return SN_ERR_UNSUPPORTED;
  return 0;
}

}  // namespace
}  // namespace sn

extern "C" {

int sn_dist_unique_id(void* id_out) {
  if (!id_out) return -1;
  if (int rc = sn::load_nccl()) return rc;
  ncclUniqueId id;
  NCK(sn::g_nccl.GetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return 0;
}

int sn_dist_init(int rank, int world, const void* unique_id, int device) {
  if (world < 1 || rank < 0 || rank >= world) return -1;
  if (!unique_id) return -3;
  std::lock_guard<std::mutex> lock(sn::g_mu);
  if (int rc = sn::load_nccl()) return rc;
  if (cudaSetDevice(device) != cudaSuccess) return SN_ERR_CUDA;
  if (sn::g_comm.ready) {
    sn::g_nccl.CommDestroy(sn::g_comm.comm);
    sn::g_comm.ready = false;
  }
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  NCK(sn::g_nccl.CommInitRank(&sn::g_comm.comm, world, id, rank));
  sn::g_comm.rank = rank;
  sn::g_comm.world = world;
  sn::g_comm.device = device;
  sn::g_comm.ready = true;
  return 0;
}

int sn_dist_finalize(void) {
  std::lock_guard<std::mutex> lock(sn::g_mu);
  if (sn::g_comm.ready) {
    sn::g_nccl.CommDestroy(sn::g_comm.comm);
    sn::g_comm.ready = false;
  }
  return 0;
}

int sn_dist_layout(int64_t n, int64_t P, int64_t col_block, int64_t rank, int64_t* user_cols, int64_t* q0,
                   int64_t* q1) {
  if (n < 0 || P < 1 || col_block < 1 || rank < 0 || rank >= P) return -1;
  sn::DistLayout lay;
  lay.n = n; lay.P = P; lay.bc = col_block;
  if (user_cols) *user_cols = lay.user_cols(rank);
  if (q0) *q0 = lay.q0(rank);
  if (q1) *q1 = lay.q1(rank);
  return 0;
}

int sn_reorder_schur_dist(const sn_opts* opts, int64_t n, int64_t col_block, double* S_loc, int64_t ldS_loc,
                          double* Q_loc, int64_t ldQ_loc, int32_t* select, int64_t* m, int8_t* bmap_out,
                          sn_stats* stats, void* stream) {
  sn_opts o;
  if (opts) o = *opts; else sn_default_opts(&o);
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->rejected_window = -1;
    stats->rejected_row = -1;
  }
  if (int rc = sn::check_common(o, n, col_block, ldS_loc, ldQ_loc, Q_loc != nullptr, select, m)) return rc;
  if (n == 0) return 0;
  if (!sn::g_comm.ready) return SN_ERR_NCCL;
  sn::DistLayout lay;
  lay.n = n; lay.P = sn::g_comm.world; lay.bc = col_block;
  const int r = sn::g_comm.rank;
  if (lay.user_cols(r) > 0 && S_loc == nullptr) return -4;
  if (Q_loc && ldQ_loc < lay.q1(r) - lay.q0(r)) return -7;
  std::lock_guard<std::mutex> lock(sn::g_mu);
  if ((S_loc && !sn::is_device_ptr(S_loc)) || (Q_loc && !sn::is_device_ptr(Q_loc))) {
    // host shards: stage through device memory (the copies are part of the call)
    const double t0 = sn::now_ms();
    const int64_t uc = std::max<int64_t>(1, lay.user_cols(r)), nq = std::max<int64_t>(1, lay.q1(r) - lay.q0(r));
    double *dS = nullptr, *dQ = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMalloc(&dS, sizeof(double) * n * uc) != cudaSuccess) return SN_ERR_CUDA;
    if (Q_loc && cudaMalloc(&dQ, sizeof(double) * nq * n) != cudaSuccess) { cudaFree(dS); return SN_ERR_CUDA; }
    int rc = SN_OK;
    if (cudaMemcpy2DAsync(dS, n * 8, S_loc, ldS_loc * 8, n * 8, lay.user_cols(r), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        (Q_loc && cudaMemcpy2DAsync(dQ, nq * 8, Q_loc, ldQ_loc * 8, (lay.q1(r) - lay.q0(r)) * 8, n,
                                    cudaMemcpyHostToDevice, s) != cudaSuccess) ||
        cudaStreamSynchronize(s) != cudaSuccess)
      rc = SN_ERR_CUDA;
    const double t1 = sn::now_ms();
    if (rc == SN_OK)
      rc = sn::run_dist(o, n, col_block, lay.P, true, {sn::RankIO{dS, dQ}}, n, nq, select, m, bmap_out, stats, s);
    const double t2 = sn::now_ms();
    if (rc == SN_OK || rc == SN_ERR_REJECTED) {
      if (cudaMemcpy2DAsync(S_loc, ldS_loc * 8, dS, n * 8, n * 8, lay.user_cols(r), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          (Q_loc && cudaMemcpy2DAsync(Q_loc, ldQ_loc * 8, dQ, nq * 8, (lay.q1(r) - lay.q0(r)) * 8, n,
                                      cudaMemcpyDeviceToHost, s) != cudaSuccess) ||
          cudaStreamSynchronize(s) != cudaSuccess)
        rc = SN_ERR_CUDA;
    }
    const double t3 = sn::now_ms();
    cudaFree(dS);
    if (dQ) cudaFree(dQ);
    if (stats) {
      stats->ms_h2d = t1 - t0;
      stats->ms_d2h = t3 - t2;
      stats->ms_total = t3 - t0;
    }
    return rc;
  }
  return sn::run_dist(o, n, col_block, lay.P, true, {sn::RankIO{S_loc, Q_loc}}, ldS_loc, ldQ_loc, select, m,
                      bmap_out, stats, (cudaStream_t)stream);
}

int sn_reorder_schur_dist_local(const sn_opts* opts, int64_t P, int64_t n, int64_t col_block, double* const* S_locs,
                                int64_t ldS_loc, double* const* Q_locs, int64_t ldQ_loc, int32_t* select,
                                int64_t* m, int8_t* bmap_out, sn_stats* stats, void* stream) {
  sn_opts o;
  if (opts) o = *opts; else sn_default_opts(&o);
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->rejected_window = -1;
    stats->rejected_row = -1;
  }
  if (P < 1 || P > 64) return -2;
  if (int rc = sn::check_common(o, n, col_block, ldS_loc, ldQ_loc, Q_locs != nullptr, select, m)) return rc;
  if (n == 0) return 0;
  if (!S_locs) return -5;
  std::lock_guard<std::mutex> lock(sn::g_mu);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return SN_ERR_CUDA;
  }
  sn::DistLayout lay;
  lay.n = n; lay.P = P; lay.bc = col_block;
  std::vector<sn::RankIO> io((size_t)P);
  for (int64_t r = 0; r < P; ++r) {
    io[r].Su = S_locs[r];
    io[r].Q = Q_locs ? Q_locs[r] : nullptr;
    if (lay.user_cols(r) > 0 && (!io[r].Su || !sn::is_device_ptr(io[r].Su))) return -5;
    if (Q_locs && lay.q1(r) > lay.q0(r) && (!io[r].Q || !sn::is_device_ptr(io[r].Q))) return -7;
    if (Q_locs && ldQ_loc < lay.q1(r) - lay.q0(r)) return -7;
  }
  return sn::run_dist(o, n, col_block, P, false, io, ldS_loc, ldQ_loc, select, m, bmap_out, stats,
                      (cudaStream_t)stream);
}

int64_t sn_dist_program(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w, int64_t col_block, int64_t P,
                        int64_t rank, int64_t cap, int64_t* rec) {
  if (n < 0) return -1;
  if (n > 0 && (!bmap || !selrow)) return -2;
  sn::Plan plan;
  int rc = sn::build_plan(n, bmap, selrow, w, 64, -1, &plan);
  if (rc) return rc;
  sn::DistLayout lay;
  lay.n = n; lay.P = P; lay.bc = col_block; lay.hc = w;
  sn::DistProgram D;
  rc = sn::build_dist_program(plan, lay, rank, sn::kStrip, &D);
  if (rc) return rc;
  // flat records of 8 int64 (see sn_reorder.h)
  int64_t cnt = 0;
  auto put = [&](int64_t a, int64_t b, int64_t c, int64_t d, int64_t e, int64_t f, int64_t g, int64_t h) {
    if (rec && cnt < cap) {
      int64_t* p = rec + 8 * cnt;
      p[0] = a; p[1] = b; p[2] = c; p[3] = d; p[4] = e; p[5] = f; p[6] = g; p[7] = h;
    }
    ++cnt;
  };
  put(0, (int64_t)D.levels.size(), (int64_t)D.wins.size(), lay.ext_cols(rank), lay.q0(rank), lay.q1(rank), lay.hc, 0);
  for (const auto& d : D.wins) put(1, d.level, d.t, d.j1, d.k, d.owner, d.partner, d.coff);
  for (int64_t l = 0; l < (int64_t)D.levels.size(); ++l) {
    const sn::DistLevel& L = D.levels[l];
    put(2, l, L.w0, L.w1, (int64_t)L.pulls.size(), L.L1 - L.L0, L.R1 - L.R0, L.Q1 - L.Q0);
    for (int64_t mi : L.pulls) {
      const sn::DistMsg& m = D.msgs[mi];
      put(3, m.w, m.src, m.dst, m.nrows, m.ncols, m.src_lcol, m.dst_lcol);
    }
    for (int64_t s = L.L0; s < L.L1; ++s) put(4, D.strips[s].w, D.strips[s].cnt, D.strips[s].x0, 0, 0, 0, 0);
    for (int64_t s = L.R0; s < L.R1; ++s) put(5, D.strips[s].w, D.strips[s].cnt, D.strips[s].x0, 0, 0, 0, 0);
    for (int64_t mi : L.pushes) {
      const sn::DistMsg& m = D.msgs[mi];
      put(7, m.w, m.src, m.dst, m.nrows, m.ncols, m.src_lcol, m.dst_lcol);
    }
    for (int64_t q = L.Lr0; q < L.Lr1; ++q) put(8, D.strips[q].w, D.strips[q].cnt, D.strips[q].x0, 0, 0, 0, 0);
    for (int64_t q = L.Rr0; q < L.Rr1; ++q) put(9, D.strips[q].w, D.strips[q].cnt, D.strips[q].x0, 0, 0, 0, 0);
    for (int64_t s = L.Q0; s < L.Q1; ++s) put(6, D.strips[s].w, D.strips[s].cnt, D.strips[s].x0, 0, 0, 0, 0);
  }
  return cnt;
}

}  // extern "C"
