// sn_kernels_panel_tma.cu -- the left/right/Q update tasks as
// warp-specialised, TMA-fed FP64 DMMA kernels for sm_100a.  Same products as
// sn_kernels_panel.cu (which remains the path for leading dimensions TMA cannot describe):
//   left  (kind 0):  S[j1:j2, strip]  <- Z^T * S[j1:j2, strip]
//   right (kind 1):  S[strip, j1:j2]  <- S[strip, j1:j2] * Z
//   Q     (kind 2):  Q[strip, j1:j2]  <- Q[strip, j1:j2] * Z
//   Q fused (kind 3, row f1): Q[strip, x1:x2] <- Q[strip, x1:x2] * Zx, then
//                     Q[strip, y1:y2] <- Q[strip, y1:y2] * Zy for two consecutive windows x, y of
//                     a chain, in one CTA pass per strip (the second pass's TMA loads wait on an
//                     mbarrier the consumer warps release after storing the first pass)
// CTA = MT/32 consumer warps (each a 32 x 64 tile of the MT x 64 strip result, MI = 2 m16
// tiles x NI = 8 n8 tiles of mma.sync.m16n8k4 f64 = DMMA) + 1 producer warp whose elected
// lane streams K chunks (16 rows of Z^T and of the strip) with cp.async.bulk.tensor (TMA)
// into a ring of NS shared-memory stages.  Stage hand-off is by mbarriers: full[s] completes
// when the TMA bytes land (expect_tx), empty[s] when every consumer warp has read the stage;
// there is no CTA-wide barrier in the main loop.  A CTA walks up to 4 strips, the producer
// running ahead into the next strip's chunks while the consumers store the previous result.
//
// The TMA boxes carry their own padding (A: 20 = 16 + 4 K elements per Z column, B: 68 = 64 + 4
// rows for right/Q, 20 K rows for left), so the shared-memory tiles have the conflict-free
// strides of the cp.async kernel (row stride == 4 mod 16 doubles) without a swizzle mode; the
// padding elements are loaded (or zero-filled out of bounds) and never read.  Out-of-bounds
// box elements (past n, past column 255 of a Z slot) are zero-filled by TMA.  The innermost
// box coordinate must be 16-byte aligned (an odd FP64 start raises an illegal-instruction
// fault): the left update's K rows start at j1, so its box starts at the even row below and
// the consumers read one element further when j1 is odd.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "sn_device.cuh"

namespace sn {
namespace {

constexpr int KC = 16;          // K chunk
constexpr int LDA = KC + 4;     // A box inner extent (Z rows per Z column, padded)
constexpr int NT = 64;          // strip width
constexpr int LDBR = NT + 4;    // right/Q: B box inner extent (strip rows, padded)
constexpr int LDBL = KC + 4;    // left: B box inner extent (K rows, padded)
constexpr int kMaxStripsPerCta = 4;

template <int MT>
struct TCfg {
  static constexpr int CONS = MT / 32;                // consumer warps (32 x 64 tiles)
  static constexpr int THREADS = (CONS + 1) * 32;     // + producer warp
  static constexpr int NS = MT == 256 ? 4 : 6;        // stages
  static constexpr int A_BYTES = 8 * LDA * MT;
  static constexpr int B_BYTES = 8 * (LDBR * KC > LDBL * NT ? LDBR * KC : LDBL * NT);
  static constexpr int STAGE = ((A_BYTES + B_BYTES + 1023) / 1024) * 1024;
  static constexpr size_t SMEM = (size_t)STAGE * NS + 1024 + 2 * 8 * NS + 8;
};

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "SN_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra SN_WAIT_%=;\n}\n" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          sa(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(sa(bar))
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.b32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

struct StripInfo {
  int w, nx, k, nk;
  int64_t x0, j1, jc;
  int slot;
  bool skip;
  // fused chain Q update (a.fuse): the predecessor's pass, applied first when pdo
  bool pdo;
  int pk, pnk, pslot;
  int64_t pjc;
};

template <int KIND>
__device__ __forceinline__ StripInfo resolve(const PanelArgs& a, int sid) {
  StripInfo s;
  int w;
  if (a.strips) {
    int lo = 0, hi = a.nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.prefix[mid] <= sid) lo = mid; else hi = mid - 1;
    }
    const StripDev sd = a.strips[lo];
    const int idx = sid - a.prefix[lo];
    w = sd.w;
    s.x0 = sd.x0 + (int64_t)idx * NT;
    s.nx = min(NT, sd.cnt - idx * NT);
  } else {
    int lo = 0, hi = a.nwin - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.prefix[mid] <= sid) lo = mid; else hi = mid - 1;
    }
    w = lo;
    int strip = sid - a.prefix[w];
    const WinDev& wq = a.wins[w];
    if (KIND == 0 && a.part == 2) strip += wq.crit_l;
    if (KIND == 1 && a.part == 1) strip += (int)((wq.j1 + NT - 1) / NT) - wq.crit_r;
    if (KIND == 0) {
      s.x0 = wq.j1 + wq.k + (int64_t)strip * NT;
      s.nx = (int)min((int64_t)NT, a.n - s.x0);
    } else {
      s.x0 = (int64_t)strip * NT;
      const int64_t lim = (KIND == 1) ? wq.j1 : a.n;
      s.nx = (int)min((int64_t)NT, lim - s.x0);
    }
  }
  s.w = w;
  s.skip = a.status[a.base + w] == kWinSkipped;
  const WinDev& wd = a.wins[w];
  s.k = wd.k;
  s.nk = (wd.k + KC - 1) / KC;
  s.j1 = wd.j1;
  s.jc = (KIND == 1) ? wd.j1 + wd.coff : wd.j1;
  s.slot = wd.slot;
  s.pdo = false;
  s.pk = 0; s.pnk = 0; s.pslot = 0; s.pjc = 0;
  if (KIND == 3 && wd.qprev > 0) {
    const int pidx = wd.qprev - 1;                 // level-sorted index (a.wins == base + a.base)
    const WinDev& pd = a.wins[pidx - a.base];
    s.pdo = a.status[pidx] != kWinSkipped;
    s.pk = pd.k;
    s.pnk = (pd.k + KC - 1) / KC;
    s.pslot = pd.slot;
    s.pjc = pd.j1 + pd.coff;
  }
  return s;
}

template <int MT, int KIND>
__global__ void __launch_bounds__(TCfg<MT>::THREADS, 1)
    panel_tma_kernel(PanelArgs a, int32_t nstrips, const __grid_constant__ CUtensorMap zmap,
                     const __grid_constant__ CUtensorMap mmap, int dbg) {
  using C = TCfg<MT>;
  constexpr bool LEFT = (KIND == 0);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align by an offset into the shared array itself (keeps the pointer in the shared window,
  // so fragment loads compile to LDS rather than generic loads)
  unsigned char* smem = smem_raw + ((1024u - (sa(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = (uint64_t*)(smem + (size_t)C::STAGE * C::NS);
  uint64_t* empty = full + C::NS;
  uint64_t* wb = empty + C::NS;     // fused Q passes: first pass stored (one arrival per consumer warp)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::CONS);
    }
    mbar_init(wb, C::CONS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int s_begin = blockIdx.x;
  const int s_step = gridDim.x;
  constexpr uint32_t kTx = 8u * (LDA * MT + (LEFT ? LDBL * NT : LDBR * KC));

  if (warp == C::CONS) {
    // ---------------- producer: one elected lane issues every TMA
    // the whole warp walks the schedule (warp-uniform values); one elected lane issues
    uint32_t it = 0, wbuse = 0;
    for (int sid = s_begin; sid < nstrips; sid += s_step) {
      const StripInfo si = resolve<KIND>(a, sid);
      // passes: the fused predecessor's Z (p = 0), then this window's (p = 1)
      for (int p = si.pdo ? 0 : 1; p < 2; ++p) {
      if (p == 1 && si.skip) break;
      if (p == 1 && si.pdo) {
        // the second pass reads columns the first pass wrote: wait until every consumer warp
        // has stored them and fenced them for the async proxy
        mbar_wait(wb, wbuse & 1);
        ++wbuse;
      }
      const int pnk = p ? si.nk : si.pnk, pslot = p ? si.slot : si.pslot;
      const int64_t pjc = p ? si.jc : si.pjc;
      for (int kc = 0; kc < pnk; ++kc, ++it) {
        const int st = it % C::NS;
        mbar_wait(&empty[st], ((it / C::NS) & 1) ^ 1);
        unsigned char* As = smem + (size_t)st * C::STAGE;
        unsigned char* Bs = As + C::A_BYTES;
        if (elect_one()) {
          if (dbg & 1) {
            mbar_arrive(&full[st]);
          } else {
            const uint32_t txA = 8u * LDA * MT, txB = kTx - txA;
            mbar_expect_tx(&full[st], (dbg & 4) ? txA : (dbg & 8) ? txB : kTx);
            // A: As[m][0..19] = Z[kc*16 + 0..19, m] of the window's slot (Z columns m < MT)
            if (!(dbg & 8)) tma_2d(As, &zmap, kc * KC, pslot * kZld, &full[st]);
            if (!(dbg & 4)) {
              // the inner box coordinate must be 16-byte aligned: start one row early for odd
              // j1 (the consumers read with the offset j1 & 1; the box has 4 rows of slack)
              if (LEFT) tma_2d(Bs, &mmap, (int)((si.j1 + kc * KC) & ~(int64_t)1), (int)si.x0, &full[st]);  // Bs[c][kk]
              else tma_2d(Bs, &mmap, (int)si.x0, (int)(pjc + kc * KC), &full[st]);           // Bs[kk][r]
            }
          }
        }
        __syncwarp();
      }
      }
    }
    __syncwarp();
    return;
  }

  // ---------------- consumers
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = warp * 32;
  uint32_t it = 0;
  for (int sid = s_begin; sid < nstrips; sid += s_step) {
    const StripInfo si = resolve<KIND>(a, sid);
    for (int p = si.pdo ? 0 : 1; p < 2; ++p) {
    if (p == 1 && si.skip) break;
    const int pk = p ? si.k : si.pk, pnk = p ? si.nk : si.pnk, pslot = p ? si.slot : si.pslot;
    const int64_t pjc = p ? si.jc : si.pjc;
    // K interval of this warp's 32 output rows (Z structure; exact zeros outside)
    int wlo, whi;
    {
      const int16_t* zr = a.zrange + (int64_t)pslot * kZrange;
      int lo = zr[wm0 + lane], hi = zr[kZld + wm0 + lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      wlo = lo;
      whi = hi;
    }
    const int boff = LEFT ? (int)(si.j1 & 1) : 0;
    double acc[2][8][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;
    for (int kc = 0; kc < pnk; ++kc, ++it) {
      const int st = it % C::NS;
      mbar_wait(&full[st], (it / C::NS) & 1);
      const double* As = (const double*)(smem + (size_t)st * C::STAGE);
      const double* Bs = (const double*)(smem + (size_t)st * C::STAGE + C::A_BYTES);
#pragma unroll
      for (int ks = 0; ks < KC; ks += 4) {
        const int kg = kc * KC + ks;
        if (kg + 3 < wlo || kg > whi) continue;   // Z^T rows of this warp are exact zeros here
        if (dbg & 2) continue;
        double a0[2], a1[2], bf[8];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double* ap = As + (wm0 + i * 16 + g) * LDA + ks + t;
          a0[i] = ap[0];
          a1[i] = ap[8 * LDA];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int xx = j * 8 + g;
          bf[j] = LEFT ? Bs[xx * LDBL + boff + ks + t] : Bs[(ks + t) * LDBR + xx];
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) mma_16x8x4(acc[i][j], a0[i], a1[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // every K chunk of this strip has landed and been consumed: overwrite in place
    double* M = a.M;
    const int64_t ld = a.ld;
    if (dbg & 32) {   // SN_TMA_DBG bit 32: no epilogue stores (timing probe only)
    } else if (!LEFT && (si.x0 & 1) == 0 && !(dbg & 16)) {   // SN_TMA_DBG bit 16: scalar stores (A/B)
      // right / Q: a lane's two accumulators of one row pair are adjacent strip rows (column-
      // major), 16-byte aligned (TMA-described M: aligned base, even ld; even x0): one 16-byte
      // store, four lanes filling 64 contiguous bytes of a column
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = wm0 + i * 16 + g + 8 * h;
            const int xx = j * 8 + 2 * t;
            if (m >= pk || xx >= si.nx) continue;
            double* dst = M + (si.x0 + xx) + (pjc + m) * ld;
            if (xx + 1 < si.nx) *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][2 * h], acc[i][j][2 * h + 1]);
            else dst[0] = acc[i][j][2 * h];
          }
    } else {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = wm0 + i * 16 + g + 8 * h;
          if (m >= pk) continue;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int xx = j * 8 + 2 * t + q;
            if (xx >= si.nx) continue;
            const double v = acc[i][j][2 * h + q];
            if (LEFT) M[(si.j1 + m) + (si.x0 + xx) * ld] = v;
            else M[(si.x0 + xx) + (pjc + m) * ld] = v;
          }
        }
    }
    if (p == 0 && !si.skip) {
      // the second pass's TMA loads read these columns: order the generic stores before the
      // async proxy, then release them to the producer
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(wb);
    }
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  return fn;
}

bool encode_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box0,
               uint32_t box1) {
  auto enc = get_encode();
  if (!enc) return false;
  if (((uintptr_t)base & 15) || ((ld_elems * 8) & 15) || inner == 0 || outer == 0) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 8};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MT, int KIND>
void launch_tma_t(const PanelArgs& a, int32_t nstrips, const PanelMaps& pm, cudaStream_t st) {
  using C = TCfg<MT>;
  static bool attr[kMaxDevices] = {};   // per device: the attribute is device state
  const int dslot = device_slot();
  if (!attr[dslot]) {
    cudaFuncSetAttribute(panel_tma_kernel<MT, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    attr[dslot] = true;
  }
  int grid = nstrips < 148 ? nstrips : 148;
  const int need = (nstrips + kMaxStripsPerCta - 1) / kMaxStripsPerCta;
  if (need > grid) grid = need;
  const CUtensorMap* mm = KIND == 0 ? &pm.mL : &pm.mRQ;
  if (std::getenv("SN_TMA_TRACE")) {
    std::vector<WinDev> w((size_t)a.nwin);
    std::vector<int32_t> pre((size_t)a.nwin + 1), stt((size_t)a.nwin);
    cudaStreamSynchronize(st);
    cudaMemcpy(w.data(), a.wins, sizeof(WinDev) * a.nwin, cudaMemcpyDeviceToHost);
    if (a.prefix) cudaMemcpy(pre.data(), a.prefix, sizeof(int32_t) * (a.nwin + 1), cudaMemcpyDeviceToHost);
    cudaMemcpy(stt.data(), a.status + a.base, sizeof(int32_t) * a.nwin, cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "tma kind %d MT %d nstrips %d n %lld ld %lld nwin %d base %d part %d M %p Z %p zr %p\n", KIND, MT,
                 nstrips, (long long)a.n, (long long)a.ld, a.nwin, a.base, a.part, (void*)a.M, (void*)a.Z,
                 (void*)a.zrange);
    for (int i = 0; i < a.nwin; ++i)
      std::fprintf(stderr, "  w%d j1 %lld k %d slot %d coff %lld sidx %d status %d prefix %d\n", i, (long long)w[i].j1,
                   w[i].k, w[i].slot, (long long)w[i].coff, w[i].sidx, stt[i], pre[i]);
  }
  // SN_TMA_DBG: timing probes (results are wrong when set); SN_TMA_DBG_KINDS: bit mask of the
  // kinds it applies to (default all)
  static const int dbg_all = [] {
    const char* e = std::getenv("SN_TMA_DBG");
    return e ? std::atoi(e) : 0;
  }();
  static const int dbg_kinds = [] {
    const char* e = std::getenv("SN_TMA_DBG_KINDS");
    return e ? std::atoi(e) : 15;
  }();
  const int dbg = (dbg_kinds >> KIND) & 1 ? dbg_all : 0;
  panel_tma_kernel<MT, KIND><<<grid, C::THREADS, C::SMEM, st>>>(a, nstrips, pm.z[MT == 256 ? 2 : MT == 128 ? 1 : 0],
                                                                *mm, dbg);
  if (std::getenv("SN_DEBUG")) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess)
      std::fprintf(stderr, "sn: panel_tma_kernel<%d,%d> grid %d smem %d: %s\n", MT, KIND, grid, (int)C::SMEM,
                   cudaGetErrorString(e));
  }
}

}  // namespace

// Tensor maps of one matrix (S or Q: rows x cols, ld) and of the Z slot array.  Returns
// false if TMA cannot describe them (then the cp.async kernel is used).
bool panel_maps_init(PanelMaps* pm, const double* Zbase, int64_t nslots, const double* M, int64_t rows, int64_t cols,
                     int64_t ld) {
  pm->valid = 0;
  if (std::getenv("SN_NO_TMA")) return false;
  bool ok = true;
  const int mts[3] = {64, 128, 256};
  for (int q = 0; q < 3; ++q)
    ok = ok && encode_2d(&pm->z[q], Zbase, kZld, (uint64_t)nslots * kZld, kZld, LDA, mts[q]);
  ok = ok && encode_2d(&pm->mL, M, rows, cols, ld, LDBL, NT);
  ok = ok && encode_2d(&pm->mRQ, M, rows, cols, ld, LDBR, KC);
  pm->valid = ok ? 1 : 0;
  return ok;
}

void launch_panel_tma(int kind, int mt, const PanelArgs& a, int32_t nstrips, const PanelMaps& pm, cudaStream_t st) {
  if (nstrips <= 0) return;
  if (mt <= 64) {
    if (kind == 0) launch_tma_t<64, 0>(a, nstrips, pm, st);
    else if (kind == 1) launch_tma_t<64, 1>(a, nstrips, pm, st);
    else if (a.fuse) launch_tma_t<64, 3>(a, nstrips, pm, st);
    else launch_tma_t<64, 2>(a, nstrips, pm, st);
  } else if (mt <= 128) {
    if (kind == 0) launch_tma_t<128, 0>(a, nstrips, pm, st);
    else if (kind == 1) launch_tma_t<128, 1>(a, nstrips, pm, st);
    else if (a.fuse) launch_tma_t<128, 3>(a, nstrips, pm, st);
    else launch_tma_t<128, 2>(a, nstrips, pm, st);
  } else {
    if (kind == 0) launch_tma_t<256, 0>(a, nstrips, pm, st);
    else if (kind == 1) launch_tma_t<256, 1>(a, nstrips, pm, st);
    else if (a.fuse) launch_tma_t<256, 3>(a, nstrips, pm, st);
    else launch_tma_t<256, 2>(a, nstrips, pm, st);
  }
}

}  // namespace sn
