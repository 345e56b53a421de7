// sn_kernels_panel.cu -- the right/left update tasks ("applies
// accumulated right-hand [left-hand] side updates using level-3 BLAS operations") and the
// Q update (Q <- Q*Q3), as in-place FP64 tensor-core GEMMs on sm_100a.
//
//   left  (kind 0):  S[j1:j2, c0:c0+NT]  <- Z^T * S[j1:j2, c0:c0+NT]     (row panel right)
//   right (kind 1):  S[r0:r0+NT, j1:j2]  <- S[r0:r0+NT, j1:j2] * Z       (column panel above)
//   Q     (kind 2):  Q[r0:r0+NT, j1:j2]  <- Q[r0:r0+NT, j1:j2] * Z
//
// One CTA owns one strip for the whole K = k extent, so the strip can be overwritten in
// place after its last K chunk is consumed (no other CTA touches it).  All three kinds are
// the same product  C[m][x] = sum_kk Z[kk][m] * B[kk][x]  with A = Z^T from the Z slot and B
// the strip (x = column for left, row for right/Q).  Operands are staged through shared
// memory with a 3-stage cp.async pipeline and multiplied with mma.sync.m16n8k4.f64 (DMMA),
// the FP64 tensor-core path of sm_100 (tcgen05 has no f64 kind).  DESIGN.md §6.
#include <cstdint>
#include <cstdlib>

#include "sn_device.cuh"

namespace sn {
namespace {

constexpr int KC = 16;        // K chunk
constexpr int LDA = KC + 4;   // As[m][kk], row stride == 4 mod 16 (conflict-free fragments)
constexpr int NSTAGE = 3;

__device__ __forceinline__ void mma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async16z(void* dst, const void* src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

template <int MT, int NT, int KIND, int THREADS>
struct Cfg {
  static constexpr bool LEFT = (KIND == 0);
  static constexpr int WN = 2, WM = THREADS / 32 / WN;
  static constexpr int MI = MT / (WM * 16);   // m16 tiles per warp
  static constexpr int NI = NT / (WN * 8);    // n8 tiles per warp
  static constexpr int LDB = LEFT ? (KC + 4) : (NT + 4);   // Bs[x][kk] (left) or Bs[kk][x]
  static constexpr int A_ELEMS = MT * LDA;
  static constexpr int B_ELEMS = LEFT ? NT * LDB : KC * LDB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = sizeof(double) * (size_t)STAGE * NSTAGE;
};

template <int MT, int NT, int KIND, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) panel_kernel(PanelArgs a) {
  using C = Cfg<MT, NT, KIND, THREADS>;
  constexpr int kThreads = THREADS;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;

  double* M = a.M;
  int w, nx;       // window index within the level; valid columns (left) or rows (right/Q)
  int64_t x0;      // first column (left) or row (right/Q) of the strip
  if (a.strips) {
    // explicit segments (sharded executor, sn_dist.h)
    const int sid = blockIdx.x;
    int lo = 0, hi = a.nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.prefix[mid] <= sid) lo = mid; else hi = mid - 1;
    }
    const StripDev sd = a.strips[lo];
    const int idx = sid - a.prefix[lo];
    w = sd.w;
    x0 = sd.x0 + (int64_t)idx * NT;
    nx = min(NT, sd.cnt - idx * NT);
  } else {
    // strip -> (window, index) by binary search over the level's prefix
    const int sid = blockIdx.x;
    int lo = 0, hi = a.nwin - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.prefix[mid] <= sid) lo = mid; else hi = mid - 1;
    }
    w = lo;
    const WinDev& wq = a.wins[w];
    int strip = sid - a.prefix[w];
    // critical strips (read by the next level's windows): a prefix of the left strips, a
    // suffix of the right strips
    if (KIND == 0 && a.part == 2) strip += wq.crit_l;
    if (KIND == 1 && a.part == 1) strip += (int)((wq.j1 + NT - 1) / NT) - wq.crit_r;
    if (C::LEFT) {
      x0 = wq.j1 + wq.k + (int64_t)strip * NT;
      nx = (int)min((int64_t)NT, a.n - x0);
    } else {
      x0 = (int64_t)strip * NT;
      const int64_t lim = (KIND == 1) ? wq.j1 : a.n;
      nx = (int)min((int64_t)NT, lim - x0);
    }
  }
  if (a.status[a.base + w] == kWinSkipped) return;
  const WinDev wd = a.wins[w];
  const int k = wd.k;
  const int64_t j1 = wd.j1, ld = a.ld;
  // first column of the window's columns in M (right update: S may be stored with a column
  // offset; Q and the left update's row index use the global index)
  const int64_t jc = (KIND == 1) ? j1 + wd.coff : j1;
  const double* Z = a.Z + (int64_t)wd.slot * kZslot;
  const int nk = (k + KC - 1) / KC;
  // Z structure: output rows m of a 16-row tile only need the K rows where
  // one of the tile's Z columns is nonzero; outside that interval the DMMAs (and the A
  // loads) are skipped.  The skipped products are exact zeros, so results are unchanged.
  __shared__ int16_t s_tlo[MT / 16], s_thi[MT / 16];
  if (tid < MT / 16) {
    const int16_t* zr = a.zrange + (int64_t)wd.slot * kZrange;
    int lo = kZld, hi = -1;
    for (int c = 16 * tid; c < 16 * tid + 16; ++c) { lo = min(lo, (int)zr[c]); hi = max(hi, (int)zr[kZld + c]); }
    s_tlo[tid] = (int16_t)lo;
    s_thi[tid] = (int16_t)hi;
  }
  __syncthreads();

  auto load_stage = [&](int stage, int kc) {
    double* As = smem + stage * C::STAGE;
    double* Bs = As + C::A_ELEMS;
    const int kk0 = kc * KC;
    // A = Z^T chunk: As[m][kk] = Z[kk0 + kk + m*256]; 16-byte copies, 8 per row
    for (int idx = tid; idx < MT * (KC / 2); idx += kThreads) {
      const int m = idx / (KC / 2), part = idx % (KC / 2);
      cp_async16(As + m * LDA + part * 2, Z + (int64_t)m * kZld + kk0 + part * 2);
    }
    if (C::LEFT) {
      // Bs[c][kk] = M[(j1 + kk0 + kk) + (x0 + c)*ld]
      for (int idx = tid; idx < NT * KC; idx += kThreads) {
        const int c = idx / KC, kk = idx % KC;
        const bool v = (c < nx) && (kk0 + kk < k);
        const double* src = v ? M + (j1 + kk0 + kk) + (x0 + c) * ld : M;
        cp_async8(Bs + c * C::LDB + kk, src, v);
      }
    } else if (a.vec16) {
      // Bs[kk][r..r+1] = M[(x0 + r) + (j1 + kk0 + kk)*ld], 16-byte copies (x0 is a multiple
      // of NT, ld is even and M 16-byte aligned), zero-filled past the strip
      for (int idx = tid; idx < NT * KC / 2; idx += kThreads) {
        const int kk = idx / (NT / 2), r = 2 * (idx % (NT / 2));
        const int nb = (kk0 + kk < k) ? 8 * max(0, min(2, nx - r)) : 0;
        const double* src = nb ? M + (x0 + r) + (jc + kk0 + kk) * ld : M;
        cp_async16z(Bs + kk * C::LDB + r, src, nb);
      }
    } else {
      // Bs[kk][r] = M[(x0 + r) + (j1 + kk0 + kk)*ld]
      for (int idx = tid; idx < NT * KC; idx += kThreads) {
        const int kk = idx / NT, r = idx % NT;
        const bool v = (r < nx) && (kk0 + kk < k);
        const double* src = v ? M + (x0 + r) + (jc + kk0 + kk) * ld : M;
        cp_async8(Bs + kk * C::LDB + r, src, v);
      }
    }
  };

  double acc[C::MI][C::NI][4];
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;

  const int wm0 = (warp % C::WM) * (MT / C::WM);
  const int wn0 = (warp / C::WM) * (NT / C::WN);
  // K interval of this warp's output rows (warp-uniform: the skip is one branch per k4 step)
  int wlo = kZld, whi = -1;
#pragma unroll
  for (int i = 0; i < C::MI; ++i) {
    wlo = min(wlo, (int)s_tlo[(wm0 >> 4) + i]);
    whi = max(whi, (int)s_thi[(wm0 >> 4) + i]);
  }

#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_wait<NSTAGE - 2>();
    __syncthreads();
    // prefetch chunk kc + NSTAGE - 1 into the stage freed by chunk kc - 1
    if (kc + NSTAGE - 1 < nk) load_stage((kc + NSTAGE - 1) % NSTAGE, kc + NSTAGE - 1);
    cp_commit();
    const double* As = smem + (kc % NSTAGE) * C::STAGE;
    const double* Bs = As + C::A_ELEMS;
    // k4-outer order: between two dependent DMMAs on one accumulator the warp issues
    // MI*NI-1 independent ones (the m16n8k8 form chains two 8x8x4 DMMAs back to back).
#pragma unroll
    for (int ks = 0; ks < KC; ks += 4) {
      const int kg = kc * KC + ks;
      if (kg + 3 < wlo || kg > whi) continue;   // Z^T rows of this warp are exact zeros here
      double a0[C::MI], a1[C::MI], bf[C::NI];
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        const double* ap = As + (wm0 + i * 16 + g) * LDA + ks + t;
        a0[i] = ap[0];
        a1[i] = ap[8 * LDA];
      }
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        const int xx = wn0 + j * 8 + g;
        bf[j] = C::LEFT ? Bs[xx * C::LDB + ks + t] : Bs[(ks + t) * C::LDB + xx];
      }
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) mma_16x8x4(acc[i][j], a0[i], a1[i], bf[j]);
    }
  }
  cp_wait<0>();
  // every K chunk of this strip has been read by this CTA: overwrite in place
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = wm0 + i * 16 + g + 8 * h;
        if (m >= k) continue;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int xx = wn0 + j * 8 + 2 * t + q;
          if (xx >= nx) continue;
          const double v = acc[i][j][2 * h + q];
          if (C::LEFT) M[(j1 + m) + (x0 + xx) * ld] = v;
          else M[(x0 + xx) + (jc + m) * ld] = v;
        }
      }
}

template <int MT, int NT, int KIND, int THREADS>
void launch_t(const PanelArgs& a, int32_t nstrips, cudaStream_t st) {
  using C = Cfg<MT, NT, KIND, THREADS>;
  static bool attr[kMaxDevices] = {};   // per device: the attribute is device state
  const int dslot = device_slot();
  if (!attr[dslot]) {
    cudaFuncSetAttribute(panel_kernel<MT, NT, KIND, THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM);
    attr[dslot] = true;
  }
  panel_kernel<MT, NT, KIND, THREADS><<<nstrips, THREADS, C::SMEM, st>>>(a);
}

template <int KIND>
void launch_kind(int mt, const PanelArgs& a, int32_t nstrips, cudaStream_t st) {
  static const int wide = [] {
    const char* e = std::getenv("SN_PANEL_THREADS");
    return e ? std::atoi(e) : 512;
  }();
  if (mt <= 64) launch_t<64, 64, KIND, 256>(a, nstrips, st);
  else if (mt <= 128) launch_t<128, 64, KIND, 256>(a, nstrips, st);
  else if (wide == 256) launch_t<256, 64, KIND, 256>(a, nstrips, st);
  else launch_t<256, 64, KIND, 512>(a, nstrips, st);
}

}  // namespace

int panel_strip_width(int kind, int mt) { (void)kind; (void)mt; return 64; }

void launch_panel(int kind, int mt, const PanelArgs& a, int32_t nstrips, cudaStream_t st) {
  if (nstrips <= 0) return;
  if (a.maps && a.maps->valid) {
    launch_panel_tma(kind, mt, a, nstrips, *a.maps, st);
    return;
  }
  if (kind == 0) launch_kind<0>(mt, a, nstrips, st);
  else if (kind == 1) launch_kind<1>(mt, a, nstrips, st);
  else launch_kind<2>(mt, a, nstrips, st);
}

}  // namespace sn
