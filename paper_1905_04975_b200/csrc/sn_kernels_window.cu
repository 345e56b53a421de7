// sn_kernels_window.cu -- the window task ("applies a set of local
// transformations inside the diagonal window ... produces updated tiles and an accumulator
// matrix as output").
//
// One CTA per window of a DAG level.  The window (k <= 256 rows) is processed as a chain of
// inner windows of <= 64 rows (the plan's inner schedule): each inner window
// is staged in shared memory, its block swaps run warp-cooperatively (sn_swap.cuh) into an
// inner accumulator Zin, and Zin is then applied with FP64 DMMA (mma.sync m16n8k8 f64) to
// the rest of the outer window and to the outer accumulator Z -- the paper's accumulated
// level-3 update, one level down.  The outer Z is left in a 256x256 slot for
// the panel kernels.
#include <cstdint>

#include "sn_device.cuh"
#include "sn_swap.cuh"

namespace sn {
namespace {

constexpr int kThreads = 256;
constexpr int LDD = 65;   // inner window (odd stride: conflict-free row walks)
constexpr int LDZ = 68;   // inner accumulator (== 4 mod 16: conflict-free DMMA fragments)
constexpr int LDT = 68;   // staging tile

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

__global__ void __launch_bounds__(kThreads, 1) window_kernel(WindowArgs a) {
  extern __shared__ __align__(16) double smem[];
  double* Din = smem;                       // kInner x LDD
  double* Zin = Din + kInner * LDD;         // kInner x LDZ
  double* Tb = Zin + kInner * LDZ;          // 64 x LDT
  __shared__ uint8_t bsz[256], bsel[256];
  __shared__ int16_t brow[257];
  __shared__ int s_rej, s_done_swaps, s_rej_row, s_rej_n1, s_rej_n2;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int widx = blockIdx.x;
  const WinDev wd = a.wins[widx];
  const int sidx = a.base + widx;
  if (*(volatile int32_t*)&a.ctl->abort) {
    if (tid == 0) a.status[sidx] = kWinSkipped;
    return;
  }
  const int k = wd.k, nb = wd.nblk;
  const uint8_t* pool = a.pool + wd.pool;
  for (int b = tid; b < nb; b += kThreads) { bsz[b] = pool[b]; bsel[b] = pool[nb + b]; }
  int64_t ioff = wd.pool + 2 * nb;
  ioff += ioff & 1;
  const uint16_t* inner = reinterpret_cast<const uint16_t*>(a.pool + ioff);
  double* S = a.S;
  const int64_t ld = a.ldS;
  const int64_t j1 = wd.j1;
  double* Z = a.Z + (int64_t)wd.slot * kZslot;
  // Z <- I (k x k, zero padded to 256 x 256)
  for (int idx = tid; idx < kZld * kZld; idx += kThreads) {
    const int r = idx & (kZld - 1), c = idx >> 8;
    Z[idx] = (r == c && r < k) ? 1.0 : 0.0;
  }
  if (tid == 0) {
    s_rej = 0; s_done_swaps = 0;
  }
  __syncthreads();
  if (tid == 0) {
    int r = 0;
    for (int b = 0; b < nb; ++b) { brow[b] = (int16_t)r; r += bsz[b]; }
    brow[nb] = (int16_t)r;
  }
  __syncthreads();

  int swaps_done = 0;
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
    if (warp == 0) {
      // movers of [top, bottom) in top-to-bottom order; mover im ends at block top+im
      int im = 0;
      bool rej = false;
      for (int b = top; b < bottom && !rej; ++b) {
        if (!bsel[b]) continue;
        for (int p = b; p > top + im; --p) {
          const int jl = brow[p - 1] - i1;
          const int n1 = bsz[p - 1], n2 = bsz[p];
          bool r = (wd.order == a.force_order && swaps_done == a.force_swap);
          if (!r) r = dev::warp_swap(Din, LDD, kin, jl, n1, n2, Zin, LDZ, kin, lane);
          if (r) {
            if (lane == 0) {
              s_rej = 1;
              s_rej_row = (int)(j1 + i1 + jl);
              s_rej_n1 = n1;
              s_rej_n2 = n2;
            }
            rej = true;
            break;
          }
          ++swaps_done;
          if (lane == 0) {
            const uint8_t ts = bsz[p - 1], tl = bsel[p - 1];
            bsz[p - 1] = bsz[p]; bsel[p - 1] = bsel[p];
            bsz[p] = ts; bsel[p] = tl;
            brow[p] = (int16_t)(brow[p - 1] + bsz[p - 1]);
          }
          __syncwarp();
        }
        ++im;
      }
      if (lane == 0) s_done_swaps = swaps_done;
    }
    __syncthreads();
    swaps_done = s_done_swaps;
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
    if (s_rej) break;
  }
  if (tid == 0) {
    if (s_rej) {
      a.ctl->abort = 1;
      a.ctl->rej_window = sidx;
      a.ctl->rej_swaps_done = swaps_done;
      a.ctl->rej_row = s_rej_row;
      a.ctl->rej_n1 = s_rej_n1;
      a.ctl->rej_n2 = s_rej_n2;
      for (int b = 0; b < nb; ++b) { a.ctl->rej_sz[b] = bsz[b]; a.ctl->rej_sel[b] = bsel[b]; }
      a.status[sidx] = kWinPartial;
    } else {
      a.status[sidx] = kWinDone;
    }
  }
}

}  // namespace

size_t window_smem_bytes() {
  return sizeof(double) * (size_t)(kInner * LDD + kInner * LDZ + 64 * LDT);
}

void launch_window(const WindowArgs& a, cudaStream_t st) {
  static bool attr = false;
  const size_t smem = window_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (a.nwin > 0) window_kernel<<<a.nwin, kThreads, smem, st>>>(a);
}

}  // namespace sn
