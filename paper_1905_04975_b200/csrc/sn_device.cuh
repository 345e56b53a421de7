// sn_device.cuh -- device-side data layout shared by the executor and the kernels.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

namespace sn {

constexpr int kZld = 256;                 // Z slots are 256 x 256, column-major, ld 256
constexpr int64_t kZslot = (int64_t)kZld * kZld;
// Structure of Z: every column c of a window's accumulator is nonzero only in
// the rows [lo[c], hi[c]] (an interval containing c: each swap mixes adjacent columns, so the
// union of their intervals is again an interval).  Per Z slot, int16 lo[256] then hi[256];
// columns >= k hold the empty interval (lo = 255, hi = 0).  Entries outside are exact zeros.
constexpr int kZrange = 2 * kZld;
constexpr int kInner = 64;                // max rows of an in-kernel inner window

// One window, as seen by the kernels (sorted by level).
struct WinDev {
  int64_t j1;        // first row of the window
  int32_t k;         // rows
  int32_t nblk;      // blocks
  int32_t ninner;    // inner windows
  int32_t slot;      // Z slot
  int64_t pool;      // byte offset of sz[nblk], sel[nblk], (pad), inner[2*ninner] (uint16)
  int64_t order;     // schedule order
  int32_t crit_l;    // left-update strips (a prefix) read by the next level's windows
  int32_t crit_r;    // right-update strips (a suffix) read by the next level's windows
  int64_t coff;      // column offset: column j of S is stored at column j + coff of the
                     // array passed (0 on one GPU; the extended local layout when sharded)
  int32_t sidx;      // index of this window in the status array (level-sorted order)
  int32_t qprev;     // fused chain Q update (PanelArgs.fuse): 1 + level-sorted index of the
                     // chain predecessor whose Q update this window's Q launch applies first
                     // (0: none)
};

// One panel segment given explicitly (the sharded executor, sn_dist.h): window index within
// the level, columns (left) or rows (right, Q), and the first column / row.  A segment is
// processed as ceil(cnt / 64) strips of 64.
struct StripDev {
  int32_t w;
  int32_t cnt;
  int64_t x0;
};

// Per-call device control block.
struct Control {
  int32_t abort;            // set by a window kernel that rejected a swap
  int32_t abort_level;      // 1 + DAG level of the rejecting window(s) (claimed by atomicCAS):
                            // windows of later levels are skipped, every window of that level
                            // runs (levels are row-disjoint), so the outcome does not depend on
                            // CTA scheduling
  int32_t rej_window;       // sorted index of the rejecting window (pencil path)
  int32_t rej_swaps_done;   // swaps completed in that window before the rejected one (pencil)
  int32_t rej_row;          // global first row of the rejected swap (pencil path)
  int32_t rej_n1, rej_n2;
  int32_t pad[2];
  unsigned long long ratio_bits;  // pencil path: largest G3 residual ratio of an accepted swap
                                  // (the bits of a non-negative double: ordered as integers)
};

// Per-window rejection record (standard path): a window that rejects a swap stores the number
// of swaps it completed, the rejected pair and its block list after the last good swap here,
// indexed by its sorted index; several windows of one level may reject.  Zero-initialised,
// written only by the owning CTA (the sharded executor combines ranks with a max all-reduce).
struct WinRec {
  int32_t done;             // swaps completed before the rejection
  int32_t row;              // global first row of the rejected swap
  int32_t n1, n2;           // its block sizes
  uint8_t sz[256];          // block list of [top, top + nblk) after the last good swap
  uint8_t sel[256];
};

// status[] of a window: 0 not executed, 1 complete, 2 partial (rejected inside; Z valid)
enum : int32_t { kWinSkipped = 0, kWinDone = 1, kWinPartial = 2 };

struct WindowArgs {
  const WinDev* wins;       // this level's windows
  int32_t nwin;
  int32_t base;             // sorted index of wins[0]
  const uint8_t* pool;
  double* S;
  int64_t ldS;
  double* Z;                // slot array base
  int16_t* zrange;          // per slot: nonzero row interval of every Z column
  int32_t* status;          // indexed by sorted index
  Control* ctl;
  WinRec* recs;             // per sorted index: rejection records
  int32_t level;            // DAG level of this launch
  unsigned long long* tprof;  // debug: per-phase cycle counters (NULL: off)
  int32_t* kwork;           // per sorted index: k4 steps the panel kernels execute per strip,
                            // summed over the 32-row groups of Z^T (Z-structure skipping)
  int64_t force_order;      // debug: schedule order of the window to reject in (-1 none)
  int32_t force_swap;       // debug: swap index (execution order) to reject
};

// TMA descriptors of one panel launch target (host side; passed to the kernels by value as
// __grid_constant__ parameters): the Z slot array for MT = 64/128/256 and the matrix M (S or Q)
// for the left (K rows x 64 columns) and right/Q (68 rows x 16 K columns) boxes.
struct PanelMaps {
  CUtensorMap z[3];
  CUtensorMap mL, mRQ;
  int valid;
};

struct PanelArgs {
  const WinDev* wins;       // this level's windows
  int32_t nwin;
  int32_t base;
  const int32_t* prefix;    // nwin+1 cumulative strip counts of this kind and part
  const StripDev* strips;   // explicit segments (sharded executor): then prefix[0..nseg] holds
                            // the strips before each segment
  int32_t nseg;
  int32_t part;             // 0 all strips, 1 the critical strips, 2 the remaining strips
  int32_t vec16;            // M is 16-byte aligned and ld is even: 16-byte row-strip copies
  const int32_t* status;
  double* M;                // S (left/right) or Q
  int64_t ld;
  int64_t n;
  const double* Z;
  const int16_t* zrange;    // per slot row intervals of Z's columns (window kernel output)
  const PanelMaps* maps;    // host pointer: TMA descriptors (NULL or !valid: cp.async kernel)
  int32_t fuse;             // Q kind, TMA kernel only: apply WinDev.qprev's Z to a strip, then
                            // this window's Z, in one pass of the CTA (row f1)
  int32_t pad;
};

// per-device launch state (function attributes are set once per device)
constexpr int kMaxDevices = 64;
inline int device_slot() {
  int d = 0;
  cudaGetDevice(&d);
  return d < kMaxDevices ? d : kMaxDevices - 1;
}

// kernel launchers (sn_kernels_*.cu)
void launch_scan(const double* S, int64_t ldS, int64_t n, int32_t validate_lower, uint8_t* subflag,
                 int32_t* bad, cudaStream_t st);
// sharded S (extended local layout, sn_dist.h): flags of the columns this rank owns
void launch_scan_dist(const double* Sx, int64_t ldx, int64_t n, int64_t P, int64_t bc, int64_t hc, int64_t rank,
                      int32_t validate_lower, uint8_t* subflag, int32_t* bad, cudaStream_t st);
void launch_window(const WindowArgs& a, cudaStream_t st);
size_t window_smem_bytes();
// kind: 0 = left update of S, 1 = right update of S, 2 = Q update; mt = 64/128/256
void launch_panel(int kind, int mt, const PanelArgs& a, int32_t nstrips, cudaStream_t st);
int panel_strip_width(int kind, int mt);
// TMA path (sn_kernels_panel_tma.cu)
bool panel_maps_init(PanelMaps* pm, const double* Zbase, int64_t nslots, const double* M, int64_t rows, int64_t cols,
                     int64_t ld);
void launch_panel_tma(int kind, int mt, const PanelArgs& a, int32_t nstrips, const PanelMaps& pm, cudaStream_t st);

}  // namespace sn
