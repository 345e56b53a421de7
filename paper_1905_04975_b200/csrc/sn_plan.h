// sn_plan.h -- host-side execution plan of the reordering (product code).
//
// The plan is the window schedule of SURVEY §8c-2 (our reading of PAPER.md P:156-158,
// P:167-175 "chains of diagonal windows", "inserted in a sequentially consistent
// order"), refined for the GPU:
//   * every window also carries an inner schedule (windows of <= inner_window rows inside
//     the outer window, executed by the window kernel from shared memory; the same chain
//     rules applied recursively to the window's own block list);
//   * windows are grouped into dependency levels of the window DAG: a window's level is
//     1 + the highest level of the earlier windows whose row range intersects its own.
//     Windows of one level touch pairwise disjoint diagonal ranges and run concurrently
//     ("multiple diagonal windows can be processed simultaneously").
#pragma once
#include <cstdint>
#include <vector>

namespace sn {

struct WindowPlan {
  int64_t j1 = 0;         // first row of the window
  int32_t k = 0;          // rows
  int32_t nblk = 0;       // blocks in the window
  int32_t ninner = 0;     // inner windows
  int32_t level = 0;      // DAG level (0-based)
  int64_t pool = 0;       // byte offset: sz[nblk], sel[nblk], pad to 2, inner (uint16 top,bottom)*ninner
  int64_t nswap = 0;
  int64_t swaps_by_type[4] = {0, 0, 0, 0};
  int64_t order = 0;      // index in schedule order
  int64_t top = 0;        // first block index of the window (block list before the window)
};

struct Plan {
  int64_t n = 0, w = 0, kin = 0;
  std::vector<WindowPlan> wins;     // schedule order
  std::vector<uint8_t> pool;
  int64_t nlevels = 0;
  int64_t nswap = 0;
  int64_t ninner = 0;
  // final block list (after all planned windows)
  std::vector<uint8_t> final_sz, final_sel;
};

// Builds the plan.  bmap: 0 = 1x1, 1/2 = rows of a 2x2; selrow: 0/1 per row (block
// consistent).  max_windows < 0: all windows.  Returns 0 or a negative error.
int build_plan(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w, int64_t kin,
               int64_t max_windows, Plan* plan);

// Lookahead split of the left/right update strips (strip width NT), per window in schedule
// order: crit_l = leading left strips, crit_r = trailing right strips that must be applied
// before the next level's window kernel.
void lookahead_strips(const Plan& plan, int64_t NT, std::vector<int32_t>& crit_l, std::vector<int32_t>& crit_r);

// Swap list of window t in kernel execution order (inner windows, movers top to bottom).
int64_t window_swaps(const Plan& plan, int64_t t, int64_t cap, int64_t* sj, int8_t* s1, int8_t* s2);

}  // namespace sn
