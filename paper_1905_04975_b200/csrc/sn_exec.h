// sn_exec.h -- host helpers shared by the one-GPU executor (sn_abi.cu) and the sharded
// executor (sn_dist_exec.cu).  Product code.
#pragma once
#include <cstdint>
#include <mutex>
#include <vector>

#include "sn_device.cuh"
#include "sn_plan.h"

namespace sn {

extern std::mutex g_mu;   // the library's device state is used by one call at a time

double now_ms();
bool is_device_ptr(const void* p);

// a1 on the host: block map and per-row selection from the subdiagonal flags (a 2x2 block is
// selected if either row is); m = selected rows.  Returns 0 or -2 (not quasi-triangular).
int structure_from_sub(int64_t n, const uint8_t* sub, const int32_t* select, int8_t* bmap, int8_t* selrow,
                       int64_t* m);

// Final block list after a run: the plan's final list, or, after a rejection, the list of the
// windows that completed plus each partial window's own record (recs, by sorted index).
// rej_sorted: the first partial window in schedule order (sorted index), or -1.
void final_blocks(const Plan& P, const std::vector<int64_t>& sorted, bool aborted, const int32_t* status,
                  const WinRec* recs, int64_t n, const int8_t* bmap, const int8_t* selrow, std::vector<uint8_t>& fsz,
                  std::vector<uint8_t>& fsel, int64_t* executed, int64_t* swaps, int64_t sbt[4], int64_t* rej_sorted);

// select (per-row achieved mask) and bmap_out (may be NULL) from a block list
void write_blocks(const std::vector<uint8_t>& fsz, const std::vector<uint8_t>& fsel, int32_t* select,
                  int8_t* bmap_out);

}  // namespace sn
