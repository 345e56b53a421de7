// sn_dist.h -- host-side program of the multi-GPU reordering (product code).
//
// Partitioning (one process per GPU, P ranks):
//   * S: 1-D block-cyclic over column blocks of width bc: global column j lives in block
//     b = j / bc on rank b % P, with all n rows.  Internally every owned block is followed
//     by a halo slot of hc = w columns (the "extended" layout), so that a window whose
//     columns straddle into the next block [c, j2) can be made contiguous on its owner.
//   * Q: contiguous row blocks of ceil(n/P) rows.
// Per dependency level of the window DAG (P:158 concurrent windows, P:184
// sequentially consistent order), every rank executes the same phase sequence:
//   1 PULL   straddling windows: partner -> owner, S[0:j2, c:j2] into the owner's halo slot
//   2 W      window tasks on the owner (the rank of column j1), Z into a slot
//   3 SYNC   broadcast of every Z from its owner (NCCL over NVLink), window status max-reduce
//   4 L      left update S[j1:j2, j2:n] <- Z^T S on every rank, its own columns (plus the
//            halo slots it holds this level, minus the columns it lent this level)
//   5 R      right update S[0:j1, j1:j2] <- S Z on the owner (contiguous via the halo slot)
//   6 PUSH   owner -> partner, S[0:j2, c:j2] back from the halo slot
//   7 Q      Q[:, j1:j2] <- Q Z on every rank, its own rows
// Lookahead: steps 4-5 run only the *critical* strips before the push -- the strips the next
// level's window tasks read, the strips on columns the next level pulls, the
// halo strips and every right strip of a straddling window; the remaining strips run on a
// second stream after the push, overlapping the next level's pulls and window tasks, and the
// next level's updates wait for them.
// The program is a pure function of (plan, n, P, bc, w, rank): identical on every rank,
// so the collectives match by construction.  It is exported (sn_dist_program) so that the
// CPU tests can interpret it with gloo (tests/test_dist_program.py).
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

#include "sn_device.cuh"
#include "sn_plan.h"

namespace sn {

struct DistLayout {
  int64_t n = 0, P = 1, bc = 256, hc = 256;
  int64_t nblocks() const { return (n + bc - 1) / bc; }
  int64_t owner_of_col(int64_t j) const { return (j / bc) % P; }
  int64_t nblk_of(int64_t r) const { return r < nblocks() ? (nblocks() - r + P - 1) / P : 0; }
  // extended (internal) layout: owned block lb at local columns [lb*(bc+hc), lb*(bc+hc)+bc),
  // its halo slot at [lb*(bc+hc)+bc, (lb+1)*(bc+hc))
  int64_t ext_cols(int64_t r) const { return nblk_of(r) * (bc + hc); }
  int64_t ext_lcol(int64_t j) const {
    const int64_t b = j / bc;
    return (b / P) * (bc + hc) + (j - b * bc);
  }
  // local column, in the halo slot of block b-1, of global column j of block b
  int64_t halo_lcol(int64_t j) const {
    const int64_t b = j / bc - 1;
    return (b / P) * (bc + hc) + bc + (j - (b + 1) * bc);
  }
  // user (compact) layout: owned block lb at local columns [lb*bc, (lb+1)*bc)
  int64_t user_cols(int64_t r) const { return nblk_of(r) * bc; }
  int64_t user_lcol(int64_t j) const {
    const int64_t b = j / bc;
    return (b / P) * bc + (j - b * bc);
  }
  int64_t qrows_per() const { return (n + P - 1) / P; }
  int64_t q0(int64_t r) const { return std::min(n, r * qrows_per()); }
  int64_t q1(int64_t r) const { return std::min(n, (r + 1) * qrows_per()); }
};

struct DistWin {            // one window, in level-sorted order
  int64_t t = 0;            // schedule order
  int64_t j1 = 0;
  int32_t k = 0;
  int32_t level = 0;
  int32_t owner = 0;        // rank of column j1
  int32_t partner = -1;     // rank of column j2-1 when the window straddles a block boundary
  int64_t c = -1;           // first column of the partner's block (straddle), else -1
  int64_t coff = 0;         // on the owner: extended local column of global j is j + coff
};

struct DistMsg {            // S[0:nrows, gcol:gcol+ncols] between two ranks
  int32_t src = 0, dst = 0;
  int64_t w = 0;            // level-sorted window index
  int64_t nrows = 0, gcol = 0, ncols = 0;
  int64_t src_lcol = 0, dst_lcol = 0;   // extended local columns on src / dst
};

// one panel strip (CTA) of a level: window index within the level, columns (L) or rows
// (R, Q), first extended local column (L) or row (R, Q)
using DistStrip = StripDev;

struct DistLevel {
  int64_t w0 = 0, w1 = 0;                       // level-sorted window range
  std::vector<int64_t> pulls, pushes;           // indices into msgs
  std::vector<int64_t> own;                     // level-sorted indices owned by this rank
  // ranges in strips: critical left/right strips (before the push and the next level's
  // pulls and window tasks), the remaining ones (overlapping the next level's window tasks),
  // and the Q strips
  int64_t L0 = 0, L1 = 0, R0 = 0, R1 = 0, Lr0 = 0, Lr1 = 0, Rr0 = 0, Rr1 = 0, Q0 = 0, Q1 = 0;
  // per group (L, R, Lr, Rr, Q): offset of its strip prefix in DistProgram::sprefix (segments + 1
  // entries) and its number of strips
  int64_t poff[5] = {0, 0, 0, 0, 0};
  int32_t nstr[5] = {0, 0, 0, 0, 0};
};

struct DistProgram {
  DistLayout lay;
  int64_t rank = 0;
  std::vector<DistWin> wins;       // level-sorted (identical on every rank)
  std::vector<int64_t> sorted;     // level-sorted index -> schedule order
  std::vector<DistMsg> msgs;       // all ranks' messages
  std::vector<DistStrip> strips;   // this rank's segments (ranges of strips of `strip`)
  std::vector<int32_t> sprefix;    // per group, strips before each segment (DistLevel::poff)
  std::vector<DistLevel> levels;
  int64_t max_level_wins = 0;
  int64_t max_msg_bytes = 0;       // largest per-level staging need of this rank (bytes)
};

// Builds rank `rank`'s program.  strip = 64 (panel CTA width).  Returns 0 or -i.
int build_dist_program(const Plan& plan, const DistLayout& lay, int64_t rank, int64_t strip, DistProgram* prog);

}  // namespace sn
