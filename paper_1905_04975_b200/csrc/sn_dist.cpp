// sn_dist.cpp -- the per-rank program of the multi-GPU reordering (see sn_dist.h).
#include "sn_dist.h"

#include <algorithm>
#include <cstdint>
#include <utility>

namespace sn {

namespace {

// split [a, b) into chunks of <= strip
void push_strips(std::vector<DistStrip>& out, int32_t w, int64_t a, int64_t b, int64_t strip) {
  for (int64_t x = a; x < b; x += strip) {
    DistStrip s;
    s.w = w;
    s.x0 = x;
    s.cnt = (int32_t)std::min(strip, b - x);
    out.push_back(s);
  }
}

}  // namespace

int build_dist_program(const Plan& plan, const DistLayout& lay, int64_t rank, int64_t strip, DistProgram* prog) {
  if (lay.P < 1 || rank < 0 || rank >= lay.P) return -1;
  if (lay.bc < plan.w || lay.hc < plan.w || lay.bc < 1) return -2;
  if (strip < 1) return -3;
  DistProgram& D = *prog;
  D = DistProgram();
  D.lay = lay;
  D.rank = rank;
  const int64_t n = lay.n, nw = (int64_t)plan.wins.size();
  D.sorted.resize(nw);
  for (int64_t i = 0; i < nw; ++i) D.sorted[i] = i;
  std::stable_sort(D.sorted.begin(), D.sorted.end(),
                   [&](int64_t x, int64_t y) { return plan.wins[x].level < plan.wins[y].level; });
  D.wins.resize(nw);
  for (int64_t i = 0; i < nw; ++i) {
    const WindowPlan& w = plan.wins[D.sorted[i]];
    DistWin& d = D.wins[i];
    d.t = D.sorted[i];
    d.j1 = w.j1;
    d.k = w.k;
    d.level = w.level;
    d.owner = (int32_t)lay.owner_of_col(w.j1);
    const int64_t j2 = w.j1 + w.k;
    if (w.j1 / lay.bc != (j2 - 1) / lay.bc) {
      d.c = (w.j1 / lay.bc + 1) * lay.bc;
      d.partner = (int32_t)lay.owner_of_col(d.c);
      if (d.partner == d.owner) { d.partner = -1; }   // P == 1: the next block is local too
    }
    d.coff = lay.ext_lcol(w.j1) - w.j1;
  }
  D.levels.resize(plan.nlevels);
  {
    int64_t i = 0;
    for (int64_t l = 0; l < plan.nlevels; ++l) {
      D.levels[l].w0 = i;
      while (i < nw && D.wins[i].level == l) ++i;
      D.levels[l].w1 = i;
      D.max_level_wins = std::max(D.max_level_wins, D.levels[l].w1 - D.levels[l].w0);
    }
  }
  // P == 1 with a straddle inside one rank: the "halo" is the next owned block itself only
  // when the blocks are adjacent in the extended layout -- they are not (a halo slot sits in
  // between), so a straddling window still needs its next-block columns in the halo slot:
  // a local copy (src == dst).  Keep partner = owner in that case.
  for (auto& d : D.wins)
    if (d.c >= 0 && d.partner < 0) d.partner = d.owner;

  for (int64_t l = 0; l < plan.nlevels; ++l) {
    DistLevel& L = D.levels[l];
    const int64_t a = L.w0, b = L.w1;
    // messages and lent / halo ranges of this level
    std::vector<std::pair<int64_t, int64_t>> lent, halo;   // global column ranges for `rank`
    int64_t bytes = 0;
    for (int64_t i = a; i < b; ++i) {
      const DistWin& d = D.wins[i];
      if (d.c < 0) continue;
      const int64_t j2 = d.j1 + d.k;
      DistMsg m;
      m.w = i;
      m.nrows = j2;
      m.gcol = d.c;
      m.ncols = j2 - d.c;
      m.src = d.partner;
      m.dst = d.owner;
      m.src_lcol = lay.ext_lcol(d.c);
      m.dst_lcol = lay.halo_lcol(d.c);
      L.pulls.push_back((int64_t)D.msgs.size());
      D.msgs.push_back(m);
      std::swap(m.src, m.dst);
      std::swap(m.src_lcol, m.dst_lcol);
      L.pushes.push_back((int64_t)D.msgs.size());
      D.msgs.push_back(m);
      if (d.partner == rank) lent.push_back({d.c, j2});
      if (d.owner == rank) halo.push_back({d.c, j2});
      if ((d.partner == rank || d.owner == rank) && d.partner != d.owner) bytes += 8 * m.nrows * m.ncols;
    }
    D.max_msg_bytes = std::max(D.max_msg_bytes, bytes);
    std::sort(lent.begin(), lent.end());
    for (int64_t i = a; i < b; ++i)
      if (D.wins[i].owner == rank) L.own.push_back(i);
    // L strips: columns [x2, n) owned by `rank`, minus lent, plus halo
    L.L0 = (int64_t)D.strips.size();
    for (int64_t i = a; i < b; ++i) {
      const DistWin& d = D.wins[i];
      const int32_t wl = (int32_t)(i - a);
      const int64_t x2 = d.j1 + d.k;
      for (int64_t blk = x2 / lay.bc; blk < lay.nblocks(); ++blk) {
        if (blk % lay.P != rank) continue;
        int64_t s = std::max(x2, blk * lay.bc);
        const int64_t e = std::min(n, (blk + 1) * lay.bc);
        for (const auto& r : lent)
          if (r.first == blk * lay.bc) s = std::max(s, r.second);   // lent prefix of this block
        if (s < e) push_strips(D.strips, wl, lay.ext_lcol(s), lay.ext_lcol(s) + (e - s), strip);
      }
      for (const auto& h : halo) {
        const int64_t s = std::max(x2, h.first), e = h.second;
        if (s < e) push_strips(D.strips, wl, lay.halo_lcol(s), lay.halo_lcol(s) + (e - s), strip);
      }
    }
    L.L1 = (int64_t)D.strips.size();
    // R strips: rows [0, j1) of the owned windows
    L.R0 = L.L1;
    for (int64_t i : L.own) push_strips(D.strips, (int32_t)(i - a), 0, D.wins[i].j1, strip);
    L.R1 = (int64_t)D.strips.size();
    // Q strips: this rank's rows, every window
    L.Q0 = L.R1;
    const int64_t nq = lay.q1(rank) - lay.q0(rank);
    for (int64_t i = a; i < b; ++i) push_strips(D.strips, (int32_t)(i - a), 0, nq, strip);
    L.Q1 = (int64_t)D.strips.size();
  }
  return 0;
}

}  // namespace sn
