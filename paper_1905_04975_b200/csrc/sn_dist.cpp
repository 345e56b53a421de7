// sn_dist.cpp -- the per-rank program of the multi-GPU reordering (see sn_dist.h).
#include "sn_dist.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <thread>
#include <utility>

namespace sn {

namespace {

struct LevelOut {            // one level of a rank's program, built independently
  std::vector<DistMsg> pulls, pushes;
  std::vector<int64_t> own;
  std::vector<DistStrip> lcrit, lrest, rcrit, rrest, q;
  int64_t bytes = 0;
};

}  // namespace

static double tnow() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int build_dist_program(const Plan& plan, const DistLayout& lay, int64_t rank, int64_t strip, DistProgram* prog) {
  const bool tr = std::getenv("SN_DIST_TIMING") != nullptr;
  const double t0 = tnow();
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

  // single-GPU lookahead counts (strips of `strip` columns / rows, schedule order)
  const double t1 = tnow();
  std::vector<int32_t> crit_l, crit_r;
  lookahead_strips(plan, strip, crit_l, crit_r);
  const double t2 = tnow();
  auto overlaps = [](int64_t a0, int64_t a1, int64_t b0, int64_t b1) { return a0 < b1 && b0 < a1; };

  auto build_level = [&](int64_t l, LevelOut& O) {
    const DistLevel& L = D.levels[l];
    const int64_t a = L.w0, b = L.w1;
    // column ranges the next level pulls (straddling windows' partner columns)
    std::vector<std::pair<int64_t, int64_t>> pulled;
    if (l + 1 < plan.nlevels)
      for (int64_t i = D.levels[l + 1].w0; i < D.levels[l + 1].w1; ++i)
        if (D.wins[i].c >= 0) pulled.push_back({D.wins[i].c, D.wins[i].j1 + D.wins[i].k});
    auto hits_pulled = [&](int64_t g0, int64_t g1) {
      for (const auto& r : pulled)
        if (overlaps(g0, g1, r.first, r.second)) return true;
      return false;
    };
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
      O.pulls.push_back(m);
      std::swap(m.src, m.dst);
      std::swap(m.src_lcol, m.dst_lcol);
      O.pushes.push_back(m);
      if (d.partner == rank) lent.push_back({d.c, j2});
      if (d.owner == rank) halo.push_back({d.c, j2});
      if ((d.partner == rank || d.owner == rank) && d.partner != d.owner) bytes += 8 * m.nrows * m.ncols;
    }
    O.bytes = bytes;
    std::sort(lent.begin(), lent.end());
    for (int64_t i = a; i < b; ++i)
      if (D.wins[i].owner == rank) O.own.push_back(i);
    std::vector<DistStrip>& lcrit = O.lcrit;
    std::vector<DistStrip>& lrest = O.lrest;
    std::vector<DistStrip>& rcrit = O.rcrit;
    std::vector<DistStrip>& rrest = O.rrest;
    // columns of the windows with critical right strips: the left strips over them must run
    // first (the one-GPU order on the corner rows(a) x cols(b))
    std::vector<std::pair<int64_t, int64_t>> rcols;
    // R strips: rows [0, j1) of the owned windows; critical if the next level's windows read
    // them (the last crit_r strips), if the window straddles (its push follows) or if its
    // columns are pulled by the next level
    for (int64_t i : O.own) {
      const DistWin& d = D.wins[i];
      const int64_t nR = (d.j1 + strip - 1) / strip;
      const bool all = d.c >= 0 || hits_pulled(d.j1, d.j1 + d.k);
      // the critical rows are a suffix [cstart, j1) in whole strips, or everything
      const int64_t cstart = all ? 0 : std::min(d.j1, strip * std::max<int64_t>(0, nR - crit_r[d.t]));
      DistStrip sd;
      sd.w = (int32_t)(i - a);
      if (cstart > 0) { sd.x0 = 0; sd.cnt = (int32_t)cstart; rrest.push_back(sd); }
      if (cstart < d.j1) {
        sd.x0 = cstart; sd.cnt = (int32_t)(d.j1 - cstart); rcrit.push_back(sd);
        if (rcols.empty() || rcols.back().first != d.j1) rcols.push_back({d.j1, d.j1 + d.k});
      }
    }
    // sorted, merged column intervals that make a left strip critical (pulled columns and the
    // columns of windows with critical right strips); binary search per strip
    std::vector<std::pair<int64_t, int64_t>> civ(pulled);
    civ.insert(civ.end(), rcols.begin(), rcols.end());
    std::sort(civ.begin(), civ.end());
    {
      std::vector<std::pair<int64_t, int64_t>> mg;
      for (const auto& r : civ) {
        if (!mg.empty() && r.first <= mg.back().second) mg.back().second = std::max(mg.back().second, r.second);
        else mg.push_back(r);
      }
      civ.swap(mg);
    }
    auto hits_crit = [&](int64_t g0, int64_t g1) {
      // first interval ending after g0
      auto it = std::upper_bound(civ.begin(), civ.end(), g0,
                                 [](int64_t v, const std::pair<int64_t, int64_t>& r) { return v < r.second; });
      return it != civ.end() && it->first < g1;
    };
    // L strips: columns [x2, n) owned by `rank`, minus lent, plus halo; critical if they meet
    // the columns [x2, x2 + strip*crit_l) the next level's windows read, a column the next
    // level pulls, or a halo slot
    auto emit_l = [&](int32_t wl, int64_t lcol, int64_t g0, int64_t len, int64_t cl_end, bool force) {
      // strips of `strip` columns from g0; runs of equal criticality become one segment
      int64_t run0 = 0;
      int run_crit = -1;
      auto flush = [&](int64_t end) {
        if (run_crit < 0 || end <= run0) return;
        DistStrip sd;
        sd.w = wl;
        sd.x0 = lcol + run0;
        sd.cnt = (int32_t)(end - run0);
        (run_crit ? lcrit : lrest).push_back(sd);
      };
      for (int64_t o = 0; o < len; o += strip) {
        const int64_t cnt = std::min(strip, len - o);
        const int c = (force || g0 + o < cl_end || hits_crit(g0 + o, g0 + o + cnt)) ? 1 : 0;
        if (c != run_crit) {
          flush(o);
          run0 = o;
          run_crit = c;
        }
      }
      flush(len);
    };
    for (int64_t i = a; i < b; ++i) {
      const DistWin& d = D.wins[i];
      const int32_t wl = (int32_t)(i - a);
      const int64_t x2 = d.j1 + d.k;
      const int64_t cl_end = x2 + strip * (int64_t)crit_l[d.t];
      for (int64_t blk = x2 / lay.bc; blk < lay.nblocks(); ++blk) {
        if (blk % lay.P != rank) continue;
        int64_t s = std::max(x2, blk * lay.bc);
        const int64_t e = std::min(n, (blk + 1) * lay.bc);
        for (const auto& r : lent)
          if (r.first == blk * lay.bc) s = std::max(s, r.second);   // lent prefix of this block
        if (s < e) emit_l(wl, lay.ext_lcol(s), s, e - s, cl_end, false);
      }
      for (const auto& h : halo) {
        const int64_t s = std::max(x2, h.first), e = h.second;
        if (s < e) emit_l(wl, lay.halo_lcol(s), s, e - s, cl_end, true);
      }
    }
    const int64_t nq = lay.q1(rank) - lay.q0(rank);
    for (int64_t i = a; i < b; ++i)
      if (nq > 0) {
        DistStrip sd;
        sd.w = (int32_t)(i - a);
        sd.x0 = 0;
        sd.cnt = (int32_t)nq;
        O.q.push_back(sd);
      }
  };
  // levels are independent given the windows: build them on host threads, then concatenate
  std::vector<LevelOut> outs((size_t)plan.nlevels);
  {
    std::atomic<int64_t> next(0);
    const int64_t nth = std::max<int64_t>(1, std::min<int64_t>(16, (int64_t)std::thread::hardware_concurrency()));
    auto worker = [&]() {
      for (int64_t l; (l = next.fetch_add(1)) < plan.nlevels;) build_level(l, outs[(size_t)l]);
    };
    std::vector<std::thread> th;
    for (int64_t q = 1; q < std::min<int64_t>(nth, plan.nlevels); ++q) th.emplace_back(worker);
    worker();
    for (auto& t : th) t.join();
  }
  const double t3 = tnow();
  for (int64_t l = 0; l < plan.nlevels; ++l) {
    DistLevel& L = D.levels[l];
    LevelOut& O = outs[(size_t)l];
    for (size_t q = 0; q < O.pulls.size(); ++q) {
      L.pulls.push_back((int64_t)D.msgs.size());
      D.msgs.push_back(O.pulls[q]);
      L.pushes.push_back((int64_t)D.msgs.size());
      D.msgs.push_back(O.pushes[q]);
    }
    D.max_msg_bytes = std::max(D.max_msg_bytes, O.bytes);
    L.own = std::move(O.own);
    auto append = [&](std::vector<DistStrip>& v, int64_t& s0, int64_t& s1, int g) {
      s0 = (int64_t)D.strips.size();
      D.strips.insert(D.strips.end(), v.begin(), v.end());
      s1 = (int64_t)D.strips.size();
      L.poff[g] = (int64_t)D.sprefix.size();
      int32_t acc = 0;
      D.sprefix.push_back(0);
      for (const auto& sd : v) {
        acc += (int32_t)((sd.cnt + strip - 1) / strip);
        D.sprefix.push_back(acc);
      }
      L.nstr[g] = acc;
      std::vector<DistStrip>().swap(v);
    };
    append(O.lcrit, L.L0, L.L1, 0);
    append(O.rcrit, L.R0, L.R1, 1);
    append(O.lrest, L.Lr0, L.Lr1, 2);
    append(O.rrest, L.Rr0, L.Rr1, 3);
    append(O.q, L.Q0, L.Q1, 4);
  }
  if (tr)
    std::fprintf(stderr, "dist program: windows %.1f ms, lookahead %.1f ms, levels %.1f ms, concat %.1f ms\n", t1 - t0,
                 t2 - t1, t3 - t2, tnow() - t3);
  return 0;
}

}  // namespace sn
