// sn_plan.cpp -- window schedule, inner schedule and DAG levels (host, product code).
// See sn_plan.h and DESIGN.md §4-5.
#include "sn_plan.h"

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <utility>

namespace sn {

namespace {

// One chain-schedule pass over a block list (sizes/flags), SURVEY §8c-2 steps (a)-(f):
// groups of at most ks rows of selected blocks are moved to the front, each by a chain of
// windows of at most wmax rows walking up the diagonal.  For every window the callback
// receives the block range [top, bottom) BEFORE the window's moves; the lists are then
// stably partitioned (movers first) inside the range.  Windows without swaps are skipped.
template <class F>
void chain_pass(std::vector<uint8_t>& sz, std::vector<uint8_t>& sel, std::vector<int64_t>* row,
                int64_t wmax, int64_t max_windows, F&& on_window) {
  const int64_t nb = (int64_t)sz.size();
  const int64_t ks = wmax / 2;
  int64_t placed = 0, emitted = 0;
  std::vector<uint8_t> tsz, tsel;
  while (placed < nb) {
    if (max_windows >= 0 && emitted >= max_windows) return;
    // (a) first unplaced selected block and the group G (<= ks rows, at least one block)
    int64_t first = placed;
    while (first < nb && !sel[first]) ++first;
    if (first == nb) return;
    int64_t grows = 0, gcount = 0, glast = first;
    for (int64_t b = first; b < nb; ++b) {
      if (!sel[b]) continue;
      if (gcount > 0 && grows + sz[b] > ks) break;
      grows += sz[b];
      ++gcount;
      glast = b;
    }
    // (b) group already in place
    if (first == placed && glast - placed + 1 == gcount) {
      placed += gcount;
      continue;
    }
    // (c)-(f): the chain
    int64_t bottom = glast + 1;
    for (;;) {
      if (max_windows >= 0 && emitted >= max_windows) return;
      int64_t top = bottom, rows = 0;
      while (top > placed && rows + sz[top - 1] <= wmax) rows += sz[--top];
      // swaps: each mover passes every unselected block above it inside [top, bottom)
      int64_t nunsel = 0, nswap = 0;
      for (int64_t b = top; b < bottom; ++b) {
        if (sel[b]) nswap += nunsel; else ++nunsel;
      }
      if (nswap > 0) {
        on_window(top, bottom);
        ++emitted;
      }
      // stable partition of [top, bottom): movers first
      tsz.clear(); tsel.clear();
      int64_t nmov = 0;
      for (int64_t b = top; b < bottom; ++b)
        if (sel[b]) { tsz.push_back(sz[b]); tsel.push_back(1); ++nmov; }
      for (int64_t b = top; b < bottom; ++b)
        if (!sel[b]) { tsz.push_back(sz[b]); tsel.push_back(0); }
      std::copy(tsz.begin(), tsz.end(), sz.begin() + top);
      std::copy(tsel.begin(), tsel.end(), sel.begin() + top);
      if (row)
        for (int64_t b = top + 1; b < bottom; ++b) (*row)[b] = (*row)[b - 1] + sz[b - 1];
      if (top == placed) { placed = top + nmov; break; }
      bottom = top + nmov;
    }
  }
}

}  // namespace

int build_plan(int64_t n, const int8_t* bmap, const int8_t* selrow, int64_t w, int64_t kin,
               int64_t max_windows, Plan* plan) {
  if (n < 0) return -1;
  if (w < 4 || w > 256) return -4;
  if (kin < 4 || kin > 64) return -5;
  Plan& P = *plan;
  P = Plan();
  P.n = n; P.w = w; P.kin = kin;
  std::vector<uint8_t> sz, sel;
  std::vector<int64_t> row;
  sz.reserve(n); sel.reserve(n); row.reserve(n + 1);
  for (int64_t i = 0; i < n;) {
    const int s = bmap[i] == 1 ? 2 : 1;
    if (s == 2 && (i + 1 >= n || bmap[i + 1] != 2)) return -2;
    sz.push_back((uint8_t)s);
    sel.push_back(selrow[i] ? 1 : 0);
    row.push_back(i);
    i += s;
  }
  row.push_back(n);
  std::vector<uint8_t> lsz, lsel;
  std::vector<uint16_t> inner;
  // row offsets: a window only permutes blocks inside its range, so the first row of the
  // range never changes and chain_pass recomputes the rows inside it.
  chain_pass(sz, sel, &row, w, max_windows, [&](int64_t top, int64_t bottom) {
    WindowPlan wp;
    wp.order = (int64_t)P.wins.size();
    wp.j1 = row[top];
    wp.top = top;
    wp.nblk = (int32_t)(bottom - top);
    int64_t k = 0;
    for (int64_t b = top; b < bottom; ++b) k += sz[b];
    wp.k = (int32_t)k;
    // swap statistics (pairs: unselected block above a mover)
    int64_t cnt_u[3] = {0, 0, 0};
    for (int64_t b = top; b < bottom; ++b) {
      if (sel[b]) {
        for (int su = 1; su <= 2; ++su) {
          wp.swaps_by_type[(su - 1) * 2 + (sz[b] - 1)] += cnt_u[su];
          wp.nswap += cnt_u[su];
        }
      } else {
        cnt_u[sz[b]]++;
      }
    }
    // inner schedule on the window's own block list
    lsz.assign(sz.begin() + top, sz.begin() + bottom);
    lsel.assign(sel.begin() + top, sel.begin() + bottom);
    inner.clear();
    chain_pass(lsz, lsel, nullptr, kin, -1, [&](int64_t it, int64_t ib) {
      inner.push_back((uint16_t)it);
      inner.push_back((uint16_t)ib);
    });
    wp.ninner = (int32_t)(inner.size() / 2);
    wp.pool = (int64_t)P.pool.size();
    P.pool.insert(P.pool.end(), sz.begin() + top, sz.begin() + bottom);
    P.pool.insert(P.pool.end(), sel.begin() + top, sel.begin() + bottom);
    if (P.pool.size() & 1) P.pool.push_back(0);
    const size_t off = P.pool.size();
    P.pool.resize(off + inner.size() * 2);
    std::memcpy(P.pool.data() + off, inner.data(), inner.size() * 2);
    while (P.pool.size() & 7) P.pool.push_back(0);
    P.nswap += wp.nswap;
    P.ninner += wp.ninner;
    P.wins.push_back(wp);
  });
  P.final_sz = sz;
  P.final_sel = sel;
  // DAG levels: 1 + max level of earlier windows sharing a row (row-range intersection)
  std::vector<int32_t> rowlev((size_t)n, -1);
  int32_t maxlev = -1;
  for (auto& wp : P.wins) {
    int32_t l = -1;
    for (int64_t r = wp.j1; r < wp.j1 + wp.k; ++r) l = std::max(l, rowlev[r]);
    wp.level = l + 1;
    for (int64_t r = wp.j1; r < wp.j1 + wp.k; ++r) rowlev[r] = wp.level;
    maxlev = std::max(maxlev, wp.level);
  }
  P.nlevels = maxlev + 1;
  return 0;
}

void lookahead_strips(const Plan& P, int64_t NT, std::vector<int32_t>& critL, std::vector<int32_t>& critR) {
  const int64_t nw = (int64_t)P.wins.size(), n = P.n;
  critL.assign(nw, 0);
  critR.assign(nw, 0);
  std::vector<std::vector<int64_t>> bylev(P.nlevels);
  for (int64_t t = 0; t < nw; ++t) bylev[P.wins[t].level].push_back(t);
  for (int64_t l = 0; l + 1 < P.nlevels; ++l) {
    // the next level's windows are row-disjoint: find the one containing a given row
    std::vector<std::pair<int64_t, int64_t>> nxt;   // (j1, j2), sorted
    for (int64_t t : bylev[l + 1]) nxt.push_back({P.wins[t].j1, P.wins[t].j1 + P.wins[t].k});
    std::sort(nxt.begin(), nxt.end());
    auto containing = [&](int64_t r) -> int64_t {
      auto it = std::upper_bound(nxt.begin(), nxt.end(), std::make_pair(r, INT64_MAX));
      if (it == nxt.begin()) return -1;
      --it;
      return (r >= it->first && r < it->second) ? (int64_t)(it - nxt.begin()) : -1;
    };
    for (int64_t t : bylev[l]) {
      const WindowPlan& x = P.wins[t];
      const int64_t x1 = x.j1, x2 = x.j1 + x.k;
      const int64_t nL = (n - x2 + NT - 1) / NT, nR = (x1 + NT - 1) / NT;
      // left strips read by y: y contains row x2 and overlaps rows(x) -> columns [x2, y2)
      int64_t q = x2 < n ? containing(x2) : -1;
      if (q >= 0 && nxt[q].first < x2) critL[t] = (int32_t)std::min(nL, (nxt[q].second - x2 + NT - 1) / NT);
      // right strips read by y: y contains row x1-1 and overlaps rows(x) -> rows [y1, x1)
      q = x1 > 0 ? containing(x1 - 1) : -1;
      if (q >= 0 && nxt[q].second > x1) critR[t] = (int32_t)(nR - nxt[q].first / NT);
    }
    // Closure.  Inside a level, the left update of a window a above a window b and the right
    // update of b meet on rows(a) x cols(b); they commute only when each is applied whole
    // there.  Critical right strips of b run before the remaining left strips, so if they
    // touch rows(a), every left strip of a over cols(b) must be critical too (the critical
    // left strips run first).
    for (int64_t tb : bylev[l]) {
      if (critR[tb] == 0) continue;
      const WindowPlan& b = P.wins[tb];
      const int64_t nRb = (b.j1 + NT - 1) / NT;
      const int64_t cr0 = (nRb - critR[tb]) * NT;     // first row of b's critical right strips
      for (int64_t ta : bylev[l]) {
        const WindowPlan& a = P.wins[ta];
        const int64_t a2 = a.j1 + a.k;
        if (a2 > b.j1 || a2 <= cr0) continue;         // a not above b, or rows(a) untouched
        const int64_t nLa = (n - a2 + NT - 1) / NT;
        critL[ta] = (int32_t)std::max<int64_t>(critL[ta], std::min(nLa, (b.j1 + b.k - a2 + NT - 1) / NT));
      }
    }
  }
}

int64_t window_swaps(const Plan& P, int64_t t, int64_t cap, int64_t* sj, int8_t* s1, int8_t* s2) {
  // Execution order of the window kernel: inner windows in order; inside one, the wavefront
  // steps in order and, within a step, the active movers top to bottom (mover i makes its
  // s-th swap at step 2i + s).
  if (t < 0 || t >= (int64_t)P.wins.size()) return -1;
  const WindowPlan& wp = P.wins[t];
  const uint8_t* base = P.pool.data() + wp.pool;
  std::vector<uint8_t> sz(base, base + wp.nblk), sel(base + wp.nblk, base + 2 * wp.nblk);
  size_t off = wp.pool + 2 * wp.nblk;
  if (off & 1) ++off;
  const uint16_t* inner = reinterpret_cast<const uint16_t*>(P.pool.data() + off);
  int64_t cnt = 0;
  for (int32_t q = 0; q < wp.ninner; ++q) {
    const int top = inner[2 * q], bottom = inner[2 * q + 1];
    int64_t rtop = wp.j1;
    for (int b = 0; b < top; ++b) rtop += sz[b];
    std::vector<int> msz, usz, mu, mrows{0}, urows{0};
    int T = 0;
    for (int b = top; b < bottom; ++b) {
      if (sel[b]) {
        const int i = (int)msz.size();
        msz.push_back(sz[b]);
        mu.push_back(b - top - i);
        mrows.push_back(mrows.back() + sz[b]);
        T = std::max(T, 2 * i + mu.back());
      } else {
        usz.push_back(sz[b]);
        urows.push_back(urows.back() + sz[b]);
      }
    }
    for (int step = 0; step < T; ++step)
      for (int i = 0; i < (int)msz.size(); ++i) {
        const int s = step - 2 * i;
        if (s < 0 || s >= mu[i]) continue;
        const int uq = mu[i] - 1 - s;
        if (cnt < cap) {
          sj[cnt] = rtop + mrows[i] + urows[uq];
          s1[cnt] = (int8_t)usz[uq];
          s2[cnt] = (int8_t)msz[i];
        }
        ++cnt;
      }
    int o = top;
    for (int x : msz) { sz[o] = (uint8_t)x; sel[o] = 1; ++o; }
    for (int x : usz) { sz[o] = (uint8_t)x; sel[o] = 0; ++o; }
  }
  return cnt;
}

}  // namespace sn
