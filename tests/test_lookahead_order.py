"""Race / ordering checker for the level executor's lookahead (-m "not gpu").

The executor runs, per dependency level l:
    stream A:  W(l) -> Lcrit(l) -> Rcrit(l) -> W(l+1) ...
    stream C:  (after Rcrit(l)) Lrest(l) -> Rrest(l)      concurrently with W(l+1)
    stream A:  W(l+1) -> [wait Rrest(l)] -> Lcrit(l+1) ...
From the library's own exported plan (schedule, levels, critical strip counts) this test
checks by brute force over footprints that
  1. no remaining (non-critical) strip of level l touches a level-(l+1) window, so the
     concurrent W(l+1) neither races with it nor misses an update it needs;
  2. inside a level, on every rectangle rows(a) x cols(b) shared by the left update of a
     window a and the right update of a window b below it, all of a's left strips run
     before all of b's right strips (the two updates commute only when applied whole);
  3. windows of one level are row-disjoint and each window's level exceeds the level of
     every earlier window sharing a row (sequential consistency).
"""
import numpy as np
import pytest

import oracle
import paper_1905_04975_b200 as sn
from tests.helpers import bmap_from_S
from workloads import make_config, make_problem

NT = 64


@pytest.fixture(scope="module", autouse=True)
def built():
    sn.build()


def _inter(a0, a1, b0, b1):
    return a0 < b1 and b0 < a1


def _check(p, w):
    n = p.n
    bm = bmap_from_S(p.S_np())
    sel, _ = oracle.select(bm, p.select)
    sch = sn.schedule(bm, sel, w)
    cl, cr = sn.lookahead(bm, sel, w, NT)
    j1, k, lev = sch["j1"], sch["k"], sch["level"]
    wins = [(int(j1[t]), int(j1[t] + k[t]), int(lev[t]), t) for t in range(len(j1))]
    bylev = [[x for x in wins if x[2] == l] for l in range(sch["nlevels"])]
    # 3. levels
    rowlev = np.full(n, -1)
    for (x1, x2, l, t) in wins:
        assert l == rowlev[x1:x2].max() + 1
        rowlev[x1:x2] = l
    nchecked = 0
    for l, ws in enumerate(bylev):
        nxt = bylev[l + 1] if l + 1 < len(bylev) else []
        for (x1, x2, _, t) in ws:
            nL, nR = -(-(n - x2) // NT), -(-x1 // NT)
            assert 0 <= cl[t] <= nL and 0 <= cr[t] <= nR
            # 1. remaining strips avoid every next-level window region
            for s in range(cl[t], nL):
                c0, c1 = x2 + s * NT, min(n, x2 + (s + 1) * NT)
                for (y1, y2, _, u) in nxt:
                    assert not (_inter(x1, x2, y1, y2) and _inter(c0, c1, y1, y2)), ("L", l, t, u, s)
                    nchecked += 1
            for s in range(0, nR - cr[t]):
                r0, r1 = s * NT, min(x1, (s + 1) * NT)
                for (y1, y2, _, u) in nxt:
                    assert not (_inter(r0, r1, y1, y2) and _inter(x1, x2, y1, y2)), ("R", l, t, u, s)
                    nchecked += 1
        # 2. corner order inside the level: Lcrit < Rcrit < Lrest < Rrest
        for (a1, a2, _, ta) in ws:
            for (b1, b2, _, tb) in ws:
                if a2 > b1:
                    continue
                nLa, nRb = -(-(n - a2) // NT), -(-b1 // NT)
                l_strips = [s for s in range(nLa) if _inter(a2 + s * NT, min(n, a2 + (s + 1) * NT), b1, b2)]
                r_strips = [s for s in range(nRb) if _inter(s * NT, min(b1, (s + 1) * NT), a1, a2)]
                if not l_strips or not r_strips:
                    continue
                any_r_crit = any(s >= nRb - cr[tb] for s in r_strips)
                any_l_rest = any(s >= cl[ta] for s in l_strips)
                assert not (any_r_crit and any_l_rest), ("corner", l, ta, tb)
                nchecked += 1
    return nchecked


@pytest.mark.parametrize("case", ["config0", "n600_w64", "n1500_w256", "n2000_w32", "all2x2", "config1"])
def test_lookahead_order(case):
    if case == "config0":
        p, w = make_config(0, seed=1), 32
    elif case == "n600_w64":
        p, w = make_problem(600, q="none", psel=0.4, w=64, seed=3), 64
    elif case == "n1500_w256":
        p, w = make_problem(1500, q="none", psel=0.35, w=256, seed=30), 256
    elif case == "n2000_w32":
        p, w = make_problem(2000, p2=0.5, q="none", psel=0.5, w=32, seed=4), 32
    elif case == "all2x2":
        p, w = make_problem(900, p2=100.0, q="none", psel=0.3, w=48, seed=5), 48
    else:
        p, w = make_problem(4096, q="none", psel=0.35, w=128, seed=1), 128
    assert _check(p, w) > 0
