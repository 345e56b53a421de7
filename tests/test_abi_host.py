"""Host-side tests of the product library (-m "not gpu"): the C ABI loads and exports every
symbol of include/sn_reorder.h, its host schedule matches the oracle's schedule, and the
compute entry points refuse to run without a GPU (no CPU fallback)."""
import os
import re

import numpy as np
import pytest
import torch

import oracle
import paper_1905_04975_b200 as sn
from tests.helpers import bmap_from_S
from workloads import make_config, make_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    sn.build()


def test_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "sn_reorder.h")).read()
    names = set(re.findall(r"\b(sn_[a-z_]+)\s*\(", hdr))
    assert names == set(sn.EXPORTS), names
    L = sn.lib()
    for nm in names:
        assert hasattr(L, nm), nm
    assert b"sm_100a" in L.sn_version()


def _pairs(sizes, flags, sj_rows, n1s, n2s):
    """Simulate a swap list on block identities; return the set of (above, below) id pairs."""
    ids = list(range(len(sizes)))
    sz = list(sizes)
    pairs = []
    for r, a, b in zip(sj_rows, n1s, n2s):
        rows = np.cumsum([0] + sz[:-1])
        p = int(np.searchsorted(rows, r))
        assert rows[p] == r and sz[p] == a and sz[p + 1] == b
        assert flags[ids[p + 1]] and not flags[ids[p]]
        pairs.append((ids[p], ids[p + 1]))
        ids[p], ids[p + 1] = ids[p + 1], ids[p]
        sz[p], sz[p + 1] = sz[p + 1], sz[p]
    return pairs, ids


@pytest.mark.parametrize("case", ["config0", "config1", "rand_a", "rand_b", "all2x2", "trailing"])
def test_schedule_matches_oracle(case):
    if case == "config0":
        p = make_config(0, seed=1)
    elif case == "config1":
        p = make_problem(4096, q="none", psel=0.35, w=128, seed=1)
    elif case == "rand_a":
        p = make_problem(700, p2=0.5, q="none", psel=0.2, w=64, seed=7)
    elif case == "rand_b":
        p = make_problem(333, p2=0.1, q="none", psel=0.8, w=10, seed=8)
    elif case == "all2x2":
        p = make_problem(300, p2=100.0, q="none", psel=0.5, w=16, seed=9)
    else:
        p = make_problem(1000, p2=0.5, q="none", sel="trailing_half", psel=None, w=256, seed=2)
    S = p.S_np()
    bm = bmap_from_S(S)
    selrow, m = oracle.select(bm, p.select)
    ref = oracle.schedule(bm, selrow, p.w)
    got = sn.schedule(bm, selrow, p.w)
    np.testing.assert_array_equal(got["j1"], ref["j1"])
    np.testing.assert_array_equal(got["j1"] + got["k"], ref["j2"])
    np.testing.assert_array_equal(got["nswap"], np.diff(ref["off"]))
    assert got["total_swaps"] == len(ref["swap_j"])
    # levels: windows of one level are row-disjoint, and a window is above every earlier
    # window sharing a row
    lev = got["level"]
    for t in range(len(lev)):
        for u in range(t):
            inter = not (got["j1"][u] + got["k"][u] <= got["j1"][t] or got["j1"][t] + got["k"][t] <= got["j1"][u])
            if inter:
                assert lev[u] < lev[t]
        if t > 400:
            break
    # the product's in-window execution order swaps the same block pairs as the oracle's
    blocks_sz = []
    i = 0
    while i < len(bm):
        blocks_sz.append(2 if bm[i] == 1 else 1)
        i += blocks_sz[-1]
    flags = []
    r = 0
    for s in blocks_sz:
        flags.append(bool(selrow[r])); r += s
    # replay window by window on a global block list, comparing pair sets
    ids = list(range(len(blocks_sz)))
    szs = list(blocks_sz)
    for t in range(min(len(ref["j1"]), 40)):
        a, b = ref["off"][t], ref["off"][t + 1]
        pj, p1, p2 = sn.window_swaps(bm, selrow, p.w, t)
        # product and oracle lists act on the same window state
        state_sz = list(szs)
        pr, ids_p = _pairs([state_sz[x] for x in range(len(state_sz))], [flags[x] for x in ids],
                           pj, p1, p2)
        orr, ids_o = _pairs([state_sz[x] for x in range(len(state_sz))], [flags[x] for x in ids],
                            ref["swap_j"][a:b], ref["swap_n1"][a:b], ref["swap_n2"][a:b])
        assert sorted(pr) == sorted(orr)
        assert ids_p == ids_o
        # advance the global state
        ids = [ids[x] for x in ids_o]
        szs = [blocks_sz[x] for x in ids]


def test_schedule_empty_and_trivial():
    bm = np.zeros(10, np.int8)
    for sel in (np.zeros(10, np.int8), np.ones(10, np.int8)):
        got = sn.schedule(bm, sel, 8)
        assert len(got["j1"]) == 0 and got["total_swaps"] == 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU refusal")
def test_no_cpu_fallback_without_gpu():
    p = make_problem(32, q="identity", psel=0.5, w=8, seed=1)
    S = p.S.clone()
    Q = p.Q.clone()
    r = sn.reorder(S, Q, p.select, window=8)
    assert r["rc"] == sn.SN_ERR_CUDA
    assert torch.equal(S, p.S) and torch.equal(Q, p.Q)
    assert sn.strerror(sn.SN_ERR_CUDA).startswith("CUDA error")


def test_argument_errors_without_gpu():
    rc, m = sn.sn_reorder_schur(-1, 0, 1, None, 1, np.zeros(1, np.int32))
    assert rc == -1
    rc, m = sn.sn_reorder_schur(4, 0, 4, None, 4, np.zeros(4, np.int32))
    assert rc == -2
    rc, m = sn.sn_reorder_schur(0, 0, 1, None, 1, np.zeros(1, np.int32))
    assert rc == 0 and m == 0


@pytest.mark.parametrize("n,ns,w,m", [(3, 2, 16, 1), (50, 8, 32, 4), (1000, 64, 160, 16), (4000, 256, 256, 32),
                                      (777, 40, 128, 12)])
def test_sweep_schedule_is_valid(n, ns, w, m):
    """The sweep plan (row f3, readings B3/B4): every reflector of every chain step lies inside
    the window executing that step (its rows p..p+2, the column p-1 it reads, the rows up to
    p+3 its right update touches), each chain's steps are covered exactly once in order, and a
    window's level exceeds that of every earlier window whose rows it meets."""
    sc = sn.sweep_schedule(n, ns, w, m)
    nb = ns // 2
    seen = {}
    rowlev = np.full(n, -1)
    for t in range(len(sc["w0"])):
        w0, k, c, t0, t1, lev = (int(sc[key][t]) for key in ("w0", "k", "chain", "tau0", "tau1", "level"))
        assert k <= w and w0 + k <= n
        mb = min(m, nb - c * m)
        assert seen.get(c, 0) == t0 and t1 > t0          # consecutive, gap-free chain steps
        seen[c] = t1
        for tau in range(t0, t1):
            for b in range(mb):
                p = tau - 4 * b
                if 0 <= p <= n - 2:
                    lo = p if p == 0 else p - 1
                    hi = min(p + 3, n - 1)
                    assert w0 <= lo and hi < w0 + k, (t, tau, b, p, w0, k)
        assert lev > rowlev[w0:w0 + k].max()
        rowlev[w0:w0 + k] = lev
    for c in range((nb + m - 1) // m):
        mb = min(m, nb - c * m)
        assert seen[c] == (n - 2) + 4 * (mb - 1) + 1     # every bulge leaves at the bottom
    assert sc["nlevels"] == rowlev.max() + 1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU refusal")
def test_rows_f3_f4_refuse_without_gpu():
    h = torch.zeros((8, 8), dtype=torch.float64)
    assert sn.qr_sweep(h, None, [1.0, 2.0], [0.0, 0.0])["rc"] == sn.SN_ERR_CUDA
    assert sn.eigenvectors(h, None, np.ones(8, np.int32))["rc"] == sn.SN_ERR_CUDA
