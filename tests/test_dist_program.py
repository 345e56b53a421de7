"""The sharded (multi-GPU) program on the CPU (-m "not gpu"): SURVEY §8e.

sn_dist_program (product host code) emits each rank's program; tests/dist_interp.py executes
it with numpy panel updates and the oracle's swap primitive, (a) all ranks in one process and
(b) as a world_size-2 torch.distributed gloo group (send/recv for the straddle messages,
broadcast for Z).  The gathered result must equal the oracle's one-process reordering (mode
(ii), same schedule) to rounding: the program moves every column to the right rank at the
right phase and covers every panel entry exactly once.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import paper_1905_04975_b200 as sn
from tests import dist_interp as DI
from workloads import make_problem

TOL = 1e-12


def problem(n, w, seed, p2=0.25, psel=0.35, sel="bernoulli"):
    p = make_problem(n, p2=p2, q="householder", sel=sel, psel=psel, w=w, seed=seed)
    return p.S_np().copy(order="F"), p.Q_np().copy(order="F"), p.select


def oracle_ref(S, Q, select, w):
    r = oracle.reorder(S, Q, select, w=w, mode=1)
    assert r["rc"] == 0
    return r


@pytest.mark.parametrize("n,w,bc,P,seed", [
    (160, 16, 16, 1, 1), (160, 16, 16, 2, 2), (200, 16, 32, 3, 3), (240, 32, 32, 4, 4),
    (250, 16, 48, 2, 5), (300, 32, 64, 3, 6), (180, 8, 8, 5, 7)])
def test_shared_interpretation_matches_oracle(n, w, bc, P, seed):
    S, Q, sel = problem(n, w, seed)
    ref = oracle_ref(S, Q, sel, w)
    Sg, Qg, progs = DI.run_shared(S, Q, sel, w, bc, P)
    nS = np.linalg.norm(S)
    dS = np.abs(Sg - ref["S"]).max() / nS
    dQ = np.abs(Qg - ref["Q"]).max()
    assert dS <= TOL and dQ <= TOL, (dS, dQ)
    # straddling windows exist in these cases (bc close to w) and exercise pull/push
    wins = progs[0][1]
    if bc <= 2 * w:
        assert any(x["partner"] >= 0 for x in wins)


def test_worst_case_chain_interpretation():
    # config-4-like: 50% 2x2 blocks, the trailing half selected (maximum swap distance)
    S, Q, sel = problem(192, 16, 11, p2=0.5, sel="trailing_half", psel=None)
    ref = oracle_ref(S, Q, sel, 16)
    Sg, Qg, _ = DI.run_shared(S, Q, sel, 16, 32, 3)
    assert np.abs(Sg - ref["S"]).max() <= TOL * np.linalg.norm(S)
    assert np.abs(Qg - ref["Q"]).max() <= TOL


def test_program_structure():
    S, Q, sel = problem(400, 32, 9)
    rc, bmap = oracle.scan(S)
    selrow, _ = oracle.select(bmap, sel)
    n, w, bc, P = 400, 32, 64, 3
    progs = [DI.parse(sn.dist_program(bmap, selrow, w, bc, P, r)) for r in range(P)]
    hdr0, wins0, levels0 = progs[0]
    for r in range(1, P):   # windows, levels and messages are identical on every rank
        assert progs[r][1] == wins0
        for l in range(hdr0["nlev"]):
            assert progs[r][2][l]["pull"] == levels0[l]["pull"]
            assert progs[r][2][l]["push"] == levels0[l]["push"]
    for x in wins0:
        j1, j2 = x["j1"], x["j1"] + x["k"]
        assert x["owner"] == (j1 // bc) % P
        assert (x["partner"] >= 0) == (j1 // bc != (j2 - 1) // bc)
        assert DI.ext_lcol(j1, P, bc, w) == j1 + x["coff"]
    for l, lev in enumerate(levels0):
        for r in range(P):
            # R strips only on the owner, covering rows [0, j1) exactly once
            rows = {}
            for (wl, cnt, x0, *_z) in progs[r][2][l]["R"] + progs[r][2][l]["Rr"]:
                assert wins0[lev["w0"] + wl]["owner"] == r
                rows.setdefault(wl, []).append((x0, cnt))
            for wl, segs in rows.items():
                segs.sort()
                assert segs[0][0] == 0 and all(a[0] + a[1] == b[0] for a, b in zip(segs, segs[1:]))
                assert segs[-1][0] + segs[-1][1] == wins0[lev["w0"] + wl]["j1"]
        # L: per window, every column >= j2 updated exactly once over all ranks (owned or
        # halo, never a lent column)
        for i in range(lev["w0"], lev["w1"]):
            x = wins0[i]
            cover = np.zeros(n, np.int32)
            for r in range(P):
                inv = {}
                for j in range(n):
                    if (j // bc) % P == r:
                        inv[DI.ext_lcol(j, P, bc, w)] = j
                for y in wins0[lev["w0"]:lev["w1"]]:
                    if y["partner"] >= 0 and y["owner"] == r:
                        c = (y["j1"] // bc + 1) * bc
                        for j in range(c, y["j1"] + y["k"]):
                            inv[DI.ext_lcol(y["j1"], P, bc, w) + (j - y["j1"])] = j
                for (wl, cnt, x0, *_z) in progs[r][2][l]["L"] + progs[r][2][l]["Lr"]:
                    if lev["w0"] + wl != i:
                        continue
                    for lc in range(x0, x0 + cnt):
                        cover[inv[lc]] += 1
            j2 = x["j1"] + x["k"]
            assert (cover[j2:] == 1).all() and (cover[:j2] == 0).all()


def test_layout_export_matches_python():
    for n, P, bc in [(1000, 3, 64), (257, 4, 32), (64, 8, 16), (100, 1, 256)]:
        for r in range(P):
            uc, q0, q1 = sn.dist_layout(n, P, bc, r)
            cols = sn.owned_columns(n, P, bc, r)
            nblk = len(range(r, (n + bc - 1) // bc, P))
            assert uc == nblk * bc and len(cols) <= uc
            assert q0 == min(n, r * -(-n // P)) and q1 == min(n, (r + 1) * -(-n // P))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, n, w, bc, seed, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S, Q, sel = problem(n, w, seed)
        me, hdr = DI.run_gloo(S, Q, sel, w, bc, rank, world)
        np.save(os.path.join(out, "S%d.npy" % rank), me["Sx"])
        np.save(os.path.join(out, "Q%d.npy" % rank), me["Q"])
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,w,bc,seed", [(2, 200, 16, 32, 21), (2, 240, 32, 32, 22), (3, 260, 16, 32, 23)])
def test_gloo_world_matches_oracle(tmp_path, world, n, w, bc, seed):
    """The sharded program (row e) executed by `world` gloo processes (send/recv + broadcast)
    equals the one-process oracle; world 3 exercises an owner cycle longer than a pair."""
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_gloo_worker, args=(world, port, n, w, bc, seed, str(tmp_path)), nprocs=world, join=True)
    S, Q, sel = problem(n, w, seed)
    ref = oracle_ref(S, Q, sel, w)
    Sg = np.zeros((n, n))
    Qg = np.zeros((n, n))
    for r in range(world):
        Sx = np.load(tmp_path / ("S%d.npy" % r))
        for j in range(n):
            if (j // bc) % world == r:
                Sg[:, j] = Sx[:, DI.ext_lcol(j, world, bc, w)]
        _, q0, q1 = sn.dist_layout(n, world, bc, r)
        Qg[q0:q1] = np.load(tmp_path / ("Q%d.npy" % r))
    assert np.abs(Sg - ref["S"]).max() <= TOL * np.linalg.norm(S)
    assert np.abs(Qg - ref["Q"]).max() <= TOL
