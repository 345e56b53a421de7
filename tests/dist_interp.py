"""A plain interpreter of the sharded program (sn_dist_program records, include/sn_reorder.h)
for the CPU tests: numpy for the panel updates, the ORACLE's swap primitive for the window
tasks, and either shared memory (all ranks in one process) or torch.distributed (gloo) for
the messages and the Z broadcast.  It checks the program -- ownership, straddle pulls and
pushes, lent and halo columns, strip coverage, phase order -- not the CUDA kernels (those are
checked on the GPU through sn_reorder_schur_dist_local).

TEST INFRASTRUCTURE: may use oracle/ (tests only).
"""
from __future__ import annotations

import numpy as np

import oracle
import paper_1905_04975_b200 as sn


def parse(rec):
    """records -> (header, windows, levels) with per-level op lists."""
    assert rec[0, 0] == 0
    nlev, nwin, ext_cols, q0, q1, hc = (int(x) for x in rec[0, 1:7])
    wins = []
    i = 1
    for _ in range(nwin):
        r = rec[i]
        assert r[0] == 1
        wins.append(dict(level=int(r[1]), t=int(r[2]), j1=int(r[3]), k=int(r[4]), owner=int(r[5]),
                         partner=int(r[6]), coff=int(r[7])))
        i += 1
    levels = []
    for _ in range(nlev):
        r = rec[i]
        assert r[0] == 2
        lev = dict(level=int(r[1]), w0=int(r[2]), w1=int(r[3]), pull=[], L=[], R=[], push=[], Q=[],
                   Lr=[], Rr=[])
        i += 1
        key = {3: "pull", 4: "L", 5: "R", 7: "push", 6: "Q", 8: "Lr", 9: "Rr"}
        while i < len(rec) and rec[i, 0] != 2:
            lev[key[int(rec[i, 0])]].append(tuple(int(x) for x in rec[i, 1:]))
            i += 1
        levels.append(lev)
    assert i == len(rec)
    return dict(nlev=nlev, ext_cols=ext_cols, q0=q0, q1=q1, hc=hc), wins, levels


def ext_lcol(j, P, bc, hc):
    b = j // bc
    return (b // P) * (bc + hc) + (j - b * bc)


def shard(S, Q, P, bc, hc, rank, hdr):
    """Extended local S (n x ext_cols, halo slots zero) and Q rows of `rank`."""
    n = S.shape[0]
    Sx = np.zeros((n, max(hdr["ext_cols"], 1)), order="F")
    for j in range(n):
        if (j // bc) % P == rank:
            Sx[:, ext_lcol(j, P, bc, hc)] = S[:, j]
    Ql = None if Q is None else np.asfortranarray(Q[hdr["q0"]:hdr["q1"], :])
    return Sx, Ql


def window_task(D, swaps):
    """The window's swaps (oracle primitive, schedule order) on D and on Z = I."""
    k = D.shape[0]
    Z = np.eye(k, order="F")
    for (j, n1, n2) in swaps:
        rc, D, Z = oracle.swap(D, j, n1, n2, Z)
        assert rc == 0
    return D, Z


class Shared:
    """All ranks in one process: messages are array copies, Z a shared dict."""

    def __init__(self, states):
        self.st = states

    def send(self, src, dst, nrows, ncols, sl, dl):
        self.st[dst]["Sx"][:nrows, dl:dl + ncols] = self.st[src]["Sx"][:nrows, sl:sl + ncols]


def do_W(me, lev, wins, Zs, sched, rank):
    Sx = me["Sx"]
    for i in range(lev["w0"], lev["w1"]):
        w = wins[i]
        if w["owner"] != rank:
            continue
        j1, k, c = w["j1"], w["k"], w["coff"]
        D = np.asfortranarray(Sx[j1:j1 + k, j1 + c:j1 + c + k])
        lo, hi = sched["off"][w["t"]], sched["off"][w["t"] + 1]
        sw = [(int(sched["swap_j"][q]) - j1, int(sched["swap_n1"][q]), int(sched["swap_n2"][q]))
              for q in range(lo, hi)]
        D, Z = window_task(D, sw)
        Sx[j1:j1 + k, j1 + c:j1 + c + k] = D
        Zs[i] = Z


def do_L(me, lev, wins, Zs, key="L"):
    Sx, w0 = me["Sx"], lev["w0"]
    for (wl, cnt, x0, *_r) in lev[key]:
        w = wins[w0 + wl]
        j1, k = w["j1"], w["k"]
        Sx[j1:j1 + k, x0:x0 + cnt] = Zs[w0 + wl].T @ Sx[j1:j1 + k, x0:x0 + cnt]


def do_R(me, lev, wins, Zs, rank, key="R"):
    Sx, w0 = me["Sx"], lev["w0"]
    for (wl, cnt, x0, *_r) in lev[key]:
        w = wins[w0 + wl]
        j1, k, c = w["j1"], w["k"], w["coff"]
        assert w["owner"] == rank
        Sx[x0:x0 + cnt, j1 + c:j1 + c + k] = Sx[x0:x0 + cnt, j1 + c:j1 + c + k] @ Zs[w0 + wl]


def do_Q(me, lev, wins, Zs):
    Ql, w0 = me["Q"], lev["w0"]
    if Ql is None:
        return
    for (wl, cnt, x0, *_r) in lev["Q"]:
        w = wins[w0 + wl]
        j1, k = w["j1"], w["k"]
        Ql[x0:x0 + cnt, j1:j1 + k] = Ql[x0:x0 + cnt, j1:j1 + k] @ Zs[w0 + wl]


def gather(states, n, P, bc, hc):
    S = np.zeros((n, n))
    for r in range(P):
        for j in range(n):
            if (j // bc) % P == r:
                S[:, j] = states[r]["Sx"][:, ext_lcol(j, P, bc, hc)]
    return S


def prepare(S, Q, select, w, bc, P):
    rc, bmap = oracle.scan(S)
    assert rc == 0
    selrow, _m = oracle.select(bmap, select)
    sched = oracle.schedule(bmap, selrow, w)
    progs = [parse(sn.dist_program(bmap, selrow, w, bc, P, r)) for r in range(P)]
    return bmap, selrow, sched, progs


def run_shared(S, Q, select, w, bc, P):
    """All P ranks in this process; returns (S, Q) gathered, and the programs."""
    n = S.shape[0]
    _bmap, _selrow, sched, progs = prepare(S, Q, select, w, bc, P)
    states = []
    for r in range(P):
        Sx, Ql = shard(S, Q, P, bc, w, r, progs[r][0])
        states.append({"Sx": Sx, "Q": Ql})
    Zs = {}
    sh = Shared(states)
    nlev = progs[0][0]["nlev"]
    prev = None
    for l in range(nlev):
        # phase by phase over the ranks, in the executor's order: the previous level's
        # remaining strips run only after this level's pulls and window tasks
        levs = [progs[r][2][l] for r in range(P)]
        for m in levs[0]["pull"]:
            sh.send(m[1], m[2], m[3], m[4], m[5], m[6])
        for r in range(P):
            do_W(states[r], levs[r], progs[r][1], Zs, sched, r)
        if prev is not None:
            for r in range(P):
                do_L(states[r], prev[r], progs[r][1], Zs, "Lr")
            for r in range(P):
                do_R(states[r], prev[r], progs[r][1], Zs, r, "Rr")
        for r in range(P):
            do_L(states[r], levs[r], progs[r][1], Zs)
        for r in range(P):
            do_R(states[r], levs[r], progs[r][1], Zs, r)
        for m in levs[0]["push"]:
            sh.send(m[1], m[2], m[3], m[4], m[5], m[6])
        for r in range(P):
            do_Q(states[r], levs[r], progs[r][1], Zs)
        prev = levs
    if prev is not None:
        for r in range(P):
            do_L(states[r], prev[r], progs[r][1], Zs, "Lr")
        for r in range(P):
            do_R(states[r], prev[r], progs[r][1], Zs, r, "Rr")
    Sg = gather(states, n, P, bc, w)
    Qg = None
    if Q is not None:
        Qg = np.zeros_like(Q)
        for r in range(P):
            Qg[progs[r][0]["q0"]:progs[r][0]["q1"], :] = states[r]["Q"]
    return Sg, Qg, progs


def run_gloo(S, Q, select, w, bc, rank, P):
    """This process is `rank` of a torch.distributed (gloo) group of P: its shard only; the
    pulls/pushes are send/recv, the Zs a broadcast from each window's owner."""
    import torch
    import torch.distributed as dist
    _bmap, _selrow, sched, progs = prepare(S, Q, select, w, bc, P)
    hdr, wins, levels = progs[rank]
    Sx, Ql = shard(S, Q, P, bc, w, rank, hdr)
    me = {"Sx": Sx, "Q": Ql}
    Zs = {}

    def exchange(msgs):
        ops = []
        for (_w, src, dst, nrows, ncols, sl, dl) in msgs:
            if src == dst:
                if src == rank:
                    Sx[:nrows, dl:dl + ncols] = Sx[:nrows, sl:sl + ncols]
                continue
            if src == rank:
                t = torch.from_numpy(np.ascontiguousarray(Sx[:nrows, sl:sl + ncols]))
                ops.append(("s", dist.isend(t, dst), None, None))
            elif dst == rank:
                t = torch.empty((nrows, ncols), dtype=torch.float64)
                ops.append(("r", dist.irecv(t, src), t, (nrows, ncols, dl)))
        for kind, h, t, meta in ops:
            h.wait()
            if kind == "r":
                nrows, ncols, dl = meta
                Sx[:nrows, dl:dl + ncols] = t.numpy()

    prev = None
    for lev in levels:
        exchange(lev["pull"])
        do_W(me, lev, wins, Zs, sched, rank)
        for i in range(lev["w0"], lev["w1"]):
            k = wins[i]["k"]
            t = torch.from_numpy(np.ascontiguousarray(Zs[i])) if wins[i]["owner"] == rank else \
                torch.empty((k, k), dtype=torch.float64)
            dist.broadcast(t, src=wins[i]["owner"])
            Zs[i] = t.numpy()
        if prev is not None:
            do_L(me, prev, wins, Zs, "Lr")
            do_R(me, prev, wins, Zs, rank, "Rr")
        do_L(me, lev, wins, Zs)
        do_R(me, lev, wins, Zs, rank)
        exchange(lev["push"])
        do_Q(me, lev, wins, Zs)
        prev = lev
    if prev is not None:
        do_L(me, prev, wins, Zs, "Lr")
        do_R(me, prev, wins, Zs, rank, "Rr")
    return me, hdr
