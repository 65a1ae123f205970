"""Multi-GPU host logic, CPU only: world_size-2 and -3 process
groups over gloo, each process deriving its own partition, ownership, halo and
row-move plans from the library (include/rsrs.h rsrs_tree_partition /
rsrs_dist_*), then exchanging them over torch.distributed and checking that
what rank a plans to send to rank b is exactly what rank b plans to receive
from a, that every foreign neighbour row a box needs is received, and that
skeleton rows reach the owner of their parent.  The GPU side of the same plans
is checked by tests/test_gpu_dist.py (emulated ranks, bit-exact against one GPU).
"""
import os
import socket

import numpy as np
import pytest

import workloads as W

NB_SEED = 123


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(kind):
    if kind == "grid":
        cfg = W.Config("g", "grid2d", 96, "log2d", "f64", leaf=16)
    else:
        cfg = W.Config("s", "sphere", 6000, "lap3d", "f64", leaf=24)
    return cfg


def _synthetic_counts(tree, rng):
    """Per level: nb (active rows) and k (skeletons <= nb) of every box, identical on all ranks."""
    out = {}
    L = tree.L
    nb = np.diff(tree.level(L)["start"]).astype(np.int32)
    for lev in range(L, 0, -1):
        k = np.minimum(nb, rng.integers(0, 9, size=nb.shape[0])).astype(np.int32)
        out[lev] = (nb.copy(), k)
        par = tree.level(lev)["parent"]
        nb = np.bincount(par, weights=k, minlength=len(tree.level(lev - 1)["keys"])).astype(np.int32)
    return out


def _worker(rank, world, port, kind, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2311_01451_b200 as R
        cfg = _problem(kind)
        X = W.points(cfg)
        t = R.Tree(X, cfg.leaf, *cfg.root())
        first, gl = t.partition(world)
        counts = _synthetic_counts(t, np.random.default_rng(NB_SEED))
        mine = {"first": first.tolist(), "gather": gl, "halo": {}, "move": {}, "owner": {}}
        ncol = 3 ** t.d
        for lev in range(t.L, 1, -1):
            lv = t.level(lev)
            nb, k = counts[lev]
            mine["owner"][lev] = t.owner(lev, world).tolist()
            for c in range(ncol):
                cnt = np.where((lv["colour"] < c) & (nb > 0), k, nb).astype(np.int32)
                mine["halo"][(lev, c)] = t.halo_plan(world, lev, c, nb, cnt, rank).tolist()
            mine["move"][lev] = t.move_plan(world, lev, k, rank).tolist()
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        q.put((rank, allp))
    finally:
        dist.destroy_process_group()


def _check(world, kind, allp):
    import paper_2311_01451_b200 as R
    cfg = _problem(kind)
    X = W.points(cfg)
    t = R.Tree(X, cfg.leaf, *cfg.root())
    N = X.shape[0]
    first = np.array(allp[0]["first"])
    # every rank derived the same partition and ownership
    for r in range(world):
        assert allp[r]["first"] == allp[0]["first"] and allp[r]["gather"] == allp[0]["gather"]
        assert allp[r]["owner"] == allp[0]["owner"]
    assert first[0] == 0 and first[-1] == N and np.all(np.diff(first) >= 0)
    gl = allp[0]["gather"]
    counts = _synthetic_counts(t, np.random.default_rng(NB_SEED))
    ncol = 3 ** t.d
    for lev in range(t.L, 1, -1):
        lv = t.level(lev)
        nb, k = counts[lev]
        own = np.array(allp[0]["owner"][lev])
        # owner = rank whose leaf range holds the box's first point (rank 0 at/above the gather level)
        starts = lv["start"][:-1]
        expect = np.searchsorted(first, starts, side="right") - 1 if lev > gl else np.zeros_like(own)
        assert np.array_equal(own, expect)
        for c in range(ncol):
            cnt = np.where((lv["colour"] < c) & (nb > 0), k, nb)
            plans = [np.array(allp[r]["halo"][(lev, c)]).reshape(-1, 4) for r in range(world)]
            for a in range(world):
                for b in range(world):
                    sa = plans[a][(plans[a][:, 0] == 0) & (plans[a][:, 1] == b)][:, 2:]
                    rb = plans[b][(plans[b][:, 0] == 1) & (plans[b][:, 1] == a)][:, 2:]
                    assert np.array_equal(sa, rb), (lev, c, a, b)
            # coverage: each colour-c box needs every foreign neighbour with active rows
            for bx in np.flatnonzero((lv["colour"] == c) & (nb > 0)):
                need = {int(j) for j in lv["neighbours"][bx] if own[j] != own[bx] and cnt[j] > 0}
                rp = plans[own[bx]]
                got = {int(j) for j in rp[rp[:, 0] == 1][:, 2]}
                assert need <= got, (lev, c, bx)
                for j in need:
                    row = rp[(rp[:, 0] == 1) & (rp[:, 2] == j)]
                    assert row.shape[0] == 1 and row[0, 1] == own[j] and row[0, 3] == cnt[j]
        # skeleton rows reach the owner of the parent
        par = lv["parent"]
        pown = np.array(allp[0]["owner"][lev - 1]) if lev - 1 >= 2 else None
        mplans = [np.array(allp[r]["move"][lev]).reshape(-1, 4) for r in range(world)]
        for bx in np.flatnonzero(k > 0):
            src = own[bx]
            dst = (0 if lev - 1 <= gl else
                   int(np.searchsorted(first, t.level(lev - 1)["start"][par[bx]], side="right") - 1))
            if pown is not None:
                assert dst == pown[par[bx]]
            sent = mplans[src][(mplans[src][:, 0] == 0) & (mplans[src][:, 2] == bx)]
            recv = mplans[dst][(mplans[dst][:, 0] == 1) & (mplans[dst][:, 2] == bx)]
            if src == dst:
                assert sent.shape[0] == 0 and recv.shape[0] == 0
            else:
                assert sent.shape[0] == 1 and sent[0, 1] == dst and sent[0, 3] == k[bx]
                assert recv.shape[0] == 1 and recv[0, 1] == src and recv[0, 3] == k[bx]


@pytest.mark.parametrize("world,kind", [(2, "grid"), (3, "sphere"), (2, "sphere")])
def test_plans_consistent_across_gloo_ranks(world, kind):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allp = dict(res)[0]
    for r, a in res:
        assert a == allp        # all_gather_object gave every rank the same view
    _check(world, kind, allp)


def test_partition_balanced():
    """Morton ranges of about equal modelled work (box + neighbour points)^2."""
    import paper_2311_01451_b200 as R
    cfg = W.CONFIGS["c1"].scaled(128)
    t = R.Tree(W.points(cfg), 16, *cfg.root())
    lv = t.level(t.L)
    sizes = np.diff(lv["start"])
    w = np.array([float(sum(sizes[j] for j in nb)) ** 2 for nb in lv["neighbours"]])
    for G in (2, 3, 4, 8):
        first, _ = t.partition(G)
        cut = np.searchsorted(lv["start"], first)
        share = np.array([w[cut[q]:cut[q + 1]].sum() for q in range(G)]) / w.sum()
        assert share.max() <= 1.0 / G + w.max() / w.sum() + 1e-12
