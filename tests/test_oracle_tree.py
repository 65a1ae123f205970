"""Pins for the oracle tree (section 4.1; Fig. 1)."""
import itertools
import json
import os

import numpy as np

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_fig1_worked_example():
    """Fig. 1: 1D tree, box 9 -> neighbours {8,9,10}, far field {11..15}."""
    g = json.load(open(os.path.join(GOLD, "fig1_tree.json")))
    X = ((np.arange(64) + 0.5) / 64.0)[:, None]       # 8 points per level-3 box
    t = O.build_tree(X, leaf=8, lo=np.zeros(1), side=1.0)
    assert t.L == 3
    for lev, ids in g["levels"].items():
        lev = int(lev)
        assert [2 ** lev + int(k) for k in t.levels[lev].keys] == ids
    b = g["box"] - 8
    lv = t.levels[3]
    assert [8 + int(j) for j in lv.neighbours[b]] == g["neighbours"]
    far = [8 + j for j in range(lv.nboxes) if j not in lv.neighbours[b]]
    assert far == g["far_field"]


def _brute(X, t, lo, side):
    N, d = X.shape
    for lev, lv in enumerate(t.levels):
        n = 1 << lev
        # every point of box j lies in the box's cell
        for j in range(lv.nboxes):
            pts = X[t.perm[lv.start[j]:lv.start[j + 1]]]
            c = np.clip(np.floor((pts - lo) / side * n).astype(int), 0, n - 1)
            assert (c == lv.coords[j]).all()
            assert lv.start[j + 1] > lv.start[j]               # nonempty boxes only
        assert lv.start[-1] == N
        # neighbours: brute force over all pairs, Chebyshev <= 1, symmetric
        C = lv.coords
        for j in range(lv.nboxes):
            brute = [q for q in range(lv.nboxes) if np.abs(C[q] - C[j]).max() <= 1]
            assert list(lv.neighbours[j]) == brute
            for q in brute:
                assert j in lv.neighbours[q]
        # parent contains child
        if lev > 0:
            pl = t.levels[lev - 1]
            assert (pl.coords[lv.parent] == lv.coords // 2).all()
        # colour classes are >= 3 apart => near sets disjoint (R10)
        for a, b in itertools.combinations(range(lv.nboxes), 2):
            if lv.colour[a] == lv.colour[b]:
                assert np.abs(C[a] - C[b]).max() >= 3
                assert not set(lv.neighbours[a]) & set(lv.neighbours[b])
    occ = np.diff(t.levels[-1].start).max()
    return occ


def test_brute_force_2d_random():
    rng = np.random.default_rng(0)
    X = rng.random((3000, 2))
    t = O.build_tree(X, leaf=40, lo=np.zeros(2), side=1.0)
    assert _brute(X, t, np.zeros(2), 1.0) <= 40
    # minimal depth: one level less violates the occupancy bound
    t2 = O.build_tree(X, leaf=40, lo=np.zeros(2), side=1.0)
    n = 1 << (t2.L - 1)
    c = np.clip(np.floor(X * n).astype(int), 0, n - 1)
    _, cnt = np.unique(c[:, 0] * n + c[:, 1], return_counts=True)
    assert cnt.max() > 40
    assert sorted(t.perm.tolist()) == list(range(3000))


def test_brute_force_sphere():
    import workloads as W
    X = W.fibonacci_sphere(4000)
    t = O.build_tree(X, leaf=64, lo=-np.ones(3), side=2.0)
    assert _brute(X, t, -np.ones(3), 2.0) <= 64


def test_uniform_grid_c1_shape():
    import workloads as W
    cfg = W.CONFIGS["c1"]
    t = O.build_tree(W.points(cfg), cfg.leaf, *cfg.root())
    assert t.L == 3
    assert [lv.nboxes for lv in t.levels] == [1, 4, 16, 64]
    assert (np.diff(t.levels[3].start) == 64).all()
    # interior leaf boxes see 9 neighbours (share an edge or corner)
    assert max(len(n) for n in t.levels[3].neighbours) == 9
    assert min(len(n) for n in t.levels[3].neighbours) == 4


def test_morton_roundtrip():
    rng = np.random.default_rng(1)
    for d in (1, 2, 3):
        c = rng.integers(0, 1 << 12, size=(200, d))
        assert (O.morton_decode(O.morton_encode(c, d), d) == c).all()
