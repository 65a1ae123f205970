"""Oracle: uniform 2^d-tree, Morton order, neighbour and colour lists.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

Follows PAPER.md:799-820 (section 4.1 "Hierarchical tree structure": split the
root into 2^d children until each node holds at most m points; uniform tree,
level l = nodes of depth l, L ~ log2(N/m)) and PAPER.md:182-184 (Fig. 1
caption: "Boxes on the same level which share an edge or corner are called
neighbors"; box 9 has neighbours {8,9,10}).

Readings:
  * depth L = smallest L with max leaf occupancy <= m; empty boxes are not
    stored (SURVEY c.2 #12);
  * box coordinate at level l: clamp(floor((x - lo) / side * 2^l), 0, 2^l - 1);
  * neighbours = nonempty boxes at Chebyshev distance <= 1 (self included),
    listed in Morton order (c.2 #13);
  * tree order = points sorted by leaf Morton key, ties by original index;
  * colour = sum_i (c_i mod 3) 3^i -- boxes of one colour are >= 3 apart, so
    their near sets are disjoint (reading R10);
  * canonical box order inside a level: colour-major, Morton inside a colour.
Written independently of the C++ tree (paper_2311_01451_b200/csrc); a test
checks the two agree.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np


def morton_encode(coords: np.ndarray, d: int) -> np.ndarray:
    """Interleave bits: bit b of coordinate i goes to bit b*d + i."""
    coords = np.asarray(coords, dtype=np.int64)
    key = np.zeros(coords.shape[0], dtype=np.int64)
    for b in range(21):
        for i in range(d):
            key |= ((coords[:, i] >> b) & 1) << (b * d + i)
    return key


def morton_decode(keys: np.ndarray, d: int) -> np.ndarray:
    keys = np.asarray(keys, dtype=np.int64)
    c = np.zeros((keys.shape[0], d), dtype=np.int64)
    for b in range(21):
        for i in range(d):
            c[:, i] |= ((keys >> (b * d + i)) & 1) << b
    return c


@dataclass
class Level:
    keys: np.ndarray        # Morton keys of the nonempty boxes, ascending
    coords: np.ndarray      # (nb, d) integer box coordinates
    start: np.ndarray       # (nb+1,) tree-position ranges of the boxes' points
    parent: np.ndarray      # index of the parent box on level-1 (-1 at level 0)
    neighbours: list        # list of int arrays (indices on this level, Morton order)
    colour: np.ndarray      # (nb,) colour in [0, 3^d)

    @property
    def nboxes(self) -> int:
        return self.keys.shape[0]

    def children_of(self, child_level: "Level"):
        out = [[] for _ in range(self.nboxes)]
        for j, pidx in enumerate(child_level.parent):
            out[pidx].append(j)
        return out


@dataclass
class Tree:
    d: int
    N: int
    L: int
    perm: np.ndarray        # tree position -> original index
    levels: list            # levels[l] for l = 0..L

    def canonical_order(self, lev: int) -> list:
        """Boxes of a level: colour-major, Morton-ascending inside a colour."""
        lv = self.levels[lev]
        order = np.lexsort((np.arange(lv.nboxes), lv.colour))
        return [int(b) for b in order]


def build_tree(X: np.ndarray, leaf: int, lo=None, side=None) -> Tree:
    X = np.asarray(X, dtype=np.float64)
    N, d = X.shape
    if lo is None or side is None:
        lo = X.min(axis=0)
        side = float((X.max(axis=0) - lo).max()) * (1 + 1e-12) or 1.0
    lo = np.asarray(lo, dtype=np.float64)

    def coords_at(lev):
        n = 1 << lev
        c = np.floor((X - lo) / side * n).astype(np.int64)
        return np.clip(c, 0, n - 1)

    L = 0
    while True:
        keys = morton_encode(coords_at(L), d) if N else np.zeros(0, np.int64)
        occ = np.bincount(np.unique(keys, return_inverse=True)[1]).max() if N else 0
        if occ <= leaf:
            break
        L += 1
        if L > 20:
            raise ValueError("tree depth exceeds 20 (coincident points?)")
    perm = np.argsort(keys, kind="stable")
    skeys = keys[perm]
    levels = []
    for lev in range(L + 1):
        lk = skeys >> (d * (L - lev))
        if N:
            change = np.flatnonzero(np.diff(lk)) + 1
            starts = np.concatenate([[0], change, [N]])
            bkeys = lk[starts[:-1]]
        else:
            starts = np.zeros(1, np.int64)
            bkeys = np.zeros(0, np.int64)
        coords = morton_decode(bkeys, d)
        colour = np.zeros(bkeys.shape[0], dtype=np.int64)
        for i in range(d):
            colour += (coords[:, i] % 3) * (3 ** i)
        lookup = {int(k): j for j, k in enumerate(bkeys)}
        neigh = []
        nside = 1 << lev
        for j in range(bkeys.shape[0]):
            nb = []
            for off in itertools.product((-1, 0, 1), repeat=d):
                c = coords[j] + np.array(off)
                if np.any(c < 0) or np.any(c >= nside):
                    continue
                k = int(morton_encode(c[None, :], d)[0])
                if k in lookup:
                    nb.append(lookup[k])
            neigh.append(np.array(sorted(nb), dtype=np.int64))
        if lev == 0:
            parent = -np.ones(bkeys.shape[0], dtype=np.int64)
        else:
            pk = bkeys >> d
            pl = levels[lev - 1]
            plook = {int(k): j for j, k in enumerate(pl.keys)}
            parent = np.array([plook[int(k)] for k in pk], dtype=np.int64)
        levels.append(Level(bkeys, coords, starts.astype(np.int64), parent, neigh, colour))
    return Tree(d=d, N=N, L=L, perm=perm.astype(np.int64), levels=levels)
