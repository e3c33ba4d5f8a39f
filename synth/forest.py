"""Seeded random tree ensembles in the flat per-node form the C ABI takes.

``Ensemble`` mirrors ``hb_ensemble`` (include/hb.h) and ``oracle_ensemble``
(oracle/oracle.h) field by field; it is a plain container with no scoring
logic. Node ids are tree-local, 0 is the root, leaves have left == right == -1
(SURVEY.md §8(b)); by default non-root ids are randomly permuted so no
consumer can rely on BFS order.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .xgen import GRID_FINE, GRID_COARSE

CMP_LT, CMP_LE = 0, 1
AGG_SUM, AGG_MEAN = 0, 1
POST_IDENTITY, POST_SIGMOID, POST_SOFTMAX, POST_ISOLATION = 0, 1, 2, 3
TASK_REGRESSION, TASK_CLASSIFICATION = 0, 1

_NCODES = {GRID_FINE: 65536, GRID_COARSE: 64}
_STEP = {GRID_FINE: 1.0 / 4096.0, GRID_COARSE: 0.25}
_ZERO = {GRID_FINE: 32768, GRID_COARSE: 32}


@dataclass
class Ensemble:
    n_trees: int
    n_features: int
    n_outputs: int
    node_offset: np.ndarray          # int64 [T+1]
    feature: np.ndarray              # int32 [N]   (-1 at leaves)
    threshold: np.ndarray            # float32 [N] (NaN at leaves; never read there)
    left: np.ndarray                 # int32 [N]   tree-local, -1 at leaves
    right: np.ndarray                # int32 [N]
    leaf_value: np.ndarray           # float32 [N * leaf_width] (NaN at internal nodes)
    leaf_width: int = 1
    tree_output: Optional[np.ndarray] = None   # int32 [T]; None => t % K
    base_score: Optional[np.ndarray] = None    # float32 [K]; None => 0
    cmp: int = CMP_LT
    agg: int = AGG_SUM
    post: int = POST_IDENTITY
    task: int = TASK_REGRESSION
    post_param: float = 0.0          # ISOLATION: c(psi)

    @property
    def n_nodes(self) -> int:
        return int(self.node_offset[-1])

    def tree(self, t: int):
        a, b = int(self.node_offset[t]), int(self.node_offset[t + 1])
        w = self.leaf_width
        return dict(feature=self.feature[a:b], threshold=self.threshold[a:b],
                    left=self.left[a:b], right=self.right[a:b],
                    leaf_value=self.leaf_value[a * w:b * w].reshape(b - a, w))

    def subset(self, t0: int, t1: int) -> "Ensemble":
        """Trees [t0, t1) as a new ensemble (same globals; used by shard tests)."""
        a, b = int(self.node_offset[t0]), int(self.node_offset[t1])
        w = self.leaf_width
        to = None if self.tree_output is None else self.tree_output[t0:t1].copy()
        if to is None and self.leaf_width == 1 and self.n_outputs > 1:
            to = (np.arange(t0, t1) % self.n_outputs).astype(np.int32)
        return Ensemble(t1 - t0, self.n_features, self.n_outputs,
                        (self.node_offset[t0:t1 + 1] - a).astype(np.int64),
                        self.feature[a:b].copy(), self.threshold[a:b].copy(),
                        self.left[a:b].copy(), self.right[a:b].copy(),
                        self.leaf_value[a * w:b * w].copy(), w, to,
                        None if self.base_score is None else self.base_score.copy(),
                        self.cmp, self.agg, self.post, self.task, self.post_param)


def from_trees(trees, n_features, n_outputs=1, leaf_width=1, **kw) -> Ensemble:
    """Build an Ensemble from a list of dicts with per-tree arrays
    (feature, threshold, left, right, leaf_value[n, w]) — used for the
    hand-built trees of the golden tests."""
    off = [0]
    F, TH, L, R, V = [], [], [], [], []
    for t in trees:
        n = len(t["left"])
        off.append(off[-1] + n)
        F.append(np.asarray(t["feature"], np.int32))
        TH.append(np.asarray(t["threshold"], np.float32))
        L.append(np.asarray(t["left"], np.int32))
        R.append(np.asarray(t["right"], np.int32))
        V.append(np.asarray(t["leaf_value"], np.float32).reshape(n * leaf_width))
    to = kw.pop("tree_output", None)
    bs = kw.pop("base_score", None)
    return Ensemble(len(trees), n_features, n_outputs, np.asarray(off, np.int64),
                    np.concatenate(F), np.concatenate(TH), np.concatenate(L),
                    np.concatenate(R), np.concatenate(V), leaf_width,
                    None if to is None else np.asarray(to, np.int32),
                    None if bs is None else np.asarray(bs, np.float32), **kw)


def gen_forest(n_trees: int, depth: int, n_features: int, *, seed: int = 0,
               family: str = "balanced", split_prob: float = 0.85,
               n_outputs: int = 1, leaf_width: int = 1,
               leaf_kind: str = "normal", leaf_sigma: float = 0.1,
               grid: int = GRID_FINE, thr_mode: str = "grid",
               tree_output: Optional[np.ndarray] = None,
               base_score=None, cmp: int = CMP_LT, agg: int = AGG_SUM,
               post: int = POST_IDENTITY, task: int = TASK_REGRESSION,
               permute: bool = True, features=None, post_param: float = 0.0) -> Ensemble:
    """Draw ``n_trees`` random trees of maximum depth ``depth``.

    family: "balanced" (XGBoost-like, every node splits down to ``depth``),
            "mixed"    (RF-like, each node splits with ``split_prob``),
            "skinny"   (LightGBM-like leaf-wise look: split prob 0.5 but at
                        least one split per level so the tree reaches ``depth``).
    leaf_kind: "normal" N(0, sigma^2); "dirichlet" (class distributions,
               needs leaf_width == n_outputs); "dyadic" (multiples of 2^-10
               in [-1, 1], sums exact in fp32); "const" (one dyadic value per
               tree).
    features: optional array of allowed feature ids (default all).
    """
    rng = np.random.default_rng(seed)
    ncodes, step, zero = _NCODES[grid], _STEP[grid], _ZERO[grid]
    feats = np.arange(n_features) if features is None else np.asarray(features)

    # frontier = nodes of the current level, across all trees
    tree_of = np.arange(n_trees, dtype=np.int64)
    path_f = np.zeros((n_trees, 0), np.int32)     # ancestor feature
    path_k = np.zeros((n_trees, 0), np.int32)     # ancestor threshold code
    path_d = np.zeros((n_trees, 0), np.int8)      # 0 = we are in its left subtree
    # per generated node (BFS id within tree assigned by order of creation)
    rec_tree, rec_parent, rec_side, rec_feat, rec_code, rec_leaf = [], [], [], [], [], []
    parent_gid = np.full(n_trees, -1, np.int64)   # global creation id of parent
    side = np.zeros(n_trees, np.int8)
    gid_next = 0
    for lvl in range(depth + 1):
        m = tree_of.size
        if m == 0:
            break
        gid = np.arange(gid_next, gid_next + m, dtype=np.int64)
        gid_next += m
        if lvl == depth:
            split = np.zeros(m, bool)
        elif family == "balanced" or lvl == 0:
            split = np.ones(m, bool)
        elif family == "mixed":
            split = rng.random(m) < split_prob
        elif family == "skinny":
            split = rng.random(m) < 0.5
            # force >= 1 split per tree per level
            order = rng.permutation(m)
            first = np.full(n_trees, -1, np.int64)
            first[tree_of[order][::-1]] = order[::-1]
            has = np.zeros(n_trees, bool)
            np.logical_or.at(has, tree_of[split], True)
            need = (~has) & (first >= 0)
            split[first[need]] = True
        else:
            raise ValueError(family)
        f = feats[rng.integers(0, feats.size, m)].astype(np.int32)
        lo = np.zeros(m, np.int64)
        hi = np.full(m, ncodes, np.int64)
        for d in range(path_f.shape[1]):
            same = path_f[:, d] == f
            k = path_k[:, d].astype(np.int64)
            right_anc = same & (path_d[:, d] == 1)
            left_anc = same & (path_d[:, d] == 0)
            lo = np.where(right_anc, np.maximum(lo, k), lo)
            hi = np.where(left_anc, np.minimum(hi, k), hi)
        span = hi - lo - 1
        code = np.where(span >= 1, lo + 1 + (rng.random(m) * np.maximum(span, 1)).astype(np.int64), lo)
        code = np.clip(code, 0, ncodes - 1).astype(np.int32)
        rec_tree.append(tree_of)
        rec_parent.append(parent_gid)
        rec_side.append(side)
        rec_feat.append(np.where(split, f, -1).astype(np.int32))
        rec_code.append(code)
        rec_leaf.append(~split)
        # children of split nodes
        s = np.nonzero(split)[0]
        ns = s.size
        tree_of = np.repeat(tree_of[s], 2)
        parent_gid = np.repeat(gid[s], 2)
        side = np.tile(np.array([0, 1], np.int8), ns)
        path_f = np.concatenate([np.repeat(path_f[s], 2, 0), np.repeat(f[s], 2)[:, None]], 1)
        path_k = np.concatenate([np.repeat(path_k[s], 2, 0), np.repeat(code[s], 2)[:, None]], 1)
        path_d = np.concatenate([np.repeat(path_d[s], 2, 0), side[:, None]], 1)

    g_tree = np.concatenate(rec_tree)
    g_parent = np.concatenate(rec_parent)
    g_side = np.concatenate(rec_side)
    g_feat = np.concatenate(rec_feat)
    g_code = np.concatenate(rec_code)
    g_leaf = np.concatenate(rec_leaf)
    G = g_tree.size
    # group nodes by tree (stable keeps BFS order within a tree: root first)
    order = np.argsort(g_tree, kind="stable")
    counts = np.bincount(g_tree, minlength=n_trees)
    off = np.zeros(n_trees + 1, np.int64)
    off[1:] = np.cumsum(counts)
    rank_in_tree = np.empty(G, np.int64)
    rank_in_tree[order] = np.arange(G) - np.repeat(off[:-1], counts)
    if permute:
        # random relabel of non-root nodes within each tree
        keys = rng.random(G)
        keys[rank_in_tree == 0] = -1.0
        o2 = np.lexsort((keys, g_tree))
        local = np.empty(G, np.int64)
        local[o2] = np.arange(G) - np.repeat(off[:-1], counts)
    else:
        local = rank_in_tree
    pos = off[g_tree] + local            # global flat slot of each node
    feature = np.full(G, -1, np.int32)
    threshold = np.full(G, np.nan, np.float32)
    left = np.full(G, -1, np.int32)
    right = np.full(G, -1, np.int32)
    internal = ~g_leaf
    feature[pos[internal]] = g_feat[internal]
    if thr_mode == "grid":
        tv = (g_code.astype(np.float64) - zero) * step
    elif thr_mode == "mid":
        tv = (g_code.astype(np.float64) - zero - 0.5) * step
    else:
        raise ValueError(thr_mode)
    threshold[pos[internal]] = tv[internal].astype(np.float32)
    has_parent = g_parent >= 0
    ch = np.nonzero(has_parent)[0]
    ppos = pos[g_parent[ch]]
    lsel = g_side[ch] == 0
    left[ppos[lsel]] = local[ch[lsel]]
    right[ppos[~lsel]] = local[ch[~lsel]]

    w = leaf_width
    leaf_value = np.full((G, w), np.nan, np.float32)
    lpos = pos[g_leaf]
    nl = lpos.size
    if leaf_kind == "normal":
        leaf_value[lpos] = (rng.standard_normal((nl, w)) * leaf_sigma).astype(np.float32)
    elif leaf_kind == "dirichlet":
        p = rng.dirichlet(np.ones(w), nl).astype(np.float32)
        leaf_value[lpos] = p / p.sum(1, keepdims=True, dtype=np.float32)
    elif leaf_kind == "dyadic":
        leaf_value[lpos] = (rng.integers(-1024, 1025, (nl, w)) / 1024.0).astype(np.float32)
    elif leaf_kind == "const":
        c = (rng.integers(-1024, 1025, (n_trees, w)) / 1024.0).astype(np.float32)
        leaf_value[lpos] = c[g_tree[g_leaf]]
    else:
        raise ValueError(leaf_kind)

    if tree_output is not None:
        tree_output = np.asarray(tree_output, np.int32)
    if base_score is not None:
        base_score = np.asarray(base_score, np.float32).reshape(n_outputs)
    return Ensemble(n_trees, n_features, n_outputs, off, feature, threshold,
                    left, right, leaf_value.reshape(G * w), w, tree_output,
                    base_score, cmp, agg, post, task, post_param)


def tree_depths(e: Ensemble) -> np.ndarray:
    """Max root->leaf edge count per tree (host helper for configs/tests)."""
    out = np.zeros(e.n_trees, np.int32)
    for t in range(e.n_trees):
        a, b = int(e.node_offset[t]), int(e.node_offset[t + 1])
        L, R = e.left[a:b], e.right[a:b]
        depth = np.zeros(b - a, np.int32)
        stack = [0]
        best = 0
        while stack:
            i = stack.pop()
            if L[i] >= 0:
                depth[L[i]] = depth[i] + 1
                depth[R[i]] = depth[i] + 1
                stack += [L[i], R[i]]
            else:
                best = max(best, depth[i])
        out[t] = best
    return out
