"""Pins of the CPU oracle to things other than itself (SURVEY.md §8(c) P-a..P-g).

P-a hand-traced trees (tests/golden/hand_trees.json)
P-b depth-1 stump closed form at ties, nextafter, +-0, +-Inf, NaN
P-c brute-force threshold regions on 2-feature toys vs an independent
    box (interval-intersection) evaluator
P-e leaf boxes partition the input space
P-f aggregation closed forms (constant trees, MEAN of identical trees,
    per-class routing, shard additivity, order independence)
P-g transform identities checked against scipy (sigmoid = expit, softmax)
"""
import math

import numpy as np
import pytest
import scipy.special

import oracle
import synth
from tests._common import load_hand_trees, small_forest


# ---------------------------------------------------------------- P-a
@pytest.mark.parametrize("cmp", [synth.CMP_LT, synth.CMP_LE])
def test_hand_traced_trees(cmp):
    e, X, exp_leaf, exp_sum = load_hand_trees(cmp)
    assert np.array_equal(oracle.leaf(e, X), exp_leaf)
    r = oracle.raw(e, X)[:, 0]
    assert np.array_equal(r, exp_sum)


# ---------------------------------------------------------------- P-b
def _stump(t, vl, vr, cmp, f=0, F=1):
    return dict(feature=[f, -1, -1], threshold=[t, np.nan, np.nan], left=[1, -1, -1],
                right=[2, -1, -1], leaf_value=[np.nan, vl, vr])


@pytest.mark.parametrize("cmp", [synth.CMP_LT, synth.CMP_LE])
def test_stump_closed_form(cmp):
    rng = np.random.default_rng(11)
    ts = np.concatenate([rng.normal(size=6).astype(np.float32),
                         np.float32([0.0, -0.0, np.inf, -np.inf, 1e-38, 3.4e38])])
    for t in ts:
        t = np.float32(t)
        xs = [t, np.nextafter(t, np.float32(-np.inf)), np.nextafter(t, np.float32(np.inf)),
              np.float32(0.0), np.float32(-0.0), np.float32(np.inf), np.float32(-np.inf),
              np.float32(np.nan), np.float32(rng.normal())]
        X = np.array(xs, np.float32)[:, None]
        e = synth.from_trees([_stump(t, -0.5, 0.25, cmp)], 1, cmp=cmp,
                             base_score=[1.0])
        got = oracle.margin(e, oracle.raw(e, X))[:, 0]
        # closed form: f(x) = base + (x < t ? vL : vR) (LE: x <= t); NaN => vR
        for x, g in zip(xs, got):
            if math.isnan(x):
                left = False
            else:
                left = (float(x) < float(t)) if cmp == synth.CMP_LT else (float(x) <= float(t))
            assert g == 1.0 + (-0.5 if left else 0.25), (t, x)


def test_stump_sum_closed_form():
    # S stumps on distinct features: sum = sum_s (x_s < t_s ? a_s : b_s)
    rng = np.random.default_rng(3)
    S = 12
    t = rng.integers(-8, 8, S).astype(np.float32)
    a = (rng.integers(-64, 64, S) / 64).astype(np.float32)
    b = (rng.integers(-64, 64, S) / 64).astype(np.float32)
    trees = [_stump(t[s], a[s], b[s], 0, f=s) for s in range(S)]
    for tr, s in zip(trees, range(S)):
        tr["feature"] = [s, -1, -1]
    e = synth.from_trees(trees, S)
    X = synth.gen_X(9, 300, S, grid=synth.GRID_COARSE)
    exp = np.where(X < t[None, :], a[None, :], b[None, :]).astype(np.float64).sum(1)
    assert np.array_equal(oracle.raw(e, X)[:, 0], exp)


# ---------------------------------------------------------------- P-c / P-e
def _boxes(tr, cmp, F):
    """Leaf -> per-feature set {x : lo <(=) x <(=) hi} (+ NaN iff no left
    constraint on that feature). Built by intersecting the path constraints;
    independent of the walk."""
    out = {}
    inf = float("inf")

    def rec(i, box):
        if tr["left"][i] == -1:
            out[int(i)] = box
            return
        f, t = int(tr["feature"][i]), float(tr["threshold"][i])
        # left: pred(x, t) true. LT: x < t ; LE: x <= t. NaN never.
        L = [list(b) for b in box]
        lo, loc, hi, hic, nan_ok = L[f]
        if (t < hi) or (t == hi and hic):
            L[f][2], L[f][3] = t, (cmp == synth.CMP_LE)
        L[f][4] = False
        rec(tr["left"][i], [tuple(b) for b in L])
        # right: pred false. LT: x >= t (or NaN) ; LE: x > t (or NaN)
        R = [list(b) for b in box]
        lo, loc, hi, hic, nan_ok = R[f]
        if (t > lo) or (t == lo and loc):
            R[f][0], R[f][1] = t, (cmp == synth.CMP_LT)
        rec(tr["right"][i], [tuple(b) for b in R])

    rec(0, [(-inf, True, inf, True, True)] * F)
    return out


def _in_box(x, box):
    for v, (lo, loc, hi, hic, nan_ok) in zip(x, box):
        v = float(v)
        if math.isnan(v):
            if not nan_ok:
                return False
            continue
        if v < lo or (v == lo and not loc):
            return False
        if v > hi or (v == hi and not hic):
            return False
    return True


def _probe_values(ts):
    ts = np.unique(np.asarray(ts, np.float32))
    vals = [np.float32(np.inf), np.float32(-np.inf), np.float32(np.nan),
            np.float32(0.0), np.float32(-0.0)]
    if ts.size:
        vals += [ts.min() - 1, ts.max() + 1]
    for i, t in enumerate(ts):
        vals += [t, np.nextafter(t, np.float32(-np.inf)), np.nextafter(t, np.float32(np.inf))]
        if i + 1 < ts.size:
            vals.append(np.float32((np.float64(t) + np.float64(ts[i + 1])) / 2))
    return np.array(vals, np.float32)


@pytest.mark.parametrize("seed,cmp", [(1, 0), (2, 1), (3, 0), (4, 1)])
def test_bruteforce_regions_and_partition(seed, cmp):
    rng = np.random.default_rng(seed)
    T = int(rng.integers(1, 17))
    D = int(rng.integers(1, 5))
    e = small_forest(seed, T=T, D=D, F=2, cmp=cmp,
                     family=["balanced", "mixed", "skinny"][seed % 3])
    internal = e.left != -1
    p0 = _probe_values(e.threshold[internal & (e.feature == 0)])
    p1 = _probe_values(e.threshold[internal & (e.feature == 1)])
    X = np.array([[a, b] for a in p0 for b in p1], np.float32)
    got = oracle.leaf(e, X)
    for t in range(e.n_trees):
        boxes = _boxes(e.tree(t), cmp, 2)
        for r in range(X.shape[0]):
            hits = [l for l, b in boxes.items() if _in_box(X[r], b)]
            assert len(hits) == 1, (t, X[r], hits)          # P-e partition
            assert hits[0] == got[r, t], (t, X[r])           # P-c


# ---------------------------------------------------------------- P-f
def test_constant_trees_closed_form():
    e = small_forest(5, T=40, D=5, F=4, leaf_kind="const", base_score=[0.375])
    consts = np.array([e.tree(t)["leaf_value"][e.tree(t)["left"] == -1][0, 0]
                       for t in range(e.n_trees)], np.float64)
    X = synth.gen_X(1, 200, 4, special_q24=1 << 20)
    m = oracle.margin(e, oracle.raw(e, X))[:, 0]
    assert np.all(m == 0.375 + consts.sum())


def test_mean_of_identical_trees_is_one_tree():
    one = small_forest(6, T=1, D=5, F=4, leaf_kind="dyadic", leaf_width=3, n_outputs=3)
    tr = one.tree(0)
    trees = [dict(feature=tr["feature"], threshold=tr["threshold"], left=tr["left"],
                  right=tr["right"], leaf_value=tr["leaf_value"]) for _ in range(8)]
    e = synth.from_trees(trees, 4, n_outputs=3, leaf_width=3, agg=synth.AGG_MEAN)
    X = synth.gen_X(2, 300, 4, grid=synth.GRID_COARSE)
    m8 = oracle.margin(e, oracle.raw(e, X))
    one.agg = synth.AGG_SUM
    m1 = oracle.raw(one, X)
    assert np.array_equal(m8, m1)


def test_per_class_routing_and_shards():
    K = 3
    e = small_forest(7, T=12, D=4, F=5, n_outputs=K, leaf_kind="dyadic")
    X = synth.gen_X(4, 257, 5, grid=synth.GRID_COARSE, special_q24=1 << 20)
    r = oracle.raw(e, X)
    exp = np.zeros_like(r)
    for t in range(e.n_trees):
        exp[:, t % K] += oracle.raw(e, X, t, t + 1)[:, t % K]
    assert np.array_equal(r, exp)
    # explicit tree_output equal to the default
    e2 = small_forest(7, T=12, D=4, F=5, n_outputs=K, leaf_kind="dyadic",
                      tree_output=np.arange(12) % K)
    assert np.array_equal(oracle.raw(e2, X), r)
    # shards add up (tree-sharding)
    s = oracle.raw(e, X, 0, 5) + oracle.raw(e, X, 5, 12)
    assert np.array_equal(s, r)     # dyadic leaves: exact


def test_tree_order_independence():
    e = small_forest(8, T=30, D=5, F=4, leaf_kind="normal")
    X = synth.gen_X(5, 100, 4)
    r = oracle.raw(e, X)[:, 0]
    perm = np.random.default_rng(0).permutation(e.n_trees)
    trees = [e.tree(int(t)) for t in perm]
    e2 = synth.from_trees([dict(feature=t["feature"], threshold=t["threshold"], left=t["left"],
                                right=t["right"], leaf_value=t["leaf_value"]) for t in trees], 4)
    r2 = oracle.raw(e2, X)[:, 0]
    assert np.allclose(r, r2, rtol=0, atol=1e-13)


def test_mean_counts_global_trees():
    # MEAN divides by #trees feeding output k in the whole ensemble
    e = small_forest(9, T=6, D=3, F=3, n_outputs=2, leaf_kind="const",
                     tree_output=[0, 0, 0, 0, 1, 1], agg=synth.AGG_MEAN)
    X = synth.gen_X(6, 10, 3)
    c = np.array([e.tree(t)["leaf_value"][e.tree(t)["left"] == -1][0, 0] for t in range(6)],
                 np.float64)
    m = oracle.margin(e, oracle.raw(e, X))
    assert np.allclose(m[:, 0], c[:4].sum() / 4, rtol=0, atol=1e-15)
    assert np.allclose(m[:, 1], c[4:].sum() / 2, rtol=0, atol=1e-15)


# ---------------------------------------------------------------- P-g
def test_transform_identities():
    e = synth.from_trees([_stump(0.0, 0.0, 0.0, 0)], 1, post=synth.POST_SIGMOID,
                         task=synth.TASK_CLASSIFICATION)
    m = np.array([[0.0], [1.5], [-1.5], [40.0], [-40.0], [1e-9]])
    p = oracle.post(e, m)[:, 0]
    assert p[0] == 0.5
    assert abs(p[1] - (1 - p[2])) < 1e-15
    assert np.allclose(p, scipy.special.expit(m[:, 0]), rtol=1e-15, atol=0)
    assert list(oracle.label(e, m)) == [0, 1, 0, 1, 0, 1]
    K = 5
    es = synth.from_trees([_stump(0.0, 0.0, 0.0, 0)], 1, n_outputs=K,
                          post=synth.POST_SOFTMAX, task=synth.TASK_CLASSIFICATION)
    rng = np.random.default_rng(1)
    M = rng.normal(size=(50, K)) * 5
    P = oracle.post(es, M)
    assert np.allclose(P, scipy.special.softmax(M, axis=1), rtol=1e-14, atol=1e-16)
    assert np.allclose(oracle.post(es, M + 123.0), P, rtol=1e-12, atol=1e-16)
    assert np.allclose(oracle.post(es, np.full((1, K), 2.0)), 1.0 / K, rtol=1e-15)
    # argmax, lowest index on ties
    T = np.array([[1.0, 3.0, 3.0, 0.0, 2.0], [5.0, 5.0, 5.0, 5.0, 5.0]])
    assert list(oracle.label(es, T)) == [1, 0]
    assert np.array_equal(oracle.label(es, M), np.argmax(M, 1))


def test_leaf_hash_consistent_with_leaves():
    e = small_forest(10, T=9, D=4, F=3)
    X = synth.gen_X(7, 64, 3, special_q24=1 << 20)
    L = oracle.leaf(e, X).astype(np.uint64)
    t = np.arange(e.n_trees, dtype=np.uint64)[None, :]
    h = synth.mix64((t << np.uint64(32)) | L)
    with np.errstate(over="ignore"):
        exp = h.sum(1, dtype=np.uint64)
    assert np.array_equal(oracle.leaf_hash(e, X), exp)
    # shard additivity of the hash
    with np.errstate(over="ignore"):
        s = oracle.leaf_hash(e, X, 0, 4) + oracle.leaf_hash(e, X, 4, 9)
    assert np.array_equal(s, exp)


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_raw_and_hash_mt_equals_single_threaded_definitions(threads):
    """oracle_raw_hash_mt (one walk per (row, tree), rows split over pthreads;
    used for every-row parity at full size) returns exactly what the
    single-threaded oracle_raw (fp64, tree order) and the hash pinned above
    (Σ mix64 over oracle_leaf) return, for vector leaves, per-class routing,
    tree shards and NaN / ±Inf cells, and for more threads than rows."""
    for e in (small_forest(21, T=13, D=5, F=4),
              small_forest(22, T=12, D=4, F=3, n_outputs=3),
              small_forest(23, T=7, D=3, F=5, n_outputs=4, leaf_width=4, leaf_kind="dirichlet",
                           agg=synth.AGG_MEAN)):
        X = synth.gen_X(31, 257, e.n_features, special_q24=1 << 20)
        for t0, t1 in ((0, e.n_trees), (2, e.n_trees - 1)):
            r, h = oracle.raw_and_hash(e, X, t0, t1, threads=threads)
            assert np.array_equal(r, oracle.raw(e, X, t0, t1))
            assert np.array_equal(h, oracle.leaf_hash(e, X, t0, t1))
        r, h = oracle.raw_and_hash(e, X[:2], threads=threads)
        assert np.array_equal(h, oracle.leaf_hash(e, X[:2]))
