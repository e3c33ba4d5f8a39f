"""P-d: the strategy invariant. The literal transcriptions of Alg. 1 (GEMM),
Alg. 2 (TreeTraversal) and Alg. 3 (PerfectTreeTraversal) in oracle/literal.py
reach the same leaf as the oracle's plain walk for every (row, tree), and
their summed leaf values equal the oracle's raw sums."""
import numpy as np
import pytest

import oracle
import synth
from oracle import literal
from tests._common import load_hand_trees, small_forest


CASES = [(s, cmp, fam) for s in range(4) for cmp in (0, 1)
         for fam in ("balanced", "mixed", "skinny")]


@pytest.mark.parametrize("seed,cmp,family", CASES)
def test_three_strategies_reach_the_walk_leaf(seed, cmp, family):
    rng = np.random.default_rng(100 + seed)
    D = int(rng.integers(1, 6))
    F = int(rng.integers(1, 6))
    e = small_forest(seed, T=int(rng.integers(1, 10)), D=D, F=F, cmp=cmp, family=family,
                     leaf_kind="dyadic")
    Dmax = int(synth.tree_depths(e).max())
    Xf = synth.gen_X(seed, 300, F, grid=synth.GRID_COARSE)               # finite, tie-heavy
    Xs = synth.gen_X(seed, 300, F, grid=synth.GRID_COARSE, special_q24=1 << 21)
    walk_f = oracle.leaf(e, Xf)
    walk_s = oracle.leaf(e, Xs)
    # Alg. 1 (finite X only: the literal dense X.A is poisoned by 0*Inf)
    for t in range(e.n_trees):
        lid, R = literal.gemm_tree(e.tree(t), Xf, F, cmp)
        assert np.array_equal(lid, walk_f[:, t])
    # Alg. 2 and Alg. 3, with specials
    for X, walk in ((Xf, walk_f), (Xs, walk_s)):
        tl, tv = literal.tt_ensemble(e, X, Dmax)
        assert np.array_equal(tl, walk)
        pl, pv = literal.ptt_ensemble(e, X, Dmax)
        assert np.array_equal(pl, walk)
        # arbitrary comparisons in the inserted perfect-padding nodes
        pl2, _ = literal.ptt_ensemble(e, X, Dmax, rng=np.random.default_rng(seed))
        assert np.array_equal(pl2, walk)
        # summed values == oracle raw (same tree order, fp64, exact for dyadic)
        r = oracle.raw(e, X)[:, 0]
        assert np.array_equal(tv[:, :, 0].sum(1), r)
        assert np.array_equal(pv[:, :, 0].sum(1), r)


def test_hand_trees_all_strategies():
    for cmp in (0, 1):
        e, X, exp_leaf, _ = load_hand_trees(cmp)
        tl, _ = literal.tt_ensemble(e, X, 4)
        pl, _ = literal.ptt_ensemble(e, X, 4)
        assert np.array_equal(tl, exp_leaf) and np.array_equal(pl, exp_leaf)
        fin = np.isfinite(X).all(1)
        for t in range(e.n_trees):
            lid, _ = literal.gemm_tree(e.tree(t), X[fin], 3, cmp)
            assert np.array_equal(lid, exp_leaf[fin, t])


def test_gemm_zero_padding_reading():
    """P:192 pads smaller trees with zeros. A padded leaf column (C = 0, D = 0)
    then matches EVERY row (reading R7 / SURVEY V2); masking pads with an
    unreachable D restores exactly one match."""
    a = small_forest(1, T=1, D=3, F=3, family="balanced")
    b = small_forest(2, T=1, D=1, F=3, family="balanced")
    trees = [a.tree(0), b.tree(0)]
    e = synth.from_trees([dict(feature=t["feature"], threshold=t["threshold"], left=t["left"],
                               right=t["right"], leaf_value=t["leaf_value"]) for t in trees], 3)
    X = synth.gen_X(3, 200, 3)
    hits, _ = literal.gemm_ensemble_padded(e, X, mask_pads=False)
    assert np.all(hits[:, 0] == 1) and np.all(hits[:, 1] == 1 + (8 - 2))
    hits, leaves = literal.gemm_ensemble_padded(e, X, mask_pads=True)
    assert np.all(hits == 1)
    assert np.array_equal(leaves, oracle.leaf(e, X))


def test_d_vector_reading():
    """Reading R5 of the garbled Table 3 D: D_j = #left edges on the
    root->leaf path. The literal 'internal nodes only' count breaks Alg. 1."""
    e = small_forest(4, T=6, D=4, F=3, family="mixed")
    X = synth.gen_X(1, 500, 3, grid=synth.GRID_COARSE)
    for t in range(e.n_trees):
        tr = e.tree(t)
        I, L, A, B, C, D, E = literal.gemm_tensors(tr, 3)
        # left-edge count by walking parents
        parent = {}
        for i in I:
            parent[int(tr["left"][i])] = (int(i), 1)
            parent[int(tr["right"][i])] = (int(i), 0)
        for j, l in enumerate(L):
            k, cnt = int(l), 0
            while k in parent:
                p, is_left = parent[k]
                cnt += is_left
                k = p
            assert D[j] == cnt
