"""The seeded generators: splitmix64 pinned to its published first output,
grid shapes, determinism, row-offset consistency, forest well-formedness."""
import numpy as np
import pytest

import synth


def test_splitmix64_reference_value():
    # SplitMix64 (Steele, Lea, Flood 2014) seeded with 0: the first output is
    # mix64(0 + 0x9E3779B97F4A7C15) = 0xE220A8397B1DCDAF (the widely quoted
    # reference value of java.util.SplittableRandom / xoshiro seeding).
    z = synth.mix64(np.array([0x9E3779B97F4A7C15], np.uint64))[0]
    assert int(z) == 0xE220A8397B1DCDAF


def test_gen_X_grid_and_determinism():
    X = synth.gen_X(7, 1000, 13)
    assert X.dtype == np.float32 and X.shape == (1000, 13)
    assert np.all(X >= -8) and np.all(X < 8)
    assert np.all(X * 4096 == np.round(X * 4096))
    assert np.array_equal(X, synth.gen_X(7, 1000, 13))
    assert not np.array_equal(X, synth.gen_X(8, 1000, 13))
    # row offset selects the same rows
    assert np.array_equal(X[300:400], synth.gen_X(7, 100, 13, row_offset=300))
    Xc = synth.gen_X(7, 1000, 13, grid=synth.GRID_COARSE)
    assert len(np.unique(Xc)) <= 64 and np.all(Xc * 4 == np.round(Xc * 4))


def test_gen_X_specials_and_ldx():
    X = synth.gen_X(3, 4000, 5, special_q24=1 << 21, ldx=8)
    assert X.shape == (4000, 8) and np.all(X[:, 5:] == 0)
    v = X[:, :5]
    assert np.isnan(v).any() and np.isposinf(v).any() and np.isneginf(v).any()
    assert (np.signbit(v) & (v == 0)).any()


@pytest.mark.parametrize("family", ["balanced", "mixed", "skinny"])
def test_forest_well_formed(family):
    e = synth.gen_forest(20, 6, 9, seed=5, family=family)
    d = synth.tree_depths(e)
    assert d.max() == 6
    if family != "mixed":
        assert np.all(d == 6)
    for t in range(e.n_trees):
        tr = e.tree(t)
        L, R = tr["left"], tr["right"]
        n = L.size
        internal = L != -1
        assert np.all((L == -1) == (R == -1))
        kids = np.concatenate([L[internal], R[internal]])
        # every non-root node has exactly one parent; root has none
        assert sorted(kids.tolist()) == list(range(1, n))
        assert np.all(tr["feature"][internal] >= 0) and np.all(tr["feature"][internal] < 9)
        assert not np.isnan(tr["threshold"][internal]).any()
        assert np.isfinite(tr["leaf_value"][~internal]).all()


def test_configs_shapes():
    c, e = synth.make_config("C1")
    assert (c.n_rows, c.n_features, e.n_trees, e.n_outputs, e.leaf_width) == (150, 4, 1, 3, 3)
    assert synth.tree_depths(e).max() == 3
    c, e = synth.make_config("C3", n_trees=10)
    assert e.n_features == 28 and synth.tree_depths(e).max() == 8
