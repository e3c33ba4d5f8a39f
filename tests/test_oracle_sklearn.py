"""P-h: third-party cross-check of the oracle against scikit-learn's own tree
code (an independent Cython implementation of the same definition).

sklearn splits with ``x <= t`` on fp32 X against fp64 thresholds, which equals
``x <= round_down_fp32(t)`` for every fp32 x (reading R4), so the
export rounds thresholds toward -inf and uses cmp = LE.
"""
import numpy as np
import pytest

sk = pytest.importorskip("sklearn")
from sklearn.ensemble import (GradientBoostingRegressor, IsolationForest,  # noqa: E402
                              RandomForestClassifier)
from sklearn.tree import DecisionTreeClassifier, DecisionTreeRegressor  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402


def _down32(t64):
    t32 = t64.astype(np.float32)
    too_big = t32.astype(np.float64) > t64
    t32[too_big] = np.nextafter(t32[too_big], np.float32(-np.inf))
    return t32


def export(estimators, n_features, values, **kw):
    trees = []
    for est, val in zip(estimators, values):
        tr = est.tree_
        leaf = tr.children_left == -1
        thr = _down32(tr.threshold)
        thr[leaf] = np.nan
        trees.append(dict(feature=np.where(leaf, -1, tr.feature), threshold=thr,
                          left=tr.children_left, right=tr.children_right,
                          leaf_value=val(tr)))
    return synth.from_trees(trees, n_features, cmp=synth.CMP_LE, **kw)


def _data(seed, n, F, k=3):
    X = synth.gen_X(seed, n, F, grid=synth.GRID_COARSE).astype(np.float32)
    # a learnable label with ties on the coarse grid
    y = ((X[:, 0] > 0).astype(int) + (X[:, 1] > 1.0).astype(int) * (k - 2)) % k
    return X, y


def test_decision_tree_classifier_apply_and_proba():
    X, y = _data(1, 3000, 6)
    clf = DecisionTreeClassifier(max_depth=8, random_state=0).fit(X, y)
    norm = lambda tr: tr.value[:, 0, :] / tr.value[:, 0, :].sum(1, keepdims=True)
    e = export([clf], 6, [norm], n_outputs=3, leaf_width=3, agg=synth.AGG_MEAN,
               task=synth.TASK_CLASSIFICATION)
    Xt = synth.gen_X(2, 2000, 6, grid=synth.GRID_COARSE)
    assert np.array_equal(oracle.leaf(e, Xt)[:, 0], clf.apply(Xt))
    s = oracle.scores(e, Xt)
    assert np.allclose(s["post"], clf.predict_proba(Xt), rtol=0, atol=1e-6)


def test_random_forest_soft_voting():
    X, y = _data(3, 3000, 8)
    rf = RandomForestClassifier(n_estimators=15, max_depth=7, random_state=0).fit(X, y)
    norm = lambda tr: tr.value[:, 0, :] / tr.value[:, 0, :].sum(1, keepdims=True)
    e = export(rf.estimators_, 8, [norm] * 15, n_outputs=3, leaf_width=3,
               agg=synth.AGG_MEAN, task=synth.TASK_CLASSIFICATION)
    Xt = synth.gen_X(4, 2000, 8)
    assert np.array_equal(oracle.leaf(e, Xt), rf.apply(Xt))
    s = oracle.scores(e, Xt)
    assert np.allclose(s["post"], rf.predict_proba(Xt), rtol=0, atol=1e-6)


def test_gradient_boosting_regression():
    X = synth.gen_X(5, 3000, 5)
    y = np.sin(X[:, 0]) + 0.1 * X[:, 1] ** 2
    gb = GradientBoostingRegressor(n_estimators=20, max_depth=4, learning_rate=0.1,
                                   random_state=0).fit(X, y)
    lr = gb.learning_rate
    vals = [lambda tr: (tr.value[:, 0, 0] * lr)[:, None]] * 20
    init = float(gb.init_.constant_.ravel()[0])
    e = export([est[0] for est in gb.estimators_], 5, vals, base_score=[init])
    Xt = synth.gen_X(6, 2000, 5)
    s = oracle.scores(e, Xt)
    # leaf values are rounded to fp32 by the ABI; the sum stays within 1e-6
    assert np.allclose(s["post"][:, 0], gb.predict(Xt), rtol=1e-6, atol=1e-6)


def test_regression_tree_apply_with_ties():
    X = synth.gen_X(7, 2000, 3, grid=synth.GRID_COARSE)
    y = X[:, 0] * 2 + X[:, 2]
    dt = DecisionTreeRegressor(max_depth=10, random_state=0).fit(X, y)
    e = export([dt], 3, [lambda tr: tr.value[:, 0, :]])
    Xt = synth.gen_X(8, 3000, 3, grid=synth.GRID_COARSE)
    assert np.array_equal(oracle.leaf(e, Xt)[:, 0], dt.apply(Xt))


def export_isolation_forest(iso, n_features):
    """IsolationForest -> ABI ensemble: leaf value = path
    length h = node depth + c(n_leaf) - 1 (sklearn _compute_score_samples),
    agg MEAN, post ISOLATION with post_param = c(max_samples)."""
    from sklearn.ensemble._iforest import _average_path_length
    vals = []
    for est in iso.estimators_:
        tr = est.tree_
        h = tr.compute_node_depths() + _average_path_length(tr.n_node_samples) - 1.0
        vals.append(lambda tr, h=h: h[:, None])
    c = float(_average_path_length([iso._max_samples])[0])
    return export(iso.estimators_, n_features, vals, agg=synth.AGG_MEAN,
                  post=synth.POST_ISOLATION, post_param=c)


def test_isolation_forest_score_samples():
    X = synth.gen_X(9, 2000, 5)
    iso = IsolationForest(n_estimators=25, max_samples=256, random_state=0).fit(X)
    e = export_isolation_forest(iso, 5)
    Xt = synth.gen_X(10, 3000, 5)
    Xt[:50] *= 40.0                                   # some clear outliers
    s = oracle.scores(e, Xt)
    assert np.allclose(s["post"][:, 0], -iso.score_samples(Xt), rtol=1e-6, atol=1e-6)
