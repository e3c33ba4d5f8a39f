"""Shared test helpers (input construction only; no scoring arithmetic)."""
from __future__ import annotations

import json
import os

import numpy as np

import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fval(v):
    return float(v) if isinstance(v, str) else float(v)


def load_hand_trees(cmp=synth.CMP_LT):
    with open(os.path.join(GOLDEN, "hand_trees.json")) as f:
        g = json.load(f)
    trees = []
    for t in g["trees"]:
        trees.append(dict(feature=t["feature"],
                          threshold=[fval(v) for v in t["threshold"]],
                          left=t["left"], right=t["right"],
                          leaf_value=[fval(v) for v in t["leaf_value"]]))
    e = synth.from_trees(trees, g["n_features"], cmp=cmp)
    X = np.array([[fval(v) for v in row] for row in g["rows"]], np.float32)
    exp = g["expected_LT" if cmp == synth.CMP_LT else "expected_LE"]
    return e, X, np.array(exp["leaf"]), np.array(exp["sum"], np.float64)


SPECIAL_Q24 = 1 << 19   # ~3% special cells (NaN, +-Inf, +-0)


def small_forest(seed, T=8, D=4, F=3, family="mixed", grid=synth.GRID_COARSE,
                 cmp=synth.CMP_LT, **kw):
    return synth.gen_forest(T, D, F, seed=seed, family=family, grid=grid, cmp=cmp, **kw)


# near-tie rows met by GPU label checks (listed, not
# failed); tests/conftest.py prints them in the terminal summary
NEAR_TIES = []


def record_near_ties(what, rows, gpu_labels, ref_labels):
    for r, g, o in zip(rows, gpu_labels, ref_labels):
        NEAR_TIES.append((what, int(r), int(g), int(o)))
