"""The five BASELINE.json workloads (C1..C5) as seeded synthetic recipes.

Shapes follow BASELINE.json ``configs`` and SURVEY.md §8(a)/(d); the paper's
workload description is PAPER.md P:330-338 (500 trees, max depth 8; balanced
XGBoost trees, skinny LightGBM trees, mixed RF trees; 10s to 2K columns).
No dataset or trained model is used.
"""
from __future__ import annotations

from dataclasses import dataclass

from .forest import (gen_forest, CMP_LT, AGG_SUM, AGG_MEAN, POST_IDENTITY,
                     POST_SIGMOID, POST_SOFTMAX, TASK_REGRESSION,
                     TASK_CLASSIFICATION)
from .xgen import GRID_FINE


@dataclass(frozen=True)
class Config:
    name: str
    n_rows: int
    n_features: int
    n_trees: int
    depth: int
    family: str
    n_outputs: int
    leaf_width: int
    leaf_kind: str
    leaf_sigma: float
    agg: int
    post: int
    task: int
    base: float
    seed_x: int
    seed_t: int
    per_class: bool = False
    note: str = ""


CONFIGS = {
    "C1": Config("C1", 150, 4, 1, 3, "balanced", 3, 3, "dirichlet", 0.0,
                 AGG_MEAN, POST_IDENTITY, TASK_CLASSIFICATION, 0.0, 0xC1, 0x1C1,
                 note="single decision tree depth 3 on 150x4 Iris-shaped rows"),
    "C2": Config("C2", 1_000_000, 90, 500, 8, "balanced", 1, 1, "normal", 0.1,
                 AGG_SUM, POST_IDENTITY, TASK_REGRESSION, 0.5, 0xC2, 0x1C2,
                 note="500-tree depth-8 GBDT regression, Year-shaped 90 features"),
    "C3": Config("C3", 10_000_000, 28, 500, 8, "balanced", 1, 1, "normal", 0.1,
                 AGG_SUM, POST_SIGMOID, TASK_CLASSIFICATION, 0.0, 0xC3, 0x1C3,
                 note="500-tree depth-8 binary GBDT, Higgs-shaped 28 features"),
    "C4": Config("C4", 5_000_000, 54, 3500, 8, "mixed", 7, 1, "normal", 0.1,
                 AGG_SUM, POST_SOFTMAX, TASK_CLASSIFICATION, 0.0, 0xC4, 0x1C4,
                 per_class=True,
                 note="3500 per-class trees (500 x 7), depth 8, Covtype-shaped 54 features"),
    "C4p": Config("C4p", 5_000_000, 54, 500, 8, "mixed", 7, 7, "dirichlet", 0.0,
                  AGG_MEAN, POST_IDENTITY, TASK_CLASSIFICATION, 0.0, 0xC4, 0x2C4,
                  note="RF variant of C4: 500 trees with 7-wide class-distribution leaves, MEAN"),
    "C5": Config("C5", 1_000_000, 2000, 10_000, 12, "mixed", 1, 1, "normal", 0.05,
                 AGG_SUM, POST_SIGMOID, TASK_CLASSIFICATION, 0.0, 0xC5, 0x1C5,
                 note="10k-tree depth-12 ensemble, Epsilon-shaped 2000 features"),
    # not a BASELINE config: the paper's Fig. 8 strategy-comparison shape
    # (synthetic, 200 features, 100 trees; depth 3, the GEMM
    # regime) at a 1M-row batch, for the GEMM (tcgen05) bench line
    "F8D3": Config("F8D3", 1_000_000, 200, 100, 3, "balanced", 1, 1, "normal", 0.1,
                   AGG_SUM, POST_SIGMOID, TASK_CLASSIFICATION, 0.0, 0xF8, 0x1F8,
                   note="Fig. 8 shape (P:537): 100 trees depth 3, 200 features, binary, 1M rows"),
}


def make_config(name: str, n_trees: int | None = None, cmp: int = CMP_LT):
    """Return (Config, Ensemble) for a named workload."""
    c = CONFIGS[name]
    T = c.n_trees if n_trees is None else n_trees
    e = gen_forest(T, c.depth, c.n_features, seed=c.seed_t, family=c.family,
                   n_outputs=c.n_outputs, leaf_width=c.leaf_width,
                   leaf_kind=c.leaf_kind, leaf_sigma=c.leaf_sigma,
                   grid=GRID_FINE, cmp=cmp, agg=c.agg, post=c.post,
                   task=c.task,
                   base_score=[c.base] * c.n_outputs if c.base else None)
    return c, e
