"""Seeded synthetic inputs shared by the tests, bench.py and smoke().

This module holds NONE of the scoring method's arithmetic: it only draws
random rows X and random tree ensembles. Both the oracle (oracle/) and the
CUDA product (paper_2010_04804_b200/) consume what it produces; neither side
imports the other.

Recipes:

* X is a counter-based draw: ``x[r, f] = grid(splitmix64(seed, r*F + f))``
  so the host (numpy, synth/xgen.py) and the device (synth/csrc/synth_dev.cu)
  produce the same bits without sharing code.
* Forests are drawn level by level. Every split node picks a feature uniformly
  and a threshold strictly inside the node's current interval on that feature
  (the interval its ancestors carve out), so both children carry traffic the
  way trained trees do (XGBoost balanced, LightGBM skinny,
  RF mixed).
"""
from .xgen import gen_X, GRID_FINE, GRID_COARSE, mix64, counter_hash  # noqa: F401
from .forest import (Ensemble, gen_forest, from_trees, tree_depths,  # noqa: F401
                     CMP_LT, CMP_LE, AGG_SUM, AGG_MEAN, POST_IDENTITY,
                     POST_SIGMOID, POST_SOFTMAX, POST_ISOLATION, TASK_REGRESSION,
                     TASK_CLASSIFICATION)
from .configs import CONFIGS, Config, make_config  # noqa: F401
