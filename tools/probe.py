"""One model, one batch, a few launches — a small target for ncu.

    python tools/probe.py --strategy gemm --trees 100 --depth 3 --features 200 --rows 1000000
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import synth.dev  # noqa: E402
import paper_2010_04804_b200 as hb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--strategy", default="auto")
ap.add_argument("--trees", type=int, default=100)
ap.add_argument("--depth", type=int, default=3)
ap.add_argument("--features", type=int, default=200)
ap.add_argument("--rows", type=int, default=1_000_000)
ap.add_argument("--family", default="balanced")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
e = synth.gen_forest(a.trees, a.depth, a.features, seed=1, family=a.family,
                     post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION)
m = hb.Model(e, strategy=a.strategy, device=0)
X = synth.dev.gen_X_device(3, a.rows, a.features)
out = torch.empty((a.rows, 2), device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(a.iters):
    ev[0].record()
    m.predict_proba(X, out=out)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"{m.info['strategy_name']} tc={m.info['tensor_cores']} {ev[0].elapsed_time(ev[1]):.3f} ms")
