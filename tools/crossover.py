"""Strategy crossover sweep on B200 (the paper's Fig. 8 setup,
PAPER.md P:533-549: synthetic 5000 x 200, 100 trees, depth 3 / 7 / 12, batch 1
and 1K — extended here to 1M rows). Every strategy is forced in turn; the
small-batch kernel (hb_small.cu) is measured as its own column.

    python tools/crossover.py [--out profiles/r01_crossover.json]

Per (depth, batch, kernel): device time per call from a replayed CUDA graph of
20 calls (launch overhead amortised the way a serving loop would), in us.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import synth.dev  # noqa: E402
import paper_2010_04804_b200 as hb  # noqa: E402


def time_calls(fn, reps=20, iters=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(iters):
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_crossover.json"))
    ap.add_argument("--trees", type=int, default=100)
    ap.add_argument("--features", type=int, default=200)
    args = ap.parse_args()
    batches = [1, 10, 100, 1000, 10_000, 100_000, 1_000_000]
    res = []
    Xall = synth.dev.gen_X_device(0xF18, batches[-1], args.features)
    for D in (3, 5, 7, 10, 12):
        e = synth.gen_forest(args.trees, D, args.features, seed=D, family="balanced",
                             post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION)
        kernels = []
        if D <= 6:
            kernels.append(("gemm", {"strategy": "gemm"}, {"HB_SMALL_BATCH": "0"}))
        if D <= 10:
            kernels.append(("ptt", {"strategy": "ptt"}, {"HB_SMALL_BATCH": "0", "HB_PTT_RANK": "0"}))
            kernels.append(("ptt-rank", {"strategy": "ptt"},
                            {"HB_SMALL_BATCH": "0", "HB_PTT_RANK": "1", "HB_RANK_PRE": "0"}))
            kernels.append(("ptt-rank-pre", {"strategy": "ptt"},
                            {"HB_SMALL_BATCH": "0", "HB_PTT_RANK": "1", "HB_RANK_PRE": "1"}))
        kernels.append(("tt", {"strategy": "tt"}, {"HB_SMALL_BATCH": "0"}))
        kernels.append(("small", {"strategy": "auto"}, {"HB_SMALL_BATCH": str(10 ** 9)}))
        # what the library picks by itself (strategy, layout and small-batch
        # threshold all default)
        kernels.append(("auto", {"strategy": "auto"}, {}))
        for name, kw, env in kernels:
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                m = hb.Model(e, device=0, **kw)
                for n in batches:
                    if name == "small" and n > 100_000:
                        continue
                    X = Xall[:n]
                    out = torch.empty((n, 2), dtype=torch.float32, device="cuda")
                    us = time_calls(lambda: m.predict_proba(X, out=out))
                    info = m.info
                    res.append({"depth": D, "batch": n, "kernel": name, "us_per_call": us,
                                "rows_per_s": n / (us * 1e-6), "layout": info["node_record_bytes"],
                                "ran": m.kernel_for(n), "strategy": info["strategy_name"],
                                "rank_prepass": info["rank_prepass"]})
                    print(f"D={D:2d} batch={n:8d} {name:9s} {us:10.1f} us  {n / us:10.2f} Mrows/s",
                          flush=True)
                m.free()
            except hb.HBError as ex:
                print(f"D={D} {name}: {ex}")
            finally:
                for k, v in old.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
    # AUTO against the best forced kernel at every (depth, batch)
    summary = []
    for D in sorted({r["depth"] for r in res}):
        for n in batches:
            rows = [r for r in res if r["depth"] == D and r["batch"] == n]
            forced = [r for r in rows if r["kernel"] != "auto"]
            auto = [r for r in rows if r["kernel"] == "auto"]
            if not forced or not auto:
                continue
            best = min(forced, key=lambda r: r["us_per_call"])
            summary.append({"depth": D, "batch": n, "best": best["kernel"], "best_us": best["us_per_call"],
                            "auto_us": auto[0]["us_per_call"], "auto_ran": auto[0]["ran"],
                            "auto_over_best": auto[0]["us_per_call"] / best["us_per_call"]})
            print(f"D={D:2d} batch={n:8d} best={best['kernel']:12s} auto/best={summary[-1]['auto_over_best']:.3f}")
    json.dump({"setup": f"{args.trees} trees, F={args.features}, balanced, sigmoid proba; "
                        "device time per call from a replayed CUDA graph of 20 calls",
               "results": res, "auto_vs_best": summary}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
