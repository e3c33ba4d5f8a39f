"""GEMM strategy probe (Alg. 1): the
paper's Fig. 8 shape (synthetic F = 200, balanced trees) at depth
3 with 100 and 500 trees, 1M rows, forced GEMM (tcgen05) against PTT / AUTO.
Prints device ms per call (CUDA events, best of 5 after warm-up) and the
GEMM kernel's fraction of its on-chip gather roof (96 B per
(row, tree) at D3 = 7 node gathers x 12 B + 12 B leaf) and of the bf16 tensor
roof (56 MAC per (row, tree)).

    python tools/gemm_probe.py [--rows 1000000] [--only gemm] [--trees 100,500]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--trees", default="100,500")
    ap.add_argument("--only", default="")
    ap.add_argument("--depth", type=int, default=3)
    ap.add_argument("--features", type=int, default=200)
    a = ap.parse_args()
    import torch
    import paper_2010_04804_b200 as hb
    import synth
    import synth.dev
    X = synth.dev.gen_X_device(0xF18, a.rows, a.features)
    peaks = {}
    try:
        import tools
        tools.build()
        peaks = tools.peaks(0)
    except Exception:
        pass
    smem = peaks.get("smem_gbs") or 148 * 128 * 1.965
    res = []
    for T in [int(t) for t in a.trees.split(",")]:
        e = synth.gen_forest(T, a.depth, a.features, seed=a.depth, family="balanced",
                             post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION)
        for name, strat, env in (("gemm", "gemm", {}), ("ptt", "ptt", {"HB_PTT_RANK": "0"}),
                                 ("ptt-rank", "ptt", {"HB_PTT_RANK": "1"}), ("auto", "auto", {})):
            if a.only and name != a.only:
                continue
            old = {k: os.environ.get(k) for k in list(env) + ["HB_SMALL_BATCH"]}
            os.environ.update(env)
            os.environ["HB_SMALL_BATCH"] = "0"
            m = hb.Model(e, strategy=strat, device=0)
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
            out = m.run(X, "proba")
            for _ in range(3):
                m.run(X, "proba", out=out)
            torch.cuda.synchronize()
            best = 1e30
            for _ in range(5):
                s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                m.run(X, "proba", out=out)
                t.record()
                torch.cuda.synchronize()
                best = min(best, s.elapsed_time(t))
            nodes = 2 ** a.depth - 1
            gather_bytes = a.rows * T * (nodes * 12 + 12)
            mac = a.rows * T * nodes * 2 ** a.depth
            r = {"trees": T, "kernel": name, "layout": m.info["kernel_name"], "ms": best,
                 "rows_per_s": a.rows / (best * 1e-3)}
            if name == "gemm":
                r["gather_roof_frac"] = gather_bytes / (best * 1e-3) / 1e9 / smem
                r["tensor_tflops"] = 2 * mac / (best * 1e-3) / 1e12
                r["tensor_roof_frac_bf16_burst"] = r["tensor_tflops"] / 1678.2
            res.append(r)
            print(json.dumps(r), flush=True)
            m.free()
    print(json.dumps({"smem_peak_gbs": smem, "results": res}))


if __name__ == "__main__":
    main()
