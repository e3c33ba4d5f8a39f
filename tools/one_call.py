"""One hb_predict call in bench.py's launch shape, for ncu (no timing here):

    ncu --set full --clock-control none --nvtx --nvtx-include "hb_call/" \\
        -o gpurun_out/tr_C3 python tools/one_call.py C3 [--emulate-gpus 8] [--rows N]

A warm call first, then the profiled call inside the NVTX range "hb_call".
Prints the layout key bench.py uses for profiles/ncu_traffic.json.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--emulate-gpus", type=int, default=0)
    a = ap.parse_args()
    import torch
    import paper_2010_04804_b200 as hb
    import synth
    import synth.dev
    from paper_2010_04804_b200.dist import tree_shard
    cfg, e = synth.make_config(a.config)
    n = a.rows or cfg.n_rows
    if a.emulate_gpus:
        t0, t1 = tree_shard(e.n_trees, 0, a.emulate_gpus, e.n_outputs, e.leaf_width)
        m = hb.Model(e, device=0, tree_range=(t0, t1))
        kind = "raw64"
    else:
        t0, t1 = 0, e.n_trees
        m = hb.Model(e, device=0)
        kind = "proba" if e.task == synth.TASK_CLASSIFICATION else "predict"
    if cfg.name == "C5" and not a.emulate_gpus:
        kind = "raw64"          # bench's trees mode scores raw partials, then finalizes
    X = synth.dev.gen_X_device(cfg.seed_x, n, cfg.n_features)
    out = m.run(X, kind)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("hb_call")
    m.run(X, kind, out=out)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    info = m.info
    layout = info["strategy_name"] + ("-rank" if info.get("node_record_bytes") == 4 else "") + \
        ("-pre" if info.get("rank_prepass") else "") + ("-chunk" if info.get("tt_chunk_trees") else "")
    if n <= info["small_batch_max_rows"]:
        layout = "small-batch"
    print(f"KEY {a.config}:{layout}:{n}:{t1 - t0}")


if __name__ == "__main__":
    main()
