"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import synth.dev  # noqa: E402
import paper_2010_04804_b200 as hb  # noqa: E402

cases = [
    ("ptt-rank", synth.gen_forest(40, 6, 12, seed=1), {"HB_PTT_RANK": "1"}, "ptt"),
    ("ptt-fp32", synth.gen_forest(40, 6, 12, seed=1), {"HB_PTT_RANK": "0"}, "ptt"),
    ("tt", synth.gen_forest(24, 11, 12, seed=2, family="mixed"), {}, "tt"),
    ("tt-wide", synth.gen_forest(24, 11, 12, seed=2, family="mixed"), {"HB_TT_WIDE": "1"}, "tt"),
    ("ptt-rank-wrap", synth.gen_forest(300, 8, 12, seed=4), {"HB_PTT_RANK": "1", "HB_CH": "8"}, "ptt"),
    ("ptt-fp32-wrap", synth.gen_forest(300, 8, 12, seed=4), {"HB_PTT_RANK": "0", "HB_CH": "8"}, "ptt"),
    ("ptt-rank-prepass-32", synth.gen_forest(40, 6, 12, seed=1),
     {"HB_PTT_RANK": "1", "HB_RANK_PRE": "1", "HB_RC_TMA": "0", "HB_RANK_CW": "32"}, "ptt"),
    ("ptt-rank-prepass-16", synth.gen_forest(40, 6, 12, seed=1),
     {"HB_PTT_RANK": "1", "HB_RANK_PRE": "1", "HB_RC_TMA": "0", "HB_RANK_CW": "16"}, "ptt"),
    ("ptt-rank-prepass-staged-16", synth.gen_forest(40, 6, 12, seed=1),
     {"HB_PTT_RANK": "1", "HB_RANK_PRE": "1", "HB_RC_TMA": "0", "HB_RANK_CW": "16", "HB_RC_STAGED": "1"}, "ptt"),
    ("ptt-rank-prepass-staged-32-rb1", synth.gen_forest(40, 6, 12, seed=1),
     {"HB_PTT_RANK": "1", "HB_RANK_PRE": "1", "HB_RC_TMA": "0", "HB_RANK_CW": "32", "HB_RC_STAGED": "1", "HB_RC_RB": "1"}, "ptt"),
    ("ptt-rank-prepass-column", synth.gen_forest(40, 6, 12, seed=1),
     {"HB_PTT_RANK": "1", "HB_RANK_PRE": "1", "HB_RC_TMA": "0", "HB_RANK_CW": "32", "HB_RC_ONEK": "1"}, "ptt"),
    ("ptt-rank-prepass-rows8", synth.gen_forest(40, 6, 12, seed=1),
     {"HB_PTT_RANK": "1", "HB_RANK_PRE": "1", "HB_RC_TMA": "0", "HB_RANK_CW": "16", "HB_RC_STAGED": "0", "HB_RC_ROWS": "8"}, "ptt"),
    ("tt-wide-chunks", synth.gen_forest(24, 11, 12, seed=2, family="mixed"),
     {"HB_TT_WIDE": "1", "HB_TT_CHUNK": "8"}, "tt"),
    ("gemm-tc", synth.gen_forest(40, 3, 12, seed=3), {}, "gemm"),
    ("gemm-tc-multiclass", synth.gen_forest(50, 3, 12, seed=5, n_outputs=3, post=synth.POST_SOFTMAX,
                                            task=synth.TASK_CLASSIFICATION), {}, "gemm"),
    ("tt-wide-multiclass", synth.gen_forest(30, 11, 12, seed=6, family="mixed", n_outputs=3,
                                            post=synth.POST_SOFTMAX, task=synth.TASK_CLASSIFICATION),
     {"HB_TT_WIDE": "1"}, "tt"),
    ("gemm-cuda", synth.gen_forest(40, 5, 12, seed=3), {}, "gemm"),
    # round 2 paths: direct pre-pass with (row, word) lanes (16-bit pair loads),
    # two rows per lane in the scorer (pre-pass, K = 1, D >= 3), interleaved units
    ("ptt-rank-prepass-16-rowword", synth.gen_forest(40, 6, 12, seed=1),
     {"HB_PTT_RANK": "1", "HB_RANK_PRE": "1", "HB_RC_TMA": "0", "HB_RANK_CW": "16", "HB_RC_STAGED": "0"}, "ptt",
     (3000, 50_000)),
    ("ptt-rank-rpl2-multiclass", synth.gen_forest(42, 7, 12, seed=8, n_outputs=3, post=synth.POST_SOFTMAX,
                                                  task=synth.TASK_CLASSIFICATION),
     {"HB_PTT_RANK": "1", "HB_RANK_PRE": "1", "HB_RANK_CW": "32"}, "ptt", (3000, 50_000)),
    # TMA pre-pass (F = 12: three 4-column groups); 250K rows wrap every
    # warp's 3-stage ring several times
    ("ptt-rank-prepass-tma-32", synth.gen_forest(4, 4, 12, seed=7),
     {"HB_PTT_RANK": "1", "HB_RANK_PRE": "1", "HB_RANK_CW": "32", "HB_RC_TMA": "1"}, "ptt", (3000, 250_000)),
    ("ptt-rank-prepass-tma-16", synth.gen_forest(4, 4, 12, seed=7),
     {"HB_PTT_RANK": "1", "HB_RANK_PRE": "1", "HB_RANK_CW": "16", "HB_RC_TMA": "1"}, "ptt", (3000, 250_000)),
]
only = set(sys.argv[1:])   # optional case names; default: every case
print("library", hb.lib_path, flush=True)
for name, e, env, strat, *rows in cases:
    if only and name not in only:
        continue
    os.environ.update(env)
    runs = [(n, "0") for n in rows[0]] if rows else [(3000, "0"), (40, "4096")]
    for n, small in runs:
        os.environ["HB_SMALL_BATCH"] = small
        m = hb.Model(e, strategy=strat, device=0)
        if env.get("HB_RC_TMA") == "1":
            assert m.info["rank_prepass_tma"] == 1, name
        X = synth.dev.gen_X_device(7, n, 12)
        for kind in ("predict", "raw", "raw64", "leaf", "leaf_hash"):
            m.run(X, kind)
        torch.cuda.synchronize()
        m.free()
    for k in env:
        os.environ.pop(k)
    print("ok", name, flush=True)
