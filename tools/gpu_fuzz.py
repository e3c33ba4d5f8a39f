"""Randomized differential test of the CUDA path against the CPU oracle
(test infrastructure).

Each iteration draws a random ensemble (depth 0-12, 1-80 trees, 1-70
features, regression / binary / per-class multiclass / vector-leaf random
forest, LT / LE, coarse or fine threshold grids with exact ties), a random
layout forced through the compile-time overrides (AUTO; PTT fp32 nodes;
rank-coded PTT with 32- / 16-bit cells, in-kernel or pre-pass codes, one or
two rows per lane, TMA / direct / staged / column pre-pass kernels,
interleaved or contiguous warp units; TT narrow / wide rows with tree chunks;
GEMM on tensor or CUDA cores; the small-batch kernel) and a random row count
and row pitch, then compares every output kind with the oracle: leaf ids and
leaf hashes bit-exact, scores within 1e-5 + 1e-5 |ref| (R23), labels exact
outside near-ties.

    python tools/gpu_fuzz.py [iterations] [seed]

Exit status 0 iff every comparison passed. With HB_LIB pointing at
libhb_checked.so the same run also exercises the device bounds checks.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import synth.dev  # noqa: E402
import paper_2010_04804_b200 as hb  # noqa: E402

LAYOUT_ENV = ("HB_PTT_RANK", "HB_RANK_CW", "HB_RANK_PRE", "HB_PTTR_RPL", "HB_RC_TMA", "HB_RC_STAGED",
              "HB_RC_ONEK", "HB_RC_RW", "HB_PTTR_INTERLEAVE", "HB_TT_WIDE", "HB_TT_CHUNK", "HB_GEMM_TC",
              "HB_SMALL_BATCH", "HB_X_BULK")


def tol_ok(got, ref):
    return np.abs(np.asarray(got, np.float64) - ref) <= 1e-5 + 1e-5 * np.abs(ref)


def near_tie(e, m):
    if e.n_outputs == 1:
        return np.abs(m[:, 0]) < 2 * (1e-5 + 1e-5 * np.abs(m[:, 0]))
    s = np.sort(m, 1)
    return (s[:, -1] - s[:, -2]) < 2 * (1e-5 + 1e-5 * np.abs(s[:, -1]))


def draw(rng):
    kind = rng.choice(["reg", "binary", "multiclass", "rf"])
    D = int(rng.integers(0, 13))
    T = int(rng.integers(1, 81))
    F = int(rng.integers(1, 71))
    cmp = int(rng.integers(0, 2))
    grid = synth.GRID_COARSE if rng.random() < 0.4 else synth.GRID_FINE
    family = rng.choice(["balanced", "mixed", "skinny"])
    common = dict(seed=int(rng.integers(1 << 30)), family=family, cmp=cmp, grid=grid)
    if kind == "reg":
        e = synth.gen_forest(T, D, F, base_score=[float(rng.normal())], **common)
    elif kind == "binary":
        e = synth.gen_forest(T, D, F, post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION, **common)
    elif kind == "multiclass":
        K = int(rng.integers(2, 8))
        e = synth.gen_forest(max(T, K), D, F, n_outputs=K, post=synth.POST_SOFTMAX,
                             task=synth.TASK_CLASSIFICATION, **common)
    else:
        K = int(rng.integers(2, 8))
        e = synth.gen_forest(T, D, F, n_outputs=K, leaf_width=K, leaf_kind="dirichlet",
                             agg=synth.AGG_MEAN, task=synth.TASK_CLASSIFICATION, **common)
    return kind, e, D, F, grid


def layout(rng):
    """(strategy, env) — a random point of the layout space."""
    r = rng.random()
    if r < 0.15:
        return "auto", {}
    if r < 0.55:
        env = {"HB_PTT_RANK": str(rng.choice(["0", "1"]))}
        if env["HB_PTT_RANK"] == "1":
            env.update({"HB_RANK_CW": str(rng.choice(["0", "32", "16"])),
                        "HB_RANK_PRE": str(rng.choice(["0", "1"])),
                        "HB_PTTR_RPL": str(rng.choice(["1", "2"])),
                        "HB_RC_TMA": str(rng.choice(["0", "1"])),
                        "HB_RC_STAGED": str(rng.choice(["-1", "0", "1"])),
                        "HB_RC_ONEK": str(rng.choice(["0", "1"])),
                        "HB_RC_RW": str(rng.choice(["0", "1"])),
                        "HB_PTTR_INTERLEAVE": str(rng.choice(["0", "1"]))})
        return "ptt", env
    if r < 0.85:
        return "tt", {"HB_TT_WIDE": str(rng.choice(["-1", "1"])), "HB_TT_CHUNK": str(rng.choice(["-1", "0", "8"]))}
    return "gemm", {"HB_GEMM_TC": str(rng.choice(["0", "1"]))}


def check(e, m, Xd, Xh, what):
    F = e.n_features
    Xo = np.ascontiguousarray(Xh[:, :F])
    s = oracle.scores(e, Xo)
    cls = e.task == synth.TASK_CLASSIFICATION
    assert np.array_equal(m.run(Xd, "leaf").cpu().numpy(), oracle.leaf(e, Xo)), what + ": leaf ids"
    assert np.array_equal(m.run(Xd, "leaf_hash").cpu().numpy().view(np.uint64), oracle.leaf_hash(e, Xo)), \
        what + ": leaf hash"
    assert tol_ok(m.run(Xd, "raw64").cpu().numpy(), s["raw"]).all(), what + ": raw64"
    assert tol_ok(m.run(Xd, "margin").cpu().numpy(), s["margin"]).all(), what + ": margin"
    if cls:
        assert tol_ok(m.run(Xd, "proba").cpu().numpy(), oracle.proba(e, s["post"])).all(), what + ": proba"
        lab = m.run(Xd, "predict").cpu().numpy()
        tie = near_tie(e, s["margin"])
        assert np.array_equal(lab[~tie], s["label"][~tie]), what + ": labels"
    else:
        assert tol_ok(m.run(Xd, "predict").cpu().numpy(), s["post"]).all(), what + ": predict"


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    print("library", hb.lib_path, flush=True)
    ran = rejected = 0
    seen = {}
    for it in range(iters):
        kind, e, D, F, grid = draw(rng)
        strat, env = layout(rng)
        for k in LAYOUT_ENV:
            os.environ.pop(k, None)
        os.environ.update(env)
        sb = str(rng.choice(["", "0", "4096"]))     # "": the default (small-batch kernel for AUTO only)
        if sb:
            os.environ["HB_SMALL_BATCH"] = sb
        try:
            m = hb.Model(e, strategy=strat, device=0)
        except hb.HBError as ex:          # a forced layout the model cannot take (e.g. GEMM beyond D 10)
            assert ex.status == 3, f"iteration {it}: {ex}"
            rejected += 1
            continue
        n = int(rng.choice([1, 31, 33, 257, 1000, 4097, 20000, 70000]))
        ldx = F + int(rng.choice([0, 0, 1, 3, 4]))
        sq = 1 << 22 if rng.random() < 0.5 else 0
        seed = int(rng.integers(1 << 30))
        Xd = synth.dev.gen_X_device(seed, n, F, grid=grid, special_q24=sq, ldx=ldx)
        Xh = synth.gen_X(seed, n, F, grid=grid, special_q24=sq, ldx=ldx)
        info = m.info
        key = (info["strategy_name"], info["kernel_name"], info["node_record_bytes"], info["rank_prepass"],
               info["code_cell_bits"], info["rows_per_lane"], info["tt_chunk_trees"] > 0,
               n <= info["small_batch_max_rows"])
        seen[key] = seen.get(key, 0) + 1
        what = f"iteration {it}: {kind} D{D} T{e.n_trees} F{F} n{n} ldx{ldx} {strat} {env} -> {key}"
        check(e, m, Xd, Xh, what)
        m.free()
        ran += 1
    torch.cuda.synchronize()
    print(f"gpu_fuzz: {ran} models checked against the oracle on every output kind, {rejected} forced "
          f"layouts rejected as unsupported, {len(seen)} distinct (strategy, kernel, record, pre-pass, "
          f"cells, rows/lane, chunked, small-batch) combinations", flush=True)
    for k, v in sorted(seen.items(), key=lambda kv: -kv[1]):
        print("  ", v, k)


if __name__ == "__main__":
    main()
