"""bench.py output contract (the driver parses one JSON line)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
             "gpu_launches"}


def _run(args, env=None, timeout=600):
    e = dict(os.environ, **(env or {}))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=e,
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0 and len(lines) == 1, out.stdout[-2000:] + out.stderr[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    """--impl reference times the CPU oracle (the only reference this tier has)."""
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1"],
             env={"HB_REF_STEP_S": "0.3"})
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "rows/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("C3")


@pytest.mark.gpu
def test_gpu_arm_contract():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--steps", "3", "--warmup", "3", "--rows", "300000"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    r = d["roofline"]
    assert r["bound"] == "smem" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert "truncated mean" in d["cpu_baseline"]["timing"]
    assert d["e2e"]["h2d_bytes_per_step"] == 300000 * 28 * 4
    # one hb_predict call per step: one launch, two when the model runs the
    # rank-code pre-pass (C3's AUTO layout does); the dominant kernel's time
    # comes from the library's per-launch events
    per_call = 2 if d["roofline"]["layout"].endswith("-pre") else 1
    assert len(d["gpu_launches_per_call"]) == per_call
    assert d["gpu_launches"] == 3 * per_call and d["scaling"] == "strong" and d["n_gpus"] == 1
    assert r["kernel"] == "pttr_kernel" and 0 < r["kernel_ms"] <= r["call_ms"] * 1.001
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    p = d["parity"]
    assert p["pass"] and p["leaf_hash_mismatches"] == 0 and p["rows"] > 0
    assert p["label_mismatches_outside_near_ties"] == 0


@pytest.mark.gpu
def test_gpu_arm_small_batch_graph_and_prepass():
    """C1 (150 rows) is timed through a CUDA graph of 200 calls per step; a
    C2-shaped run (rank-code pre-pass) counts two launches per call."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--config", "C1", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e"])
    assert d["gpu_launches"] == 3 * 200 and "CUDA graph" in d["config"]["timing"]
    assert d["roofline"]["kernel"] == "small_batch_kernel" and d["value"] > 0
    assert d["roofline"]["layout"] == "small-batch"
    d = _run(["--config", "C2", "--steps", "3", "--warmup", "3", "--rows", "200000", "--no-cpu",
              "--no-e2e"])
    assert d["roofline"]["layout"] == "ptt-rank-pre" and d["gpu_launches"] == 6


def _torchrun(args, timeout=900):
    env = dict(os.environ, HB_BENCH_ONE_DEVICE="1", HB_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"),
           "--gpus", "2"] + args
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0 and len(lines) == 1, out.stdout[-2000:] + out.stderr[-3000:]
    return json.loads(lines[0])


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,extra", [("C3", []), ("C5", ["--rows", "2000"])])
def test_multi_rank_bench_on_one_device(cfg, extra):
    """The torchrun path of bench.py (2 ranks; both on this box's one GPU,
    gloo for the collectives): row shards with no data-path collective (C3),
    tree shards + one reduce of fp64 partials + finalize on rank 0 (C5). C3
    is strong-scaled: its 10M rows are split over the two ranks."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _torchrun(["--config", cfg, "--steps", "2", "--warmup", "3", "--no-e2e"]
                  + (["--no-cpu"] if cfg == "C3" else []) + extra)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["scaling"] == "strong"
    assert d["config"]["trees_per_gpu"] == (500 if cfg == "C3" else 5000)
    if cfg == "C5":   # the reduced, finalized output of all 10k trees against the oracle
        fo = d["parity"]["final_output"]
        assert fo["outside_tol"] == 0 and fo["rows"] == 2000 and d["parity"]["pass"]
    if cfg == "C3":   # BASELINE C3: 10M rows sharded over the GPUs (strong scaling)
        assert d["config"]["rows_total"] == 10_000_000 and d["config"]["rows_per_gpu"] == 5_000_000
        assert d["value"] == pytest.approx(10_000_000 / (d["ms_per_step"] * 1e-3), rel=1e-6)
