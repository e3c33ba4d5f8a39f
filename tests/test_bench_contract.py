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
    assert d["e2e"]["h2d_bytes_per_step"] == 300000 * 28 * 4
    assert d["gpu_launches"] == 3 and d["scaling"] == "weak" and d["n_gpus"] == 1
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
