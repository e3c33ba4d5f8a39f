"""A compiled C consumer of the boundary: tests/c/abi_smoke.c
is built with gcc against include/hb.h (C, not C++), linked to libhb.so, and
on a GPU calls every entry point — hb_validate, hb_compile /
hb_compile_range, hb_predict / _proba / _raw / _leaf / hb_predict_ex (RAW64,
LEAF_HASH), hb_finalize / hb_finalize64, hb_predict_host, hb_model_get_info,
hb_free, hb_last_error, hb_abi_version — on the hand-traced trees of
tests/golden/hand_trees.json, checking leaf ids bit-exact and scores within
the R23 tolerance."""
import os
import subprocess

import numpy as np
import pytest

import synth
from tests._common import GOLDEN, load_hand_trees

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "abi_smoke.c")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    import paper_2010_04804_b200 as hb
    exe = str(tmp_path / "abi_smoke")
    libdir = os.path.dirname(hb.lib_path)
    cmd = ["gcc", "-std=c11", "-O1", "-Wall", "-Wextra", "-Werror", "-pedantic",
           "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CUDA, "include"),
           SRC, "-o", exe, "-L" + libdir, "-l:libhb.so", "-Wl,-rpath," + libdir,
           "-L" + os.path.join(CUDA, "lib64"), "-lcudart", "-Wl,-rpath," + os.path.join(CUDA, "lib64"),
           "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return exe


def test_c_consumer_compiles_and_links(tmp_path):
    """include/hb.h is valid C11 (-pedantic -Werror) and every call the C
    consumer makes resolves against libhb.so at link time."""
    exe = _build(tmp_path)
    assert os.path.exists(exe)


def _dump(path):
    e_lt, X, leaf_lt, sum_lt = load_hand_trees(synth.CMP_LT)
    _, _, leaf_le, sum_le = load_hand_trees(synth.CMP_LE)
    def fl(a):
        return " ".join(repr(float(v)) if np.isfinite(v) else ("nan" if np.isnan(v) else ("inf" if v > 0 else "-inf"))
                        for v in np.asarray(a, np.float64).ravel())
    def it(a):
        return " ".join(str(int(v)) for v in np.asarray(a).ravel())
    n = int(e_lt.node_offset[-1])
    with open(path, "w") as f:
        f.write(f"{e_lt.n_trees} {e_lt.n_features} {n} {X.shape[0]}\n")
        for a in (e_lt.node_offset, e_lt.feature):
            f.write(it(a) + "\n")
        f.write(fl(e_lt.threshold) + "\n")
        for a in (e_lt.left, e_lt.right):
            f.write(it(a) + "\n")
        f.write(fl(e_lt.leaf_value) + "\n")
        f.write(fl(X) + "\n")
        for leaf, s in ((leaf_lt, sum_lt), (leaf_le, sum_le)):
            f.write(it(leaf) + "\n" + fl(s) + "\n")


@pytest.mark.gpu
def test_c_consumer_on_hand_traced_trees(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build(tmp_path)
    dump = str(tmp_path / "golden.txt")
    _dump(dump)
    r = subprocess.run([exe, dump], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
