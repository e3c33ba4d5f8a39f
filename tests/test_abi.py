"""CPU-side checks of the C ABI: libhb.so loads, exports every symbol
include/hb.h declares, and the host-only validator (hb_validate) accepts good
ensembles and rejects each malformed-tree class."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hb_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    import paper_2010_04804_b200 as hb
    declared = _declared()
    assert len(declared) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", hb.lib_path], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (hb_\w+)", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert sorted(hb.exported_symbols) == declared
    assert hb.lib.hb_abi_version() == 6


def test_sm100a_cubin_embedded():
    import paper_2010_04804_b200 as hb
    out = subprocess.run(["cuobjdump", "--list-elf", hb.lib_path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _ok_forest():
    return synth.gen_forest(4, 4, 5, seed=1, family="mixed")


def _bad(mut):
    e = _ok_forest()
    mut(e)
    return e


def test_validate_accepts_generated_and_configs():
    from paper_2010_04804_b200.hb import validate
    validate(_ok_forest())
    for name in ("C1", "C2"):
        validate(synth.make_config(name, n_trees=3)[1])


@pytest.mark.parametrize("what,mut,status", [
    ("one child -1", lambda e: e.right.__setitem__(0, -1), 2),
    ("child out of range", lambda e: e.left.__setitem__(0, 999), 2),
    ("feature out of range", lambda e: e.feature.__setitem__(0, 5), 2),
    ("NaN threshold", lambda e: e.threshold.__setitem__(0, np.nan), 2),
    ("non-finite leaf", lambda e: e.leaf_value.__setitem__(int(np.nonzero(e.left == -1)[0][0]), np.inf), 2),
    ("double parent", lambda e: e.left.__setitem__(0, e.right[0]), 2),
    ("tree_output range", lambda e: setattr(e, "tree_output", np.array([0, 1, 0, 0], np.int32)), 2),
    ("sigmoid with K=2", lambda e: (setattr(e, "n_outputs", 2), setattr(e, "post", 1)), 2),
    ("GT cmp", lambda e: setattr(e, "cmp", 2), 3),
    ("classification identity K=1", lambda e: setattr(e, "task", 1), 2),
    ("isolation without c(psi)", lambda e: (setattr(e, "post", 3), setattr(e, "agg", 1)), 2),
    ("isolation K=2", lambda e: (setattr(e, "post", 3), setattr(e, "post_param", 8.0),
                                 setattr(e, "n_outputs", 2)), 2),
])
def test_validate_rejects(what, mut, status):
    from paper_2010_04804_b200.hb import validate, HBError
    with pytest.raises(HBError) as ei:
        validate(_bad(mut))
    assert ei.value.status == status, what


def test_validate_rejects_cycle():
    from paper_2010_04804_b200.hb import validate, HBError
    # root 0 -> (1, 2); nodes 3 and 4 form a cycle 3 -> (4, 5), 4 -> (3, 6)
    tr = dict(feature=[0, -1, -1, 0, 0, -1, -1], threshold=[0, np.nan, np.nan, 0, 0, np.nan, np.nan],
              left=[1, -1, -1, 4, 3, -1, -1], right=[2, -1, -1, 5, 6, -1, -1],
              leaf_value=[np.nan, 1, 2, np.nan, np.nan, 3, 4])
    e = synth.from_trees([tr], 1)
    with pytest.raises(HBError) as ei:
        validate(e)
    assert ei.value.status == 2 and "reachable" in str(ei.value)


def test_compile_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_2010_04804_b200 as hb
    with pytest.raises(hb.HBError) as ei:
        hb.Model(_ok_forest(), device=0)
    assert ei.value.status == 1   # HB_E_INVALID: not a CUDA device


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: a copy of the package without libhb.so imports (so the
    build module works on a clean tree) but any API use raises ImportError."""
    import shutil
    pkg = os.path.join(ROOT, "paper_2010_04804_b200")
    dst = tmp_path / "paper_2010_04804_b200"
    shutil.copytree(pkg, dst, ignore=shutil.ignore_patterns("*.so", "build", "csrc"))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_2010_04804_b200 as hb\n"
            "import paper_2010_04804_b200.build\n"
            "try:\n    hb.Model\nexcept ImportError as e:\n    print('IMPORTERROR', e)\n") % str(tmp_path)
    out = subprocess.run([__import__("sys").executable, "-c", code], capture_output=True, text=True)
    assert "IMPORTERROR" in out.stdout and "libhb.so is missing" in out.stdout, out.stdout + out.stderr
