"""ASan + UBSan build of the host-side boundary code with a mutation fuzzer
(SURVEY.md §4 levels 2 and 4): tests/fuzz/fuzz_layout.cpp links hb_validate
and the whole compile path (hb_host.cpp, hb_compile.cpp) in their host-only
mode, compiles random valid ensembles under every strategy and layout option,
interprets every built layout against a plain tree walk, and checks that
corrupted ensembles are rejected — any sanitizer report fails the run."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2010_04804_b200", "csrc")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def test_fuzz_layout_asan_ubsan(tmp_path):
    exe = str(tmp_path / "fuzz_layout")
    cmd = ["g++", "-std=c++17", "-O1", "-g", "-fsanitize=address,undefined",
           "-fno-sanitize-recover=all", "-fno-omit-frame-pointer", "-Wall",
           "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I" + os.path.join(CUDA, "include"),
           os.path.join(ROOT, "tests", "fuzz", "fuzz_layout.cpp"),
           os.path.join(CSRC, "hb_host.cpp"), os.path.join(CSRC, "hb_compile.cpp"),
           "-L" + os.path.join(CUDA, "lib64"), "-lcudart", "-lpthread",
           "-Wl,-rpath," + os.path.join(CUDA, "lib64"), "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1")
    for seed in (1, 2):
        r = subprocess.run([exe, "800", str(seed)], capture_output=True, text=True, env=env, timeout=600)
        assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
        assert "0 failures" in r.stdout, r.stdout
        # the TMA pre-pass grouping (rank_code_tma_kernel) was built and interpreted
        m = re.search(r"TMA groups (\d+)", r.stdout)
        assert m and int(m.group(1)) > 0, r.stdout
