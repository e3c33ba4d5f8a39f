"""Device-side X generation (synth/csrc/synth_dev.cu -> synth/libhbsynth.so):
same bits as synth.gen_X, written straight into a torch CUDA tensor so the
bench never moves its inputs over PCIe (except for the e2e leg)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(_HERE, "libhbsynth.so")
SRC = os.path.join(_HERE, "csrc", "synth_dev.cu")


def build(force=False):
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode",
                               "arch=compute_100a,code=sm_100a", "-O3", "-Xcompiler", "-fPIC",
                               "-shared", "-o", SO, SRC, "-lcudart_static"])
    return SO


_lib = None


def _L():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise ImportError(f"{SO} missing; run __graft_entry__.build()")
        _lib = C.CDLL(SO)
        _lib.hbsynth_gen_X.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int64, C.c_int,
                                       C.c_uint32, C.c_int64, C.c_void_p, C.c_void_p]
        _lib.hbsynth_gen_X.restype = C.c_int
    return _lib


def gen_X_device(seed, n_rows, n_features, grid=0, special_q24=0, row_offset=0, ldx=None,
                 device=0):
    import torch
    ldx = n_features if ldx is None else ldx
    out = torch.empty((n_rows, ldx), dtype=torch.float32, device=f"cuda:{device}")
    st = torch.cuda.current_stream(out.device)
    rc = _L().hbsynth_gen_X(seed & 0xFFFFFFFFFFFFFFFF, n_rows, n_features, ldx, grid,
                            special_q24, row_offset, C.c_void_p(out.data_ptr()),
                            C.c_void_p(st.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"hbsynth_gen_X failed: cuda error {rc}")
    return out
