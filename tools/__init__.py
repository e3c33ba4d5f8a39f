"""Measurement helpers for bench.py (not on the scoring path)."""
import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(_HERE, "libhbpeaks.so")
SRC = os.path.join(_HERE, "peaks.cu")


def build(force=False):
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode",
                               "arch=compute_100a,code=sm_100a", "-O3", "-Xcompiler", "-fPIC",
                               "-shared", "-o", SO, SRC, "-lcudart_static"])
    return SO


def peaks(device=0):
    L = C.CDLL(SO)
    L.hbpeaks_smem_gbs.restype = C.c_double
    L.hbpeaks_l2_gbs.restype = C.c_double
    return {"smem_gbs": L.hbpeaks_smem_gbs(device), "l2_gbs": L.hbpeaks_l2_gbs(device)}


def l2_chase(device=0, nbytes=16 << 20, chains=4):
    """Dependent random 16-B gathers per second from an `nbytes` buffer, in
    tt_wide_kernel's launch shape (1024 threads per SM, `chains` walks per
    thread): the latency-bound roof of a tree walk whose records live in L2."""
    L = C.CDLL(SO)
    L.hbpeaks_l2_chase.restype = C.c_double
    L.hbpeaks_l2_chase.argtypes = [C.c_int, C.c_longlong, C.c_int]
    return L.hbpeaks_l2_chase(device, nbytes, chains)
