"""ctypes front-end of the C oracle (oracle/oracle.c) plus the literal
transcriptions of Alg. 1-3 (oracle/literal.py).

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package. The product
(paper_2010_04804_b200) never imports it, and this package never imports the
product.

Parity status per function:
  leaf, raw, margin, post, label, leaf_hash — pinned (tests/test_oracle_*.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               "-fno-fast-math", "-Wall", "-o", _SO, src, "-lm",
                               "-lpthread"])
    return _SO


class _Ens(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("n_features", C.c_int32), ("n_outputs", C.c_int32),
                ("node_offset", C.c_void_p), ("feature", C.c_void_p),
                ("threshold", C.c_void_p), ("left", C.c_void_p), ("right", C.c_void_p),
                ("leaf_value", C.c_void_p), ("leaf_width", C.c_int32),
                ("tree_output", C.c_void_p), ("base_score", C.c_void_p),
                ("cmp", C.c_int32), ("agg", C.c_int32), ("post", C.c_int32),
                ("post_param", C.c_double)]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i64, i32, vp = C.c_int64, C.c_int32, C.c_void_p
        P = C.POINTER(_Ens)
        _lib.oracle_leaf.argtypes = [P, vp, i64, i64, i32, i32, vp]
        _lib.oracle_raw.argtypes = [P, vp, i64, i64, i32, i32, vp]
        _lib.oracle_margin.argtypes = [P, vp, i64, vp]
        _lib.oracle_post.argtypes = [P, vp, i64, vp]
        _lib.oracle_label.argtypes = [P, vp, i64, vp]
        _lib.oracle_leaf_hash.argtypes = [P, vp, i64, i64, i32, i32, vp]
        _lib.oracle_raw_mt.argtypes = [P, vp, i64, i64, i32, i32, vp, C.c_int]
        _lib.oracle_raw_mt.restype = C.c_int
        _lib.oracle_raw_hash_mt.argtypes = [P, vp, i64, i64, i32, i32, vp, vp, C.c_int]
        _lib.oracle_raw_hash_mt.restype = C.c_int
        _lib.oracle_predict_mt.argtypes = [P, vp, i64, i64, vp, C.c_int]
        _lib.oracle_predict_mt.restype = C.c_int
    return _lib


class _Handle:
    """Keeps contiguous copies of the ensemble arrays alive with the struct."""

    def __init__(self, e):
        self.keep = []

        def arr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            self.keep.append(a)
            return a.ctypes.data

        self.s = _Ens(int(e.n_trees), int(e.n_features), int(e.n_outputs),
                      arr(e.node_offset, np.int64), arr(e.feature, np.int32),
                      arr(e.threshold, np.float32), arr(e.left, np.int32),
                      arr(e.right, np.int32), arr(e.leaf_value, np.float32),
                      int(e.leaf_width), arr(e.tree_output, np.int32),
                      arr(e.base_score, np.float32), int(e.cmp), int(e.agg),
                      int(e.post), float(getattr(e, "post_param", 0.0)))
        self.K = int(e.n_outputs)
        self.T = int(e.n_trees)


def _X(X):
    X = np.asarray(X, dtype=np.float32)
    if X.ndim != 2 or X.strides[1] != 4:
        X = np.ascontiguousarray(X)
    return X, X.strides[0] // 4


def leaf(e, X, t0=0, t1=None):
    """int32 [n, t1-t0]: tree-local original id of the reached leaf."""
    h = _Handle(e)
    t1 = h.T if t1 is None else t1
    X, ldx = _X(X)
    out = np.empty((X.shape[0], t1 - t0), np.int32)
    _L().oracle_leaf(C.byref(h.s), X.ctypes.data, X.shape[0], ldx, t0, t1, out.ctypes.data)
    return out


def raw(e, X, t0=0, t1=None, threads=1):
    """fp64 [n, K]: sum of reached leaf values over trees [t0, t1)."""
    h = _Handle(e)
    t1 = h.T if t1 is None else t1
    X, ldx = _X(X)
    out = np.empty((X.shape[0], h.K), np.float64)
    if threads == 1:
        _L().oracle_raw(C.byref(h.s), X.ctypes.data, X.shape[0], ldx, t0, t1, out.ctypes.data)
    else:
        _L().oracle_raw_mt(C.byref(h.s), X.ctypes.data, X.shape[0], ldx, t0, t1,
                           out.ctypes.data, threads)
    return out


def margin(e, raw_sum):
    h = _Handle(e)
    raw_sum = np.ascontiguousarray(raw_sum, np.float64)
    out = np.empty_like(raw_sum)
    _L().oracle_margin(C.byref(h.s), raw_sum.ctypes.data, raw_sum.shape[0], out.ctypes.data)
    return out


def post(e, m):
    h = _Handle(e)
    m = np.ascontiguousarray(m, np.float64)
    out = np.empty_like(m)
    _L().oracle_post(C.byref(h.s), m.ctypes.data, m.shape[0], out.ctypes.data)
    return out


def label(e, m):
    h = _Handle(e)
    m = np.ascontiguousarray(m, np.float64)
    out = np.empty(m.shape[0], np.int32)
    _L().oracle_label(C.byref(h.s), m.ctypes.data, m.shape[0], out.ctypes.data)
    return out


def leaf_hash(e, X, t0=0, t1=None):
    h = _Handle(e)
    t1 = h.T if t1 is None else t1
    X, ldx = _X(X)
    out = np.empty(X.shape[0], np.uint64)
    _L().oracle_leaf_hash(C.byref(h.s), X.ctypes.data, X.shape[0], ldx, t0, t1, out.ctypes.data)
    return out


def raw_and_hash(e, X, t0=0, t1=None, threads=0):
    """(raw fp64 [n, K], leaf hash uint64 [n]) over trees [t0, t1) with one
    walk per (row, tree) on `threads` pthreads (0: all cores) — the same values
    as raw() and leaf_hash(); for every-row parity at full size."""
    h = _Handle(e)
    t1 = h.T if t1 is None else t1
    X, ldx = _X(X)
    out = np.empty((X.shape[0], h.K), np.float64)
    hs = np.empty(X.shape[0], np.uint64)
    _L().oracle_raw_hash_mt(C.byref(h.s), X.ctypes.data, X.shape[0], ldx, t0, t1,
                            out.ctypes.data, hs.ctypes.data, threads)
    return out, hs


def scores(e, X, threads=1):
    """Everything a caller gets: dict(raw, margin, post, label) in fp64/int32."""
    r = raw(e, X, threads=threads)
    m = margin(e, r)
    return dict(raw=r, margin=m, post=post(e, m), label=label(e, m))


def proba(e, post_scores):
    """Class probabilities as the ABI returns them (reading R27):
    binary sigmoid models give [1-p, p]; K >= 2 gives the post scores."""
    if e.n_outputs == 1:
        p = post_scores[:, 0]
        return np.stack([1.0 - p, p], 1)
    return post_scores


def predict_mt(e, X, threads=0):
    """Multi-threaded full scoring (raw -> margin -> post); returns
    (scores fp64 [n, K], threads used). Used only for the CPU baseline."""
    h = _Handle(e)
    X, ldx = _X(X)
    out = np.empty((X.shape[0], h.K), np.float64)
    used = _L().oracle_predict_mt(C.byref(h.s), X.ctypes.data, X.shape[0], ldx,
                                  out.ctypes.data, threads)
    return out, used
