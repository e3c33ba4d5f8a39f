"""ctypes binding of libhb.so (include/hb.h). Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# HB_LIB: another build of the same library (tests: the bounds-checked
# libhb_checked.so); never a fallback — a missing library still fails loudly
lib_path = os.environ.get("HB_LIB") or os.path.join(_PKG, "libhb.so")

CMP_LT, CMP_LE = 0, 1
AGG_SUM, AGG_MEAN = 0, 1
POST_IDENTITY, POST_SIGMOID, POST_SOFTMAX, POST_ISOLATION = 0, 1, 2, 3
TASK_REGRESSION, TASK_CLASSIFICATION = 0, 1
STRATEGY = {"auto": 0, "gemm": 1, "tt": 2, "ptt": 3}
STRATEGY_NAME = {v: k for k, v in STRATEGY.items()}
ABI_VERSION = 6
KERNEL_NAME = {0: "ptt_kernel", 1: "pttr_kernel", 2: "tt_kernel", 3: "tt_wide_kernel",
               4: "gemm_tc_kernel", 5: "gemm_kernel"}
OUT = {"predict": 0, "proba": 1, "raw": 2, "margin": 3, "leaf": 4, "leaf_hash": 5, "raw64": 6}

# every symbol include/hb.h declares (checked by tests/test_abi.py)
exported_symbols = ["hb_validate", "hb_compile", "hb_compile_range", "hb_predict_ex",
                    "hb_predict_ex_events", "hb_predict", "hb_predict_proba", "hb_predict_raw", "hb_predict_leaf",
                    "hb_finalize", "hb_finalize64", "hb_predict_host", "hb_model_get_info", "hb_free",
                    "hb_last_error", "hb_abi_version"]


class HBError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"hb status {status}: {msg}")
        self.status = status


class _Ens(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("n_features", C.c_int32), ("n_outputs", C.c_int32),
                ("node_offset", C.c_void_p), ("feature", C.c_void_p),
                ("threshold", C.c_void_p), ("left", C.c_void_p), ("right", C.c_void_p),
                ("leaf_value", C.c_void_p), ("leaf_width", C.c_int32),
                ("tree_output", C.c_void_p), ("base_score", C.c_void_p),
                ("cmp", C.c_int32), ("agg", C.c_int32), ("post", C.c_int32),
                ("task", C.c_int32), ("post_param", C.c_float)]


class _Info(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("max_depth", C.c_int32), ("tree_begin", C.c_int32),
                ("n_trees", C.c_int32), ("n_trees_total", C.c_int32),
                ("n_features", C.c_int32), ("n_outputs", C.c_int32),
                ("leaf_width", C.c_int32), ("device", C.c_int32), ("x_in_smem", C.c_int32),
                ("device_bytes", C.c_int64), ("tree_stride_bytes", C.c_int64),
                ("tensor_cores", C.c_int32), ("node_record_bytes", C.c_int32),
                ("kernel", C.c_int32), ("rows_per_cta", C.c_int32),
                ("code_cell_bits", C.c_int32), ("rank_prepass", C.c_int32),
                ("tt_sector", C.c_int32), ("tt_chunk_trees", C.c_int32),
                ("small_batch_max_rows", C.c_int32), ("tt_walks_per_lane", C.c_int32),
                ("tt_record_bytes", C.c_int64), ("rank_prepass_tma", C.c_int32), ("rows_per_lane", C.c_int32)]


def _load():
    if not os.path.exists(lib_path):
        raise ImportError(f"{lib_path} is missing: build it with "
                          "`python -m paper_2010_04804_b200.build` (no CPU fallback exists)")
    L = C.CDLL(lib_path)
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
    P = C.POINTER(_Ens)
    sig = {
        "hb_validate": ([P], C.c_int),
        "hb_compile": ([P, i32, i32, C.POINTER(vp)], C.c_int),
        "hb_compile_range": ([P, i32, i32, i32, i32, C.POINTER(vp)], C.c_int),
        "hb_predict_ex": ([vp, vp, i64, i64, i32, vp, vp], C.c_int),
        "hb_predict_ex_events": ([vp, vp, i64, i64, i32, vp, vp, C.POINTER(vp), i32, C.POINTER(i32)],
                                 C.c_int),
        "hb_predict": ([vp, vp, i64, i64, vp, vp], C.c_int),
        "hb_predict_proba": ([vp, vp, i64, i64, vp, vp], C.c_int),
        "hb_predict_raw": ([vp, vp, i64, i64, vp, vp], C.c_int),
        "hb_predict_leaf": ([vp, vp, i64, i64, vp, vp], C.c_int),
        "hb_finalize": ([vp, vp, i64, i32, vp, vp], C.c_int),
        "hb_finalize64": ([vp, vp, i64, i32, vp, vp], C.c_int),
        "hb_predict_host": ([vp, vp, i64, i64, i32, vp], C.c_int),
        "hb_model_get_info": ([vp, C.POINTER(_Info)], C.c_int),
        "hb_free": ([vp], None),
        "hb_last_error": ([], C.c_char_p),
        "hb_abi_version": ([], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if L.hb_abi_version() != ABI_VERSION:     # hb_model_info layout of this binding
        raise ImportError(f"{lib_path}: ABI {L.hb_abi_version()}, binding expects {ABI_VERSION}: rebuild it")
    return L


lib = _load()


def _check(st):
    if st != 0:
        raise HBError(st, lib.hb_last_error().decode())


class _EnsHandle:
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
                      int(e.post), int(getattr(e, "task", 0)),
                      float(getattr(e, "post_param", 0.0)))


def validate(e) -> None:
    """Host-only validation (hb_validate); raises HBError."""
    h = _EnsHandle(e)
    _check(lib.hb_validate(C.byref(h.s)))


class Model:
    """A compiled ensemble on one GPU (hb_compile / hb_compile_range)."""

    def __init__(self, ensemble, strategy="auto", device=0, tree_range=None):
        h = _EnsHandle(ensemble)
        p = C.c_void_p()
        s = STRATEGY[strategy] if isinstance(strategy, str) else int(strategy)
        if tree_range is None:
            _check(lib.hb_compile(C.byref(h.s), s, int(device), C.byref(p)))
        else:
            _check(lib.hb_compile_range(C.byref(h.s), int(tree_range[0]), int(tree_range[1]),
                                        s, int(device), C.byref(p)))
        self._p = p
        self.device = int(device)
        self.info = self._info()
        self.task = int(getattr(ensemble, "task", 0))

    def _info(self):
        i = _Info()
        _check(lib.hb_model_get_info(self._p, C.byref(i)))
        d = {k: getattr(i, k) for k, _ in _Info._fields_}
        d["strategy_name"] = STRATEGY_NAME[d["strategy"]]
        d["kernel_name"] = KERNEL_NAME.get(d["kernel"], "?")
        return d

    def kernel_for(self, n_rows):
        """Name of the scoring kernel a call with n_rows rows launches: the
        small-batch (trees-across-threads) kernel up to small_batch_max_rows,
        else the model's row-tile scorer."""
        if n_rows <= self.info["small_batch_max_rows"]:
            return "small_batch_kernel"
        return self.info["kernel_name"]

    def free(self):
        if getattr(self, "_p", None):
            lib.hb_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    # ------------------------------------------------------------ device API
    def out_shape(self, n, kind):
        K = self.info["n_outputs"]
        if kind == "predict":
            return ((n,), "int32") if self.task == TASK_CLASSIFICATION else ((n, K), "float32")
        if kind == "proba":
            return ((n, 2 if K == 1 else K), "float32")
        if kind in ("raw", "margin"):
            return ((n, K), "float32")
        if kind == "raw64":
            return ((n, K), "float64")
        if kind == "leaf":
            return ((n, self.info["n_trees"]), "int32")
        if kind == "leaf_hash":
            return ((n,), "int64")
        raise ValueError(kind)

    def _out(self, n, kind, out, device):
        """Allocate `out`, or check a caller-supplied one: the C ABI cannot see
        a buffer's length, so a wrong shape/dtype/device would be an
        out-of-bounds device write."""
        import torch
        shape, dt = self.out_shape(n, kind)
        want = getattr(torch, dt)
        if out is None:
            return torch.empty(shape, dtype=want, device=device)
        if not isinstance(out, torch.Tensor) or tuple(out.shape) != tuple(shape) or out.dtype != want \
                or not out.is_contiguous() or out.device != torch.device(device):
            raise ValueError(f"out must be a contiguous {dt} tensor of shape {shape} on {device}, got "
                             f"{getattr(out, 'dtype', type(out))} {tuple(getattr(out, 'shape', ()))} "
                             f"on {getattr(out, 'device', '?')}")
        return out

    def run(self, X, kind="predict", out=None, stream=None):
        """One fused scoring launch (hb_predict_ex; two with the rank-code pre-pass) on torch CUDA tensors.
        X: float32 [n, >= F] with unit column stride. Returns `out`."""
        import torch
        if X.dtype != torch.float32 or X.dim() != 2 or X.stride(1) != 1:
            raise ValueError("X must be a 2-D float32 tensor with unit column stride")
        n = X.shape[0]
        out = self._out(n, kind, out, X.device)
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        _check(lib.hb_predict_ex(self._p, C.c_void_p(X.data_ptr()), n, X.stride(0), OUT[kind],
                                 C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream)))
        return out

    def run_events(self, X, kind, out, events, stream):
        """hb_predict_ex_events: the same call as run(), recording torch
        CUDA events (already created, enable_timing) at the start of every
        kernel launch and after the last one; returns the launch count."""
        n = X.shape[0]
        out = self._out(n, kind, out, X.device)
        arr = (C.c_void_p * len(events))(*[C.c_void_p(ev.cuda_event) for ev in events])
        nl = C.c_int32(0)
        _check(lib.hb_predict_ex_events(self._p, C.c_void_p(X.data_ptr()), n, X.stride(0), OUT[kind],
                                        C.c_void_p(out.data_ptr()), C.c_void_p(stream.cuda_stream),
                                        arr, len(events), C.byref(nl)))
        return nl.value

    def predict(self, X, **kw):
        return self.run(X, "predict", **kw)

    def predict_proba(self, X, **kw):
        return self.run(X, "proba", **kw)

    def predict_raw(self, X, **kw):
        return self.run(X, "raw", **kw)

    def predict_raw64(self, X, **kw):
        return self.run(X, "raw64", **kw)

    def predict_margin(self, X, **kw):
        return self.run(X, "margin", **kw)

    def predict_leaf(self, X, **kw):
        return self.run(X, "leaf", **kw)

    def predict_leaf_hash(self, X, **kw):
        return self.run(X, "leaf_hash", **kw)

    def finalize(self, raw, kind="predict", out=None, stream=None):
        """hb_finalize (float32 raw) / hb_finalize64 (float64 raw): epilogue
        from device raw sums over all trees, shape (n, K)."""
        import torch
        K = self.info["n_outputs"]
        if raw.dtype not in (torch.float32, torch.float64) or raw.dim() != 2 or raw.shape[1] != K \
                or not raw.is_contiguous():
            raise ValueError(f"raw must be a contiguous float32/float64 tensor of shape (n, {K})")
        n = raw.shape[0]
        out = self._out(n, kind, out, raw.device)
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        fn = lib.hb_finalize64 if raw.dtype == torch.float64 else lib.hb_finalize
        _check(fn(self._p, C.c_void_p(raw.data_ptr()), n, OUT[kind],
                  C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream)))
        return out

    # ------------------------------------------------------------ host API
    def predict_host(self, X, kind="predict", out=None):
        """hb_predict_host: end-to-end from host memory (numpy array or CPU
        torch tensor, ideally pinned). Synchronous."""
        try:
            import torch
            is_t = isinstance(X, torch.Tensor)
        except ImportError:
            is_t = False
        n = X.shape[0]
        shape, dt = self.out_shape(n, kind)
        if is_t:
            import torch
            assert X.device.type == "cpu" and X.dtype == torch.float32 and X.stride(1) == 1
            ldx = X.stride(0)
            if out is None:
                out = torch.empty(shape, dtype=getattr(torch, dt))
            xp, op = X.data_ptr(), out.data_ptr()
        else:
            X = np.asarray(X, np.float32)
            if X.strides[1] != 4:
                X = np.ascontiguousarray(X)
            ldx = X.strides[0] // 4
            if out is None:
                out = np.empty(shape, dtype=dt)
            xp, op = X.ctypes.data, out.ctypes.data
        _check(lib.hb_predict_host(self._p, C.c_void_p(xp), n, ldx, OUT[kind], C.c_void_p(op)))
        return out
