"""B200-native (sm_100a) batch scoring of decision-tree ensembles with the three
strategies of Hummingbird (arXiv 2010.04804): GEMM, TreeTraversal and
PerfectTreeTraversal.

All computation happens in libhb.so (CUDA kernels behind the C ABI declared in
include/hb.h). This module only marshals arguments: numpy arrays for the
ensemble, torch CUDA tensors for X / outputs and the current CUDA stream.
There is no CPU fallback: the first use of any API name loads libhb.so and
raises ImportError if it is missing. (Attributes are resolved lazily so that
the build module, `python -m paper_2010_04804_b200.build`, imports on a clean
tree.)
"""
import importlib

_API = ("HBError", "Model", "validate", "lib", "lib_path", "exported_symbols", "STRATEGY",
        "OUT", "KERNEL_NAME", "CMP_LT", "CMP_LE", "AGG_SUM", "AGG_MEAN", "POST_IDENTITY",
        "POST_SIGMOID", "POST_SOFTMAX", "POST_ISOLATION", "TASK_REGRESSION",
        "TASK_CLASSIFICATION")

__all__ = list(_API)


def __getattr__(name):
    if name in _API:
        hb = importlib.import_module(".hb", __name__)
        return getattr(hb, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
