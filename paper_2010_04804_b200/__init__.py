"""B200-native (sm_100a) batch scoring of decision-tree ensembles with the three
strategies of Hummingbird (arXiv 2010.04804): GEMM, TreeTraversal and
PerfectTreeTraversal.

All computation happens in libhb.so (CUDA kernels behind the C ABI declared in
include/hb.h). This module only marshals arguments: numpy arrays for the
ensemble, torch CUDA tensors for X / outputs and the current CUDA stream.
There is no CPU fallback: if libhb.so is missing, importing the binding raises.
"""
from .hb import (HBError, Model, validate, lib, lib_path, exported_symbols,  # noqa: F401
                 STRATEGY, OUT, CMP_LT, CMP_LE, AGG_SUM, AGG_MEAN, POST_IDENTITY,
                 POST_SIGMOID, POST_SOFTMAX, POST_ISOLATION, TASK_REGRESSION, TASK_CLASSIFICATION)
