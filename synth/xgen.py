"""Counter-based generator for input rows X (host side, numpy).

The device twin is ``synth/csrc/synth_dev.cu`` (same formula, written
separately); ``tests/test_synth.py`` checks a prefix of the host bits and the
GPU tests check host == device on every parity input.

Definition (all arithmetic mod 2^64)::

    z      = mix64(seed * 0x9E3779B97F4A7C15 + c * 0xD1B54A32D192ED03),  c = r*F + f
    fine   : x = ((z & 0xFFFF) - 32768) * 2^-12        (65536 dyadic values in [-8, 8))
    coarse : x = ((z & 0x3F)   - 32)    * 0.25          (64 values, tie-heavy)
    special: if (z >> 40) < special_q24:  x = [NaN, +Inf, -Inf, -0.0, +0.0][(z >> 16) % 5]

``mix64`` is the splitmix64 finaliser.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

GRID_FINE = 0
GRID_COARSE = 1

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)
_H = np.uint64(0xD1B54A32D192ED03)

_SPECIALS = np.array([np.nan, np.inf, -np.inf, -0.0, 0.0], dtype=np.float32)


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def counter_hash(seed: int, c: np.ndarray) -> np.ndarray:
    s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        return mix64(s * _G + np.asarray(c, dtype=np.uint64) * _H)


def _rows(seed, n_features, grid, special_q24, r0, r1, out):
    c = (np.arange(r0, r1, dtype=np.uint64)[:, None] * np.uint64(n_features)
         + np.arange(n_features, dtype=np.uint64)[None, :])
    z = counter_hash(seed, c)
    if grid == GRID_FINE:
        code = (z & np.uint64(0xFFFF)).astype(np.int32) - 32768
        x = code.astype(np.float32) * np.float32(1.0 / 4096.0)
    elif grid == GRID_COARSE:
        code = (z & np.uint64(0x3F)).astype(np.int32) - 32
        x = code.astype(np.float32) * np.float32(0.25)
    else:
        raise ValueError(f"unknown grid {grid}")
    if special_q24:
        sel = (z >> np.uint64(40)) < np.uint64(special_q24)
        kind = ((z >> np.uint64(16)) % np.uint64(5)).astype(np.int64)
        x = np.where(sel, _SPECIALS[kind], x)
    out[:, :n_features] = x


def gen_X(seed: int, n_rows: int, n_features: int, grid: int = GRID_FINE,
          special_q24: int = 0, row_offset: int = 0, ldx: int | None = None,
          threads: int | None = None) -> np.ndarray:
    """Rows [row_offset, row_offset+n_rows) of the seeded matrix, fp32.

    Returns an array of shape (n_rows, ldx) whose first ``n_features`` columns
    hold X (extra columns, if ``ldx > n_features``, are zero padding).
    ``special_q24`` = expected fraction of special cells times 2^24.
    """
    ldx = n_features if ldx is None else ldx
    if ldx < n_features:
        raise ValueError("ldx < n_features")
    out = np.zeros((n_rows, ldx), dtype=np.float32)
    if n_rows == 0:
        return out
    block = max(1, (1 << 22) // max(1, n_features))
    spans = [(r, min(n_rows, r + block)) for r in range(0, n_rows, block)]
    threads = threads or min(8, os.cpu_count() or 1)

    def work(span):
        a, b = span
        _rows(seed, n_features, grid, special_q24, row_offset + a,
              row_offset + b, out[a:b])

    if len(spans) == 1 or threads == 1:
        for s in spans:
            work(s)
    else:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, spans))
    return out
