"""Synthetic inputs: uniform(0,1) tables from the counter-based
SplitMix64 generator, produced on the GPU (jq_gen.cu), bit-identical to the
recipe documented in oracle/datagen.py (first outputs for seed 1234567 are the
generator's published test vector, tests/test_oracle_golden.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from .joins import Table


@dataclass
class GenSpec:
    rows: int
    cols: int
    seed: int
    key_groups: Optional[int] = None


def uniform(seed: int, rows: int, cols: int, row0: int = 0, out=None):
    """rows x cols block (from table row row0) into `out` (numpy or torch CUDA)."""
    if out is None:
        out = np.empty((rows, cols))
    N.use_torch_stream(out)
    N.check(N.lib().jq_gen_uniform(N.ctx(), seed & 0xFFFFFFFFFFFFFFFF, rows, cols, row0, N.ptr(out)))
    return out


def near_equal_keys(rows: int, key_groups: int) -> np.ndarray:
    """Sorted keys, first rows % key_groups groups one row larger."""
    if not 1 <= key_groups <= rows:
        raise ValueError("key_groups must lie in 1..rows")
    q, r = divmod(rows, key_groups)
    i = np.arange(rows, dtype=np.int64)
    big = r * (q + 1)
    return np.where(i < big, i // (q + 1), r + (i - big) // max(q, 1)).astype(np.int64)


def zipf_cdf(s: float, universe: int) -> np.ndarray:
    cdf = np.cumsum(np.arange(1, universe + 1, dtype=np.float64) ** (-s))
    return cdf / cdf[-1]


def zipf_sorted_keys(seed: int, rows: int, s: float = 1.1, universe: int = 1_000_000, out=None):
    """Sorted Zipf(s) keys: the sorted multiset of searchsorted(cdf, u_row, 'right')."""
    cdf = zipf_cdf(s, universe)
    if out is None:
        out = np.empty(rows, dtype=np.int64)
    N.use_torch_stream(out)
    N.check(N.lib().jq_gen_zipf_sorted_keys(N.ctx(), seed & 0xFFFFFFFFFFFFFFFF, rows,
                                            cdf.ctypes.data, universe, N.ptr(out)))
    return out


def zipf_keys(seed: int, rows: int, s: float = 1.1, universe: int = 1_000_000, out=None):
    """Unsorted Zipf(s) keys, one per row: searchsorted(cdf, u_row, 'right')."""
    cdf = zipf_cdf(s, universe)
    if out is None:
        out = np.empty(rows, dtype=np.int64)
    N.use_torch_stream(out)
    N.check(N.lib().jq_gen_zipf_keys(N.ctx(), seed & 0xFFFFFFFFFFFFFFFF, rows, cdf.ctypes.data, universe,
                                     N.ptr(out)))
    return out


def zipf_table(seed_keys: int, seed_data: int, rows: int, cols: int, device=None, s: float = 1.1,
               universe: int = 1_000_000) -> Table:
    """C3 recipe: per-row Zipf keys and uniform rows in generation
    order, then a stable sort of (key, row) permutes the data rows (GPU radix sort +
    row gather).  device=None: numpy tables; else torch tensors on that device."""
    from .joins import argsort_keys, gather_rows
    if device is None:
        keys, data = zipf_keys(seed_keys, rows, s, universe), uniform(seed_data, rows, cols)
    else:
        import torch
        keys = zipf_keys(seed_keys, rows, s, universe,
                         out=torch.empty(rows, dtype=torch.int64, device=device))
        data = uniform(seed_data, rows, cols, out=torch.empty((rows, cols), dtype=torch.float64, device=device))
    sk, perm = argsort_keys(keys)
    return Table(gather_rows(data, perm), sk)


def gen_uniform(spec: GenSpec) -> Table:
    """rows x cols uniform(0,1), same spec -> bit-identical table."""
    if spec.rows < 1 or spec.cols < 1:
        raise ValueError("gen_uniform needs rows >= 1 and cols >= 1")
    data = uniform(spec.seed, spec.rows, spec.cols)
    keys = None if spec.key_groups is None else near_equal_keys(spec.rows, spec.key_groups)
    return Table(data, keys)
