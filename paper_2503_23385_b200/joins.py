"""Claim-1 join reduction on the GPU.

`reduce_cartesian` / `reduce_natural_join` / `reduce_join` return the reduced
matrix in SPEC row order (group by group in ascending key order, top block
[sqrt(m2g) A_g | head(B_g)] then bottom block [0 | sqrt(m1g) tail(B_g)]).
`group_keys` exposes the bit-exact device grouping.
figaro_r never materialises this matrix: it streams the same rows into the
TSQR (qr.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N
from ._arrays import as_keys, like
from .matrix import as_matrix


@dataclass
class Table:
    """Data columns plus an optional int64 key column sorted non-decreasing
    (SPEC.md:174-179).  `data` / `keys` may be numpy arrays or torch CUDA tensors."""

    data: object
    keys: Optional[object] = None

    def __post_init__(self):
        self.data = as_matrix(self.data)
        self.keys = as_keys(self.keys, self.data.shape[0])


@dataclass
class ReducedMatrix:
    """(sum_g (m1g+m2g-1)) x (n1+n2) matrix plus provenance."""

    matrix: object
    group_boundaries: List[Tuple[int, int]] = field(default_factory=list)
    n1: int = 0
    n2: int = 0


def _reduce(a, ka, b, kb) -> ReducedMatrix:
    m1, n1 = a.shape
    m2, n2 = b.shape
    if ka is None:
        total, gb = m1 + m2 - 1, [(0, m1 + m2 - 1)]
    else:
        red_off = group_keys(ka, kb)[5]
        total = int(red_off[-1])
        ro = red_off.tolist()
        gb = list(zip(ro[:-1], ro[1:]))
    out = like((total, n1 + n2), a, b)
    if total:
        rows = np.zeros(1, dtype=np.int64)
        N.use_torch_stream(a, b, ka, kb)
        N.check(N.lib().jq_reduce(N.ctx(), N.ptr(a), m1, n1, N.ptr(ka), N.ptr(b), m2, n2, N.ptr(kb),
                                  N.ptr(out), total, rows.ctypes.data, None))
    return ReducedMatrix(out, gb, n1, n2)


def reduce_cartesian(a, b) -> ReducedMatrix:
    """empty input -> ValueError."""
    a, b = as_matrix(a), as_matrix(b)
    if a.shape[0] == 0 or b.shape[0] == 0:
        raise ValueError("reduce_cartesian needs non-empty inputs")
    return _reduce(a, None, b, None)


def reduce_natural_join(a: Table, b: Table, sort: bool = False) -> ReducedMatrix:
    """missing keys / unsorted keys -> ValueError.  ``sort=True``
    (opt-in, not in the reference) first sorts both tables by key on the GPU
    (sort_by_key); group_boundaries then refer to the sorted tables."""
    if a.keys is None or b.keys is None:
        raise ValueError("reduce_natural_join needs keys on both tables")
    if sort:
        a, b = sort_by_key(a), sort_by_key(b)
    return _reduce(a.data, a.keys, b.data, b.keys)


def reduce_join(a: Table, b: Table, sort: bool = False) -> ReducedMatrix:
    """Dispatcher exported by the reference (pkg/src/joinqr/__init__.py:38)."""
    if (a.keys is None) != (b.keys is None):
        raise ValueError("both tables must carry keys, or neither")
    if a.keys is None:
        return reduce_cartesian(a.data, b.data)
    return reduce_natural_join(a, b, sort=sort)


def argsort_keys(keys):
    """(sorted keys, permutation) of an int64 key column by the GPU stable LSD radix
    sort (jq_sort.cu): perm equals np.argsort(keys, kind="stable") bit for bit and
    sorted = keys[perm].  numpy in -> numpy out, torch CUDA in -> torch CUDA out."""
    k = as_keys(keys, len(keys))
    out_k = like((len(k),), k, dtype="i8")
    perm = like((len(k),), k, dtype="i8")
    N.use_torch_stream(k)
    N.check(N.lib().jq_sort_keys(N.ctx(), N.ptr(k), len(k), N.ptr(out_k), N.ptr(perm)))
    return out_k, perm


def gather_rows(x, perm):
    """x[perm] for a row-major table on the GPU (jq_gather_rows)."""
    x = as_matrix(x)
    perm = as_keys(perm, len(perm))
    rows, cols = x.shape
    if len(perm) != rows:
        raise ValueError("permutation length does not match the row count")
    out = like((rows, cols), x)
    N.use_torch_stream(x, perm)
    N.check(N.lib().jq_gather_rows(N.ctx(), N.ptr(x), rows, cols, N.ptr(perm), N.ptr(out)))
    return out


def sort_by_key(t: Table) -> Table:
    """The table with its rows stably sorted by key (GPU radix sort + row gather).
    The reference requires sorted keys and raises otherwise; this is
    the opt-in way to feed it unsorted tables.  Keyless tables are returned as is."""
    if t.keys is None:
        return t
    keys, perm = argsort_keys(t.keys)
    return Table(gather_rows(t.data, perm), keys)


def group_keys(keys_a, keys_b):
    """(matched_keys, a_start, a_count, b_start, b_count, red_off) as int64 numpy
    arrays, computed on the GPU (bit-exact with the reference grouping)."""
    ka = as_keys(keys_a, len(keys_a))
    kb = as_keys(keys_b, len(keys_b))
    cap = max(1, min(len(ka), len(kb)))
    # np.empty: only the first ng entries are written (no 5 x cap zero fill on the host)
    outs = [np.empty(cap, dtype=np.int64) for _ in range(5)]
    red = np.empty(cap + 1, dtype=np.int64)
    ng = np.zeros(1, dtype=np.int64)
    N.use_torch_stream(ka, kb)
    N.check(N.lib().jq_group_keys(N.ctx(), N.ptr(ka), len(ka), N.ptr(kb), len(kb), cap,
                                  ng.ctypes.data, *[o.ctypes.data for o in outs], red.ctypes.data))
    g = int(ng[0])
    return tuple(o[:g] for o in outs) + (red[:g + 1],)
