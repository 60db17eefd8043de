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


def reduce_natural_join(a: Table, b: Table) -> ReducedMatrix:
    """missing keys / unsorted keys -> ValueError."""
    if a.keys is None or b.keys is None:
        raise ValueError("reduce_natural_join needs keys on both tables")
    return _reduce(a.data, a.keys, b.data, b.keys)


def reduce_join(a: Table, b: Table) -> ReducedMatrix:
    """Dispatcher exported by the reference (pkg/src/joinqr/__init__.py:38)."""
    if (a.keys is None) != (b.keys is None):
        raise ValueError("both tables must carry keys, or neither")
    if a.keys is None:
        return reduce_cartesian(a.data, b.data)
    return reduce_natural_join(a, b)


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
