"""Claim-1 join reduction, restated from SPEC.md:169-238.

Test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from .headtail import head, tail
from .matrix import as_matrix


@dataclass
class Table:
    """Data columns plus an optional int64 key column."""

    data: np.ndarray
    keys: Optional[np.ndarray] = None

    def __post_init__(self):
        self.data = as_matrix(self.data)
        if self.keys is not None:
            self.keys = np.ascontiguousarray(self.keys, dtype=np.int64).reshape(-1)
            if self.keys.shape[0] != self.data.shape[0]:
                raise ValueError("key column length does not match the row count")


@dataclass
class ReducedMatrix:
    """(sum_g (m1g+m2g-1)) x (n1+n2) reduced matrix plus provenance."""

    matrix: np.ndarray
    group_boundaries: List[Tuple[int, int]] = field(default_factory=list)
    n1: int = 0
    n2: int = 0


def reduce_cartesian(a, b) -> ReducedMatrix:
    """Top m1 rows [sqrt(m2) A | head(B)], bottom m2-1 rows [0 | sqrt(m1) tail(B)]
    (zero block dropped).  NB SPEC.md:200 misprints the
    m1 = 1 example; the Gram-consistent top-left entry is sqrt(2)."""
    a = as_matrix(a)
    b = as_matrix(b)
    if a.shape[0] == 0 or b.shape[0] == 0:
        raise ValueError("reduce_cartesian needs non-empty inputs")
    m1, n1 = a.shape
    m2, n2 = b.shape
    top = np.hstack([a * float(np.sqrt(m2)), np.repeat(head(b), m1, axis=0)])
    bottom = np.hstack([np.zeros((m2 - 1, n1)), tail(b) * float(np.sqrt(m1))])
    mat = np.vstack([top, bottom])
    return ReducedMatrix(mat, [(0, m1 + m2 - 1)], n1, n2)


def _check_sorted(keys: np.ndarray, side: str) -> None:
    if keys.size > 1 and np.any(keys[1:] < keys[:-1]):
        raise ValueError(f"{side} table keys are not sorted non-decreasing")


def group_keys(keys_a: np.ndarray, keys_b: np.ndarray):
    """Grouping of two sorted key columns, ascending matched keys.

    Returns int64 arrays (matched_keys, a_start, a_count, b_start, b_count, red_off)
    with red_off = [0, cumsum(a_count + b_count - 1)].  This is the
    bit-exact target of the GPU grouping kernels (SURVEY.md §8c fixture recipe).
    """
    ka = np.ascontiguousarray(keys_a, dtype=np.int64)
    kb = np.ascontiguousarray(keys_b, dtype=np.int64)
    _check_sorted(ka, "left")
    _check_sorted(kb, "right")
    ua, ia, ca = np.unique(ka, return_index=True, return_counts=True)
    ub, ib, cb = np.unique(kb, return_index=True, return_counts=True)
    keys, xa, xb = np.intersect1d(ua, ub, assume_unique=True, return_indices=True)
    a_start = ia[xa].astype(np.int64)
    a_count = ca[xa].astype(np.int64)
    b_start = ib[xb].astype(np.int64)
    b_count = cb[xb].astype(np.int64)
    red_off = np.concatenate([[0], np.cumsum(a_count + b_count - 1)]).astype(np.int64)
    return keys.astype(np.int64), a_start, a_count, b_start, b_count, red_off


def reduce_natural_join(a: Table, b: Table) -> ReducedMatrix:
    """Stack reduce_cartesian(A_v, B_v) over keys present on both sides, ascending
    key order; disjoint keys -> 0 x (n1+n2)."""
    if a.keys is None or b.keys is None:
        raise ValueError("reduce_natural_join needs keys on both tables")
    n1, n2 = a.data.shape[1], b.data.shape[1]
    keys, a_start, a_count, b_start, b_count, red_off = group_keys(a.keys, b.keys)
    blocks, bounds = [], []
    for g in range(keys.shape[0]):
        ag = a.data[a_start[g]:a_start[g] + a_count[g]]
        bg = b.data[b_start[g]:b_start[g] + b_count[g]]
        blocks.append(reduce_cartesian(ag, bg).matrix)
        bounds.append((int(red_off[g]), int(red_off[g + 1])))
    mat = np.vstack(blocks) if blocks else np.zeros((0, n1 + n2))
    return ReducedMatrix(mat, bounds, n1, n2)


def reduce_join(a: Table, b: Table) -> ReducedMatrix:
    """Dispatcher (exported at pkg/src/joinqr/__init__.py:38): keys on both sides ->
    natural join, on neither -> Cartesian product, mixed -> error."""
    if (a.keys is None) != (b.keys is None):
        raise ValueError("both tables must carry keys, or neither")
    if a.keys is None:
        return reduce_cartesian(a.data, b.data)
    return reduce_natural_join(a, b)
