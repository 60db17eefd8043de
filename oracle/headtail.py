"""QR head / tail operators, restated from SPEC.md:107-165.

Prefix sums are accumulated sequentially in row order, in plain double
 — ``np.cumsum`` along axis 0 is a sequential accumulate.
Test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np

from .matrix import as_matrix


def _check(m: np.ndarray) -> np.ndarray:
    m = as_matrix(m)
    if m.shape[0] == 0:
        raise ValueError("head/tail undefined for a matrix with 0 rows")
    return m


def head(m) -> np.ndarray:
    """(1/sqrt(rows)) * sum_i M[i,:] as a 1 x n matrix."""
    m = _check(m)
    s = np.cumsum(m, axis=0)[-1]
    return (s / np.sqrt(m.shape[0]))[None, :]


def tail(m) -> np.ndarray:
    """Rows r = 0..m-2 with i = r+1: (sqrt(i) M[i] - S_i / sqrt(i)) / sqrt(i+1),
    S_i = sum_{k<i} M[k] (empty 0 x n for one row)."""
    m = _check(m)
    rows = m.shape[0]
    if rows == 1:
        return np.zeros((0, m.shape[1]))
    s_excl = np.cumsum(m, axis=0)[:-1]                 # S_1 .. S_{m-1}
    i = np.arange(1, rows, dtype=np.float64)[:, None]
    si = np.sqrt(i)
    return (si * m[1:] - s_excl / si) / np.sqrt(i + 1.0)


def head_tail(m) -> np.ndarray:
    """Row 0 = head, rows 1.. = tail, sharing one prefix-sum pass."""
    m = _check(m)
    return np.vstack([head(m), tail(m)])
