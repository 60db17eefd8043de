"""Matrix-core helpers, restated from /root/reference/pkg/src/joinqr/matrix.py.

Test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np


def as_matrix(values) -> np.ndarray:
    """C-contiguous 2-D float64; a 1-D input becomes a single row.

    Follows matrix.py:13-22 (`as_matrix`): 1-D of length n -> 1 x n, 1-D of
    length 0 -> 0 x 0, anything not 2-D afterwards -> ValueError.
    """
    a = np.ascontiguousarray(values, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape((1, a.shape[0]) if a.shape[0] else (0, 0))
    if a.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={a.ndim}")
    return a


def gram(a: np.ndarray) -> np.ndarray:
    """A^T A made symmetric to the bit from its upper triangle (matrix.py:31-34)."""
    g = a.T @ a
    up = np.triu(g)
    return up + np.triu(g, 1).T


def max_abs_diff(a: np.ndarray, b: np.ndarray) -> float:
    """Max |a_ij - b_ij| (matrix.py:37-42); 0.0 for empty, ValueError on shape mismatch."""
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    return float(np.max(np.abs(a - b))) if a.size else 0.0


def frobenius_norm(a: np.ndarray) -> float:
    """sqrt(sum a_ij^2) (matrix.py:49-50)."""
    return float(np.sqrt(np.sum(a * a)))


def is_upper_triangular(r: np.ndarray) -> bool:
    """Square with EXACT zeros strictly below the diagonal (matrix.py:73-75)."""
    return r.ndim == 2 and r.shape[0] == r.shape[1] and not np.any(np.tril(r, -1))
