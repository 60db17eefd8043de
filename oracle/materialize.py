"""Brute-force ground truth, restated from SPEC.md:375-429.

Test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np

from .joins import Table, group_keys
from .matrix import as_matrix
from .qr import canonicalize, householder_r
from .svd import svd_of_r


def materialize_cartesian(a, b) -> np.ndarray:
    """Block i stacks [A_i | B_j] for j = 1..m2."""
    a, b = as_matrix(a), as_matrix(b)
    if a.shape[0] == 0 or b.shape[0] == 0:
        raise ValueError("materialize_cartesian needs non-empty inputs")
    m1, m2 = a.shape[0], b.shape[0]
    return np.hstack([np.repeat(a, m2, axis=0), np.tile(b, (m1, 1))])


def materialize_natural_join(a: Table, b: Table) -> np.ndarray:
    """Sort-merge join ordered by key, left row, right row."""
    if a.keys is None or b.keys is None:
        raise ValueError("materialize_natural_join needs keys on both tables")
    n = a.data.shape[1] + b.data.shape[1]
    keys, a_start, a_count, b_start, b_count, _ = group_keys(a.keys, b.keys)
    blocks = [materialize_cartesian(a.data[a_start[g]:a_start[g] + a_count[g]],
                                    b.data[b_start[g]:b_start[g] + b_count[g]])
              for g in range(keys.shape[0])]
    return np.vstack(blocks) if blocks else np.zeros((0, n))


def baseline_r(j) -> np.ndarray:
    """canonicalize(householder_r(J)) on the materialised join."""
    return canonicalize(householder_r(j))


def baseline_svd(j, want_vectors: bool = False):
    return svd_of_r(baseline_r(j), want_vectors)


def det_lu(j) -> float:
    """Determinant by partially pivoted elimination."""
    a = as_matrix(j).copy()
    n = a.shape[0]
    if a.shape[1] != n:
        raise ValueError("det_lu needs a square matrix")
    det = 1.0
    for k in range(n):
        p = k + int(np.argmax(np.abs(a[k:, k])))
        if a[p, k] == 0.0:
            return 0.0
        if p != k:
            a[[k, p]] = a[[p, k]]
            det = -det
        det *= a[k, k]
        a[k + 1:, k:] -= np.outer(a[k + 1:, k] / a[k, k], a[k, k:])
    return float(det)
