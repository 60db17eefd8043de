"""QR finishing step, restated from SPEC.md:242-312.

``householder_r`` follows the LAPACK dlarfg/dgeqr2 reflector convention
(beta = -sign(alpha) * ||x||, tau = (beta - alpha) / beta, v = [1; x2 / (alpha - beta)])
in a column loop; ``householder_r_lapack`` is the same algorithm through numpy's
LAPACK (dgeqrf) for sizes where the Python loop is too slow (CPU baseline).
Test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np

from .joins import reduce_join
from .matrix import as_matrix


def _pad(m: np.ndarray) -> np.ndarray:
    rows, cols = m.shape
    if cols == 0:
        raise ValueError("householder_r needs at least one column")
    if rows < cols:
        m = np.vstack([m, np.zeros((cols - rows, cols))])
    return m


def householder_r(m) -> np.ndarray:
    """N x N upper-triangular R with R^T R = M^T M, not sign-canonical."""
    a = _pad(as_matrix(m)).copy()
    rows, n = a.shape
    for j in range(n):
        alpha = a[j, j]
        x2 = a[j + 1:, j]
        s = float(x2 @ x2)
        if s == 0.0:
            continue                                   # tau = 0: H = I
        beta = -np.copysign(np.sqrt(alpha * alpha + s), alpha)
        tau = (beta - alpha) / beta
        v = x2 / (alpha - beta)
        a[j, j] = beta
        a[j + 1:, j] = 0.0
        if j + 1 < n:
            w = a[j, j + 1:] + v @ a[j + 1:, j + 1:]
            a[j, j + 1:] -= tau * w
            a[j + 1:, j + 1:] -= tau * np.outer(v, w)
    return np.triu(a[:n])


def householder_r_lapack(m) -> np.ndarray:
    """Same contract via numpy.linalg.qr (LAPACK dgeqrf, Householder)."""
    a = _pad(as_matrix(m))
    return np.triu(np.linalg.qr(a, mode="r")[: a.shape[1]])


def givens_r(m) -> np.ndarray:
    """Independent Givens reference with the householder_r contract."""
    a = _pad(as_matrix(m)).copy()
    rows, n = a.shape
    for j in range(n):
        for i in range(rows - 1, j, -1):
            x, y = a[i - 1, j], a[i, j]
            if y == 0.0:
                continue
            r = np.hypot(x, y)
            c, s = x / r, y / r
            top, bot = a[i - 1, j:].copy(), a[i, j:].copy()
            a[i - 1, j:] = c * top + s * bot
            a[i, j:] = -s * top + c * bot
            a[i, j] = 0.0
    return np.triu(a[:n])


def canonicalize(r) -> np.ndarray:
    """Negate every row whose diagonal entry is negative."""
    r = as_matrix(r).copy()
    neg = np.diag(r) < 0
    r[neg] *= -1.0
    return r


def figaro_r(a, b, lapack: bool = False) -> np.ndarray:
    """reduce -> householder_r -> canonicalize."""
    red = reduce_join(a, b).matrix
    qr = householder_r_lapack if lapack else householder_r
    return canonicalize(qr(red))
