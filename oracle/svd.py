"""Singular values / right vectors of R, restated from SPEC.md:316-371.

One-sided Jacobi on the columns of R, cyclic-by-rows pair order, converged
when every |a_p . a_q| / sqrt(|a_p|^2 |a_q|^2) < 1e-14, hard cap of 64 sweeps
then an error.  Test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .matrix import as_matrix
from .qr import figaro_r

TOL = 1e-14
MAX_SWEEPS = 64


@dataclass
class SvdResult:
    """Descending non-negative values, optional n x n V."""

    values: np.ndarray
    right_vectors: Optional[np.ndarray] = None


def rotation(alpha: float, beta: float, gamma: float):
    """(c, s) so that [a_p, a_q] <- [c a_p - s a_q, s a_p + c a_q] makes them orthogonal."""
    zeta = (beta - alpha) / (2.0 * gamma)
    t = 1.0 / (zeta + np.sqrt(1.0 + zeta * zeta)) if zeta >= 0 else \
        -1.0 / (-zeta + np.sqrt(1.0 + zeta * zeta))
    c = 1.0 / np.sqrt(1.0 + t * t)
    return c, c * t


def svd_of_r(r, want_vectors: bool = False, tol: float = TOL,
             max_sweeps: int = MAX_SWEEPS) -> SvdResult:
    a = as_matrix(r).copy()
    n = a.shape[1]
    v = np.eye(n)
    # Negligible-column guard (refines SPEC.md:356, whose ratio is 0/0 for a null
    # column): a column with |a|^2 <= (n eps |R|_F)^2 is numerically zero and is
    # never rotated; without it rank-deficient R (e.g. m1+m2-1 < n1+n2) never
    # meets the 1e-14 bar because two noise columns stay parallel.
    tiny = (n * np.finfo(np.float64).eps) ** 2 * float(np.sum(a * a))
    for _ in range(max_sweeps):
        rotated = False
        for p in range(n - 1):
            for q in range(p + 1, n):
                ap, aq = a[:, p], a[:, q]
                alpha, beta, gamma = float(ap @ ap), float(aq @ aq), float(ap @ aq)
                if alpha <= tiny or beta <= tiny:
                    continue
                if gamma == 0.0 or abs(gamma) < tol * (np.sqrt(alpha) * np.sqrt(beta)):
                    continue
                rotated = True
                c, s = rotation(alpha, beta, gamma)
                a[:, p], a[:, q] = c * ap - s * aq, s * ap + c * aq
                vp, vq = v[:, p].copy(), v[:, q].copy()
                v[:, p], v[:, q] = c * vp - s * vq, s * vp + c * vq
        if not rotated:
            break
    else:
        raise RuntimeError(f"Jacobi SVD did not converge in {max_sweeps} sweeps")
    sigma = np.sqrt(np.sum(a * a, axis=0))
    order = np.argsort(-sigma, kind="stable")
    return SvdResult(sigma[order], v[:, order] if want_vectors else None)


def figaro_svd(a, b, want_vectors: bool = False, lapack: bool = False) -> SvdResult:
    """figaro_r -> svd_of_r."""
    return svd_of_r(figaro_r(a, b, lapack=lapack), want_vectors)
