"""Singular values / right vectors on the GPU.

One-sided Jacobi on R (jq_svd.cu): SPEC.md:356 stopping rule (1e-14, 64 sweeps,
RuntimeError after that), values descending, optional V (n x n).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

from . import _native as N
from ._arrays import like
from .matrix import as_matrix
from .qr import _tables


@dataclass
class SvdResult:
    """Descending non-negative values, optional V."""

    values: object
    right_vectors: Optional[object] = None


def svd_of_r(r, want_vectors: bool = False) -> SvdResult:
    r = as_matrix(r)
    if r.shape[0] != r.shape[1]:
        raise ValueError(f"svd_of_r needs a square upper-triangular R, got {r.shape[0]}x{r.shape[1]}")
    n = r.shape[1]
    if n > 512:
        raise ValueError(f"svd_of_r supports n <= 512 (got {n})")
    vals = like((n,), r)
    v = like((n, n), r) if want_vectors else None
    N.use_torch_stream(r)
    N.check(N.lib().jq_svd_of_r(N.ctx(), N.ptr(r), n, int(bool(want_vectors)), N.ptr(vals), N.ptr(v)))
    return SvdResult(vals, v)


def figaro_svd(a, b, want_vectors: bool = False, sort: bool = False) -> SvdResult:
    """figaro_r followed by svd_of_r, in one device pipeline;
    ``sort`` as in figaro_r."""
    a, b = _tables(a, b, sort)
    m1, n1 = a.data.shape
    m2, n2 = b.data.shape
    n = n1 + n2
    vals = like((n,), a.data, b.data)
    v = like((n, n), a.data, b.data) if want_vectors else None
    N.use_torch_stream(a.data, b.data, a.keys, b.keys)
    N.check(N.lib().jq_figaro_svd(N.ctx(), N.ptr(a.data), m1, n1, N.ptr(a.keys), N.ptr(b.data), m2,
                                  n2, N.ptr(b.keys), int(bool(want_vectors)), N.ptr(vals), N.ptr(v),
                                  None))
    return SvdResult(vals, v)
