"""QR finishing step on the GPU.

`householder_r` — streaming Householder TSQR on the FP64 tensor pipe (DMMA),
`canonicalize` — row-sign normalisation, `figaro_r` — grouping, head/tail scan
and the fused Claim-1 assembly + TSQR (jq_tsqr.cu), canonical R out.  The
reduced matrix is never materialised on this path.
"""

from __future__ import annotations

from . import _native as N
from ._arrays import like
from .joins import Table
from .matrix import as_matrix


def householder_r(m):
    """N x N upper-triangular R with R^T R = M^T M, not sign-canonical."""
    m = as_matrix(m)
    rows, cols = m.shape
    if cols == 0:
        raise ValueError("householder_r needs at least one column")
    out = like((cols, cols), m)
    N.use_torch_stream(m)
    N.check(N.lib().jq_householder_r(N.ctx(), N.ptr(m), rows, cols, N.ptr(out)))
    return out


def canonicalize(r):
    """Negate each row whose diagonal entry is negative."""
    r = as_matrix(r)
    n = r.shape[0]
    if r.shape[0] != r.shape[1]:
        raise ValueError("canonicalize needs a square matrix")
    out = like((n, n), r)
    N.use_torch_stream(r)
    N.check(N.lib().jq_canonicalize(N.ctx(), N.ptr(r), n, N.ptr(out)))
    return out


def _tables(a: Table, b: Table, sort: bool = False):
    if not isinstance(a, Table):
        a = Table(a)
    if not isinstance(b, Table):
        b = Table(b)
    if (a.keys is None) != (b.keys is None):
        raise ValueError("both tables must carry keys, or neither")
    if sort and a.keys is not None:
        from .joins import sort_by_key
        a, b = sort_by_key(a), sort_by_key(b)
    return a, b


def figaro_r(a: Table, b: Table, sort: bool = False):
    """Canonical R of the join matrix, join never materialised.
    ``sort=True`` (opt-in) sorts unsorted keyed tables on the GPU first (sort_by_key);
    by default unsorted keys raise ValueError as in the reference."""
    a, b = _tables(a, b, sort)
    m1, n1 = a.data.shape
    m2, n2 = b.data.shape
    out = like((n1 + n2, n1 + n2), a.data, b.data)
    N.use_torch_stream(a.data, b.data, a.keys, b.keys)
    N.check(N.lib().jq_figaro_r(N.ctx(), N.ptr(a.data), m1, n1, N.ptr(a.keys),
                                N.ptr(b.data), m2, n2, N.ptr(b.keys), N.ptr(out)))
    return out
