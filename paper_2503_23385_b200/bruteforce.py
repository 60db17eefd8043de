"""Brute-force oracle names of the reference on the GPU.

`materialize_cartesian` / `materialize_natural_join` write the join matrix
itself (rows ordered by key, then left row, then right row).  `baseline_r` /
`baseline_svd` decompose a given matrix directly, with the same TSQR and Jacobi
kernels figaro_r uses.  `join_r_bruteforce` is baseline_r of the join without
materialising it: the TSQR data warps generate the join rows from A and B
(jq_join.cu).  That is the performance foil of figaro_r, in the role the paper
gives cuSOLVER.  The CPU checker of all of these lives in
oracle/.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from ._arrays import like
from .joins import Table
from .matrix import as_matrix
from .qr import _tables, canonicalize, householder_r
from .svd import SvdResult, svd_of_r


def _materialize(a, ka, b, kb):
    m1, n1 = a.shape
    m2, n2 = b.shape
    rows = np.zeros(1, dtype=np.int64)
    N.use_torch_stream(a, b, ka, kb)
    if ka is None:
        total = m1 * m2
    else:
        N.check(N.lib().jq_materialize(N.ctx(), N.ptr(a), m1, n1, N.ptr(ka), N.ptr(b), m2, n2, N.ptr(kb),
                                       None, 0, rows.ctypes.data))
        total = int(rows[0])
    out = like((total, n1 + n2), a, b)
    if total:
        N.check(N.lib().jq_materialize(N.ctx(), N.ptr(a), m1, n1, N.ptr(ka), N.ptr(b), m2, n2, N.ptr(kb),
                                       N.ptr(out), total, rows.ctypes.data))
    return out


def materialize_cartesian(a, b):
    """m1*m2 x (n1+n2): block i stacks [A_i | B_j] for j = 1..m2."""
    a, b = as_matrix(a), as_matrix(b)
    if a.shape[0] == 0 or b.shape[0] == 0:
        raise ValueError("materialize_cartesian needs non-empty inputs")
    return _materialize(a, None, b, None)


def materialize_natural_join(a: Table, b: Table):
    """One row [A-data | B-data] per matching key pair, ordered by key, then left row,
    then right row.  Missing / unsorted keys -> ValueError."""
    if a.keys is None or b.keys is None:
        raise ValueError("materialize_natural_join needs keys on both tables")
    return _materialize(a.data, a.keys, b.data, b.keys)


def baseline_r(j):
    """Canonical R of the matrix j by direct decomposition."""
    return canonicalize(householder_r(as_matrix(j)))


def baseline_svd(j, want_vectors: bool = False) -> SvdResult:
    """svd_of_r(baseline_r(j))."""
    return svd_of_r(baseline_r(j), want_vectors)


def join_r_bruteforce(a: Table, b: Table):
    """baseline_r of the join matrix of a and b, its rows generated inside the TSQR
    (never materialised): the full O(|J| (n1+n2)^2) cost, no Figaro reduction."""
    a, b = _tables(a, b)
    m1, n1 = a.data.shape
    m2, n2 = b.data.shape
    out = like((n1 + n2, n1 + n2), a.data, b.data)
    N.use_torch_stream(a.data, b.data, a.keys, b.keys)
    N.check(N.lib().jq_join_r_bruteforce(N.ctx(), N.ptr(a.data), m1, n1, N.ptr(a.keys),
                                         N.ptr(b.data), m2, n2, N.ptr(b.keys), N.ptr(out)))
    return out
