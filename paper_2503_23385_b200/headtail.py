"""QR head / tail operators on the GPU.

`head_tail` is one device pass (jq_head_tail -> segmented prefix scan +
emit kernels, jq_headtail.cu); `head` / `tail` are its first row / the rest,
exactly as SPEC.md:135-141 defines them.  rows = 0 raises ValueError
(SPEC.md:119, :129); a single row has an empty 0 x n tail.
"""

from __future__ import annotations

from . import _native as N
from ._arrays import like
from .matrix import as_matrix


def head_tail(m):
    m = as_matrix(m)
    rows, cols = m.shape
    if rows == 0:
        raise ValueError("head/tail undefined for a matrix with 0 rows")
    out = like((rows, cols), m)
    N.use_torch_stream(m)
    N.check(N.lib().jq_head_tail(N.ctx(), N.ptr(m), rows, cols, N.ptr(out)))
    return out


def head(m):
    return head_tail(m)[:1]


def tail(m):
    return head_tail(m)[1:]
