"""Wide tables (256 < n1 + n2 <= 512, "n <= a few
hundred"): head_tail, reduce_*, householder_r, figaro_r, svd_of_r and figaro_svd
against the oracle at n = 300 and 512 (the wide TSQR of jq_wide.cu, the 16-column-per
lane scan / emit kernels, the cooperative Jacobi kernel for n > 256)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2503_23385_b200 as P
    return P


def rel(x, y):
    return np.linalg.norm(np.asarray(x) - np.asarray(y)) / max(np.linalg.norm(np.asarray(y)), 1e-300)


def check_r(r, r_ref, tol=1e-10):
    r = np.asarray(r)
    assert np.all(np.tril(r, -1) == 0.0) and np.all(np.diag(r) >= 0)
    assert rel(np.abs(r), np.abs(r_ref)) <= tol
    assert rel(r.T @ r, r_ref.T @ r_ref) <= tol


@pytest.mark.parametrize("n", [300, 512])
def test_head_tail_wide(P, n):
    rng = np.random.default_rng(n)
    m = rng.random((3001, n))
    ht = np.asarray(P.head_tail(m))
    ref = O.head_tail(m)
    assert np.abs(ht - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("n1,n2", [(150, 150), (200, 312), (512, 0)])
def test_reduce_wide(P, n1, n2):
    rng = np.random.default_rng(n1 + n2)
    A, B = rng.random((700, n1)), rng.random((500, n2))
    red = np.asarray(P.reduce_cartesian(A, B).matrix)
    ref = O.reduce_cartesian(A, B).matrix
    assert red.shape == ref.shape and np.abs(red - ref).max() <= 1e-12 * np.abs(ref).max()
    ka, kb = np.sort(rng.integers(0, 30, 700)), np.sort(rng.integers(0, 30, 500))
    red = P.reduce_natural_join(P.Table(A, ka), P.Table(B, kb))
    ref = O.reduce_join(O.Table(A, ka), O.Table(B, kb))
    assert red.group_boundaries == ref.group_boundaries
    assert np.abs(np.asarray(red.matrix) - ref.matrix).max() <= 1e-12 * np.abs(ref.matrix).max()


@pytest.mark.parametrize("rows,n", [(5000, 300), (3000, 512), (400, 300), (100_000, 260)])
def test_householder_r_wide(P, rows, n):
    rng = np.random.default_rng(rows)
    m = rng.random((rows, n))
    r = np.asarray(P.canonicalize(P.householder_r(m)))
    check_r(r, O.canonicalize(O.householder_r_lapack(m)))


@pytest.mark.parametrize("n1,n2,keys", [(150, 150, False), (256, 256, False), (200, 112, True)])
def test_figaro_r_wide(P, n1, n2, keys):
    rng = np.random.default_rng(n1 * 3 + n2)
    m1, m2 = 2000, 1500
    ka = np.sort(rng.integers(0, 20, m1)) if keys else None
    kb = np.sort(rng.integers(0, 20, m2)) if keys else None
    a, b = O.Table(rng.random((m1, n1)), ka), O.Table(rng.random((m2, n2)), kb)
    r = np.asarray(P.figaro_r(P.Table(a.data, a.keys), P.Table(b.data, b.keys)))
    red = O.reduce_join(a, b).matrix
    check_r(r, O.canonicalize(O.householder_r_lapack(red)))


@pytest.mark.parametrize("n", [300, 512])
def test_svd_of_r_wide(P, n):
    rng = np.random.default_rng(n)
    r = np.triu(rng.random((n, n))) + np.eye(n) * 3.0
    s = P.svd_of_r(r, True)
    vals, v = np.asarray(s.values), np.asarray(s.right_vectors)
    ref = np.linalg.svd(r, compute_uv=False)
    assert np.max(np.abs(vals - ref)) <= 1e-10 * ref[0]
    assert np.abs(v.T @ v - np.eye(n)).max() <= 1e-10
    assert rel(v @ np.diag(vals ** 2) @ v.T, r.T @ r) <= 1e-10


def test_figaro_svd_wide(P):
    rng = np.random.default_rng(9)
    a, b = rng.random((1200, 160)), rng.random((900, 140))
    s = P.figaro_svd(P.Table(a), P.Table(b), want_vectors=True)
    red = O.reduce_cartesian(a, b).matrix
    ref = np.linalg.svd(red, compute_uv=False)
    assert np.max(np.abs(np.asarray(s.values) - ref)) <= 1e-10 * ref[0]


def test_wide_caps(P):
    with pytest.raises(ValueError):
        P.householder_r(np.ones((600, 513)))
    with pytest.raises(ValueError):
        P.svd_of_r(np.eye(513))
