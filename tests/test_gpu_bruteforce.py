"""Brute-force names of the reference's oracle module on the GPU:
the join matrix (bit-exact: it is a copy), baseline_r / baseline_svd, and the
streamed brute-force R against figaro_r and the CPU oracle."""

import numpy as np
import pytest

import oracle as O
from test_gpu_parity import check_r, rand_tables, to_p

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2503_23385_b200 as P
    return P


def test_spec_examples(P):
    # SPEC.md:382-384, :397-399
    assert np.array_equal(P.materialize_cartesian([[1.0, 2.0]], [[3.0], [4.0]]), [[1, 2, 3], [1, 2, 4]])
    j = P.materialize_cartesian([[1.0], [2.0]], [[3.0], [4.0]])
    assert np.array_equal(j, [[1, 3], [1, 4], [2, 3], [2, 4]])
    assert np.abs(P.baseline_r(j) - [[3.162278, 6.640783], [0, 2.428992]]).max() < 1e-6
    s = P.baseline_svd(j)
    assert np.abs(np.asarray(s.values) - [np.sqrt(59.0), 1.0]).max() < 1e-12
    assert np.array_equal(P.baseline_r(np.eye(5)), np.eye(5))
    # keys [1,1,2] / [1,2,2] -> (1,3), (2,3), (5,7), (5,8)
    a = P.Table(np.array([[1.0], [2.0], [5.0]]), [1, 1, 2])
    b = P.Table(np.array([[3.0], [7.0], [8.0]]), [1, 2, 2])
    assert np.array_equal(P.materialize_natural_join(a, b), [[1, 3], [2, 3], [5, 7], [5, 8]])
    # disjoint keys -> 0 x (n1+n2)
    e = P.materialize_natural_join(P.Table(np.ones((2, 2)), [1, 2]), P.Table(np.ones((3, 1)), [3, 4, 5]))
    assert e.shape == (0, 3)
    with pytest.raises(ValueError):
        P.materialize_cartesian(np.zeros((0, 2)), np.ones((2, 2)))
    with pytest.raises(ValueError):
        P.materialize_natural_join(P.Table(np.ones((2, 1))), P.Table(np.ones((2, 1))))


@pytest.mark.parametrize("m1,n1,m2,n2,groups", [(37, 3, 53, 4, None), (300, 5, 200, 6, 20), (800, 9, 700, 7, 3)])
def test_materialize_matches_oracle_bit_exact(P, m1, n1, m2, n2, groups):
    rng = np.random.default_rng(m1 * m2 + n1)
    a, b = rand_tables(rng, m1, n1, m2, n2, groups)
    if groups is None:
        got, ref = P.materialize_cartesian(a.data, b.data), O.materialize_cartesian(a.data, b.data)
    else:
        got, ref = P.materialize_natural_join(to_p(P, a), to_p(P, b)), O.materialize_natural_join(a, b)
    assert got.shape == ref.shape and np.array_equal(got, ref)


def test_materialize_device_tensors(P):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    a, b = rng.random((40, 3)), rng.random((50, 2))
    got = P.materialize_cartesian(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    assert got.is_cuda and np.array_equal(got.cpu().numpy(), O.materialize_cartesian(a, b))


@pytest.mark.parametrize("m1,n1,m2,n2,groups", [(60, 3, 70, 4, None), (400, 8, 300, 8, None),
                                                (1000, 12, 900, 20, 30), (500, 30, 400, 34, 5),
                                                (200, 64, 300, 64, None)])
def test_join_r_bruteforce_matches_oracle_and_figaro(P, m1, n1, m2, n2, groups):
    rng = np.random.default_rng(m1 + m2 + n1 + n2)
    a, b = rand_tables(rng, m1, n1, m2, n2, groups)
    r = np.asarray(P.join_r_bruteforce(to_p(P, a), to_p(P, b)))
    j = O.materialize_cartesian(a.data, b.data) if groups is None else O.materialize_natural_join(a, b)
    if j.shape[0] >= j.shape[1] and np.linalg.matrix_rank(j) == j.shape[1]:
        check_r(r, O.baseline_r(j))
    g = j.T @ j
    assert np.abs(r.T @ r - g).max() <= 1e-10 * max(1.0, np.abs(g).max())
    rf = np.asarray(P.figaro_r(to_p(P, a), to_p(P, b)))
    assert np.abs(rf.T @ rf - r.T @ r).max() <= 1e-10 * max(1.0, np.abs(g).max())
    # baseline_r of the materialised join: the same canonical R
    rb = np.asarray(P.baseline_r(j))
    assert np.abs(rb.T @ rb - g).max() <= 1e-10 * max(1.0, np.abs(g).max())
