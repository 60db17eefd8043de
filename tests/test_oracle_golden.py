"""Pin the CPU oracle against the SPEC's worked examples and the reference's matrix.py.

Golden file: tests/golden/spec_examples.json (tests/golden/make_golden.py).
Acceptance criteria: SPEC.md:551-561 (1-5, 8).
"""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
A = np.asarray


def close(x, y, tol=1e-12):
    x, y = A(x, dtype=float), A(y, dtype=float)
    assert x.shape == y.shape, (x.shape, y.shape)
    assert np.max(np.abs(x - y), initial=0.0) <= tol * max(1.0, np.max(np.abs(y), initial=0.0))


def test_head_tail_examples():
    for c in GOLD["head"]:
        close(O.head(c["in"]), c["out"])
        if "printed" in c:
            close(O.head(c["in"]), c["printed"], 1e-6)
    for c in GOLD["tail"]:
        if "out_shape" in c:
            assert O.tail(c["in"]).shape == tuple(c["out_shape"])
        else:
            close(O.tail(c["in"]), c["out"])
            close(O.tail(c["in"]), c["printed"], 1e-6)
    for c in GOLD["head_tail"]:
        close(O.head_tail(c["in"]), c["out"])
    with pytest.raises(ValueError):
        O.head(np.zeros((0, 3)))


def test_reduce_examples():
    for c in GOLD["reduce_cartesian"]:
        red = O.reduce_cartesian(c["a"], c["b"])
        close(red.matrix, c["out"])
        if "gram" in c:
            close(O.gram(red.matrix), c["gram"])
    for c in GOLD["reduce_natural_join"]:
        ta, tb = O.Table(c["a"], c["ka"]), O.Table(c["b"], c["kb"])
        red = O.reduce_natural_join(ta, tb)
        assert red.matrix.shape == (c["rows"], 2)
        if c["rows"]:
            j = O.materialize_natural_join(ta, tb)
            close(j, c["join"])
            close(O.gram(red.matrix), O.gram(j), 1e-12)


def test_qr_svd_examples():
    for c in GOLD["householder_r"]:
        close(O.canonicalize(O.householder_r(c["in"])), c["canonical"])
        close(O.canonicalize(O.givens_r(c["in"])), c["canonical"])
    for c in GOLD["canonicalize"]:
        close(O.canonicalize(c["in"]), c["out"])
    for c in GOLD["figaro_r"]:
        r = O.figaro_r(O.Table(c["a"]), O.Table(c["b"]))
        close(r, c["out"])
        close(r, c["printed"], 1e-6)
        assert O.is_upper_triangular(r)
    for c in GOLD["svd_of_r"]:
        res = O.svd_of_r(c["in"], True)
        close(res.values, c["values"])
        close(res.right_vectors, c["v"])
    for c in GOLD["figaro_svd"]:
        res = O.figaro_svd(O.Table(c["a"]), O.Table(c["b"]))
        close(res.values, c["values"])
        close(res.values, c["printed"], 1e-6)
    for c in GOLD["materialize_cartesian"]:
        close(O.materialize_cartesian(c["a"], c["b"]), c["out"])
    for c in GOLD["det_lu"]:
        assert abs(O.det_lu(c["in"]) - c["out"]) < 1e-12
    for c in GOLD["gen_keys"]:
        assert O.near_equal_keys(c["rows"], c["key_groups"]).tolist() == c["out"]


def test_reference_matrix_module_agrees():
    for c in GOLD["reference_matrix_py"]:
        m = A(c["matrix"], dtype=float)
        close(O.gram(m), c["gram"], 0)
        assert O.is_upper_triangular(m) == c["is_upper_triangular"]


def test_splitmix64_published_vector():
    # SplitMix64 reference output for seed 1234567 (the generator's published test vector).
    from oracle.datagen import _mix64, GAMMA
    with np.errstate(over="ignore"):
        x = _mix64(np.uint64(1234567) + np.arange(1, 6, dtype=np.uint64) * GAMMA)
    assert x.tolist() == [6457827717110365317, 3203168211198807973, 9817491932198370423,
                          4593380528125082431, 16408922859458223821]
    u = O.splitmix64_uniform(7, 0, 40000)
    assert np.all((u > 0) & (u < 1)) and abs(u.mean() - 0.5) < 0.02
    t1, t2 = O.gen_uniform(O.GenSpec(3, 2, 42)), O.gen_uniform(O.GenSpec(3, 2, 42))
    assert np.array_equal(t1.data, t2.data)


# ---- property invariants (acceptance 1-5) ----

def test_head_tail_gram_preservation_500():
    rng = np.random.default_rng(0)
    for _ in range(500):
        m = rng.standard_normal((rng.integers(1, 51), rng.integers(1, 9)))
        g = O.gram(m)
        assert O.max_abs_diff(O.gram(O.head_tail(m)), g) <= 1e-12 * max(1, np.abs(g).max())
    c = np.tile(rng.random(5), (7, 1))
    assert np.abs(O.tail(c)).max() <= 1e-14 * 10


def _instance(rng, keyed):
    n1, n2 = rng.integers(1, 6, size=2)
    if not keyed:
        m1, m2 = rng.integers(1, 13, size=2)
        return O.Table(rng.random((m1, n1))), O.Table(rng.random((m2, n2)))
    g = rng.integers(1, 6)
    ca, cb = rng.integers(0, 7, size=g), rng.integers(0, 7, size=g)
    if ca.sum() == 0:
        ca[0] = 1
    if cb.sum() == 0:
        cb[0] = 1
    ka = np.repeat(np.arange(g), ca)
    kb = np.repeat(np.arange(g), cb)
    return O.Table(rng.random((len(ka), n1)), ka), O.Table(rng.random((len(kb), n2)), kb)


def _join(a, b):
    return (O.materialize_cartesian(a.data, b.data) if a.keys is None
            else O.materialize_natural_join(a, b))


def test_claim1_gram_identity_500():
    rng = np.random.default_rng(1)
    for i in range(500):
        a, b = _instance(rng, keyed=bool(i % 2))
        j = _join(a, b)
        gj = O.gram(j)
        red = O.reduce_join(a, b).matrix
        assert O.max_abs_diff(O.gram(red), gj) <= 1e-10 * max(1, np.abs(gj).max())
        if a.keys is None:
            m1, n1 = a.data.shape
            assert red.shape[0] == m1 + b.data.shape[0] - 1
            assert np.all(red[m1:, :n1] == 0.0)                # SPEC.md:215 exact zeros


def test_oracle_equivalence_r_sigma_200():
    rng = np.random.default_rng(2)
    for i in range(200):
        a, b = _instance(rng, keyed=bool(i % 2))
        j = _join(a, b)
        r = O.figaro_r(a, b)
        rb = O.baseline_r(j)
        assert O.is_upper_triangular(r)
        gj = O.gram(j)
        assert O.max_abs_diff(O.gram(r), gj) <= 1e-10 * max(1, np.abs(gj).max())
        if j.shape[0] >= j.shape[1] and np.linalg.matrix_rank(j) == j.shape[1]:
            assert O.max_abs_diff(r, rb) <= 1e-8 * max(1, np.abs(r).max())
        s = O.svd_of_r(r, True)
        sb = O.baseline_svd(j)
        assert np.all(np.abs(s.values - sb.values) <= 1e-8 * max(1, sb.values[0]))
        v = s.right_vectors
        assert np.abs(v.T @ v - np.eye(v.shape[0])).max() <= 1e-10
        rec = v @ np.diag(s.values ** 2) @ v.T
        assert np.abs(r.T @ r - rec).max() <= 1e-8 * max(1, s.values[0] ** 2)


def test_determinant_and_lapack_agree():
    rng = np.random.default_rng(3)
    for i in range(50):
        # 2x2 |x| 2x2 has rank <= m1+m2-1 = 3 < 4, so det = 0; the
        # full-rank square joins are 1 x 1 |x| k x (k-1).
        a, b = O.Table(rng.random((2, 2))), O.Table(rng.random((2, 2)))
        assert abs(O.det_lu(O.materialize_cartesian(a.data, b.data))) < 1e-12
        assert abs(np.prod(np.diag(O.figaro_r(a, b)))) < 1e-12
        k = 3 + i % 4
        n1 = 1                      # n1 >= 2 would repeat one direction (rank-deficient)
        a, b = O.Table(rng.random((1, n1))), O.Table(rng.random((k, k - n1)))
        j = O.materialize_cartesian(a.data, b.data)
        r = O.figaro_r(a, b)
        d = abs(O.det_lu(j))
        assert abs(np.prod(np.diag(r)) - d) <= 1e-8 * d
        assert abs(np.prod(O.svd_of_r(r).values) - d) <= 1e-8 * d
        assert O.max_abs_diff(O.figaro_r(a, b, lapack=True), r) <= 1e-12


def test_grouping_fixture():
    ka = np.array([1, 1, 2, 4, 4, 4, 7])
    kb = np.array([0, 1, 2, 2, 4, 9])
    keys, a_s, a_c, b_s, b_c, off = O.group_keys(ka, kb)
    assert keys.tolist() == [1, 2, 4]
    assert a_s.tolist() == [0, 2, 3] and a_c.tolist() == [2, 1, 3]
    assert b_s.tolist() == [1, 2, 4] and b_c.tolist() == [1, 2, 1]
    assert off.tolist() == [0, 2, 4, 7]
    with pytest.raises(ValueError):
        O.group_keys(np.array([2, 1]), kb)


def test_factorised_gram_oracle():
    rng = np.random.default_rng(4)
    for keyed in (False, True):
        a, b = _instance(rng, keyed)
        j = _join(a, b)
        assert O.max_abs_diff(O.factorised_gram(a, b), O.gram(j)) <= 1e-10 * max(1, np.abs(O.gram(j)).max())
    a, b = O.config_tables(2, rows=20_000)
    g = O.factorised_gram(a, b)
    r = O.figaro_r(a, b, lapack=True)
    assert np.abs(O.gram_r(g) - r).max() <= 1e-10 * np.abs(r).max()


def test_c_gram_oracle_with_permuted_rows():
    """oracle/c gram with row permutations (the C3 recipe's stable key sort) equals
    the numpy factorised Gram of the permuted tables."""
    from oracle import cgram
    if not cgram.available():
        pytest.skip("oracle/c not built")
    t_a, pa = O.datagen.zipf_sorted_table(77, 78, 3000, 3, universe=50)
    t_b, pb = O.datagen.zipf_sorted_table(79, 80, 2000, 4, universe=50)
    assert np.array_equal(pa, np.argsort(O.zipf_keys(77, 3000, universe=50), kind="stable"))
    g = cgram.join_gram(78, 3000, 3, 80, 2000, 4, t_a.keys, t_b.keys, pa, pb)
    g_ref = O.factorised_gram(t_a, t_b)
    assert np.abs(g - g_ref).max() <= 1e-12 * np.abs(g_ref).max()


def test_c_gram_oracle_cartesian_matches_numpy():
    from oracle import cgram
    if not cgram.available():
        pytest.skip("oracle/c not built")
    g = cgram.join_gram(4001, 20000, 5, 4002, 15000, 6)
    a = O.Table(O.datagen.uniform_matrix(4001, 20000, 5))
    b = O.Table(O.datagen.uniform_matrix(4002, 15000, 6))
    g_ref = O.factorised_gram(a, b)
    assert np.abs(g - g_ref).max() <= 1e-12 * np.abs(g_ref).max()
