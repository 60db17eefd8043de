"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): grouping bit-exact; |R| (row signs normalised)
and R^T R within 1e-10 relative Frobenius; singular values within 1e-10
relative.  Head/tail and the reduced matrix are checked entrywise at 1e-12
(their only difference from the oracle is the blocked vs sequential prefix sum).
"""
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def P():
    import paper_2503_23385_b200 as P
    return P


def rel_fro(x, y):
    x, y = np.asarray(x), np.asarray(y)
    return np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)


def check_r(r, r_ref, tol=1e-10):
    r, r_ref = np.asarray(r), np.asarray(r_ref)
    assert np.all(np.tril(r, -1) == 0.0), "R must have exact zeros below the diagonal"
    assert np.all(np.diag(r) >= 0), "R must be canonical"
    assert rel_fro(np.abs(r), np.abs(r_ref)) <= tol, rel_fro(np.abs(r), np.abs(r_ref))
    assert rel_fro(r.T @ r, r_ref.T @ r_ref) <= tol


def rand_tables(rng, m1, n1, m2, n2, groups=None):
    if groups is None:
        return O.Table(rng.random((m1, n1))), O.Table(rng.random((m2, n2)))
    ka = np.sort(rng.integers(0, groups, m1))
    kb = np.sort(rng.integers(0, groups, m2))
    return O.Table(rng.random((m1, n1)), ka), O.Table(rng.random((m2, n2)), kb)


def to_p(P, t):
    return P.Table(t.data, t.keys)


# ------------------------------------------------------------ SPEC golden examples
def test_spec_examples_on_gpu(P):
    for c in GOLD["head"]:
        assert np.allclose(P.head(c["in"]), c["out"], rtol=0, atol=1e-14)
    for c in GOLD["tail"]:
        t = P.tail(c["in"])
        if "out_shape" in c:
            assert t.shape == tuple(c["out_shape"])
        else:
            assert np.allclose(t, c["out"], rtol=0, atol=1e-14)
    for c in GOLD["reduce_cartesian"]:
        assert np.allclose(P.reduce_cartesian(c["a"], c["b"]).matrix, c["out"], rtol=0, atol=1e-14)
    for c in GOLD["reduce_natural_join"]:
        red = P.reduce_natural_join(P.Table(c["a"], c["ka"]), P.Table(c["b"], c["kb"]))
        assert red.matrix.shape == (c["rows"], 2)
    for c in GOLD["householder_r"]:
        assert np.allclose(P.canonicalize(P.householder_r(c["in"])), c["canonical"], atol=1e-14)
    for c in GOLD["canonicalize"]:
        assert np.array_equal(P.canonicalize(c["in"]), np.array(c["out"], dtype=float))
    for c in GOLD["figaro_r"]:
        r = P.figaro_r(P.Table(c["a"]), P.Table(c["b"]))
        assert np.allclose(r, c["out"], rtol=1e-14, atol=1e-14)
        assert P.is_upper_triangular(r)
    for c in GOLD["svd_of_r"]:
        s = P.svd_of_r(c["in"], True)
        assert np.allclose(s.values, c["values"], atol=1e-14)
        assert np.allclose(np.abs(s.right_vectors), np.abs(np.array(c["v"])), atol=1e-14)
    for c in GOLD["figaro_svd"]:
        s = P.figaro_svd(P.Table(c["a"]), P.Table(c["b"]))
        assert np.allclose(s.values, c["values"], rtol=1e-13)


# ------------------------------------------------------------ head / tail
@pytest.mark.parametrize("rows,cols", [(1, 3), (2, 1), (7, 5), (1023, 8), (1024, 8), (1025, 17),
                                       (5000, 64), (3000, 256)])
def test_head_tail(P, rows, cols):
    rng = np.random.default_rng(rows * 7 + cols)
    m = rng.standard_normal((rows, cols))
    got = P.head_tail(m)
    ref = O.head_tail(m)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1, np.abs(ref).max())
    g = O.gram(m)
    assert O.max_abs_diff(O.gram(got), g) <= 1e-12 * max(1, np.abs(g).max())


def test_head_tail_constant_rows(P):
    m = np.tile(np.array([0.3, -2.0, 5.5]), (3000, 1))
    assert np.abs(P.tail(m)).max() <= 1e-12


# ------------------------------------------------------------ grouping (bit-exact)
@pytest.mark.parametrize("m1,m2,universe", [(1, 1, 1), (10, 7, 5), (1000, 1500, 37), (200_000, 150_000, 50_000),
                                            (100_000, 100_000, 10)])
def test_group_keys_bit_exact(P, m1, m2, universe):
    rng = np.random.default_rng(m1 + m2)
    ka = np.sort(rng.integers(-universe, universe, m1))
    kb = np.sort(rng.integers(-universe, universe, m2))
    got = P.group_keys(ka, kb)
    ref = O.group_keys(ka, kb)
    for x, y in zip(got, ref):
        assert x.dtype == np.int64 and np.array_equal(x, y)


def test_group_keys_disjoint_and_extremes(P):
    got = P.group_keys(np.array([1, 1, 3]), np.array([2, 4]))
    assert len(got[0]) == 0 and got[5].tolist() == [0]
    big = np.array([np.iinfo(np.int64).min, -1, 0, np.iinfo(np.int64).max])
    for x, y in zip(P.group_keys(big, big), O.group_keys(big, big)):
        assert np.array_equal(x, y)


def test_unsorted_keys_raise(P):
    with pytest.raises(ValueError, match="sorted"):
        P.group_keys(np.array([2, 1]), np.array([1, 2]))
    with pytest.raises(ValueError, match="sorted"):
        P.figaro_r(P.Table(np.ones((2, 1)), [1, 1]), P.Table(np.ones((2, 1)), [3, 2]))


# ------------------------------------------------------------ reduce (SPEC order)
@pytest.mark.parametrize("case", ["cart_small", "cart_m1", "cart_m2", "cart_big", "nat", "nat_big"])
def test_reduce_matches_oracle(P, case):
    rng = np.random.default_rng(hash(case) % 2**32)
    shapes = {"cart_small": (5, 3, 7, 2, None), "cart_m1": (1, 2, 9, 3, None),
              "cart_m2": (6, 2, 1, 4, None), "cart_big": (3000, 8, 5000, 16, None),
              "nat": (60, 3, 80, 2, 9), "nat_big": (20000, 4, 30000, 5, 700)}
    m1, n1, m2, n2, groups = shapes[case]
    a, b = rand_tables(rng, m1, n1, m2, n2, groups)
    ref = O.reduce_join(a, b)
    got = P.reduce_join(to_p(P, a), to_p(P, b))
    assert got.matrix.shape == ref.matrix.shape
    assert np.max(np.abs(got.matrix - ref.matrix), initial=0) <= 1e-12 * max(1, np.abs(ref.matrix).max(initial=0))
    assert got.group_boundaries == ref.group_boundaries
    if groups is None:
        assert np.all(got.matrix[m1:, :n1] == 0.0)   # exact zeros


# ------------------------------------------------------------ householder_r / figaro_r
@pytest.mark.parametrize("rows,cols", [(1, 1), (3, 5), (7, 3), (64, 16), (1000, 31), (20000, 64),
                                       (5000, 100), (3000, 128), (2000, 200), (1500, 256)])
def test_householder_r(P, rows, cols):
    rng = np.random.default_rng(rows + 1000 * cols)
    m = rng.standard_normal((rows, cols))
    r = np.asarray(P.householder_r(m))
    assert P.is_upper_triangular(r)
    ref = O.householder_r_lapack(m)
    g = m.T @ m
    assert np.abs(r.T @ r - g).max() <= 1e-10 * max(1, np.abs(g).max())
    if rows >= cols:
        check_r(P.canonicalize(r), O.canonicalize(ref))


@pytest.fixture(params=["dense", "footnote"])
def variant(request, P):
    P.set_variant(request.param)
    yield request.param
    P.set_variant("auto")


@pytest.mark.parametrize("m1,n1,m2,n2,groups", [
    (2, 1, 2, 1, None), (1, 3, 1, 2, None), (1, 1, 9, 4, None), (7, 4, 1, 3, None),
    (1000, 4, 1000, 4, None), (3000, 8, 2000, 8, None), (4000, 32, 5000, 32, None),
    (2500, 64, 2500, 64, None), (3000, 100, 2000, 120, None), (5000, 128, 4000, 128, None),
    (400, 5, 300, 6, 40), (6000, 16, 7000, 16, 600), (20000, 32, 20000, 32, 100),
    (3000, 7, 2000, 3, 2500),
    # footnote: B's scan tiles on the spare warps of A's leaf (33..64 columns), a B side
    # with many more tiles than A has spare warps, keyed groups spanning tiles
    (2000, 50, 50000, 60, None), (3000, 40, 40000, 56, 30), (30000, 48, 25000, 40, 70),
    # footnote with few join groups: head rows absorbed by Givens rotations
    (5000, 20, 4000, 24, 3), (3000, 100, 3000, 120, 5),
    # Cartesian footnote, carry-free leaves: many between-block row elements (NP = 16,
    # sides with different leaf counts: separate trees), an odd leaf count (147 leaves,
    # three dense elements, both trees in shared launches), a partial last block
    (200000, 8, 150000, 12, None), (150001, 64, 150001, 64, None),
    # sides of different leaf widths (NP 64 ws2 leaves / NP 128 ws2 direct-load leaves)
    (200000, 40, 150000, 100, None),
    # keyed tile passes of <= 16 columns (several rows per warp load), groups spanning
    # 1024-row tiles, 1 / 3 / 8 / 9 / 16 columns
    (5000, 1, 4000, 3, 700), (6000, 8, 5000, 9, 40), (9000, 16, 7000, 1, 5),
    # N = 128 direct-load leaves on keyed joins: group starts inside chunks, rows
    # without a partner group
    (9000, 70, 8000, 58, 900), (20000, 128, 3000, 128, 17),
    # N = 128 leaves with fewer rows than one chunk / a leaf, and single rows
    (3, 100, 2, 120, None), (130, 64, 7, 64, None), (1, 128, 200, 128, None), (145, 65, 1, 63, 2)])
def test_figaro_r_matches_oracle(P, variant, m1, n1, m2, n2, groups):
    rng = np.random.default_rng(m1 + 3 * m2 + n1 + (groups or 0))
    a, b = rand_tables(rng, m1, n1, m2, n2, groups)
    r = np.asarray(P.figaro_r(to_p(P, a), to_p(P, b)))
    red = O.reduce_join(a, b).matrix
    if red.shape[0] >= red.shape[1] and np.linalg.matrix_rank(red) == red.shape[1]:
        check_r(r, O.canonicalize(O.householder_r_lapack(red)))
    g = O.gram(red)
    assert np.abs(r.T @ r - g).max() <= 1e-10 * max(1, np.abs(g).max())


@pytest.mark.parametrize("m,n", [(150001, 64), (70000, 128), (3000, 20)])
def test_carry_free_leaves_match_scan_carried(P, m, n):
    """The Cartesian footnote default (carry-free leaves + between-block rows) against
    the scan-carried leaves (JQ_FOOTNOTE_CARRY=scan, read once per process: run in a
    child process) on the same device-generated tables: same R to rounding."""
    import subprocess
    import sys
    code = ("import sys, numpy as np, torch; sys.path.insert(0, %r); import paper_2503_23385_b200 as P; "
            "from paper_2503_23385_b200 import datagen; P.set_variant('footnote'); "
            "A = torch.empty((%d, %d), dtype=torch.float64, device='cuda'); B = torch.empty_like(A); "
            "datagen.uniform(11, %d, %d, out=A); datagen.uniform(12, %d, %d, out=B); "
            "np.save(sys.argv[1], P.figaro_r(P.Table(A), P.Table(B)).cpu().numpy())"
            % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), m, n, m, n, m, n))
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        out = {}
        for mode in ("scan", "blocks"):
            f = os.path.join(d, mode + ".npy")
            env = dict(os.environ, JQ_FOOTNOTE_CARRY=mode)
            subprocess.run([sys.executable, "-c", code, f], env=env, check=True, timeout=300)
            out[mode] = np.load(f)
    check_r(out["blocks"], out["scan"], tol=1e-12)


def test_figaro_r_empty_join_and_materialised(P, variant):
    a = P.Table(np.ones((2, 2)), [1, 1])
    b = P.Table(np.ones((3, 1)), [2, 2, 2])
    assert np.array_equal(P.figaro_r(a, b), np.zeros((3, 3)))
    rng = np.random.default_rng(5)
    ta, tb = rand_tables(rng, 30, 2, 25, 3, 4)
    j = O.materialize_natural_join(ta, tb)
    check_r(P.figaro_r(to_p(P, ta), to_p(P, tb)), O.baseline_r(j))


# ------------------------------------------------------------ svd
@pytest.mark.parametrize("n", [1, 2, 3, 8, 33, 64, 128, 256])
def test_svd_of_r(P, n):
    rng = np.random.default_rng(n)
    r = np.triu(rng.standard_normal((n, n)))
    s = P.svd_of_r(r, True)
    ref = np.linalg.svd(r, compute_uv=False)
    assert np.max(np.abs(s.values - ref)) <= 1e-10 * ref[0]
    v = np.asarray(s.right_vectors)
    assert np.abs(v.T @ v - np.eye(n)).max() <= 1e-10
    rec = v @ np.diag(s.values ** 2) @ v.T
    assert np.abs(r.T @ r - rec).max() <= 1e-8 * max(1, s.values[0] ** 2)
    if n <= 64:
        so = O.svd_of_r(r)
        assert np.max(np.abs(s.values - so.values)) <= 1e-10 * so.values[0]


def test_svd_rank_deficient_and_zero(P):
    s = P.svd_of_r(np.zeros((4, 4)), True)
    assert np.array_equal(s.values, np.zeros(4)) and np.array_equal(s.right_vectors, np.eye(4))
    rng = np.random.default_rng(9)
    a, b = O.Table(rng.random((2, 3))), O.Table(rng.random((2, 3)))  # rank <= 3 < 6
    s = P.figaro_svd(to_p(P, a), to_p(P, b), True)
    ref = np.linalg.svd(O.materialize_cartesian(a.data, b.data), compute_uv=False)
    ref = np.concatenate([ref, np.zeros(6 - len(ref))])      # J is 4 x 6: two zero values
    assert np.max(np.abs(s.values - ref)) <= 1e-10 * ref[0]


@pytest.mark.parametrize("n", [40, 200, 256])
def test_svd_rank_deficient_cluster(P, n):
    # rank n/2: half the columns go numerically to zero and are never rotated again
    rng = np.random.default_rng(100 + n)
    m = rng.standard_normal((2 * n, n // 2)) @ rng.standard_normal((n // 2, n))
    r = np.linalg.qr(m, mode="r")
    s = P.svd_of_r(r, True)
    ref = np.linalg.svd(r, compute_uv=False)
    assert np.max(np.abs(s.values - ref)) <= 1e-10 * ref[0]
    v = np.asarray(s.right_vectors)
    assert np.abs(v.T @ v - np.eye(n)).max() <= 1e-10
    rec = v @ np.diag(s.values ** 2) @ v.T
    assert np.abs(r.T @ r - rec).max() <= 1e-8 * s.values[0] ** 2


@pytest.mark.parametrize("m,n,groups", [(1000, 4, None), (3000, 16, None), (5000, 64, None), (4000, 16, 300)])
def test_figaro_svd_matches_oracle(P, variant, m, n, groups):
    rng = np.random.default_rng(m + n)
    a, b = rand_tables(rng, m, n, m + 17, n, groups)
    s = P.figaro_svd(to_p(P, a), to_p(P, b), True)
    red = O.reduce_join(a, b).matrix
    ref = np.linalg.svd(red, compute_uv=False)
    assert np.max(np.abs(np.asarray(s.values) - ref)) <= 1e-10 * ref[0]


# ------------------------------------------------------------ generator (bit-exact)
def test_gen_uniform_bit_exact(P):
    t = P.gen_uniform(P.GenSpec(1000, 7, 1234567, key_groups=10))
    ot = O.gen_uniform(O.GenSpec(1000, 7, 1234567, key_groups=10))
    assert np.array_equal(np.asarray(t.data), ot.data)
    assert np.array_equal(np.asarray(t.keys), ot.keys)
    from paper_2503_23385_b200 import datagen
    blk = datagen.uniform(42, 33, 5, row0=1001)
    assert np.array_equal(blk, O.datagen.uniform_matrix(42, 33, 5, row0=1001))


def test_zipf_keys_bit_exact(P):
    from paper_2503_23385_b200 import datagen
    got = datagen.zipf_sorted_keys(3003, 200_000, 1.1, 50_000)
    ref = np.sort(O.zipf_keys(3003, 200_000, 1.1, 50_000), kind="stable")
    assert np.array_equal(got, ref)


# ------------------------------------------------------------ shard building blocks
@pytest.mark.parametrize("variant", ["dense", "footnote"])
def test_shard_r_and_stack_equal_single_device(P, variant):
    """Row-sharded Cartesian figaro_r == unsharded figaro_r."""
    from paper_2503_23385_b200 import _native as N
    rng = np.random.default_rng(11)
    m1, n1, m2, n2 = 5000, 6, 7000, 5
    A, B = rng.random((m1, n1)), rng.random((m2, n2))
    n = n1 + n2
    ref = np.asarray(P.figaro_r(P.Table(A), P.Table(B)))
    P.set_variant(variant)
    try:
        for parts in (1, 2, 3, 5):
            ab = np.linspace(0, m1, parts + 1).astype(int)
            bb = np.linspace(0, m2, parts + 1).astype(int)
            sa = np.stack([A[ab[p]:ab[p + 1]].sum(axis=0) for p in range(parts)])
            sb = np.stack([B[bb[p]:bb[p + 1]].sum(axis=0) for p in range(parts)])
            ta, tb = sa.sum(axis=0), sb.sum(axis=0)
            rs = np.zeros((parts, n, n))
            for p in range(parts):
                pa = np.ascontiguousarray(sa[:p].sum(axis=0)) if p else np.zeros(n1)
                pb = np.ascontiguousarray(sb[:p].sum(axis=0)) if p else np.zeros(n2)
                a_sh = np.ascontiguousarray(A[ab[p]:ab[p + 1]])
                b_sh = np.ascontiguousarray(B[bb[p]:bb[p + 1]])
                N.check(N.lib().jq_figaro_r_shard(N.ctx(), a_sh.ctypes.data, len(a_sh), n1, m1, int(ab[p]),
                                                  pa.ctypes.data, ta.ctypes.data, b_sh.ctypes.data, len(b_sh), n2,
                                                  m2, int(bb[p]), pb.ctypes.data, tb.ctypes.data, int(p == 0),
                                                  rs[p].ctypes.data))
            r = np.zeros((n, n))
            N.check(N.lib().jq_tsqr_stack(N.ctx(), rs.ctypes.data, parts, n, r.ctypes.data))
            check_r(r, ref, 1e-12)
    finally:
        P.set_variant("dense")


@pytest.mark.parametrize("m1,n1,m2,n2", [(5000, 6, 7000, 5), (300000, 64, 250000, 64), (40000, 128, 40000, 128)])
def test_shard_local_carry_free_equal_single_device(P, m1, n1, m2, n2):
    """Carry-free shards (jq_figaro_r_shard_local + between_shard_rows + the stack):
    the orchestration of sharded.figaro_r_sharded_local, ranks played in turn on one
    device, == unsharded figaro_r."""
    import torch
    from paper_2503_23385_b200 import sharded
    rng = np.random.default_rng(m1 + n1)
    A, B = rng.random((m1, n1)), rng.random((m2, n2))
    n = n1 + n2
    ref = np.asarray(P.figaro_r(P.Table(A), P.Table(B)))
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    for parts in (1, 2, 3, 8):
        rs, sums = [], []
        for p in range(parts):
            a0, a1 = sharded.shard_range(m1, parts, p)
            b0, b1 = sharded.shard_range(m2, parts, p)
            r, s = sharded._native_shard_local(dA[a0:a1].contiguous(), dB[b0:b1].contiguous(), m1, m2)
            rs.append(r)
            sums.append(s)
        sizes_a = [sharded.shard_range(m1, parts, p)[1] - sharded.shard_range(m1, parts, p)[0] for p in range(parts)]
        sizes_b = [sharded.shard_range(m2, parts, p)[1] - sharded.shard_range(m2, parts, p)[0] for p in range(parts)]
        extra = sharded._native_householder(
            sharded.between_shard_rows(torch.stack(sums), sizes_a, sizes_b, m1, m2, n1).contiguous())
        r = sharded._native_stack(torch.cat([torch.stack(rs), extra.reshape(1, n, n)]).contiguous())
        check_r(r.cpu().numpy(), ref, 1e-12)


def test_colsums(P):
    from paper_2503_23385_b200 import _native as N
    x = np.random.default_rng(1).random((10_000, 40))
    s = np.zeros(40)
    N.check(N.lib().jq_colsums(N.ctx(), x.ctypes.data, 10_000, 40, s.ctypes.data))
    assert np.allclose(s, x.sum(axis=0), rtol=1e-13)


def test_device_tensors_in_place(P):
    import torch
    rng = np.random.default_rng(3)
    A, B = rng.random((3000, 8)), rng.random((2000, 8))
    ta = P.Table(torch.from_numpy(A).cuda())
    tb = P.Table(torch.from_numpy(B).cuda())
    r = P.figaro_r(ta, tb)
    assert r.is_cuda
    check_r(r.cpu().numpy(), np.asarray(P.figaro_r(P.Table(A), P.Table(B))), 1e-14)


def test_determinism(P, variant):
    rng = np.random.default_rng(8)
    a, b = P.Table(rng.random((30000, 16))), P.Table(rng.random((30000, 16)))
    r1, r2 = P.figaro_r(a, b), P.figaro_r(a, b)
    assert np.array_equal(r1, r2)


@pytest.mark.parametrize("variant", ["dense", "footnote"])
def test_streamed_host_path_matches_device_path(P, variant):
    """>= 1 GiB of host input takes the pipelined H2D path (pieces of 512 MB on a copy
    stream overlapped with the per-piece scan + TSQR); same R as the device path."""
    import torch
    from paper_2503_23385_b200 import datagen
    m, n = 1_100_000, 64                       # 2 x 563 MB of host input, 2 pieces per table
    a = datagen.uniform(77, m, n)
    b = datagen.uniform(78, m + 3, n)
    P.set_variant(variant)
    try:
        r_host = np.asarray(P.figaro_r(P.Table(a), P.Table(b)))
        r_dev = P.figaro_r(P.Table(torch.from_numpy(a).cuda()), P.Table(torch.from_numpy(b).cuda())).cpu().numpy()
    finally:
        P.set_variant("dense")
    check_r(r_host, r_dev, 1e-12)


@pytest.mark.parametrize("variant", ["dense", "footnote"])
@pytest.mark.parametrize("pieces", [(1, 1), (2, 3), (3, 2), (4, 7), (5, 5), (7, 1)], ids=lambda p: f"{p[0]}x{p[1]}")
def test_streamed_host_path_piece_sweep(P, variant, pieces, monkeypatch):
    """The streamed host path (the one bench.py's e2e times) with 1-7 pieces per table,
    odd counts and unequal sides: JQ_STREAM_MIN_BYTES forces the path at small sizes,
    JQ_PIECE_BYTES sets 1024-row pieces.  R must match LAPACK on the reduced matrix and
    the device-resident path."""
    import torch
    n1, n2 = 12, 20
    pa, pb = pieces
    m1, m2 = 1024 * (pa - 1) + 517, 1024 * (pb - 1) + 1000    # last piece partial
    rng = np.random.default_rng(100 * pa + pb)
    A, B = rng.random((m1, n1)), rng.random((m2, n2))
    # pieces of exactly 1024 rows on both sides: piece_bytes / (8 * cols) rounded to 1024
    monkeypatch.setenv("JQ_STREAM_MIN_BYTES", "1")
    monkeypatch.setenv("JQ_PIECE_BYTES", str(8 * max(n1, n2) * 1024 + 8 * 1023))
    P.set_variant(variant)
    try:
        r_host = np.asarray(P.figaro_r(P.Table(A), P.Table(B)))
        monkeypatch.delenv("JQ_STREAM_MIN_BYTES")
        r_dev = P.figaro_r(P.Table(torch.from_numpy(A).cuda()), P.Table(torch.from_numpy(B).cuda())).cpu().numpy()
    finally:
        P.set_variant("dense")
    red = O.reduce_cartesian(A, B).matrix
    check_r(r_host, O.canonicalize(O.householder_r_lapack(red)))
    check_r(r_host, r_dev, 1e-12)


def test_async_torch_producer_is_ordered(P):
    """a tensor produced by a non_blocking H2D copy and a large torch
    kernel on torch's default stream, handed to the library with no sync in between,
    must be read after it lands (the library runs on cudaStreamLegacy, not its own
    non-blocking stream)."""
    import torch
    rng = np.random.default_rng(5)
    m, n = 2_000_000, 16
    ha = torch.from_numpy(rng.random((m, n))).pin_memory()
    hb = torch.from_numpy(rng.random((m, n))).pin_memory()
    ref = np.asarray(P.figaro_r(P.Table(ha.numpy()), P.Table(hb.numpy())))
    for _ in range(3):
        A = torch.empty((m, n), dtype=torch.float64, device="cuda")
        B = torch.empty((m, n), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        A.copy_(ha, non_blocking=True)
        B.copy_(hb, non_blocking=True)
        B.mul_(1.0).add_(0.0)                   # producer kernels queued behind the copies
        r = P.figaro_r(P.Table(A), P.Table(B)).cpu().numpy()
        check_r(r, ref, 1e-12)


@pytest.mark.gpu
def test_auto_variant_large_join_matches_oracle_gram(P):
    """Default variant ("auto") above its 1e8-element threshold takes the footnote
    path; R must still match the factorised Gram of the join."""
    import oracle as O
    rng = np.random.default_rng(7)
    m, n = 450_000, 120
    a, b = rng.random((m, n // 2)), rng.random((m, n // 2))
    P.set_variant("auto")
    r = np.asarray(P.figaro_r(P.Table(a), P.Table(b)))
    g = O.factorised_gram(O.Table(a), O.Table(b))
    err = np.linalg.norm(r.T @ r - g) / np.linalg.norm(g)
    assert err < 1e-10, err


@pytest.mark.gpu
@pytest.mark.parametrize("keys", [False, True], ids=["cartesian", "keyed"])
def test_figaro_r_mixed_gram_and_explicit_panels(P, variant, keys):
    """Near-duplicate columns make the Gram-panel guard reject the panels that hold
    them (explicit fallback, then a direct Gram for the next tile) while the other
    panels stay on the Gram path: R must still match LAPACK on the reduced matrix."""
    rng = np.random.default_rng(11 + keys)
    m, n = 60_000, 24
    A, B = rng.random((m, n)), rng.random((m, n))
    # kappa ~ 1e4 pairs: the guard rejects the panels holding them in every chunk
    # (residual |x'|^2 ~ 1e-8 of the column), yet R stays determined to ~1e-12
    A[:, 9] = A[:, 8] + 1e-4 * rng.standard_normal(m)     # panel 1 of the A side
    B[:, 17] = B[:, 16] + 1e-4 * rng.standard_normal(m)   # panel 2 of the B side
    ka = kb = None
    if keys:
        ka = np.sort(rng.integers(0, 50, m)); kb = np.sort(rng.integers(0, 50, m))
    a, b = O.Table(A, ka), O.Table(B, kb)
    r = np.asarray(P.figaro_r(to_p(P, a), to_p(P, b)))
    red = O.reduce_join(a, b).matrix
    check_r(r, O.canonicalize(O.householder_r_lapack(red)))
    g = O.gram(red)
    assert np.abs(r.T @ r - g).max() <= 1e-12 * np.abs(g).max()


@pytest.mark.parametrize("scale", [1e-150, 1e-60, 1e-8, 1e8, 1e60, 1e150])
def test_extreme_scales_fall_back_correctly(P, scale):
    """Data scaled so that the Cholesky panel's minors (~ S^8) leave the MUFU range or
    overflow: the guard must route those panels to the reflector chain / explicit path,
    and R must still match LAPACK relatively (SPEC.md:250-258 has no scale limit)."""
    rng = np.random.default_rng(int(abs(np.log10(scale))))
    m = rng.random((20_000, 24)) * scale
    r = np.asarray(P.canonicalize(P.householder_r(m)))
    r_ref = O.canonicalize(O.householder_r_lapack(m))
    assert np.all(np.isfinite(r))
    assert rel_fro(np.abs(r), np.abs(r_ref)) <= 1e-10
    a, b = rng.random((5000, 10)) * scale, rng.random((4000, 12)) * scale
    P.set_variant("footnote")
    try:
        rf = np.asarray(P.figaro_r(P.Table(a), P.Table(b)))
    finally:
        P.set_variant("dense")
    g = O.factorised_gram(O.Table(a), O.Table(b))
    rg = O.gram_r(g) if scale < 1e100 and scale > 1e-100 else None
    if rg is not None:
        assert rel_fro(np.abs(rf), np.abs(rg)) <= 1e-10
    else:  # the Gram itself over/underflows in float64: compare with LAPACK on the reduced matrix
        red = O.reduce_cartesian(a, b).matrix
        assert rel_fro(np.abs(rf), np.abs(O.canonicalize(O.householder_r_lapack(red)))) <= 1e-10
