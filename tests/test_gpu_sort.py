"""GPU stable LSD radix sort of join keys (jq_sort.cu) against np.argsort(kind="stable"),
bit-exact, and the opt-in sorted path of figaro_r / reduce_natural_join (SPEC.md:202-207:
the reference raises on unsorted keys; sort=True sorts on the GPU first)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
I64 = np.iinfo(np.int64)


@pytest.fixture(scope="module")
def P():
    import paper_2503_23385_b200 as P
    return P


def ref_sort(k):
    perm = np.argsort(k, kind="stable")
    return k[perm], perm


@pytest.mark.parametrize("m", [1, 2, 31, 4095, 4096, 4097, 100_003, 1_000_000])
def test_radix_sort_random_full_range(P, m):
    rng = np.random.default_rng(m)
    k = rng.integers(I64.min, I64.max, m, dtype=np.int64, endpoint=True)
    k[: m // 3] = k[m // 3: 2 * (m // 3)]                # duplicates (stability matters)
    sk, perm = P.argsort_keys(k)
    rk, rp = ref_sort(k)
    assert np.array_equal(perm, rp) and np.array_equal(sk, rk)


@pytest.mark.parametrize("case", ["equal", "two_values", "extremes", "sorted", "reversed", "small_range",
                                  "negative"])
def test_radix_sort_edge_cases(P, case):
    rng = np.random.default_rng(1)
    m = 50_000
    k = {"equal": np.full(m, 7, np.int64),
         "two_values": rng.integers(0, 2, m).astype(np.int64) * (1 << 40),
         "extremes": rng.choice(np.array([I64.min, -1, 0, 1, I64.max], np.int64), m),
         "sorted": np.sort(rng.integers(-1000, 1000, m)).astype(np.int64),
         "reversed": np.sort(rng.integers(-1000, 1000, m))[::-1].astype(np.int64).copy(),
         "small_range": rng.integers(0, 300, m).astype(np.int64),
         "negative": -rng.integers(0, 1 << 20, m).astype(np.int64)}[case]
    sk, perm = P.argsort_keys(k)
    rk, rp = ref_sort(k)
    assert np.array_equal(perm, rp) and np.array_equal(sk, rk)


def test_radix_sort_empty(P):
    sk, perm = P.argsort_keys(np.zeros(0, np.int64))
    assert len(sk) == 0 and len(perm) == 0


def test_radix_sort_torch_device(P):
    import torch
    rng = np.random.default_rng(3)
    k = rng.integers(-(1 << 30), 1 << 30, 300_000).astype(np.int64)
    sk, perm = P.argsort_keys(torch.from_numpy(k).cuda())
    assert sk.is_cuda and perm.is_cuda
    rk, rp = ref_sort(k)
    assert np.array_equal(perm.cpu().numpy(), rp) and np.array_equal(sk.cpu().numpy(), rk)


def test_gather_rows_rejects_bad_permutation(P):
    x = np.ones((100, 4))
    with pytest.raises(ValueError, match="out of range"):
        P.gather_rows(x, np.r_[np.arange(99), 100].astype(np.int64))
    with pytest.raises(ValueError, match="out of range"):
        P.gather_rows(x, np.r_[-1, np.arange(1, 100)].astype(np.int64))


@pytest.mark.parametrize("cols", [1, 3, 16, 33])
def test_gather_rows_bit_exact(P, cols):
    rng = np.random.default_rng(cols)
    x = rng.random((20_001, cols))
    perm = rng.permutation(20_001).astype(np.int64)
    assert np.array_equal(np.asarray(P.gather_rows(x, perm)), x[perm])


def test_unsorted_keys_raise_by_default_and_sort_opt_in(P):
    rng = np.random.default_rng(4)
    ka, kb = rng.integers(0, 40, 3000), rng.integers(0, 40, 2500)
    A, B = rng.random((3000, 5)), rng.random((2500, 6))
    with pytest.raises(ValueError):
        P.figaro_r(P.Table(A, ka), P.Table(B, kb))
    r = np.asarray(P.figaro_r(P.Table(A, ka), P.Table(B, kb), sort=True))
    pa, pb = np.argsort(ka, kind="stable"), np.argsort(kb, kind="stable")
    a_s, b_s = O.Table(A[pa], ka[pa]), O.Table(B[pb], kb[pb])
    r_ref = O.figaro_r(a_s, b_s, lapack=True)
    assert np.linalg.norm(np.abs(r) - np.abs(r_ref)) <= 1e-10 * np.linalg.norm(r_ref)
    red = P.reduce_natural_join(P.Table(A, ka), P.Table(B, kb), sort=True)
    red_ref = O.reduce_join(a_s, b_s)
    assert red.group_boundaries == red_ref.group_boundaries
    assert np.abs(np.asarray(red.matrix) - red_ref.matrix).max() <= 1e-12 * np.abs(red_ref.matrix).max()
    s = P.figaro_svd(P.Table(A, ka), P.Table(B, kb), want_vectors=False, sort=True)
    s_ref = np.linalg.svd(r_ref, compute_uv=False)
    assert np.max(np.abs(np.asarray(s.values) - s_ref)) <= 1e-10 * s_ref[0]


def test_zipf_table_recipe_matches_oracle(P):
    """C3 recipe at 1e6 rows: per-row Zipf keys, stable sort, permuted data rows --
    keys, permutation and data bit-exact with the numpy restatement."""
    from paper_2503_23385_b200 import datagen
    t = datagen.zipf_table(3003, 3001, 1_000_000, 4)
    ref, perm = O.datagen.zipf_sorted_table(3003, 3001, 1_000_000, 4)
    assert np.array_equal(np.asarray(t.keys), ref.keys)
    assert np.array_equal(np.asarray(t.data), ref.data)
    assert np.array_equal(datagen.zipf_keys(3003, 1_000_000), O.zipf_keys(3003, 1_000_000))
