"""Key-range co-partition of key-sorted tables (sharded.co_partition):
contiguous covering row ranges, every non-split key wholly on one rank (both sides),
split (giant) keys covered exactly by parts that hold rows of both sides, <= 2 parts
per rank.  Host-only (numpy)."""
import numpy as np
import pytest

from paper_2503_23385_b200.sharded import co_partition


def check_plan(ka, kb, world):
    plan = co_partition(ka, kb, world)
    assert plan.a_ranges[0][0] == 0 and plan.a_ranges[-1][1] == len(ka)
    assert plan.b_ranges[0][0] == 0 and plan.b_ranges[-1][1] == len(kb)
    for p in range(world - 1):
        assert plan.a_ranges[p][1] == plan.a_ranges[p + 1][0]
        assert plan.b_ranges[p][1] == plan.b_ranges[p + 1][0]
    split = {pp.key for pp in plan.parts}
    for pp in plan.parts:
        assert pp.a_hi > pp.a_lo and pp.b_hi > pp.b_lo
        assert np.all(ka[pp.a_lo:pp.a_hi] == pp.key) and np.all(kb[pp.b_lo:pp.b_hi] == pp.key)
        lo, hi = plan.a_ranges[pp.rank]
        assert lo <= pp.a_lo and pp.a_hi <= hi
    for p in range(world):
        assert len(plan.rank_parts(p)) <= 2
        a0, a1, b0, b1 = plan.interior(p)
        keys = set(ka[a0:a1].tolist()) | set(kb[b0:b1].tolist())
        assert not (keys & split)
        for k in keys:  # wholly on this rank, both sides
            ia, ib = np.nonzero(ka == k)[0], np.nonzero(kb == k)[0]
            assert ia.size == 0 or (ia.min() >= a0 and ia.max() < a1)
            assert ib.size == 0 or (ib.min() >= b0 and ib.max() < b1)
    for k in split:
        ps = [pp for pp in plan.parts if pp.key == k]
        assert sum(pp.a_hi - pp.a_lo for pp in ps) == np.sum(ka == k)
        assert sum(pp.b_hi - pp.b_lo for pp in ps) == np.sum(kb == k)
    return plan


def test_co_partition_random_shapes():
    rng = np.random.default_rng(0)
    for t in range(300):
        world = int(rng.integers(1, 9))
        m1, m2 = int(rng.integers(1, 400)), int(rng.integers(1, 400))
        kmax = int(rng.integers(1, 40))
        if t % 3 == 0:
            ka, kb = np.sort(rng.integers(0, kmax, m1)), np.sort(rng.integers(0, kmax, m2))
        elif t % 3 == 1:
            ka, kb = np.sort(np.minimum(rng.zipf(1.5, m1), kmax)), np.sort(np.minimum(rng.zipf(1.5, m2), kmax))
        else:
            ka, kb = np.zeros(m1), np.zeros(m2)
        check_plan(ka.astype(np.int64), kb.astype(np.int64), world)


def test_co_partition_giant_key_is_split_and_balanced():
    ka, kb = np.zeros(100, np.int64), np.zeros(50, np.int64)
    plan = check_plan(ka, kb, 4)
    assert len(plan.parts) == 4
    assert [hi - lo for lo, hi in plan.a_ranges] == [25, 25, 25, 25]


@pytest.mark.parametrize("world", [2, 3, 8])
def test_co_partition_lopsided_giant(world):
    """A giant key with fewer B rows than ranks: parts without B rows merge away."""
    ka = np.sort(np.r_[np.zeros(1000), np.arange(1, 100)]).astype(np.int64)
    kb = np.sort(np.r_[np.zeros(3), np.arange(1, 100)]).astype(np.int64)
    plan = check_plan(ka, kb, world)
    assert all(pp.b_hi - pp.b_lo >= 1 for pp in plan.parts)
