"""Multi-GPU orchestration with the NATIVE callbacks (jq_figaro_r_shard_local,
jq_split_group_rows, jq_householder_r, jq_tsqr_stack, figaro_r on the interior) in
2-3 processes sharing the one B200 of the test box; the collectives run over gloo
(host copies of the packed R's and sums, sharded._all_gather), so no rank's kernel
waits on another's.  Every rank must hold the identical R, equal to the single-device
R of the whole join within 1e-12."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def tables(kind, seed=0):
    rng = np.random.default_rng(seed)
    if kind == "cartesian":
        return rng.random((30_011, 24)), None, rng.random((20_003, 20)), None
    m1, m2 = 40_000, 30_000
    if kind == "keyed":
        ka, kb = np.sort(rng.integers(0, 500, m1)), np.sort(rng.integers(100, 700, m2))
    else:  # giant: one key holds most rows of both sides and is split over the ranks
        ka = np.sort(np.r_[np.full(m1 - 3000, 77), rng.integers(0, 300, 3000)])
        kb = np.sort(np.r_[np.full(m2 - 2000, 77), rng.integers(0, 300, 2000)])
    return rng.random((m1, 12)), ka.astype(np.int64), rng.random((m2, 10)), kb.astype(np.int64)


def _worker(rank, world, port, kind, variant, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2503_23385_b200 as P
    from paper_2503_23385_b200 import sharded, _native as N
    torch.cuda.set_device(0)
    N.set_device(0)
    P.set_variant(variant)
    A, ka, B, kb = tables(kind)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    if ka is None:
        a0, a1 = sharded.shard_range(len(A), world, rank)
        b0, b1 = sharded.shard_range(len(B), world, rank)
        r = sharded.figaro_r_sharded_local(dev(A[a0:a1]), dev(B[b0:b1]), len(A), len(B), a0, b0)
    else:
        plan = sharded.co_partition(ka, kb, world)
        (a0, a1), (b0, b1) = plan.a_ranges[rank], plan.b_ranges[rank]
        r = sharded.figaro_r_sharded_join(dev(A[a0:a1]), dev(ka[a0:a1]), dev(B[b0:b1]), dev(kb[b0:b1]), plan)
        out[("parts", rank)] = len(plan.rank_parts(rank))
    out[rank] = r.cpu().numpy()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["cartesian", "keyed", "giant"])
def test_sharded_native_matches_single_device(world, kind):
    import paper_2503_23385_b200 as P
    variant = "footnote"
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), kind, variant, out), nprocs=world, join=True)
    A, ka, B, kb = tables(kind)
    P.set_variant(variant)
    ref = np.asarray(P.figaro_r(P.Table(A, ka), P.Table(B, kb)))
    rs = [np.asarray(out[r]) for r in range(world)]
    for r in rs[1:]:
        assert np.array_equal(r, rs[0]), "ranks must hold the identical R"
    assert np.all(np.tril(rs[0], -1) == 0) and np.all(np.diag(rs[0]) >= 0)
    err = np.linalg.norm(rs[0] - ref) / np.linalg.norm(ref)
    assert err <= 1e-12, err
    if kind == "giant":
        assert sum(out[("parts", r)] for r in range(world)) >= 2
