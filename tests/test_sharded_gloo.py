"""Multi-process (gloo, world_size 2 and 3) check of the row-sharded orchestration
(paper_2503_23385_b200/sharded.py): carry exchange of B column sums, per-rank local
R, R all-gather and the TSQR tree must reproduce the unsharded oracle R.

The per-rank compute is injected as a CPU restatement (this container has no GPU);
on a B200 box the same orchestration runs with the native callbacks (bench.py).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def cpu_colsums(x):
    return x.sum(0)


def cpu_shard_r(a, b, m1, m2, a_row0, b_row0, a_prefix, a_total, prefix, total, include_head):
    """Local reduced rows of a Cartesian shard (SPEC.md:189-200 with a global prefix)."""
    a, b = a.numpy(), b.numpy()
    n1, n2 = a.shape[1], b.shape[1]
    top = np.hstack([a * np.sqrt(m2), np.repeat((total.numpy() / np.sqrt(m2))[None], len(a), 0)])
    s = prefix.numpy().copy()
    rows = []
    for k in range(len(b)):
        i = b_row0 + k
        if i == 0:
            s = b[k].copy()
            continue
        rows.append(np.concatenate([np.zeros(n1), (np.sqrt(i) * b[k] - s / np.sqrt(i)) / np.sqrt(i + 1) * np.sqrt(m1)]))
        s = s + b[k]
    red = np.vstack([top] + ([np.array(rows)] if rows else []))
    return torch.from_numpy(O.householder_r_lapack(red))


def cpu_shard_local(a, b, m1, m2):
    """Carry-free shard (jq_figaro_r_shard_local): the shard's own tails of A (scale
    sqrt(m2)) and of B (scale sqrt(m1)) -- the shard is one block -- and its sums."""
    a, b = a.numpy(), b.numpy()
    n1, n2 = a.shape[1], b.shape[1]
    ta, tb = O.tail(a) * np.sqrt(m2), O.tail(b) * np.sqrt(m1)
    red = np.vstack([np.hstack([ta, np.zeros((len(ta), n2))]), np.hstack([np.zeros((len(tb), n1)), tb])])
    r = O.householder_r_lapack(red) if len(red) else np.zeros((n1 + n2, n1 + n2))
    return torch.from_numpy(r), torch.from_numpy(np.concatenate([a.sum(0), b.sum(0)]))


def cpu_householder(rows):
    return torch.from_numpy(O.householder_r_lapack(rows.numpy()))


def cpu_stack(rs):
    return torch.from_numpy(O.canonicalize(O.householder_r_lapack(rs.reshape(-1, rs.shape[-1]).numpy())))


def cpu_split_rows(part_sums, part_rows, part_group, n1, n2):
    from oracle.sharded import split_group_rows
    return torch.from_numpy(split_group_rows(part_sums.numpy(), part_rows, part_group, n1, n2))


def cpu_interior_r(a, ka, b, kb):
    n = a.shape[1] + b.shape[1]
    r = O.figaro_r(O.Table(a.numpy(), ka.numpy()), O.Table(b.numpy(), kb.numpy()), lapack=True)
    return torch.from_numpy(np.asarray(r)).reshape(n, n)


def _worker(rank, world, port, m1, m2, n1, n2, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_23385_b200 import sharded
    rng = np.random.default_rng(0)
    A, B = rng.random((m1, n1)), rng.random((m2, n2))
    a0, a1 = sharded.shard_range(m1, world, rank)
    b0, b1 = sharded.shard_range(m2, world, rank)
    r = sharded.figaro_r_sharded(torch.from_numpy(A[a0:a1].copy()), torch.from_numpy(B[b0:b1].copy()),
                                 m1, m2, a0, b0, colsums=cpu_colsums, shard_r=cpu_shard_r, stack=cpu_stack)
    out[rank] = r.numpy().tolist()
    r2 = sharded.figaro_r_sharded_local(torch.from_numpy(A[a0:a1].copy()), torch.from_numpy(B[b0:b1].copy()),
                                        m1, m2, a0, b0, shard_local=cpu_shard_local, householder=cpu_householder,
                                        stack=cpu_stack, split_rows=cpu_split_rows)
    out[("local", rank)] = r2.numpy().tolist()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m1,m2,n1,n2", [(2, 50, 37, 3, 4), (3, 11, 40, 2, 5), (2, 3, 2, 2, 2)])
def test_sharded_matches_single(world, m1, m2, n1, n2):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), m1, m2, n1, n2, out), nprocs=world, join=True)
    rng = np.random.default_rng(0)
    A, B = rng.random((m1, n1)), rng.random((m2, n2))
    ref = O.figaro_r(O.Table(A), O.Table(B), lapack=True)
    rs = [np.array(out[r]) for r in range(world)]
    for r in rs[1:]:
        assert np.array_equal(r, rs[0]), "ranks must hold the identical R"
    g = O.gram(O.reduce_cartesian(A, B).matrix)
    assert np.abs(rs[0].T @ rs[0] - g).max() <= 1e-10 * np.abs(g).max()
    if m1 + m2 - 1 >= n1 + n2:
        assert np.linalg.norm(np.abs(rs[0]) - np.abs(ref)) <= 1e-10 * np.linalg.norm(ref)
    # carry-free shards: one all-gather of R + sums, between-shard rows on every rank
    rl = [np.array(out[("local", r)]) for r in range(world)]
    for r in rl[1:]:
        assert np.array_equal(r, rl[0]), "ranks must hold the identical R (carry-free shards)"
    assert np.abs(rl[0].T @ rl[0] - g).max() <= 1e-10 * np.abs(g).max()
    if m1 + m2 - 1 >= n1 + n2:
        assert np.linalg.norm(np.abs(rl[0]) - np.abs(ref)) <= 1e-10 * np.linalg.norm(ref)


def join_tables(seed, m1, m2, n1, n2, kind):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        ka, kb = np.sort(rng.integers(0, 12, m1)), np.sort(rng.integers(3, 15, m2))
    elif kind == "giant":     # one key holds most rows on both sides: split over ranks
        ka = np.sort(np.r_[np.full(m1 - 20, 5), rng.integers(0, 12, 20)])
        kb = np.sort(np.r_[np.full(m2 - 15, 5), rng.integers(0, 12, 15)])
    else:                     # "lopsided": a giant key with 2 B rows (parts merge)
        ka = np.sort(np.r_[np.full(m1 - 10, 4), rng.integers(0, 9, 10)])
        kb = np.sort(np.r_[np.full(2, 4), rng.integers(5, 9, m2 - 2)])
    return rng.random((m1, n1)), ka.astype(np.int64), rng.random((m2, n2)), kb.astype(np.int64)


def _join_worker(rank, world, port, args, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_23385_b200 import sharded
    A, ka, B, kb = join_tables(*args)
    plan = sharded.co_partition(ka, kb, world)
    (a0, a1), (b0, b1) = plan.a_ranges[rank], plan.b_ranges[rank]
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x))
    r = sharded.figaro_r_sharded_join(t(A[a0:a1]), t(ka[a0:a1]), t(B[b0:b1]), t(kb[b0:b1]), plan,
                                      interior_r=cpu_interior_r, shard_local=cpu_shard_local,
                                      householder=cpu_householder, stack=cpu_stack, split_rows=cpu_split_rows)
    out[rank] = r.numpy().tolist()
    out[("parts", rank)] = len(plan.rank_parts(rank))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "uniform"), (3, "uniform"), (2, "giant"), (3, "giant"),
                                        (3, "lopsided")])
def test_sharded_natural_join_matches_single(world, kind):
    """Key-range co-partition (giant keys split by rows) reproduces the single-device
    natural-join R on every rank, identically."""
    args = (world * 7, 160, 120, 3, 4, kind)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_join_worker, args=(world, _free_port(), args, out), nprocs=world, join=True)
    A, ka, B, kb = join_tables(*args)
    a, b = O.Table(A, ka), O.Table(B, kb)
    red = O.reduce_join(a, b).matrix
    g = O.gram(red)
    rs = [np.array(out[r]) for r in range(world)]
    for r in rs[1:]:
        assert np.array_equal(r, rs[0]), "ranks must hold the identical R"
    assert np.abs(rs[0].T @ rs[0] - g).max() <= 1e-10 * np.abs(g).max()
    ref = O.canonicalize(O.householder_r_lapack(red))
    assert np.linalg.norm(np.abs(rs[0]) - np.abs(ref)) <= 1e-10 * np.linalg.norm(ref)
    if kind == "giant":
        assert sum(out[("parts", r)] for r in range(world)) >= 2, "the giant key must be split"
