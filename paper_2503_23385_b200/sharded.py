"""Row-sharded multi-GPU figaro_r: one process per GPU, NCCL over
NVLink / NVSwitch for the two real exchange steps.

For a Cartesian product the single key group is split by rows: rank p holds A
rows [a0, a1) and B rows [b0, b1).  The only cross-shard dependencies of the
Claim-1 reduction are
  * head(B) = sum of ALL B rows / sqrt(m2), needed by every top row, and
  * the tail prefix S_i of the first B row of the shard,
so each rank all-gathers its B column sums (P x n2 doubles: the carry exchange),
builds its local reduced rows with the exclusive prefix of the ranks before it,
runs the fused TSQR on them (jq_figaro_r_shard), all-gathers the P local R
factors (P x N x N doubles) and runs the same fixed binary TSQR tree
(jq_tsqr_stack), so every rank ends with the identical canonical R.

figaro_r_sharded_local (footnote variant, carry-free shards) needs no carry at all:
each rank factors its shard alone, one all-gather carries the local R's and the
shard column sums, and the head row plus the between-shard rows are rebuilt from
the sums on every rank.

figaro_r_sharded_join (natural joins) co-partitions the key-sorted tables by key range
(co_partition): every key group lies on one rank except giant keys, which are split by
rows over consecutive ranks; the ranks factor their complete groups with figaro_r and
their giant-key parts as carry-free blocks, and one all-gather plus the split keys'
head / between-part rows (a kernel) complete the Gram.

The compute callbacks default to the GPU library; tests inject CPU
restatements to check the orchestration with the gloo backend.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(m: int, world: int, rank: int):
    """Contiguous, balanced row range of `rank` (same rule for A and B)."""
    return m * rank // world, m * (rank + 1) // world


def _native_colsums(x: torch.Tensor) -> torch.Tensor:
    from . import _native as N
    out = torch.empty(x.shape[1], dtype=torch.float64, device=x.device)
    N.use_torch_stream(x)
    N.check(N.lib().jq_colsums(N.ctx(), N.ptr(x), x.shape[0], x.shape[1], N.ptr(out)))
    return out


def _native_shard_r(a, b, m1, m2, a_row0, b_row0, a_prefix, a_total, b_prefix, b_total,
                    include_head) -> torch.Tensor:
    from . import _native as N
    n = a.shape[1] + b.shape[1]
    out = torch.empty((n, n), dtype=torch.float64, device=a.device)
    N.use_torch_stream(a)
    N.check(N.lib().jq_figaro_r_shard(N.ctx(), N.ptr(a), a.shape[0], a.shape[1], m1, a_row0, N.ptr(a_prefix),
                                      N.ptr(a_total), N.ptr(b), b.shape[0], b.shape[1], m2, b_row0,
                                      N.ptr(b_prefix), N.ptr(b_total), int(bool(include_head)), N.ptr(out)))
    return out


def _native_stack(rs: torch.Tensor) -> torch.Tensor:
    from . import _native as N
    p, n, _ = rs.shape
    out = torch.empty((n, n), dtype=torch.float64, device=rs.device)
    N.use_torch_stream(rs)
    N.check(N.lib().jq_tsqr_stack(N.ctx(), N.ptr(rs), p, n, N.ptr(out)))
    return out


def _native_shard_local(a, b, m1, m2):
    from . import _native as N
    n = a.shape[1] + b.shape[1]
    r = torch.empty((n, n), dtype=torch.float64, device=a.device)
    sums = torch.empty(n, dtype=torch.float64, device=a.device)
    N.use_torch_stream(a)
    N.check(N.lib().jq_figaro_r_shard_local(N.ctx(), N.ptr(a), a.shape[0], a.shape[1], m1, N.ptr(b), b.shape[0],
                                            b.shape[1], m2, N.ptr(r), N.ptr(sums)))
    return r, sums


def _native_householder(rows: torch.Tensor) -> torch.Tensor:
    from . import _native as N
    n = rows.shape[1]
    out = torch.empty((n, n), dtype=torch.float64, device=rows.device)
    N.use_torch_stream(rows)
    N.check(N.lib().jq_householder_r(N.ctx(), N.ptr(rows), rows.shape[0], n, N.ptr(out)))
    return out


def _native_split_rows(part_sums: torch.Tensor, part_rows, part_group, n1: int, n2: int) -> torch.Tensor:
    """jq_split_group_rows: head + between-part rows of the split groups (a kernel)."""
    import numpy as np
    from . import _native as N
    pr = np.ascontiguousarray(np.asarray(part_rows, dtype=np.int64).reshape(-1))
    pg = np.ascontiguousarray(np.asarray(part_group, dtype=np.int64).reshape(-1))
    nparts = len(pg)
    cnt = np.zeros(1, dtype=np.int64)
    N.use_torch_stream(part_sums)
    N.check(N.lib().jq_split_group_rows(N.ctx(), N.ptr(part_sums), pr.ctypes.data, pg.ctypes.data, nparts, n1, n2,
                                        None, 0, cnt.ctypes.data))
    out = torch.empty((int(cnt[0]), n1 + n2), dtype=torch.float64, device=part_sums.device)
    N.check(N.lib().jq_split_group_rows(N.ctx(), N.ptr(part_sums), pr.ctypes.data, pg.ctypes.data, nparts, n1, n2,
                                        N.ptr(out), int(cnt[0]), cnt.ctypes.data))
    return out


def between_shard_rows(all_sums: torch.Tensor, a_sizes, b_sizes, m1: int, m2: int, n1: int,
                       split_rows: Callable = None) -> torch.Tensor:
    """Rows whose Gram is what the per-shard local R's miss (carry-free Cartesian
    shards): the head row [sqrt(m2) hA | sqrt(m1) hB] and, per side, one row per shard
    k >= 1 (the pairwise scatter update).  The Cartesian product is ONE key group split
    over every rank, so this is jq_split_group_rows with a single group (a kernel;
    split_rows injects a restatement for CPU tests).  all_sums: (world, n1 + n2)."""
    split_rows = split_rows or _native_split_rows
    world, n = all_sums.shape
    rows = [[int(a_sizes[k]), int(b_sizes[k])] for k in range(world)]
    return split_rows(all_sums.contiguous(), rows, [0] * world, n1, n - n1)


def _all_gather(x: torch.Tensor, group=None) -> torch.Tensor:
    """all_gather_into_tensor of a (1, L) tensor -> (world, L).  NCCL gathers device
    tensors in place; gloo (CPU tests, or several ranks sharing one GPU) goes through
    host copies."""
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    if x.is_cuda and backend != "nccl":
        xc = x.cpu()
        out = torch.empty((world,) + tuple(x.shape[1:]), dtype=x.dtype)
        dist.all_gather_into_tensor(out, xc, group=group)
        return out.to(x.device)
    out = torch.empty((world,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    dist.all_gather_into_tensor(out, x, group=group)
    return out


def figaro_r_sharded_local(a: torch.Tensor, b: torch.Tensor, m1: int, m2: int, a_row0: int, b_row0: int,
                           group: Optional[dist.ProcessGroup] = None,
                           shard_local: Callable = _native_shard_local, householder: Callable = _native_householder,
                           stack: Callable = _native_stack, split_rows: Callable = None) -> torch.Tensor:
    """Footnote variant with carry-free shards: every rank factors its own shard with
    no prefix (jq_figaro_r_shard_local: local R + shard column sums), ONE all-gather
    carries R and sums, and every rank turns the sums into the head row and the
    between-shard rows (between_shard_rows -> jq_split_group_rows), factors them
    (householder) and runs the fixed TSQR tree over [R_0; ...; R_{P-1}; R_extra] -- no
    carry exchange, no column-sum pass.  Shards are contiguous and ordered by rank
    (shard_range)."""
    world = dist.get_world_size(group)
    n1, n2 = a.shape[1], b.shape[1]
    n = n1 + n2
    r_loc, sums = shard_local(a, b, m1, m2)
    packed = torch.cat([r_loc.reshape(-1), sums.reshape(-1)]).reshape(1, n * n + n).contiguous()
    allp = _all_gather(packed, group)  # R and sums, one collective
    r_all = allp[:, :n * n].reshape(world, n, n)
    all_sums = allp[:, n * n:]
    a_sizes = [shard_range(m1, world, k)[1] - shard_range(m1, world, k)[0] for k in range(world)]
    b_sizes = [shard_range(m2, world, k)[1] - shard_range(m2, world, k)[0] for k in range(world)]
    r_extra = householder(between_shard_rows(all_sums, a_sizes, b_sizes, m1, m2, n1, split_rows).contiguous())
    return stack(torch.cat([r_all, r_extra.reshape(1, n, n)]).contiguous())


# ------------------------------------------------------------------ natural joins
@dataclass
class SplitPart:
    """Rows [a_lo, a_hi) of A and [b_lo, b_hi) of B of split key `key` held by `rank`."""

    group: int
    key: int
    rank: int
    a_lo: int
    a_hi: int
    b_lo: int
    b_hi: int


@dataclass
class JoinPlan:
    """Key-range co-partition of two key-sorted tables over `world` ranks (SURVEY.md
    §8e): rank p holds A rows a_ranges[p] and B rows b_ranges[p]; every key lies wholly
    on one rank (both sides) except the giant keys in `parts`, split by rows over
    consecutive ranks, each part holding >= 1 row of both sides."""

    world: int
    m1: int
    m2: int
    a_ranges: List[Tuple[int, int]]
    b_ranges: List[Tuple[int, int]]
    parts: List[SplitPart] = field(default_factory=list)

    def rank_parts(self, rank: int) -> List[SplitPart]:
        return [p for p in self.parts if p.rank == rank]

    def interior(self, rank: int):
        """(a_lo, a_hi, b_lo, b_hi) of the rank's rows outside its split parts."""
        a_lo, a_hi = self.a_ranges[rank]
        b_lo, b_hi = self.b_ranges[rank]
        for p in self.rank_parts(rank):
            if p.a_lo == a_lo and p.b_lo == b_lo:
                a_lo, b_lo = p.a_hi, p.b_hi
            if p.a_hi == a_hi and p.b_hi == b_hi:
                a_hi, b_hi = max(p.a_lo, a_lo), max(p.b_lo, b_lo)
        return a_lo, max(a_lo, a_hi), b_lo, max(b_lo, b_hi)


def co_partition(keys_a, keys_b, world: int, giant_fraction: float = 0.25) -> JoinPlan:
    """Key-range co-partition of key-sorted tables (host, numpy, deterministic).

    Keys in merged order carry weight m1k + m2k rows; rank p targets the rows
    [p W / P, (p+1) W / P).  A key inside one target range goes to that rank; a key
    straddling a boundary goes whole to the rank with the largest overlap unless it is
    a matched giant (weight >= giant_fraction W / P), which is split by rows at the
    boundaries, A and B proportionally; a part left without rows of one side is merged
    into its neighbour, so every part has both sides."""
    import numpy as np
    ka = np.asarray(keys_a, dtype=np.int64)
    kb = np.asarray(keys_b, dtype=np.int64)
    m1, m2 = len(ka), len(kb)
    keys = np.union1d(ka, kb)
    a_st = np.searchsorted(ka, keys, "left")
    a_ct = np.searchsorted(ka, keys, "right") - a_st
    b_st = np.searchsorted(kb, keys, "left")
    b_ct = np.searchsorted(kb, keys, "right") - b_st
    w = a_ct + b_ct
    S = np.concatenate([[0], np.cumsum(w)])
    W = int(S[-1])
    cuts = np.array([W * p // world for p in range(world + 1)], dtype=np.int64)
    first = np.searchsorted(cuts, S[:-1], "right") - 1
    last = np.searchsorted(cuts, np.maximum(S[1:] - 1, S[:-1]), "right") - 1
    owner = first.copy()
    parts: List[SplitPart] = []
    # per-rank boundary positions inside split keys: rank -> (a_pos, b_pos)
    inner_cut = {}
    for k in np.nonzero(last > first)[0]:
        lo, hi = int(S[k]), int(S[k + 1])
        ranks = list(range(int(first[k]), int(last[k]) + 1))
        ov = [min(hi, int(cuts[p + 1])) - max(lo, int(cuts[p])) for p in ranks]
        giant = a_ct[k] > 0 and b_ct[k] > 0 and w[k] * world >= giant_fraction * W
        if not giant:
            owner[k] = ranks[int(np.argmax(ov))]
            continue
        # proportional row cuts at the rank boundaries inside the key
        bounds_a, bounds_b = [int(a_st[k])], [int(b_st[k])]
        for p in ranks[1:]:
            f = (int(cuts[p]) - lo) / w[k]
            bounds_a.append(int(a_st[k]) + int(round(f * a_ct[k])))
            bounds_b.append(int(b_st[k]) + int(round(f * b_ct[k])))
        bounds_a.append(int(a_st[k] + a_ct[k]))
        bounds_b.append(int(b_st[k] + b_ct[k]))
        segs = [[ranks[i], bounds_a[i], bounds_a[i + 1], bounds_b[i], bounds_b[i + 1]] for i in range(len(ranks))]
        # merge parts without rows of one side into a neighbour (keeps >= 1 part)
        i = 0
        while len(segs) > 1 and i < len(segs):
            sg = segs[i]
            if sg[2] > sg[1] and sg[4] > sg[3]:
                i += 1
                continue
            if i > 0:
                segs[i - 1][2], segs[i - 1][4] = sg[2], sg[4]
            else:
                segs[1][1], segs[1][3] = sg[1], sg[3]
            segs.pop(i)
            i = max(i - 1, 0)
        if len(segs) == 1:
            owner[k] = segs[0][0]
            continue
        owner[k] = segs[0][0]
        gi = len({pp.group for pp in parts})
        for sg in segs:
            parts.append(SplitPart(gi, int(keys[k]), sg[0], sg[1], sg[2], sg[3], sg[4]))
        for sg in segs[1:]:
            inner_cut[sg[0]] = (sg[1], sg[3])
        # ranks inside the key without a part start where the next part starts
        held = {sg[0] for sg in segs}
        for p in ranks[1:]:
            if p not in held:
                nxt = next((sg for sg in segs if sg[0] > p), None)
                inner_cut[p] = (nxt[1], nxt[3]) if nxt else (int(a_st[k] + a_ct[k]), int(b_st[k] + b_ct[k]))
        last[k] = segs[-1][0]
    a_cut, b_cut = [0], [0]
    for p in range(1, world):
        if p in inner_cut:
            a_cut.append(inner_cut[p][0])
            b_cut.append(inner_cut[p][1])
            continue
        k = int(np.searchsorted(owner, p, "left")) if len(owner) else 0
        # keys whose split parts end before p do not count as starting at p
        a_cut.append(int(a_st[k]) if k < len(keys) else m1)
        b_cut.append(int(b_st[k]) if k < len(keys) else m2)
    a_cut.append(m1)
    b_cut.append(m2)
    for p in range(1, world + 1):  # monotone (empty ranks allowed)
        a_cut[p] = max(a_cut[p], a_cut[p - 1])
        b_cut[p] = max(b_cut[p], b_cut[p - 1])
    return JoinPlan(world, m1, m2, [(a_cut[p], a_cut[p + 1]) for p in range(world)],
                    [(b_cut[p], b_cut[p + 1]) for p in range(world)], parts)


def _native_interior_r(a, ka, b, kb) -> torch.Tensor:
    """Canonical R of the rank's complete key groups (figaro_r, keyed)."""
    from .qr import figaro_r
    from .joins import Table
    return figaro_r(Table(a, ka), Table(b, kb))


def figaro_r_sharded_join(a: torch.Tensor, ka: torch.Tensor, b: torch.Tensor, kb: torch.Tensor, plan: JoinPlan,
                          group: Optional[dist.ProcessGroup] = None,
                          interior_r: Callable = _native_interior_r, shard_local: Callable = _native_shard_local,
                          householder: Callable = _native_householder, stack: Callable = _native_stack,
                          split_rows: Callable = None) -> torch.Tensor:
    """Canonical R of the natural join of key-sorted tables
    co-partitioned by `plan` (co_partition): this rank passes its rows
    a = A[plan.a_ranges[rank]], b = B[plan.b_ranges[rank]] with their keys.

    Per rank: figaro_r of its complete key groups (R_int), and for each split part of a
    giant key the carry-free part factor (jq_figaro_r_shard_local with the key's global
    m1g, m2g: local tails, no head) plus its column sums.  ONE all-gather carries
    [R_int, R_part0, R_part1, sums0, sums1]; every rank then builds the split keys' head
    and between-part rows (jq_split_group_rows), factors them and runs the fixed TSQR
    tree over all R's -- every rank ends with the identical canonical R."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n1, n2 = a.shape[1], b.shape[1]
    n = n1 + n2
    dev = a.device
    a_lo, _ = plan.a_ranges[rank]
    b_lo, _ = plan.b_ranges[rank]
    ia0, ia1, ib0, ib1 = plan.interior(rank)
    zeros = torch.zeros((n, n), dtype=torch.float64, device=dev)
    if ia1 > ia0 and ib1 > ib0:
        r_int = interior_r(a[ia0 - a_lo:ia1 - a_lo], ka[ia0 - a_lo:ia1 - a_lo],
                           b[ib0 - b_lo:ib1 - b_lo], kb[ib0 - b_lo:ib1 - b_lo])
    else:
        r_int = zeros
    mine = plan.rank_parts(rank)
    if len(mine) > 2:
        raise ValueError("a rank holds at most two split parts")
    tot = {}
    for p in plan.parts:
        t = tot.setdefault(p.group, [0, 0])
        t[0] += p.a_hi - p.a_lo
        t[1] += p.b_hi - p.b_lo
    slots_r = [zeros, zeros]
    slots_s = [torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(2)]
    for i, p in enumerate(mine):
        m1g, m2g = tot[p.group]
        slots_r[i], slots_s[i] = shard_local(a[p.a_lo - a_lo:p.a_hi - a_lo], b[p.b_lo - b_lo:p.b_hi - b_lo], m1g, m2g)
    packed = torch.cat([r_int.reshape(-1), slots_r[0].reshape(-1), slots_r[1].reshape(-1),
                        slots_s[0].reshape(-1), slots_s[1].reshape(-1)]).reshape(1, -1).contiguous()
    allp = _all_gather(packed, group)
    r_ints = allp[:, :n * n].reshape(world, n, n)
    blocks = [r_ints]
    if plan.parts:
        r_parts, sums, prow, pgrp = [], [], [], []
        for p in plan.parts:   # ordered by (group, rank)
            slot = plan.rank_parts(p.rank).index(p)
            r_parts.append(allp[p.rank, n * n * (1 + slot):n * n * (2 + slot)].reshape(n, n))
            sums.append(allp[p.rank, 3 * n * n + slot * n:3 * n * n + (slot + 1) * n])
            prow.append([p.a_hi - p.a_lo, p.b_hi - p.b_lo])
            pgrp.append(p.group)
        extra = (split_rows or _native_split_rows)(torch.stack(sums).contiguous(), prow, pgrp, n1, n2)
        blocks += [torch.stack(r_parts), householder(extra.contiguous()).reshape(1, n, n)]
    return stack(torch.cat(blocks).contiguous())


def figaro_r_sharded(a: torch.Tensor, b: torch.Tensor, m1: int, m2: int, a_row0: int, b_row0: int,
                     group: Optional[dist.ProcessGroup] = None,
                     colsums: Callable = _native_colsums, shard_r: Callable = _native_shard_r,
                     stack: Callable = _native_stack) -> torch.Tensor:
    """Canonical R of the Cartesian join of the full A (m1 rows) and B (m2 rows),
    given this rank's contiguous row shards `a` (from global row a_row0) and `b`
    (from b_row0); shards are ordered by rank.  One all-gather of the shards' column
    sums (n1 + n2 doubles per rank) gives every rank its exclusive prefixes and the
    global heads; one all-gather of the local R factors feeds the TSQR tree."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n1, n2 = a.shape[1], b.shape[1]
    sums = torch.cat([colsums(a), colsums(b)]).reshape(1, n1 + n2).contiguous()
    all_sums = torch.empty((world, n1 + n2), dtype=torch.float64, device=b.device)
    dist.all_gather_into_tensor(all_sums, sums, group=group)          # carry exchange
    prefix = all_sums[:rank].sum(0) if rank else torch.zeros(n1 + n2, dtype=torch.float64, device=b.device)
    total = all_sums.sum(0)
    r_loc = shard_r(a, b, m1, m2, a_row0, b_row0, prefix[:n1].contiguous(), total[:n1].contiguous(),
                    prefix[n1:].contiguous(), total[n1:].contiguous(), rank == 0).contiguous()
    n = r_loc.shape[0]
    r_all = torch.empty((world, n, n), dtype=torch.float64, device=r_loc.device)
    dist.all_gather_into_tensor(r_all, r_loc.reshape(1, n, n), group=group)  # R all-gather
    return stack(r_all)
