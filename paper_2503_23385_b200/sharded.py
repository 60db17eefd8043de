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

The compute callbacks default to the GPU library; tests inject CPU
restatements to check the orchestration with the gloo backend.
"""

from __future__ import annotations

from typing import Callable, Optional

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


def between_shard_rows(all_sums: torch.Tensor, a_sizes, b_sizes, m1: int, m2: int, n1: int) -> torch.Tensor:
    """Rows whose Gram is what the per-shard local R's miss (carry-free shards): the
    head row [sqrt(m2) hA | sqrt(m1) hB] and, per side, one row per shard k >= 1
        v_k = scale sqrt(W_k m_k / (W_k + m_k)) (s_k / m_k - S_k / W_k)
    (W_k, S_k: rows and column sums of the shards before k; the pairwise scatter
    update, the same rule as the blocks inside a shard).  Fixed shard order, float64:
    identical on every rank.  all_sums: (world, n1 + n2) shard column sums."""
    world, n = all_sums.shape
    out = []
    tot = []
    for side, sizes, scale in ((0, a_sizes, m2 ** 0.5), (1, b_sizes, m1 ** 0.5)):
        cols = slice(0, n1) if side == 0 else slice(n1, n)
        W, S = 0.0, torch.zeros(cols.stop - cols.start, dtype=torch.float64, device=all_sums.device)
        for k in range(world):
            mk = float(sizes[k])
            sk = all_sums[k, cols]
            if W > 0 and mk > 0:
                row = torch.zeros(n, dtype=torch.float64, device=all_sums.device)
                row[cols] = scale * (W * mk / (W + mk)) ** 0.5 * (sk / mk - S / W)
                out.append(row)
            W += mk
            S = S + sk
        tot.append(S)
    head = torch.cat([(m2 ** 0.5) * tot[0] / (m1 ** 0.5), (m1 ** 0.5) * tot[1] / (m2 ** 0.5)])
    return torch.stack([head] + out)


def figaro_r_sharded_local(a: torch.Tensor, b: torch.Tensor, m1: int, m2: int, a_row0: int, b_row0: int,
                           group: Optional[dist.ProcessGroup] = None,
                           shard_local: Callable = _native_shard_local, householder: Callable = _native_householder,
                           stack: Callable = _native_stack) -> torch.Tensor:
    """Footnote variant with carry-free shards: every rank factors its own shard with
    no prefix (jq_figaro_r_shard_local: local R + shard column sums), ONE all-gather
    carries R and sums, and every rank turns the sums into the head row and the
    between-shard rows (between_shard_rows), factors them (householder) and runs the
    fixed TSQR tree over [R_0; ...; R_{P-1}; R_extra] -- no carry exchange, no
    column-sum pass.  Shards are contiguous and ordered by rank (shard_range)."""
    world = dist.get_world_size(group)
    n1, n2 = a.shape[1], b.shape[1]
    n = n1 + n2
    r_loc, sums = shard_local(a, b, m1, m2)
    packed = torch.cat([r_loc.reshape(-1), sums.reshape(-1)]).reshape(1, n * n + n).contiguous()
    allp = torch.empty((world, n * n + n), dtype=torch.float64, device=packed.device)
    dist.all_gather_into_tensor(allp, packed, group=group)  # R and sums, one collective
    r_all = allp[:, :n * n].reshape(world, n, n)
    all_sums = allp[:, n * n:]
    a_sizes = [shard_range(m1, world, k)[1] - shard_range(m1, world, k)[0] for k in range(world)]
    b_sizes = [shard_range(m2, world, k)[1] - shard_range(m2, world, k)[0] for k in range(world)]
    r_extra = householder(between_shard_rows(all_sums, a_sizes, b_sizes, m1, m2, n1).contiguous())
    return stack(torch.cat([r_all, r_extra.reshape(1, n, n)]).contiguous())


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
