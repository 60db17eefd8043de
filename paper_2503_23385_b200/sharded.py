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
