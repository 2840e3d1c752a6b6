"""The one exchange step of the path: the per-rank fp64
group totals [R+1][X][K] are summed across ranks.  Each rank owns a
contiguous range of segments (synth.shard / the caller's partition), so its
rows of regions it does not touch are zero and the SUM is the global result.
Integer statistics (requests, opted-out, per-level counts and tokens) are
carried in fp64 and are exact below 2^53, so their sum is exact in any order;
the fp64 energy/carbon/time/quality sums depend on the order only at the
1e-16 level.  `deterministic=True` gathers every rank's partial and adds them
in rank order instead (bit-identical across runs and backends).

Plumbing only (torch.distributed; NCCL over NVLink on B200, gloo in the CPU
tests): no arithmetic of the method happens here.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def allreduce_totals(group_totals: torch.Tensor, deterministic: bool = False, group=None) -> torch.Tensor:
    """In-place SUM of `group_totals` over the ranks of `group`."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return group_totals
    if not deterministic:
        dist.all_reduce(group_totals, op=dist.ReduceOp.SUM, group=group)
        return group_totals
    parts = [torch.empty_like(group_totals) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, group_totals, group=group)
    acc = torch.zeros_like(group_totals)
    for p in parts:          # rank order
        acc += p
    group_totals.copy_(acc)
    return group_totals


def max_over_ranks(value: float, device, group=None) -> float:
    """Max of a per-rank scalar (device timings: the job takes as long as its slowest rank)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
