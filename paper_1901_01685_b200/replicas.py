"""Multi-GPU use of the solve path: replicas only.

The smoothers and the ILUT factorisation are global sequential recurrences, so a single
solve does not shard across GPUs without changing the mathematics (block-ILUT is a SPEC
non-goal).  N GPUs therefore run independent solves -- one process per GPU,
independent configs / sweep cells or replicas of the same system -- and
the only collectives are the timing reductions of the bench (no data-path collective).
"""
from __future__ import annotations


def cells_for_rank(cells: list, rank: int, world: int) -> list:
    """Deterministic round-robin assignment of independent solves to ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return [c for i, c in enumerate(cells) if i % world == rank]


def job_throughput(local_units: float, local_seconds: float, device=None) -> tuple[float, float, float]:
    """Whole-job throughput of independent replicas: (sum of units over ranks) / (max time over
    ranks).  Uses the initialised torch.distributed group (NCCL on GPUs, gloo in the CPU tests);
    single-process when none is initialised.  Returns (units/s, total_units, max_seconds)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local_units / local_seconds, local_units, local_seconds
    t = torch.tensor([local_units, local_seconds], dtype=torch.float64, device=device)
    s = t.clone()
    dist.all_reduce(s[:1], op=dist.ReduceOp.SUM)
    dist.all_reduce(t[1:], op=dist.ReduceOp.MAX)
    units, secs = float(s[0]), float(t[1])
    return units / secs, units, secs
