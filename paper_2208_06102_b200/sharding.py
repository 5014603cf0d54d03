"""Trial sharding across ranks and the cross-GPU curve reduction.

Trials are independent and RNG counters use the GLOBAL trial index (NC-3), so a
rank only needs its [begin, end) range; the one collective is an all-reduce
(SUM) of the curves' exact fixed-point sums (NCCL on GPUs, gloo in CPU tests).
"""
from __future__ import annotations


def shard_range(trials_per_gpu: int, world: int, rank: int, scaling: str = "weak"):
    """Returns (global_trials, begin, end) of this rank.

    weak:   every rank owns trials_per_gpu trials; the job has world * trials_per_gpu.
    strong: one job of trials_per_gpu trials split as evenly as possible.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if scaling == "weak":
        return trials_per_gpu * world, trials_per_gpu * rank, trials_per_gpu * (rank + 1)
    if scaling == "strong":
        n = trials_per_gpu
        return n, n * rank // world, n * (rank + 1) // world
    raise ValueError(scaling)


def reduce_curves(curves_fixed, group=None):
    """All-reduce (SUM) of every rank's fixed-point curve sums, [cells][R][7][3] int64 limbs
    (zeus_results.curves_fixed).  Integer addition is exact and associative, so the sum has the
    same bits for any world size and any reduction order; the library then rounds it once to
    fp64 curves (zeus_sim_curves_from_fixed), giving N ranks the bits of one."""
    import torch
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        nvtx = torch.cuda.nvtx if curves_fixed.is_cuda else None   # NVTX range
        if nvtx:
            nvtx.range_push("zeus_reduce_curves")
        dist.all_reduce(curves_fixed, op=dist.ReduceOp.SUM, group=group)
        if nvtx:
            nvtx.range_pop()
    return curves_fixed
