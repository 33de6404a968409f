"""Multi-GPU sharding of the hot path: segments are independent, so rank r enhances its own
shard on its own GPU and the results are gathered on the host in plan order. No data-path collective.

`torch.distributed` (NCCL on GPUs, gloo in the CPU tests) is used only for the ordered gather of the small
per-segment outputs; the enhancement itself never communicates."""
from __future__ import annotations


def segment_cost(frames: int, channels: int, classes: int, bss_iterations: int, wpe_taps: int = 0,
                 wpe_iterations: int = 0) -> float:
    """Relative cost model ~ FLOPs of one segment: EM sweeps + WPE Grams."""
    m, k = channels, classes
    em = (bss_iterations + 1) * (3 * m * m + 4 * m * m * k + 20 * k)
    km = wpe_taps * m
    wpe = wpe_iterations * 8 * (km * (km + 1) / 2 + 2 * km * m)
    return float(frames) * (em + wpe)


def shard(costs, world_size: int):
    """Static longest-processing-time-first assignment. Returns, per rank, the ascending list of segment
    indices it owns. Deterministic (ties -> lowest index, lowest rank)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * world_size
    owned = [[] for _ in range(world_size)]
    for i in order:
        r = min(range(world_size), key=lambda q: (load[q], q))
        owned[r].append(i)
        load[r] += costs[i]
    return [sorted(o) for o in owned]


def enhance_sharded(segments, cfg, enhance_fn, rank: int, world_size: int, group=None, dst: int = 0):
    """Enhance `segments` (the same list on every rank) across `world_size` ranks.

    `enhance_fn(list_of_segments, cfg) -> list_of_results` runs on this rank's device (normally
    gss.scheduler.enhance_batches). Rank `dst` returns the results in the original order (the analogue of the
    reference's OrderedBatchQueue, scheduler.hpp:383-412); other ranks return None."""
    import torch.distributed as dist
    costs = [segment_cost(s.activity.frames, s.audio.num_channels(), s.activity.num_classes(), cfg.bss_iterations,
                          cfg.wpe.taps if cfg.enable_wpe else 0, cfg.wpe.iterations if cfg.enable_wpe else 0)
             for s in segments]
    owned = shard(costs, world_size)
    mine = owned[rank]
    local = enhance_fn([segments[i] for i in mine], cfg) if mine else []
    if world_size == 1:
        return local
    gathered = [None] * world_size if rank == dst else None
    dist.gather_object(list(zip(mine, local)), gathered, dst=dst, group=group)
    if rank != dst:
        return None
    out = [None] * len(segments)
    for part in gathered:
        for i, r in part:
            out[i] = r
    return out
