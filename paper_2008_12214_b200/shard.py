"""Multi-GPU work split for the sharded configs.

Batch GS targets and OSPR jobs are independent, so every rank owns whole
units and there is no data-path collective; the only collective is the final
gather of per-unit results to rank 0 (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [start, start + count) of `total` units for `rank`."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def unit_seeds(first_unit: int, count: int, seed0: int = 1) -> np.ndarray:
    """Seeds of units first_unit .. first_unit+count-1 (BASELINE: seed = 1 + t)."""
    return np.arange(seed0 + first_unit, seed0 + first_unit + count, dtype=np.uint64)


def gather_to_root(values, dist, world: int, rank: int):
    """Gather equally-sized 1-D tensors to rank 0 in rank order (None elsewhere)."""
    import torch
    if world == 1:
        return values
    out = [torch.empty_like(values) for _ in range(world)] if rank == 0 else None
    dist.gather(values, out, dst=0)
    return torch.cat(out) if rank == 0 else None


def gather_batch_results(levels, traces, dist, world: int, rank: int, total: int):
    """rank 0 receives every target's levels and MSE trace, the
    result set of cmd_batch (runner.cpp:365-451), in target order.

    levels: [count][ny][nx] uint8 (or int16/int32) tensor of this rank's
    targets, traces: [count][K] float64 tensor; both on the rank's device
    (NCCL) or on the CPU (gloo).  Ranks own contiguous shard_range blocks that
    differ by at most one target, so every rank pads to the largest block and
    one gather per array moves everything.  Returns (levels [total][ny][nx],
    traces [total][K]) as tensors on rank 0, None elsewhere."""
    import torch
    first, count = shard_range(total, world, rank)
    if levels.shape[0] != count or traces.shape[0] != count:
        raise ValueError("gather_batch_results: arrays do not match this rank's shard")
    if world == 1:
        return levels, traces
    cmax = shard_range(total, world, 0)[1]
    lv = torch.zeros((cmax,) + tuple(levels.shape[1:]), dtype=levels.dtype, device=levels.device)
    tr = torch.zeros((cmax,) + tuple(traces.shape[1:]), dtype=traces.dtype, device=traces.device)
    lv[:count] = levels
    tr[:count] = traces
    lv_all = gather_to_root(lv.reshape(-1), dist, world, rank)
    tr_all = gather_to_root(tr.reshape(-1), dist, world, rank)
    if rank != 0:
        return None
    lv_all = lv_all.reshape((world, cmax) + tuple(levels.shape[1:]))
    tr_all = tr_all.reshape((world, cmax) + tuple(traces.shape[1:]))
    keep = [shard_range(total, world, g)[1] for g in range(world)]
    return (torch.cat([lv_all[g, :keep[g]] for g in range(world)]),
            torch.cat([tr_all[g, :keep[g]] for g in range(world)]))


def run_batch_sharded(cfg, amplitude, total: int, dist, world: int, rank: int, seed0: int = 1, stream=None):
    """Batch GS over `total` independent targets sharded across ranks (SURVEY
    §8 e1, BASELINE config 5): rank g runs targets shard_range(total, world, g)
    (seed = seed0 + t) as one batched plan with no collective inside the
    iterations, then rank 0 gathers the levels and traces (NCCL).  Returns
    {"levels": [total][ny][nx], "trace": [total][K]} numpy arrays on rank 0,
    None elsewhere."""
    import torch
    from .api import IftaPlan
    amp = np.ascontiguousarray(amplitude, np.float64)
    ny, nx = amp.shape[-2:]
    first, count = shard_range(total, world, rank)
    if count == 0:
        raise ValueError("run_batch_sharded: more ranks than targets")
    amps = np.broadcast_to(amp, (count, ny, nx)) if amp.ndim == 2 else amp[first:first + count]
    plan = IftaPlan(cfg, nx, ny, count)
    plan.upload(amps, seeds=unit_seeds(first, count, seed0))
    st = stream or torch.cuda.Stream()
    plan.execute(st.cuda_stream)
    st.synchronize()
    _, lv, tr = plan.device_arrays()
    levels = torch.as_tensor(lv, device="cuda").clone()
    traces = torch.as_tensor(tr, device="cuda").clone()
    plan.close()
    got = gather_batch_results(levels, traces, dist, world, rank, total)
    if got is None:
        return None
    return {"levels": got[0].cpu().numpy(), "trace": got[1].cpu().numpy()}


def run_ospr_sharded(cfg, dist, world: int, rank: int, stream=None) -> dict | None:
    """ONE plain OSPR job split into contiguous subframe blocks, one per rank
    (SURVEY §8 e2).  Rank g runs global subframes shard_range(N, world, g)
    from the jump-ahead stream position; the only exchange is one all-gather
    of the block intensity sums (npix fp32 per rank, NCCL over NVLink), after
    which each rank finishes its cumulative MSEs locally.  Rank 0 gathers the
    level frames and traces and returns the whole run's arrays (None on other
    ranks).  `stream`: a torch.cuda.Stream to run on (default: a new one)."""
    import torch
    from .api import OsprBlockPlan
    N = cfg.subframes
    first, count = shard_range(N, world, rank)
    if count == 0:
        raise ValueError("run_ospr_sharded: more ranks than subframes")
    amp = np.ascontiguousarray(cfg.target.amplitude, np.float64)
    ny, nx = amp.shape
    roi = getattr(cfg.target, "roi", None)
    plan = OsprBlockPlan(cfg, nx, ny, first, count)
    plan.upload(amp, roi=roi)
    st = stream or torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan.execute(st.cuda_stream)
        B = torch.as_tensor(plan.block_sum(), device="cuda")
        gathered = torch.empty((world, B.numel()), dtype=torch.float32, device="cuda")
        if world == 1:
            gathered[0].copy_(B)
        else:
            dist.all_gather_into_tensor(gathered, B)
        plan.finish(gathered.data_ptr(), world, rank, st.cuda_stream)
        out = plan.download()
    plan.close()
    # gather to rank 0: pad every block to the largest count (shard_range blocks differ by <= 1)
    cmax = shard_range(N, world, 0)[1]
    npix = nx * ny
    lv = np.zeros((cmax, npix), out["levels"].dtype)
    lv[:count] = out["levels"].reshape(count, npix)
    tr = np.zeros((cmax, 2))
    tr[:count, 0], tr[:count, 1] = out["frame_mse"][0], out["cumulative_mse"][0]
    if world == 1:
        lv_all, tr_all = lv[None], tr[None]
    else:
        lv_t = torch.as_tensor(lv if lv.dtype == np.uint8 else lv.astype(np.int32), device="cuda")
        tr_t = torch.as_tensor(tr, device="cuda")
        lv_g = gather_to_root(lv_t.reshape(-1), dist, world, rank)
        tr_g = gather_to_root(tr_t.reshape(-1), dist, world, rank)
        if rank != 0:
            return None
        lv_all = lv_g.cpu().numpy().reshape(world, cmax, npix).astype(out["levels"].dtype)
        tr_all = tr_g.cpu().numpy().reshape(world, cmax, 2)
    levels, fm, cm = [], [], []
    for g in range(world):
        c = shard_range(N, world, g)[1]
        levels.append(lv_all[g, :c])
        fm.append(tr_all[g, :c, 0])
        cm.append(tr_all[g, :c, 1])
    return {"levels": np.concatenate(levels).reshape(N, ny, nx), "frame_mse": np.concatenate(fm),
            "cumulative_mse": np.concatenate(cm), "mean_intensity": out["mean_intensity"][0],
            "final_error": float(np.concatenate(cm)[-1])}
