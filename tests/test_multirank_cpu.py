"""CPU: the N>1 host logic of the sharded configs with world size 2 over gloo.

Each rank takes its shard of a batch of GS targets (shard.shard_range), runs
them (on the CPU oracle here — the GPU ranks run the same split on the
kernels), and rank 0 gathers the per-target final errors.  The gathered
vector must equal a single-process run over all targets, in target order.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2008_12214_b200 import patterns
from paper_2008_12214_b200.shard import gather_to_root, shard_range, unit_seeds

TOTAL, N, K = 6, 32, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _final_errors(seeds):
    from pyoracle import Oracle
    from paper_2008_12214_b200.types import SlmSpec
    o = Oracle("restatement")
    amp = patterns.bench_target(N)
    return np.array([o.ifta(amp, SlmSpec.binary_phase(), K, seed=int(s)).trace[-1] for s in seeds])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, count = shard_range(TOTAL, world, rank)
    errs = torch.tensor(_final_errors(unit_seeds(start, count)), dtype=torch.float64)
    got = gather_to_root(errs, dist, world, rank)
    if rank == 0:
        q.put(got.numpy())
    dist.destroy_process_group()


def test_shard_range_covers_exactly():
    for total in (1, 5, 64):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s, c = shard_range(total, world, r)
                seen += list(range(s, s + c))
            assert seen == list(range(total))


def test_two_rank_gather_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _final_errors(unit_seeds(0, TOTAL))
    assert np.array_equal(got, want)


# ---- one OSPR job split into subframe blocks (world size 2, gloo)
OSPR_N, OSPR_NPX = 5, 32


def _ospr_block_worker(rank, world, port, q):
    """Each rank owns subframes shard_range(N, world, rank) of one job, forms
    its block intensity sum B_g, all-gathers B (the only exchange), and
    finishes its cumulative MSEs from the prefix of earlier blocks — the
    protocol of shard.run_ospr_sharded / hgc_ospr_block_finish, with the
    oracle's frames standing in for the GPU block."""
    from pyoracle import Oracle
    from paper_2008_12214_b200.types import SlmSpec
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle("restatement")
    amp = patterns.bench_target(OSPR_NPX)
    full = o.ospr(amp, SlmSpec.binary_phase(), OSPR_N, seed=1, keep_frames=True)
    first, count = shard_range(OSPR_N, world, rank)
    inten = [np.abs(o.fft2(full.frames[k], -1)).astype(np.float64) ** 2 for k in range(first, first + count)]
    snaps = np.cumsum(np.array(inten), axis=0)  # local running sums after each block frame
    B = torch.tensor(snaps[-1].ravel())
    gathered = [torch.empty_like(B) for _ in range(world)]
    dist.all_gather(gathered, B)
    prefix = sum((gathered[h].numpy() for h in range(rank)), np.zeros_like(B.numpy())).reshape(amp.shape)
    cum = np.array([o.mse(amp, np.sqrt((prefix + snaps[k]) / (first + k + 1)).astype(np.complex64))
                    for k in range(count)])
    pad = np.zeros(shard_range(OSPR_N, world, 0)[1])
    pad[:count] = cum
    got = gather_to_root(torch.tensor(pad), dist, world, rank)
    if rank == 0:
        parts = got.numpy().reshape(world, -1)
        q.put((np.concatenate([parts[g, :shard_range(OSPR_N, world, g)[1]] for g in range(world)]),
               full.cumulative_mse))
    dist.destroy_process_group()


def test_two_rank_ospr_subframe_blocks_match_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ospr_block_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got.shape == want.shape
    assert np.max(np.abs(got - want) / want) < 1e-5


# ---- rank 0 gathers every target's levels and MSE trace
# (cmd_batch's result set, runner.cpp:365-451) over uneven shards
BATCH_TOTAL = 5


def _batch_results(seeds):
    from pyoracle import Oracle
    from paper_2008_12214_b200.types import SlmSpec
    o = Oracle("restatement")
    amp = patterns.bench_target(N)
    runs = [o.ifta(amp, SlmSpec.full_circle_phase(16), K, seed=int(s)) for s in seeds]
    return np.stack([r.levels.astype(np.uint8) for r in runs]), np.stack([r.trace for r in runs])


def _batch_worker(rank, world, port, q):
    from paper_2008_12214_b200.shard import gather_batch_results
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, count = shard_range(BATCH_TOTAL, world, rank)
    lv, tr = _batch_results(unit_seeds(start, count))
    got = gather_batch_results(torch.from_numpy(lv), torch.from_numpy(tr), dist, world, rank, BATCH_TOTAL)
    if rank == 0:
        q.put((got[0].numpy(), got[1].numpy()))
    else:
        assert got is None
    dist.destroy_process_group()


def test_two_rank_batch_levels_and_traces_gathered_in_target_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    lv, tr = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_lv, want_tr = _batch_results(unit_seeds(0, BATCH_TOTAL))
    assert lv.shape == want_lv.shape and tr.shape == want_tr.shape
    assert np.array_equal(lv, want_lv) and np.array_equal(tr, want_tr)
