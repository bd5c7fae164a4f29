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
