#!/usr/bin/env python
"""Benchmark of the B200 HoloGen hot path (BASELINE.json metric:
"GS iterations/sec at 4096^2 and OSPR subframes/sec; % of HBM roofline").

Workload (BASELINE config 5, the largest single-GPU config): batch GS,
4096x4096, 256-level full-circle phase SLM, K = 25 iterations (reference
default, config.hpp:35), smooth_blobs + UnitEnergy targets (the reference's
bench target, bench.cpp:115-116), target t seeded with 1 + t.  The 64 targets
(--total-targets) are sharded over the GPUs: one step = one
full batched run per GPU (random-phase init + K iterations + trace reduction)
of its shard; value = target-iterations per second over all GPUs ("strong":
the total is fixed).  --targets T instead runs T targets per GPU ("weak").
OSPR (config 3: 1024^2 binary, 24 subframes) is reported in the "ospr" object.

  python bench.py [--gpus N --steps K --warmup W]          ours
  python bench.py --impl reference [...]                  reference CPU path

Multi-GPU: one process per GPU.  Under torchrun the world comes from
WORLD_SIZE (and must equal --gpus); a bare `bench.py --gpus N` re-launches
itself under torch.distributed.run with N ranks.  Whole targets per GPU, no
data-path collective; after the timed steps NCCL gathers every target's
levels and MSE trace to rank 0 (cmd_batch's result set).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GS iterations/sec at 4096² and OSPR subframes/sec; % of HBM roofline"
E2E_MIN_STEPS = 20  # the exposed first upload (~0.2 s at 4096^2 x 64) is amortised over the loop
GS_BYTES_PER_PX = {"row": 16, "col": 20, "iteration": 36}  # 2 fused round trips + fp32 target
OSPR_BYTES_PER_PX = {"seed": 8, "col_inv": 16, "row": 17, "col_acc": 20, "subframe": 49}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--levels", type=int, default=256)
    ap.add_argument("--total-targets", type=int, default=64,
                    help="targets per step over all GPUs, sharded (BASELINE config 5: 64)")
    ap.add_argument("--targets", type=int, default=None,
                    help="targets per GPU per step instead (weak scaling); default: --total-targets sharded")
    ap.add_argument("--dry-run", action="store_true",
                    help="exercise the launch / sharding / gather plumbing only (gloo, no GPU work)")
    ap.add_argument("--iters", type=int, default=25)
    ap.add_argument("--ospr-n", type=int, default=1024)
    ap.add_argument("--ospr-jobs", type=int, default=148, help="OSPR jobs per GPU per step (one MT stream per SM)")
    ap.add_argument("--ospr-subframes", type=int, default=24)
    ap.add_argument("--no-ospr", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------- distributed
class Dist:
    def __init__(self, collectives: bool = True, backend: str = "nccl"):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.device = "cuda" if backend == "nccl" else "cpu"
        if self.world > 1 and collectives:
            import torch
            import torch.distributed as dist
            if backend == "nccl":
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        import torch
        t = torch.tensor([v], device=self.device, dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------- clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev, self.rows, self.proc = dev, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------- GS (ours)
def shard_of(args, d: Dist):
    """This rank's targets: a contiguous block of --total-targets (strong
    scaling, BASELINE config 5 sharded over the GPUs) or --targets per GPU."""
    from paper_2008_12214_b200.shard import shard_range
    if args.targets:
        return d.rank * args.targets, args.targets, args.targets * d.world, "weak"
    first, count = shard_range(args.total_targets, d.world, d.rank)
    return first, count, args.total_targets, "strong"


def timed_steps(plan, stream, steps):
    """Back-to-back graph launches with an event pair around each: total ms and
    the per-step times (for the dispersion)."""
    import torch
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    torch.cuda.synchronize()
    ev[0].record(stream)
    for i in range(steps):
        plan.execute(stream.cuda_stream)
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    return ev[0].elapsed_time(ev[-1]), per


def gs_ours(args, d: Dist):
    import torch
    import paper_2008_12214_b200 as hg
    from paper_2008_12214_b200.shard import gather_batch_results, unit_seeds
    n, K = args.n, args.iters
    first, B, total, scaling = shard_of(args, d)
    hg.set_device(d.local)
    amp1 = hg.patterns.bench_target(n)
    seeds = unit_seeds(first, B)
    slm = hg.SlmSpec.full_circle_phase(args.levels) if args.levels > 2 else hg.SlmSpec.binary_phase()
    cfg = hg.IftaConfig(iterations=K, slm=slm, target=hg.TargetSpec(amp1))
    npix = n * n
    # pinned host inputs [B][n][n] (every target its own buffer, as cmd_batch jobs are)
    amps = torch.empty((B, n, n), dtype=torch.float64, pin_memory=True)
    amps[:] = torch.from_numpy(amp1)
    plan = hg.IftaPlan(cfg, n, n, B)
    plan.set_kernel_timing(True)  # CUDA events around each pass inside the graph (roofline kernel times)
    plan.upload(amps.numpy(), seeds=seeds)
    stream = torch.cuda.Stream()  # the graph runs on this stream; events are recorded on it
    for _ in range(args.warmup):
        plan.execute(stream.cuda_stream)
    torch.cuda.synchronize()
    d.barrier()
    with Clocks(d.local) as clk:
        ms, per_step = timed_steps(plan, stream, args.steps)
    d.barrier()
    ms_max = d.max(ms)
    launches = plan.launches() * args.steps
    # rank 0 gathers every target's levels and MSE trace (NCCL), after the timed steps
    _, lv, tr = plan.device_arrays()
    levels = torch.as_tensor(lv, device="cuda")
    trace = torch.as_tensor(tr, device="cuda")
    got = gather_batch_results(levels, trace, d.pg, d.world, d.rank, total)
    check = None
    if got is not None:
        glv, gtr = got
        check = {"gathered_targets": int(gtr.shape[0]), "gathered_level_bytes": int(glv.numel() * glv.element_size()),
                 "traces_finite_and_decreasing": bool(torch.isfinite(gtr).all().item()
                                                      and (gtr[:, -1] < gtr[:, 0]).all().item()),
                 "final_mse_mean": float(gtr[:, -1].mean().item()),
                 "levels_checksum": int(glv.sum(dtype=torch.int64).item())}
    kt = plan.kernel_times()  # the last timed step's passes, measured inside its graph
    prof = plan.profile(reps=5)
    prof["graph_row"], prof["graph_col"] = kt["row"], kt["col"]
    prof["iteration_in_graph"] = in_graph_iteration_ms(args, plan, amps, seeds, stream, ms / args.steps, B)
    res = {"ms": ms_max, "per_step_ms": per_step, "launches": launches, "clocks": clk.summary(),
           "profile_ms": prof, "check": check, "npix": npix, "B": B, "total": total, "scaling": scaling}
    if not args.no_e2e:
        res["e2e"] = gs_e2e(args, plan, amps, seeds, d, total)
    plan.close()
    return res


def in_graph_iteration_ms(args, plan, amps, seeds, stream, ms_step, B):
    """Per-iteration device time inside the real launch sequence: the same
    batch run with K1 = K/5 iterations, timed like the step, and
    (t(K) - t(K1)) / (K - K1); init, seed and trace reduction cancel."""
    import torch
    import paper_2008_12214_b200 as hg
    K = args.iters
    K1 = max(1, K // 5)
    if K - K1 < 4:
        return None
    cfg = hg.IftaConfig(iterations=K1, slm=plan.cfg.slm, target=plan.cfg.target)
    p1 = hg.IftaPlan(cfg, args.n, args.n, B)
    p1.upload(amps.numpy(), seeds=seeds)
    p1.execute(stream.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        p1.execute(stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    t1 = e0.elapsed_time(e1) / args.steps
    p1.close()
    return (ms_step - t1) / (K - K1)


def gs_e2e(args, plan, amps, seeds, d: Dist, total: int):
    """Same metric through the C ABI with host buffers.  Every step uploads
    that step's targets from pinned memory (H2D, validated on the device),
    runs, and reads back the levels and the MSE traces (D2H).  Two plans are
    used double-buffered, as a serving loop would: batch s+1 is uploaded while
    batch s computes, and batch s's results are read back while s+1 computes."""
    import torch
    import paper_2008_12214_b200 as hg
    from paper_2008_12214_b200 import _lib
    B, n, K = plan.batch, args.n, args.iters
    plan2 = hg.IftaPlan(plan.cfg, n, n, B)
    plans = [plan, plan2]
    lvs = [torch.empty((B, n, n), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    trs = [np.empty((B, K), np.float64) for _ in range(2)]
    ios = []
    for i in range(2):
        io = _lib.HgcIftaIo()
        io.amplitude = amps.data_ptr()
        io.seeds = seeds.ctypes.data
        io.levels8 = lvs[i].data_ptr()
        io.trace = trs[i].ctypes.data
        ios.append(io)
    L = _lib.lib
    h = [p._h for p in plans]

    def run(steps):
        _lib.check(L.hgc_ifta_plan_upload(h[0], C.byref(ios[0])))
        _lib.check(L.hgc_ifta_plan_execute(h[0], None))
        for s_ in range(steps):
            cur, nxt = s_ % 2, (s_ + 1) % 2
            if s_ + 1 < steps:
                _lib.check(L.hgc_ifta_plan_upload(h[nxt], C.byref(ios[nxt])))  # overlaps batch s on the GPU
                _lib.check(L.hgc_ifta_plan_execute(h[nxt], None))
            _lib.check(L.hgc_ifta_plan_download(h[cur], C.byref(ios[cur])))  # overlaps batch s+1

    run(2)  # warm (graph instantiation of the second plan)
    d.barrier()
    # steady-state serving loop: at least E2E_MIN_STEPS batches, so the first
    # batch's upload (exposed, nothing to overlap it with) is amortised as in
    # a long-running service; it is still inside the timed region
    steps = max(E2E_MIN_STEPS, args.steps)
    t0 = time.perf_counter()
    run(steps)
    dt = d.max(time.perf_counter() - t0)
    ok = bool(np.isfinite(trs[0]).all() and (trs[0][:, -1] < trs[0][:, 0]).all())
    plan2.close()
    units = total * K * steps
    return {"value": units / dt, "unit": "iterations/s", "h2d_bytes_per_step": int(B * n * n * 8 + B * 8),
            "d2h_bytes_per_step": int(B * n * n + B * K * 8), "steps": steps, "check_ok": ok,
            "api": "hgc_ifta_plan_upload/execute/download (C ABI, pinned host buffers, two plans double-buffered)"}


# ------------------------------------------------------------- OSPR (ours)
def ospr_ours(args, d: Dist):
    import torch
    import paper_2008_12214_b200 as hg
    from paper_2008_12214_b200 import _lib
    n, J, N = args.ospr_n, args.ospr_jobs, args.ospr_subframes
    amp = hg.patterns.bench_target(n)
    cfg = hg.OsprConfig(subframes=N, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp))
    seeds = np.arange(1 + d.rank * J, 1 + (d.rank + 1) * J, dtype=np.uint64)
    plan = hg.OsprPlan(cfg, n, n, J)
    plan.upload(amp, seeds=seeds)
    stream = torch.cuda.Stream()
    for _ in range(max(1, args.warmup)):
        plan.execute(stream.cuda_stream)
    torch.cuda.synchronize()
    d.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    steps = max(1, args.steps)
    for _ in range(steps):
        plan.execute(stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = d.max(e0.elapsed_time(e1))
    prof = plan.profile(reps=5)
    res = {"ms": ms, "steps": steps, "launches": plan.launches() * steps, "profile_ms": prof}
    if not args.no_e2e:  # double-buffered plans, as in gs_e2e
        plan2 = hg.OsprPlan(cfg, n, n, J)
        h = [plan._h, plan2._h]
        # binary frames come back as bit-planes (what a binary FLC SLM is fed): npix/8 bytes per frame
        lvs = [torch.empty((J, N, n * n // 8), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        fms = [np.empty((J, N)) for _ in range(2)]
        cms = [np.empty((J, N)) for _ in range(2)]
        ios = []
        for i in range(2):
            io = _lib.HgcOsprIo()
            io.amplitude = amp.ctypes.data
            io.seeds = seeds.ctypes.data
            io.levels1 = lvs[i].data_ptr()
            io.frame_mse, io.cumulative_mse = fms[i].ctypes.data, cms[i].ctypes.data
            ios.append(io)
        L = _lib.lib

        def run(k):
            _lib.check(L.hgc_ospr_plan_upload(h[0], C.byref(ios[0])))
            _lib.check(L.hgc_ospr_plan_execute(h[0], None))
            for s_ in range(k):
                cur, nxt = s_ % 2, (s_ + 1) % 2
                if s_ + 1 < k:
                    _lib.check(L.hgc_ospr_plan_upload(h[nxt], C.byref(ios[nxt])))
                    _lib.check(L.hgc_ospr_plan_execute(h[nxt], None))
                _lib.check(L.hgc_ospr_plan_download(h[cur], C.byref(ios[cur])))

        run(2)
        d.barrier()
        es = max(E2E_MIN_STEPS, steps)
        t0 = time.perf_counter()
        run(es)
        dt = d.max(time.perf_counter() - t0)
        plan2.close()
        res["e2e"] = {"value": d.world * J * N * es / dt, "unit": "subframes/s",
                      "h2d_bytes_per_step": int(n * n * 8 + J * 8), "d2h_bytes_per_step": int(J * N * n * n // 8 + 2 * J * N * 8),
                      "steps": es, "api": "hgc_ospr_plan_upload/execute/download (C ABI, pinned host buffers, "
                                          "two plans double-buffered; frames read back as bit-planes)"}
    plan.close()
    return res


def ospr_single_job(args, d: Dist):
    """ONE config-3 OSPR job (1024^2 binary, 24 subframes, seed 1) split into
    subframe blocks over the ranks (SURVEY §8 e2, strong scaling): per step
    each rank runs its block (jump-ahead stream start, chunked seeds), one
    NCCL all-gather of the block intensity sums, then its cumulative-MSE
    finish.  Device time per job, max over ranks."""
    import torch
    import paper_2008_12214_b200 as hg
    from paper_2008_12214_b200.shard import shard_range
    n, N = args.ospr_n, args.ospr_subframes
    amp = hg.patterns.bench_target(n)
    cfg = hg.OsprConfig(subframes=N, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=1)
    first, count = shard_range(N, d.world, d.rank)
    plan = hg.OsprBlockPlan(cfg, n, n, first, count)
    plan.upload(amp)
    st = torch.cuda.Stream()
    B = torch.as_tensor(plan.block_sum(), device="cuda")
    gathered = torch.empty((d.world, B.numel()), dtype=torch.float32, device="cuda")

    def job():
        plan.execute(st.cuda_stream)
        if d.pg:
            d.pg.all_gather_into_tensor(gathered, B)
        else:
            gathered[0].copy_(B)
        plan.finish(gathered.data_ptr(), d.world, d.rank, st.cuda_stream)

    with torch.cuda.stream(st):
        for _ in range(max(3, args.warmup)):
            job()
        torch.cuda.synchronize()
        d.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(st)
        for _ in range(reps):
            job()
        e1.record(st)
        torch.cuda.synchronize()
    ms = d.max(e0.elapsed_time(e1) / reps)
    out = plan.download()
    plan.close()
    return {"metric": "OSPR single-job latency", "ms_per_job": ms, "subframes_per_s": N / (ms / 1e3),
            "unit": "ms", "scaling": "strong", "n_gpus": d.world,
            "config": {"workload": f"ospr_{n}_binary single job (BASELINE config 3)", "subframes": N, "seed": 1,
                       "split": "contiguous subframe blocks per rank, one all-gather of npix fp32 block sums"},
            "final_error": float(out["final_error"][0]) if d.world == 1 else None}


def single_target_configs(args, d: Dist, peak: float):
    """BASELINE configs 1, 2 and 4: one target per run (replicas only across
    GPUs).  Device time of a whole run (init + K iterations +
    trace), resident inputs, best of 3 after a warm-up; roofline from the
    algorithmic bytes per iteration (GS 36 B/px, WGS 44 B/px)."""
    import torch
    import paper_2008_12214_b200 as hg
    out = {}
    specs = [("config1_gs_512_binary", 512, hg.SlmSpec.binary_phase(), hg.IftaVariant.GS, 100, None, 36),
             ("config2_wgs_1024_256level", 1024, hg.SlmSpec.full_circle_phase(256), hg.IftaVariant.WeightedGS, 200,
              None, 44),
             ("config4_fresnel_gs_2048_256level", 2048, hg.SlmSpec.full_circle_phase(256), hg.IftaVariant.GS, 100,
              hg.FresnelParams(532e-9, 0.1, 8e-6, 8e-6), 36)]
    st = torch.cuda.Stream()
    for name, n, slm, var, K, fr, bpp in specs:
        amp = hg.patterns.bench_target(n)
        cfg = hg.IftaConfig(variant=var, iterations=K, slm=slm, target=hg.TargetSpec(amp), seed=1)
        plan = hg.IftaPlan(cfg, n, n, 1, prop=hg.Propagator.fresnel(n, n, fr) if fr else None)
        plan.upload(amp[None], seeds=[1])
        plan.execute(st.cuda_stream)
        torch.cuda.synchronize()
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            plan.execute(st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        gbs = bpp * n * n * K / (best * 1e-3) / 1e9
        out[name] = {"ms_per_run": best, "iterations_per_s": K / (best * 1e-3), "achieved_gbs": gbs,
                     "frac_of_hbm_peak": gbs / peak, "bytes_per_px_iteration": bpp,
                     "note": "working set L2-resident (126 MB L2): the fraction can exceed what HBM alone allows"
                     if n * n * (bpp / 2) < 100e6 else "HBM-resident"}
        plan.close()
    return out


# ---------------------------------------------------- reference CPU path
# The reference's own run_ifta<float> / run_ospr (oracle/_ref/libhgref.so: its
# unmodified headers compiled here; a substitute f32 FFT since FFTW is absent
# on these hosts).  Nothing from the product package is imported on this path:
# the target comes from the reference's patterns::smooth_blobs +
# normalize_image (UnitEnergy), the SLM is a plain SlmSpec record.
TWO_PI = 6.283185307179586476925286766559


def ref_oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle
    ref = Oracle("reference")
    ref.set_fast_fft(True)  # the substitute's fast f32 path (FFTW stand-in); labelled in `sample`
    return ref


def ref_slm(levels):
    """SlmSpec::full_circle_phase(L) / binary_phase() (quantise.hpp:33-58)."""
    if levels > 2:
        return SimpleNamespace(mode=1, levels=levels, min_arg=0.0, max_arg=TWO_PI, full_circle=True, min_amp=0.0,
                               max_amp=1.0, illumination=None)
    return SimpleNamespace(mode=1, levels=2, min_arg=0.0, max_arg=TWO_PI / 2, full_circle=False, min_amp=0.0,
                           max_amp=1.0, illumination=None)


def ref_target(ref, n):
    return ref.normalize(ref.smooth_blobs(n, n), True)  # patterns.hpp:55-80, target.hpp:15-30


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def ref_gs_batch(ref, amp, slm, K, jobs, threads):
    """`jobs` independent run_ifta<float> jobs (seeds 1..jobs) on `threads` host
    threads (cmd_batch's job pool, runner.cpp:388-421); wall seconds + reports."""
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        reps = list(ex.map(lambda sd: ref.ifta(amp, slm, K, seed=int(sd)), range(1, jobs + 1)))
    return time.perf_counter() - t0, reps


def ref_gs_throughput(ref, n, levels, K_run, threads, k_lo=1, k_hi=3):
    """All-core throughput of the reference GS on a bounded sample (BASELINE.md
    §3): one job per host thread, each timed at k_lo and k_hi iterations.  The
    difference gives the per-iteration cost and the rest the per-job init
    (random-phase seed); `value` is the K_run-iteration job rate they imply,
    i.e. the same target-iterations/s the GPU line reports (init included)."""
    amp, slm = ref_target(ref, n), ref_slm(levels)
    t_lo, _ = ref_gs_batch(ref, amp, slm, k_lo, threads, threads)
    t_hi, reps = ref_gs_batch(ref, amp, slm, k_hi, threads, threads)
    t_it = max(t_hi - t_lo, 1e-9) / (k_hi - k_lo)  # wall per iteration of the whole job pool
    t_init = max(t_lo - k_lo * t_it, 0.0)
    value = threads * K_run / (K_run * t_it + t_init)
    return {"value": value, "per_iteration_rate": threads / t_it, "init_s_per_job_pool": t_init,
            "wall_s": t_lo + t_hi, "jobs": threads, "k": [k_lo, k_hi],
            "check_ok": all(np.isfinite(r.trace).all() for r in reps)}


def ref_gs_single_core(ref, n, levels, K=3):
    """One job on one thread, K iterations: the reference's own RunReport
    seconds and PhaseProfile (report.hpp:38-65) — seconds per iteration =
    (transform + constraint + metric) / K; the rest ("other") is the init."""
    r = ref.ifta(ref_target(ref, n), ref_slm(levels), K, seed=1)
    tr, cn, me, ot = r.profile
    return {"seconds_per_iteration": (tr + cn + me) / K, "iterations_per_s": K / (tr + cn + me),
            "run_seconds": r.seconds, "init_and_other_s": ot, "iterations": K,
            "profile": {"transform": tr, "constraint": cn, "metric": me, "other": ot}}


def ref_ospr_throughput(ref, n, subframes, threads):
    amp, slm = ref_target(ref, n), ref_slm(2)
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(lambda sd: ref.ospr(amp, slm, subframes, seed=int(sd)), range(1, threads + 1)))
    return threads * subframes / (time.perf_counter() - t0)


def base_config(args, d, total, scaling):
    per = args.targets if args.targets else f"{total} sharded over {d.world} GPU(s) (shard_range)"
    return {"workload": f"batch_gs_{args.n}_{args.levels}level (BASELINE config 5)", "resolution": args.n,
            "levels": args.levels, "iterations": args.iters, "total_targets": total, "targets_per_gpu": per,
            "seeds": "1 + target index", "target": "smooth_blobs + UnitEnergy (bench.cpp:115-116)",
            "scaling": scaling,
            "l2": "inputs larger than L2 (per GPU: targets x 128 MiB field + 64 MiB fp32 target)"}


def run_reference(args, d: Dist):
    """--impl reference: the reference's own CPU path on this host's cores,
    rank 0 only, on the same config / metric as our arm (bounded samples)."""
    if d.rank != 0:
        d.close()
        return
    ref = ref_oracle()
    threads = cpu_threads()
    total = args.targets * d.world if args.targets else args.total_targets
    for _ in range(args.warmup):
        ref_gs_throughput(ref, args.n, args.levels, args.iters, threads, 1, 2)
    runs = [ref_gs_throughput(ref, args.n, args.levels, args.iters, threads) for _ in range(args.steps)]
    vals = [r["value"] for r in runs]
    value = statistics.mean(vals)
    single = ref_gs_single_core(ref, args.n, args.levels)
    sample = (f"per step: {threads} concurrent jobs (one per host thread) of GS {args.n}^2 {args.levels}-level at "
              f"1 and 3 iterations; per-iteration cost = difference, init = remainder; value = the "
              f"{args.iters}-iteration job rate they imply; reference headers unmodified + substitute f32 FFT "
              f"(FFTW absent); CPU {cpu_model()}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": d.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(r["wall_s"] for r in runs),
            "value_sigma": statistics.stdev(vals) if len(vals) > 1 else 0.0,
            "higher_is_better": True, "scaling": "strong" if not args.targets else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": base_config(args, d, total, "strong" if not args.targets else "weak"),
            "product_package_imported": "paper_2008_12214_b200" in sys.modules,
            "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": threads, "kind": "reference",
                             "sample": sample, "cpu_model": cpu_model(), "single_core": single,
                             "per_iteration_rate_all_cores": statistics.mean(r["per_iteration_rate"] for r in runs)},
            "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    d.close()


def relaunch_if_needed(args):
    """--gpus N without torchrun: re-run this command under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous).  Under torchrun
    WORLD_SIZE must equal --gpus."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={ws}"}), flush=True)
            sys.exit(2)
        return
    if args.gpus <= 1:
        return
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def dry_run(args):
    """The multi-GPU plumbing without GPU work (gloo): world size, target
    shards, and the rank-0 gather of per-target levels + traces."""
    import torch
    from paper_2008_12214_b200.shard import gather_batch_results
    d = Dist(backend="gloo")
    first, B, total, scaling = shard_of(args, d)
    lv = torch.full((B, 4, 4), d.rank, dtype=torch.uint8)
    tr = torch.arange(first, first + B, dtype=torch.float64)[:, None].repeat(1, args.iters)
    got = gather_batch_results(lv, tr, d.pg, d.world, d.rank, total)
    if d.rank == 0:
        order_ok = bool((got[1][:, 0] == torch.arange(total, dtype=torch.float64)).all().item())
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": None, "n_gpus": d.world, "scaling": scaling,
                          "config": base_config(args, d, total, scaling),
                          "shards": [list(__import__("paper_2008_12214_b200.shard", fromlist=["x"]).shard_range(
                              total, d.world, r)) for r in range(d.world)] if not args.targets else None,
                          "gathered_targets": int(got[1].shape[0]), "gather_in_target_order": order_ok}), flush=True)
    d.close()


def main():
    args = parse()
    relaunch_if_needed(args)
    if args.dry_run:
        return dry_run(args)
    if args.impl == "reference":  # rank 0 alone works on the host cores: no process group needed
        return run_reference(args, Dist(collectives=False))
    d = Dist()
    peak, peak_kind = peaks()
    gs = gs_ours(args, d)
    weak = None
    if d.world > 1 and not args.targets:  # secondary line: 64 targets on EVERY GPU (weak scaling)
        wa = argparse.Namespace(**{**vars(args), "targets": args.total_targets, "no_e2e": True})
        w = gs_ours(wa, d)
        weak = {"value": w["total"] * args.iters * args.steps / (w["ms"] / 1e3), "unit": "iterations/s",
                "targets_per_gpu": args.total_targets, "ms_per_step": w["ms"] / args.steps, "scaling": "weak"}
    osp = None if args.no_ospr else ospr_ours(args, d)
    single = None if args.no_ospr else ospr_single_job(args, d)
    singles = single_target_configs(args, d, peak) if d.rank == 0 and not args.no_ospr else None
    cpu = None
    if d.rank == 0 and d.world == 1 and not args.no_cpu:
        ref = ref_oracle()
        threads = cpu_threads()
        r = ref_gs_throughput(ref, args.n, args.levels, args.iters, threads)
        cpu = {"value": r["value"], "unit": "iterations/s", "cores": threads, "kind": "reference",
               "sample": f"{threads} concurrent jobs (one per host thread) of GS {args.n}^2 {args.levels}-level at "
                         f"1 and 3 iterations; per-iteration cost = difference, init = remainder; value = the "
                         f"{args.iters}-iteration job rate they imply; reference headers + substitute f32 FFT "
                         f"(FFTW absent)",
               "cpu_model": cpu_model(), "per_iteration_rate_all_cores": r["per_iteration_rate"],
               "single_core": ref_gs_single_core(ref, args.n, args.levels)}
        if osp is not None:
            cpu["ospr"] = {"value": ref_ospr_throughput(ref, args.ospr_n, 2, threads), "unit": "subframes/s",
                           "cores": threads,
                           "sample": f"{threads} concurrent jobs x 2 subframes of OSPR {args.ospr_n}^2 binary"}
    if d.rank != 0:
        d.close()
        return
    B, K, npix = gs["B"], args.iters, gs["npix"]
    units = gs["total"] * K * args.steps
    value = units / (gs["ms"] / 1e3)
    per = gs["per_step_ms"]
    sigma_ms = statistics.stdev(per) if len(per) > 1 else 0.0
    pr = gs["profile_ms"]
    # pass times: CUDA events around each pass inside the timed step's graph
    # (the last timed step, iterations 1..K-1); repeated isolated launches of
    # each pass are reported beside them ("isolated_ms")
    g_row, g_col = pr["graph_row"], pr["graph_col"]
    row_gbs = GS_BYTES_PER_PX["row"] * npix * B / (g_row * 1e-3) / 1e9
    col_gbs = GS_BYTES_PER_PX["col"] * npix * B / (g_col * 1e-3) / 1e9
    dom = "col" if g_col >= g_row else "row"
    ach = col_gbs if dom == "col" else row_gbs
    it_ms = g_row + g_col
    it_gbs = GS_BYTES_PER_PX["iteration"] * npix * B / (it_ms * 1e-3) / 1e9
    step_gbs = GS_BYTES_PER_PX["iteration"] * npix * B * K / (gs["ms"] / args.steps * 1e-3) / 1e9
    ig = pr.get("iteration_in_graph")
    in_graph = None
    if ig:
        ig_gbs = GS_BYTES_PER_PX["iteration"] * npix * B / (ig * 1e-3) / 1e9
        in_graph = {"ms": ig, "achieved": ig_gbs, "frac": ig_gbs / peak, "per_gpu_it_per_s": 1e3 / ig * B,
                    "how": "(t(K) - t(K/5)) / (4K/5): whole batched runs on the bench stream, CUDA events"}
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(f"gs_{dom}")
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": d.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": gs["ms"] / args.steps,
        "ms_per_step_sigma": sigma_ms, "value_sigma": value * sigma_ms / (gs["ms"] / args.steps),
        "ms_per_step_each": per, "higher_is_better": True, "scaling": gs["scaling"],
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": base_config(args, d, gs["total"], gs["scaling"]),
        "roofline": {"bound": "hbm", "kernel": f"k_{dom} (fused {'replay-plane column' if dom == 'col' else 'aperture-plane row'} pass)",
                     "achieved": ach, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": ach / peak,
                     "traffic": traffic, "bytes_per_px": GS_BYTES_PER_PX[dom],
                     "kernel_ms": g_row if dom == "row" else g_col,
                     "kernel_ms_how": "CUDA events around the pass inside the timed step's graph, mean over iterations 1..K-1",
                     "iteration": {"bytes_per_px": 36, "kernel_ms": it_ms, "achieved": it_gbs, "frac": it_gbs / peak,
                                   "per_gpu_it_per_s": 1e3 / it_ms * B,
                                   "note": "kernel_ms = row + column pass inside the graph"},
                     "iteration_in_graph": in_graph,
                     "step_including_init": {"achieved": step_gbs, "frac": step_gbs / peak},
                     "row": {"ms": g_row, "achieved": row_gbs, "frac": row_gbs / peak, "isolated_ms": pr["row"]},
                     "col": {"ms": g_col, "achieved": col_gbs, "frac": col_gbs / peak, "isolated_ms": pr["col"]},
                     "seed_ms": pr["seed"]},
        "cpu_baseline": cpu, "e2e": gs.get("e2e"), "gpu_launches": gs["launches"], "clocks": gs["clocks"],
        "check": gs["check"], "weak_scaling": weak,
    }
    if osp is not None:
        J, N, on = args.ospr_jobs, args.ospr_subframes, args.ospr_n
        sub = d.world * J * N * osp["steps"] / (osp["ms"] / 1e3)
        po = osp["profile_ms"]
        onpx = on * on
        parts = {k: {"ms": po[k], "achieved": OSPR_BYTES_PER_PX[k] * onpx * J / (po[k] * 1e-3) / 1e9}
                 for k in ("seed", "col_inv", "row", "col_acc")}
        sf_ms = sum(po.values())
        sf_gbs = OSPR_BYTES_PER_PX["subframe"] * onpx * J / (sf_ms * 1e-3) / 1e9
        line["ospr"] = {"metric": "OSPR subframes/s", "value": sub, "unit": "subframes/s",
                        "config": {"workload": f"ospr_{on}_binary (BASELINE config 3)", "subframes": N,
                                   "jobs_per_gpu": J, "seeds": "1 + job index"},
                        "ms_per_step": osp["ms"] / osp["steps"], "gpu_launches": osp["launches"],
                        "roofline": {"bound": "hbm", "bytes_per_px": 49, "subframe_kernel_ms": sf_ms,
                                     "achieved": sf_gbs, "peak": peak, "frac": sf_gbs / peak, "kernels": parts},
                        "e2e": osp.get("e2e")}
        if cpu and "ospr" in cpu:
            line["ospr"]["cpu_baseline"] = cpu.pop("ospr")
        if single is not None:
            line["ospr"]["single_job"] = single
        line["gpu_launches"] += osp["launches"]
    if singles:
        line["configs"] = singles
    print(json.dumps(line), flush=True)
    d.close()


if __name__ == "__main__":
    main()
