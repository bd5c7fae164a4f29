"""GPU parity of OSPR subframe generation (run_ospr_impl, ospr.hpp:68-164).

Binary OSPR is checked free-running (0 level differences between
f32 and f64 FFTs), at the BASELINE config 3 size (1024^2, 24 subframes).
"""
import numpy as np
import pytest

from helpers import level_mismatches, mismatch_classes, record, rel

pytestmark = pytest.mark.gpu
hg = pytest.importorskip("paper_2008_12214_b200")


def ocfg(amp, N, seed, adaptive=False, gain=1.0):
    return hg.OsprConfig(variant=hg.OsprVariant.AdaptiveOspr if adaptive else hg.OsprVariant.Ospr, subframes=N,
                         slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=seed, feedback_gain=gain)


def ospr_frame_classes(oracle, amp, N, seed, got_levels, ref_levels, name):
    """Plain OSPR frames are independent given the seed (ospr.hpp:118-124):
    frame n's pre-quantisation field is P^-1 of draws [(n-1) npix, n npix) of
    Rng(seed).fork(0), which the oracle seeds bit-exactly.  Mismatches must be
    near / lowf (helpers.mismatch_classes), counted over all frames."""
    npix = amp.size
    slm = hg.SlmSpec.binary_phase()
    tot = {}
    for n in range(N):
        pre = oracle.fft2(oracle.seed_random_phase(amp, seed, n * npix).astype(np.complex128), +1)
        c = mismatch_classes(level_mismatches(got_levels[n], ref_levels[n]), pre, slm)
        for k, v in c.items():
            tot[k] = tot.get(k, 0) + v
    return record(name, tot)


def test_ospr_small_matches_reference_fixture(oracle):
    g = np.load(__file__.replace("test_gpu_ospr.py", "golden/ref_runs.npz"))
    run = hg.run_ospr(ocfg(g["amp32"], 6, 42))
    cls = ospr_frame_classes(oracle, g["amp32"], 6, 42, run.set.levels, g["ospr32_levels"], "ospr32_binary_6_fixture")
    assert cls["bad"] == 0, cls
    assert np.max(np.abs(np.array(run.set.per_frame_mse) - g["ospr32_frame_mse"]) / g["ospr32_frame_mse"]) < 1e-4
    assert np.max(np.abs(run.report.trace.values() - g["ospr32_cum_mse"]) / g["ospr32_cum_mse"]) < 1e-4
    assert np.allclose(run.set.mean_intensity, g["ospr32_mean_intensity"], rtol=1e-4, atol=1e-7)


def test_config3_ospr_1024_binary_24_subframes(oracle):
    amp = hg.patterns.bench_target(1024)
    run = hg.run_ospr(ocfg(amp, 24, 1))
    ref = oracle.ospr(amp, hg.SlmSpec.binary_phase(), 24, seed=1)
    cls = ospr_frame_classes(oracle, amp, 24, 1, run.set.levels, ref.levels, "config3_ospr_1024_binary_24")
    assert cls["bad"] == 0, cls  # SURVEY §0.5 probe: 0 of 1,572,864 at 256^2
    assert np.max(np.abs(np.array(run.set.per_frame_mse) - ref.frame_mse) / ref.frame_mse) < 1e-4
    assert np.max(np.abs(run.report.trace.values() - ref.cumulative_mse) / ref.cumulative_mse) < 1e-4
    assert rel(hg.subframe_mse_statistic(run.set.per_frame_mse), oracle.subframe_mse_statistic(ref.frame_mse)) < 1e-4


def test_single_subframe_is_one_shot_pipeline():
    # test_ospr.cpp:25-42: N=1 == quantise(ifft(seed(fork(0))))
    amp = hg.patterns.bench_target(64)
    run = hg.run_ospr(ocfg(amp, 1, 41))
    f = hg.quantise_field(hg.fft_inverse(hg.seed_random_phase(amp, 41)), hg.SlmSpec.binary_phase())
    assert np.array_equal(run.set.frames[0], f)
    R = hg.fft_forward(f)
    assert rel(run.set.per_frame_mse[0], hg.mse(amp, R)) < 1e-5


def test_adaptive_matches_oracle_and_reductions(oracle):
    amp = hg.patterns.bench_target(64)
    plain = hg.run_ospr(ocfg(amp, 6, 42))
    a0 = hg.run_adaptive_ospr(ocfg(amp, 6, 42, adaptive=True, gain=0.0))
    assert np.array_equal(a0.set.levels, plain.set.levels)  # test_ospr.cpp:44-58
    assert a0.report.algorithm == "adaptive_ospr" and plain.report.algorithm == "ospr"
    a1 = hg.run_adaptive_ospr(ocfg(amp, 4, 43, adaptive=True, gain=1.0))
    ref = oracle.ospr(amp, hg.SlmSpec.binary_phase(), 4, seed=43, adaptive=True, gain=1.0)
    assert level_mismatches(a1.set.levels, ref.levels).sum() <= 8
    assert np.max(np.abs(a1.report.trace.values() - ref.cumulative_mse) / ref.cumulative_mse) < 1e-3


def test_batch_jobs_equal_single_runs():
    amp = hg.patterns.bench_target(128)
    runs = hg.run_ospr_batch(ocfg(amp, 5, 1), seeds=[1, 2, 3])
    for j, s in enumerate([1, 2, 3]):
        single = hg.run_ospr(ocfg(amp, 5, s))
        assert np.array_equal(runs[j].set.levels, single.set.levels)
        assert runs[j].report.final_error == single.report.final_error


def test_traces_and_averaging():
    amp = hg.patterns.bench_target(64)
    run = hg.run_ospr(ocfg(amp, 16, 1))
    tr = run.report.trace.values()
    assert run.report.trace.name == "cumulative_mse" and len(tr) == 16
    assert run.report.extra_traces[0].name == "frame_mse"
    assert tr[-1] < 0.5 * tr[0]  # test_ospr.cpp:466-479
    assert run.report.evaluations == 16
    for fr in run.set.frames:
        d = np.minimum(np.abs(fr - 1), np.abs(fr + 1))
        assert np.max(d) < 1e-6


def test_ospr_validation():
    amp = hg.patterns.bench_target(16)
    with pytest.raises(ValueError, match="subframes"):
        hg.run_ospr(ocfg(amp, 0, 1))
    with pytest.raises(ValueError, match="feedback_gain"):
        hg.run_adaptive_ospr(ocfg(amp, 3, 1, adaptive=True, gain=1.5))
    with pytest.raises(ValueError, match="variant mismatch"):
        hg.run_adaptive_ospr(ocfg(amp, 3, 1))


@pytest.mark.parametrize("adaptive", [False, True])
def test_ospr_chunked_stream_matches_oracle(oracle, monkeypatch, adaptive):
    """Each subframe's draws split across 5 CTAs; the chunk start states move
    by npix draws per subframe (k_mt_jump in place).  Same levels as the
    sequential stream (ospr.hpp:89, :118)."""
    monkeypatch.setenv("HG_SEED_CHUNKS", "5")
    amp = hg.patterns.bench_target(64)
    N = 5
    run = (hg.run_adaptive_ospr if adaptive else hg.run_ospr)(ocfg(amp, N, 17, adaptive=adaptive, gain=0.7))
    ref = oracle.ospr(amp, hg.SlmSpec.binary_phase(), N, seed=17, adaptive=adaptive, gain=0.7)
    assert level_mismatches(run.set.levels, ref.levels).sum() <= 2 * N
    assert np.max(np.abs(run.report.trace.values() - ref.cumulative_mse) / ref.cumulative_mse) < 1e-3


def _block_run(cfg, amp, G):
    """Subframe-block sharding with G blocks on one GPU: the
    all-gather is a stack of the block sums (the GPU ranks use NCCL)."""
    import torch
    ny, nx = amp.shape
    N = cfg.subframes
    plans = []
    for g in range(G):
        first, count = hg.shard.shard_range(N, G, g)
        p = hg.OsprBlockPlan(cfg, nx, ny, first, count)
        p.upload(amp)
        p.execute()
        plans.append(p)
    torch.cuda.synchronize()
    gathered = torch.stack([torch.as_tensor(p.block_sum(), device="cuda") for p in plans]).contiguous()
    outs = []
    for g, p in enumerate(plans):
        p.finish(gathered.data_ptr(), G, g)
        outs.append(p.download())
    return outs


@pytest.mark.parametrize("n,N,G", [(64, 7, 1), (64, 7, 3), (256, 8, 4), (1024, 24, 8)])
def test_ospr_subframe_blocks_match_unsharded(oracle, n, N, G):
    amp = hg.patterns.bench_target(n)
    cfg = ocfg(amp, N, 1)
    outs = _block_run(cfg, amp, G)
    levels = np.concatenate([o["levels"][0] for o in outs])
    fm = np.concatenate([o["frame_mse"][0] for o in outs])
    cm = np.concatenate([o["cumulative_mse"][0] for o in outs])
    ref = oracle.ospr(amp, hg.SlmSpec.binary_phase(), N, seed=1)
    assert level_mismatches(levels, ref.levels).sum() <= N
    assert np.max(np.abs(fm - ref.frame_mse) / ref.frame_mse) < 1e-4
    assert np.max(np.abs(cm - ref.cumulative_mse) / ref.cumulative_mse) < 1e-4
    for o in outs:  # every block holds the job's mean intensity after finish
        assert np.allclose(o["mean_intensity"][0], ref.mean_intensity, rtol=1e-4, atol=1e-7)


def test_ospr_sharded_driver_world1(oracle):
    """shard.run_ospr_sharded end to end at world size 1 (no process group)."""
    amp = hg.patterns.bench_target(128)
    cfg = ocfg(amp, 6, 3)
    out = hg.shard.run_ospr_sharded(cfg, None, 1, 0)
    ref = oracle.ospr(amp, hg.SlmSpec.binary_phase(), 6, seed=3)
    assert level_mismatches(out["levels"], ref.levels).sum() <= 6
    assert np.max(np.abs(out["cumulative_mse"] - ref.cumulative_mse) / ref.cumulative_mse) < 1e-4


def test_ospr_roi_with_tma_tiles_matches_oracle(oracle):
    """OSPR with an ROI (masked MSE, ospr.hpp:138-145) at 512^2, where the
    accumulating column pass lands its tiles by TMA."""
    n = 512
    amp = np.zeros((n, n))
    roi = np.zeros((n, n), np.uint8)
    amp[128:384, 128:384] = hg.patterns.letter_a(256, 256)
    roi[128:384, 128:384] = 1
    amp = hg.normalize_image(amp, hg.Normalization.UnitEnergy)
    cfg = ocfg(amp, 4, 12)
    cfg.target.roi = roi
    run = hg.run_ospr(cfg)
    ref = oracle.ospr(amp, hg.SlmSpec.binary_phase(), 4, seed=12, roi=roi)
    assert level_mismatches(run.set.levels, ref.levels).sum() <= 8
    assert np.max(np.abs(run.report.trace.values() - ref.cumulative_mse) / ref.cumulative_mse) < 1e-4
    assert np.max(np.abs(np.array(run.set.per_frame_mse) - ref.frame_mse) / ref.frame_mse) < 1e-4


def test_fresnel_ospr_matches_composed_oracle(oracle):
    # extension: OSPR with the Fresnel propagator.  The reference
    # rejects it (src/config.cpp:443-445), so the oracle is composed from its
    # pinned parts: seed_random_phase (rng.hpp:54-67), Propagator::inverse /
    # forward (propagation.hpp:81-95), the quantiser and the OSPR accumulation
    # (ospr.hpp:118-146), in double.  Parity-unpinned by construction.
    n, N, seed = 256, 6, 11
    amp = hg.patterns.bench_target(n)
    fr = (532e-9, 0.1, 8e-6, 8e-6)
    prop = hg.Propagator.fresnel(n, n, hg.FresnelParams(*fr))
    slm = hg.SlmSpec.binary_phase()
    run = hg.run_ospr(ocfg(amp, N, seed), prop=prop)
    q = oracle.fresnel_q(n, n, *fr).astype(np.complex128)
    states = np.array([1.0 + 0j, -1.0 + 0j])
    S = np.zeros((n, n))
    tot = {}
    for k in range(N):
        pre = oracle.fft2(oracle.seed_random_phase(amp, seed, k * amp.size).astype(np.complex128), +1) * np.conj(q)
        cls = mismatch_classes(level_mismatches(run.set.levels[k], _binary_levels(pre)), pre, slm)
        for key, v in cls.items():
            tot[key] = tot.get(key, 0) + v
        R = oracle.fft2(states[run.set.levels[k].astype(np.int64)] * q, -1)  # the GPU's own frame, forward-propagated
        I = np.abs(R) ** 2
        S += I
        assert rel(run.set.per_frame_mse[k], float(np.mean((amp - np.sqrt(I)) ** 2))) < 1e-4
        assert rel(run.report.trace.values()[k], float(np.mean((amp - np.sqrt(S / (k + 1))) ** 2))) < 1e-4
    record("fresnel_ospr_256_binary_6", tot)
    assert tot["bad"] == 0, tot
    assert np.allclose(run.set.mean_intensity, S / N, rtol=1e-4, atol=1e-9)


def _binary_levels(f):
    # binary_phase decision: level 1 iff Re(f) < 0 (quantise.hpp:175-198)
    return (f.real < 0).astype(np.int64)
