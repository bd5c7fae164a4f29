"""GPU parity of the IFTA loop (run_ifta, ifta.hpp:86-235) against the oracle.

Parity contract (BASELINE north_star): quantised levels
bit-exact except pixels whose pre-quantisation angle lies within 1e-5 rad of a
decision threshold; replay-field MSE within 1e-4 relative.  Multi-level GS is
chaotic at the level granularity between ANY two differently-rounded FFTs
(SURVEY §0.5), so multi-level configs are checked lock-step: one GPU iteration
from the oracle's own replay snapshot R_{k-1}.  Binary GS is checked
free-running.
"""
import numpy as np
import pytest

from helpers import level_mismatches, mismatch_classes, phase_threshold_distance, record, rel

pytestmark = pytest.mark.gpu
hg = pytest.importorskip("paper_2008_12214_b200")

MSE_TOL = 1e-4
NEAR = 1e-5


def cfg_for(amp, slm, K, seed=1, variant=None, **kw):
    c = hg.IftaConfig(iterations=K, slm=slm, target=hg.TargetSpec(amp), seed=seed, **kw)
    if variant is not None:
        c.variant = variant
    return c


def lockstep(oracle, amp, slm, k, variant="gs", fresnel=None, scale_free=False):
    """Oracle runs to iteration k with a snapshot of R_{k-1}; GPU runs one
    iteration from it.  Returns (mismatch mask, near-threshold mask, mse pair)."""
    ref_k = oracle.ifta(amp, slm, k, seed=5, variant=variant, snapshot_iter=k, fresnel=fresnel,
                        scale_freedom=scale_free)
    # the oracle's pre-quantisation field of iteration k (f before snapping)
    pre = oracle.fft2(ref_k.snap_r, +1)
    if fresnel is not None:
        q = oracle.fresnel_q(amp.shape[1], amp.shape[0], *fresnel)
        pre = pre * np.conj(q)
    c = cfg_for(amp, slm, 1, variant=hg.IftaVariant.WeightedGS if variant == "wgs" else None)
    c.init_phase = hg.InitPhase.Given
    c.target.freedoms.scale = scale_free
    prop = None if fresnel is None else hg.Propagator.fresnel(amp.shape[1], amp.shape[0], hg.FresnelParams(*fresnel))
    w = None if ref_k.snap_w is None else ref_k.snap_w.astype(np.float32)
    rep = hg.run_ifta(c, prop, init_field=ref_k.snap_r, init_weights=w)
    mism = level_mismatches(rep.levels, ref_k.levels)
    cls = mismatch_classes(mism, pre, slm)
    near = phase_threshold_distance(pre, slm) < NEAR
    return mism, near, (rep.final_error, ref_k.trace[-1]), rep, ref_k, cls


def free_running_classes(oracle, amp, slm, K, seed, name, variant=None, gpu_levels=None, **okw):
    """Free-running GPU vs oracle after K iterations.  The GPU's own state
    before iteration K (checkpoint of a K-1 run, bit-identical to the K run's)
    predicts its pre-quantisation field P^-1(R_{K-1}); the oracle's comes from
    its R_{K-1} snapshot.  Mismatches must be near / lowf / propagated
    (helpers.mismatch_classes); returns the counts (recorded)."""
    _, snaps = oracle.ifta_snaps(amp, slm, K, [K], seed=seed, variant=variant or "gs", **okw)
    R_ref, _, lv_ref = snaps[K]
    pre = oracle.fft2(R_ref.astype(np.complex128), +1)
    pred = None
    if K > 1:
        c = cfg_for(amp, slm, K - 1, seed=seed,
                    variant=hg.IftaVariant.WeightedGS if variant == "wgs" else None)
        ck = hg.run_ifta(c, checkpoint=True)
        pred = oracle.fft2(ck.replay.astype(np.complex128), +1)
    return record(name, mismatch_classes(level_mismatches(gpu_levels, lv_ref), pre, slm, pred))


def test_gs_small_free_running_matches_reference_fixture(oracle):
    g = np.load(__file__.replace("test_gpu_ifta.py", "golden/ref_runs.npz"))
    amp = g["amp64"]
    slm = hg.SlmSpec.binary_phase()
    rep = hg.run_gs(cfg_for(amp, slm, 20, seed=1))
    # the fixture is the reference's own run (tests/golden/make_golden.py)
    assert np.array_equal(oracle.ifta(amp, slm, 20, seed=1).levels, g["gs64_bin_levels"])
    cls = free_running_classes(oracle, amp, slm, 20, 1, "gs64_binary_20it_fixture", gpu_levels=rep.levels)
    assert cls["bad"] == 0, cls
    assert np.max(np.abs(rep.trace.values() - g["gs64_bin_trace"]) / g["gs64_bin_trace"]) < MSE_TOL


def test_config1_gs_512_binary_100it_free_running(oracle):
    # BASELINE config 1: GS Fourier 512x512 binary phase, 100 iterations
    amp = hg.patterns.bench_target(512)
    slm = hg.SlmSpec.binary_phase()
    rep = hg.run_gs(cfg_for(amp, slm, 100, seed=1))
    ref = oracle.ifta(amp, slm, 100, seed=1)
    cls = free_running_classes(oracle, amp, slm, 100, 1, "config1_gs_512_binary_100it", gpu_levels=rep.levels)
    assert cls["bad"] == 0, cls  # SURVEY §0.5 probe: 0 of 262,144 expected
    tr = rep.trace.values()
    assert np.max(np.abs(tr - ref.trace) / ref.trace) < MSE_TOL
    assert rep.final_error == tr[-1] and len(tr) == 100


@pytest.mark.parametrize("k", [1, 2, 10])
def test_gs_256level_lockstep(oracle, k):
    amp = hg.patterns.bench_target(256)
    *_, (m_gpu, m_ref), _, _, cls = lockstep(oracle, amp, hg.SlmSpec.full_circle_phase(256), k)
    record(f"gs256_256level_lockstep/k={k}", cls)
    assert cls["bad"] == 0, cls
    assert rel(m_gpu, m_ref) < MSE_TOL


@pytest.mark.parametrize("k", [1, 3])
def test_config2_wgs_1024_256level_lockstep(oracle, k):
    # BASELINE config 2 geometry: WGS 1024x1024, 256 levels (lock-step at iteration k;
    # the weight rule inside the window: tests/test_gpu_lockstep.py)
    amp = hg.patterns.bench_target(1024)
    *_, (m_gpu, m_ref), _, _, cls = lockstep(oracle, amp, hg.SlmSpec.full_circle_phase(256), k, variant="wgs")
    record(f"config2_wgs_1024_lockstep1/k={k}", cls)
    assert cls["bad"] == 0, cls
    assert rel(m_gpu, m_ref) < MSE_TOL


@pytest.mark.parametrize("k", [1, 2])
def test_config4_fresnel_lockstep(oracle, k):
    # BASELINE config 4 physics (lambda 532 nm, z 0.1 m, 8 um pitch) at 512^2
    amp = hg.patterns.bench_target(512)
    fr = (532e-9, 0.1, 8e-6, 8e-6)
    *_, (m_gpu, m_ref), _, _, cls = lockstep(oracle, amp, hg.SlmSpec.full_circle_phase(256), k, fresnel=fr)
    record(f"fresnel512_lockstep1/k={k}", cls)
    assert cls["bad"] == 0, cls
    assert rel(m_gpu, m_ref) < MSE_TOL


def test_config5_gs_4096_256level_lockstep(oracle):
    # BASELINE config 5 geometry at full size (4096^2, 256 levels): the
    # benchmark's own kernels run one iteration from the oracle's R_1
    amp = hg.patterns.bench_target(4096)
    *_, (m_gpu, m_ref), _, _, cls = lockstep(oracle, amp, hg.SlmSpec.full_circle_phase(256), 2)
    record("config5_gs_4096_lockstep1/k=2", cls)
    assert cls["bad"] == 0, cls
    assert rel(m_gpu, m_ref) < MSE_TOL


def test_config4_fresnel_2048_lockstep(oracle):
    # BASELINE config 4 at full size: Fresnel GS 2048^2, 256 levels, typical physics
    amp = hg.patterns.bench_target(2048)
    fr = (532e-9, 0.1, 8e-6, 8e-6)
    *_, (m_gpu, m_ref), _, _, cls = lockstep(oracle, amp, hg.SlmSpec.full_circle_phase(256), 1, fresnel=fr)
    record("config4_fresnel_2048_lockstep1/k=1", cls)
    assert cls["bad"] == 0, cls
    assert rel(m_gpu, m_ref) < MSE_TOL


def test_multilevel_free_running_band(oracle):
    # f32 vs f64 GS band of the reference (test_ifta.cpp:282-288): 2e-2 relative
    amp = hg.patterns.bench_target(128)
    slm = hg.SlmSpec.full_circle_phase(256)
    rep = hg.run_gs(cfg_for(amp, slm, 50, seed=2))
    ref = oracle.ifta(amp, slm, 50, seed=2)
    assert rel(rep.final_error, ref.trace[-1]) < 2e-2
    assert rep.final_error < rep.trace.points[0][1]


def test_wgs_unit_clamp_equals_gs():
    # test_ifta.cpp:154-168
    amp = hg.patterns.smooth_blobs(64, 64)
    slm = hg.SlmSpec.full_circle_phase(256)
    gs = hg.run_gs(cfg_for(amp, slm, 12, seed=7))
    w = cfg_for(amp, slm, 12, seed=7, variant=hg.IftaVariant.WeightedGS, weight_clamp_lo=1.0, weight_clamp_hi=1.0)
    wgs = hg.run_weighted_gs(w)
    assert np.array_equal(wgs.levels, gs.levels) and wgs.final_error == gs.final_error
    assert wgs.algorithm == "wgs"


def test_lt_full_area_equals_gs():
    # test_ifta.cpp:170-184
    amp = hg.normalize_image(hg.patterns.letter_a(64, 64), hg.Normalization.UnitEnergy)
    slm = hg.SlmSpec.full_circle_phase(256)
    gs = hg.run_gs(cfg_for(amp, slm, 12, seed=7))
    lt = hg.run_liu_taghizadeh(cfg_for(amp, slm, 12, seed=7, variant=hg.IftaVariant.LiuTaghizadeh,
                                       lt_initial_fraction=1.0))
    assert np.array_equal(lt.levels, gs.levels) and lt.final_error == gs.final_error


def test_lt_roi_matches_oracle(oracle):
    amp = np.zeros((64, 64))
    roi = np.zeros((64, 64), np.uint8)
    amp[16:48, 16:48] = hg.patterns.letter_a(32, 32)
    roi[16:48, 16:48] = 1
    amp = hg.normalize_image(amp, hg.Normalization.UnitEnergy)
    slm = hg.SlmSpec.binary_phase()
    c = cfg_for(amp, slm, 30, seed=2, variant=hg.IftaVariant.LiuTaghizadeh)
    c.target.roi = roi
    c.target.freedoms.amplitude_outside_roi = True
    rep = hg.run_liu_taghizadeh(c)
    ref = oracle.ifta(amp, slm, 30, seed=2, variant="lt", roi=roi, amp_outside_roi=True)
    # (LT's schedule depends on K, so no K-1 checkpoint prediction: near / lowf classes only)
    _, snaps = oracle.ifta_snaps(amp, slm, 30, [30], seed=2, variant="lt", roi=roi, amp_outside_roi=True)
    pre = oracle.fft2(snaps[30][0].astype(np.complex128), +1)
    cls = record("lt_roi_64_binary_30it", mismatch_classes(level_mismatches(rep.levels, ref.levels), pre, slm))
    assert cls["bad"] == 0, cls
    assert np.max(np.abs(rep.trace.values() - ref.trace) / ref.trace) < MSE_TOL


def test_roi_strict_and_scale_free_match_oracle(oracle):
    amp = np.zeros((64, 64))
    roi = np.zeros((64, 64), np.uint8)
    amp[16:48, 16:48] = hg.patterns.checkerboard(32, 32, 4)
    roi[16:48, 16:48] = 1
    amp = hg.normalize_image(amp, hg.Normalization.UnitEnergy)
    slm = hg.SlmSpec.binary_phase()
    c = cfg_for(amp, slm, 10, seed=21)
    c.target.roi = roi
    c.target.freedoms.scale = True
    rep = hg.run_gs(c)
    ref = oracle.ifta(amp, slm, 10, seed=21, roi=roi, scale_freedom=True)
    _, snaps = oracle.ifta_snaps(amp, slm, 10, [10], seed=21, roi=roi, scale_freedom=True)
    pre = oracle.fft2(snaps[10][0].astype(np.complex128), +1)
    c9 = cfg_for(amp, slm, 9, seed=21)
    c9.target.roi = roi
    c9.target.freedoms.scale = True
    pred = oracle.fft2(hg.run_ifta(c9, checkpoint=True).replay.astype(np.complex128), +1)
    cls = record("roi_scale_free_64_binary_10it",
                 mismatch_classes(level_mismatches(rep.levels, ref.levels), pre, slm, pred))
    assert cls["bad"] == 0, cls
    assert np.max(np.abs(rep.trace.values() - ref.trace) / ref.trace) < MSE_TOL


def test_fixed_point_target_phase(oracle):
    # test_ifta.cpp:59-91: exactly representable target with phase, no phase freedom
    r = np.random.default_rng(800)
    h = np.exp(1j * r.uniform(0, hg.TWO_PI, (32, 32))).astype(np.complex64)
    slm = hg.SlmSpec.full_circle_phase(256)
    h = hg.quantise_field(h, slm)
    R = oracle.fft2(h.astype(np.complex128), -1)
    amp = np.abs(R)
    turns = np.angle(R) / hg.TWO_PI
    turns -= np.floor(turns)
    c = cfg_for(amp, slm, 1, seed=0)
    c.target.phase = turns
    c.target.freedoms.phase = False
    rep = hg.run_gs(c)
    assert rep.final_error < 1e-10
    assert np.count_nonzero(rep.hologram != h) <= 2


def test_replay_is_transform_of_hologram():
    # test_ifta.cpp:129-139 (same pass order -> bit-identical)
    amp = hg.normalize_image(hg.patterns.letter_a(64, 64), hg.Normalization.UnitEnergy)
    rep = hg.run_gs(cfg_for(amp, hg.SlmSpec.full_circle_phase(256), 8, seed=5))
    R = hg.fft_forward(rep.hologram)
    assert np.max(np.abs(R - rep.replay)) <= 1e-6 * np.max(np.abs(R))
    assert rel(hg.mse(amp, rep.replay), rep.final_error) < 1e-5


def test_fresnel_replay_is_propagation_of_hologram():
    # test_ifta.cpp:322-336
    p = hg.FresnelParams(532e-9, 0.15, 8e-6, 8e-6)
    prop = hg.Propagator.fresnel(64, 64, p)
    amp = hg.normalize_image(hg.patterns.letter_a(64, 64), hg.Normalization.UnitEnergy)
    rep = hg.run_gs(cfg_for(amp, hg.SlmSpec.full_circle_phase(256), 15, seed=9), prop)
    assert rep.final_error < rep.trace.points[0][1]
    R = prop.forward(rep.hologram)
    assert np.max(np.abs(R - rep.replay)) <= 1e-6 * np.max(np.abs(R))


def test_determinism_and_seed_sensitivity():
    amp = hg.patterns.smooth_blobs(64, 64)
    slm = hg.SlmSpec.full_circle_phase(256)
    a = hg.run_gs(cfg_for(amp, slm, 10, seed=99))
    b = hg.run_gs(cfg_for(amp, slm, 10, seed=99))
    assert np.array_equal(a.levels, b.levels) and a.final_error == b.final_error
    assert np.array_equal(a.replay.view(np.uint32), b.replay.view(np.uint32))
    c = hg.run_gs(cfg_for(amp, slm, 10, seed=100))
    assert not np.array_equal(a.levels, c.levels)
    e = cfg_for(amp, slm, 5, seed=1); e.init_phase = hg.InitPhase.Flat
    f = cfg_for(amp, slm, 5, seed=2); f.init_phase = hg.InitPhase.Flat
    assert np.array_equal(hg.run_gs(e).levels, hg.run_gs(f).levels)


def test_batch_equals_single():
    n = 128
    amps = np.stack([hg.patterns.bench_target(n) * (1 + 0.1 * t) for t in range(3)])
    slm = hg.SlmSpec.full_circle_phase(256)
    cfg = cfg_for(amps[0], slm, 6, seed=1)
    reps = hg.run_ifta_batch(cfg, amps, seeds=[1, 2, 3])
    for t in range(3):
        single = hg.run_gs(cfg_for(amps[t], slm, 6, seed=1 + t))
        assert np.array_equal(reps[t].levels, single.levels)
        # the launch's column width may differ between batch and single runs
        # (col_width_rt), which only reorders the MSE partial sums
        assert abs(reps[t].final_error - single.final_error) <= 1e-7 * single.final_error


def test_validation_errors():
    amp = hg.patterns.checkerboard(16, 16, 2)
    with pytest.raises(ValueError, match="iterations"):
        hg.run_gs(cfg_for(amp, hg.SlmSpec.binary_phase(), 0))
    bad = cfg_for(amp, hg.SlmSpec.binary_phase(), 3)
    bad.weight_clamp_lo = 0.0
    with pytest.raises(ValueError, match="clamp"):
        hg.run_gs(bad)
    neg = amp.copy(); neg[0, 3] = -0.5
    with pytest.raises(ValueError, match="non-negative"):
        hg.run_gs(cfg_for(neg, hg.SlmSpec.binary_phase(), 3))
    with pytest.raises(ValueError, match="variant mismatch"):
        hg.run_weighted_gs(cfg_for(amp, hg.SlmSpec.binary_phase(), 3))
    with pytest.raises(hg.HgcUnsupported):
        hg.run_gs(cfg_for(np.ones((12, 12)), hg.SlmSpec.binary_phase(), 3))


def test_plan_upload_is_async_and_download_reports_invalid_target():
    """Plan API: upload no longer blocks on target validation; a non-finite
    target is reported (same message as TargetSpec::validate) by download,
    and a valid re-upload on the same plan runs normally."""
    amp = hg.patterns.bench_target(64)
    cfg = hg.IftaConfig(iterations=3, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=1)
    p = hg.IftaPlan(cfg, 64, 64, 2)
    bad = np.broadcast_to(amp, (2, 64, 64)).copy()
    bad[1, 3, 5] = np.nan
    p.upload(bad, seeds=[1, 2])
    p.execute()
    with pytest.raises(ValueError, match="non-finite"):
        p.download()
    p.upload(np.broadcast_to(amp, (2, 64, 64)), seeds=[1, 2])
    p.execute()
    out = p.download()
    assert np.isfinite(out.trace).all()


def _roi_target(n, inner):
    amp = np.zeros((n, n))
    roi = np.zeros((n, n), np.uint8)
    a, b = n // 4, n // 4 + inner
    amp[a:b, a:b] = hg.patterns.letter_a(inner, inner)
    roi[a:b, a:b] = 1
    return hg.normalize_image(amp, hg.Normalization.UnitEnergy), roi


@pytest.mark.parametrize("case", ["lt_roi", "roi_scale_free", "wgs_roi", "target_phase"])
def test_generic_constraint_with_tma_tiles_matches_oracle(oracle, case):
    """The generic replay-plane constraint (ROI, LT rectangle, scale freedom,
    WGS weights, fixed target phase; ifta.hpp:185-224) at 512^2, where the
    column pass moves its tiles by TMA: binary free-running vs the oracle."""
    n = 512
    amp, roi = _roi_target(n, 256)
    slm = hg.SlmSpec.binary_phase()
    K = 8
    if case == "lt_roi":
        c = cfg_for(amp, slm, K, seed=2, variant=hg.IftaVariant.LiuTaghizadeh)
        c.target.roi = roi
        c.target.freedoms.amplitude_outside_roi = True
        rep = hg.run_liu_taghizadeh(c)
        ref = oracle.ifta(amp, slm, K, seed=2, variant="lt", roi=roi, amp_outside_roi=True)
    elif case == "roi_scale_free":
        c = cfg_for(amp, slm, K, seed=21)
        c.target.roi = roi
        c.target.freedoms.scale = True
        rep = hg.run_gs(c)
        ref = oracle.ifta(amp, slm, K, seed=21, roi=roi, scale_freedom=True)
    elif case == "wgs_roi":
        c = cfg_for(amp, slm, K, seed=4, variant=hg.IftaVariant.WeightedGS)
        c.target.roi = roi
        rep = hg.run_weighted_gs(c)
        ref = oracle.ifta(amp, slm, K, seed=4, variant="wgs", roi=roi)
    else:
        turns = np.random.default_rng(5).uniform(0, 1, (n, n))
        c = cfg_for(hg.patterns.bench_target(n), slm, K, seed=6)
        c.target.phase = turns
        c.target.freedoms.phase = False
        rep = hg.run_gs(c)
        ref = oracle.ifta(c.target.amplitude, slm, K, seed=6, phase_turns=turns, phase_freedom=False)
    mism = level_mismatches(rep.levels, ref.levels).sum()
    assert mism <= 16, (case, mism)
    assert np.max(np.abs(rep.trace.values() - ref.trace) / ref.trace) < MSE_TOL, case


def test_plan_kernel_timing_inside_graph():
    """Per-pass CUDA events inside the plan's graph (bench roofline): positive
    times over iterations 1..K-1, and the results are those of an untimed plan."""
    n, B, K = 256, 2, 4
    amp = hg.patterns.bench_target(n)
    cfg = hg.IftaConfig(iterations=K, slm=hg.SlmSpec.full_circle_phase(16), target=hg.TargetSpec(amp))
    outs = []
    for timed in (True, False):
        p = hg.IftaPlan(cfg, n, n, B)
        if timed:
            p.set_kernel_timing(True)
        p.upload(np.broadcast_to(amp, (B, n, n)), seeds=np.arange(1, B + 1))
        p.execute()
        r = p.download()
        outs.append((np.array(r.levels, copy=True), np.array(r.trace, copy=True)))
        if timed:
            kt = p.kernel_times()
            assert kt["iterations"] == K - 1 and kt["row"] > 0 and kt["col"] > 0
        else:
            with pytest.raises(Exception):
                p.kernel_times()
        p.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("roi", [False, True])
def test_efficiency_of_final_replay(roi):
    # extension (no reference counterpart): sum_{T>0, roi} |R|^2 / sum |R|^2 of the
    # final (unconstrained) replay, reduced in the last column pass; checked
    # against the returned replay in double
    amp = np.zeros((128, 128))
    amp[32:96, 32:96] = hg.patterns.smooth_blobs(64, 64)
    amp = hg.normalize_image(amp, hg.Normalization.UnitEnergy)
    c = cfg_for(amp, hg.SlmSpec.full_circle_phase(16), 8, seed=3)
    if roi:
        m = np.zeros((128, 128), np.uint8)
        m[24:104, 24:104] = 1
        c.target.roi = m
    rep = hg.run_gs(c)
    p = np.abs(rep.replay.astype(np.complex128)) ** 2
    sup = amp > 0
    if roi:
        sup &= m.astype(bool)
    want = p[sup].sum() / p.sum()
    assert 0 < rep.efficiency < 1 and abs(rep.efficiency - want) < 1e-5, (rep.efficiency, want)


@pytest.mark.parametrize("name", ["fc256_offset", "fc64", "fc6", "fc3_offset"])
def test_fused_quantiser_kinds_lockstep(oracle, name):
    """The fused row pass's full-circle fast path decides in level units with a
    mask for mod L (QK_FULL, L a power of two, any min_arg); other L take the
    generic quantiser.  One lock-step iteration at 512^2 for each."""
    slm = {"fc256_offset": lambda: hg.SlmSpec.full_circle_phase(256, 0.3),
           "fc64": lambda: hg.SlmSpec.full_circle_phase(64, 5.9),
           "fc6": lambda: hg.SlmSpec.full_circle_phase(6),
           "fc3_offset": lambda: hg.SlmSpec.full_circle_phase(3, 2.0)}[name]()
    amp = hg.patterns.bench_target(512)
    *_, (m_gpu, m_ref), _, _, cls = lockstep(oracle, amp, slm, 3)
    record(f"quantiser_{name}_512_lockstep1/k=3", cls)
    assert cls["bad"] == 0, cls
    assert rel(m_gpu, m_ref) < MSE_TOL
