"""GPU: the double-precision device loops against the
reference's own run_ifta<double> / run_ospr_variant<double> (oracle/_ref).
Both sides compute in double; only the transforms' rounding differs (the
device f64 FFT vs the reference build's double substitute FFT), so binary /
first-iteration levels agree exactly and MSE traces to ~1e-9."""
import numpy as np
import pytest

from helpers import level_mismatches

pytestmark = pytest.mark.gpu
hg = pytest.importorskip("paper_2008_12214_b200")


def _target(ny, nx, roi_frac=None):
    amp = hg.patterns.smooth_blobs(nx, ny) if ny == nx else np.random.default_rng(3).uniform(0, 1, (ny, nx))
    amp = hg.normalize_image(np.asarray(amp, np.float64), hg.Normalization.UnitEnergy)
    roi = None
    if roi_frac:
        roi = np.zeros((ny, nx), np.uint8)
        roi[ny // 4: ny // 4 + ny // 2, nx // 4: nx // 4 + nx // 2] = 1
    return amp, roi


CASES = {
    "gs_binary": dict(slm=lambda: hg.SlmSpec.binary_phase(), K=20),
    "gs_256_first": dict(slm=lambda: hg.SlmSpec.full_circle_phase(256), K=1),
    "wgs_16": dict(slm=lambda: hg.SlmSpec.full_circle_phase(16), K=4, variant="wgs"),
    "lt_roi": dict(slm=lambda: hg.SlmSpec.binary_phase(), K=15, variant="lt", roi=True, amp_out=True),
    "roi_scale_free": dict(slm=lambda: hg.SlmSpec.binary_phase(), K=10, roi=True, scale=True),
    "fresnel": dict(slm=lambda: hg.SlmSpec.binary_phase(), K=10, fresnel=(532e-9, 0.1, 8e-6, 8e-6)),
    "target_phase": dict(slm=lambda: hg.SlmSpec.binary_phase(), K=6, phase=True),
    "amplitude_slm": dict(slm=lambda: hg.SlmSpec.amplitude(8, 0.0, 1.0), K=1),
    "non_pow2": dict(slm=lambda: hg.SlmSpec.binary_phase(), K=10, shape=(40, 48)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_ifta_f64_matches_reference_double(ref_oracle, name):
    c = CASES[name]
    ny, nx = c.get("shape", (64, 64))
    amp, roi = _target(ny, nx, c.get("roi"))
    slm = c["slm"]()
    variant = c.get("variant", "gs")
    cfg = hg.IftaConfig(iterations=c["K"], slm=slm, target=hg.TargetSpec(amp), seed=7,
                        variant={"gs": hg.IftaVariant.GS, "wgs": hg.IftaVariant.WeightedGS,
                                 "lt": hg.IftaVariant.LiuTaghizadeh}[variant])
    cfg.target.roi = roi
    cfg.target.freedoms.amplitude_outside_roi = bool(c.get("amp_out"))
    cfg.target.freedoms.scale = bool(c.get("scale"))
    turns = None
    if c.get("phase"):
        turns = np.random.default_rng(9).uniform(0, 1, (ny, nx))
        cfg.target.phase = turns
        cfg.target.freedoms.phase = False
    prop = None
    if c.get("fresnel"):
        prop = hg.Propagator.fresnel(nx, ny, hg.FresnelParams(*c["fresnel"]))
    rep = hg.run_ifta_f64(cfg, prop)
    ref = ref_oracle.ifta64(amp, slm, c["K"], seed=7, variant=variant, roi=roi, amp_outside_roi=bool(c.get("amp_out")),
                            scale_freedom=bool(c.get("scale")), phase_turns=turns, phase_freedom=not c.get("phase"),
                            fresnel=c.get("fresnel"))
    assert rep.hologram.dtype == np.complex128
    mism = level_mismatches(rep.levels, ref.levels).sum()
    assert mism <= 2, (name, mism)
    rel = np.max(np.abs(rep.trace.values() - ref.trace) / ref.trace)
    assert rel < 1e-8, (name, rel)


@pytest.mark.parametrize("adaptive", [False, True])
def test_ospr_f64_matches_reference_double(ref_oracle, adaptive):
    amp, _ = _target(64, 64)
    cfg = hg.OsprConfig(variant=hg.OsprVariant.AdaptiveOspr if adaptive else hg.OsprVariant.Ospr, subframes=5,
                        slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=3, feedback_gain=0.8)
    run = hg.run_ospr_f64(cfg)
    ref = ref_oracle.ospr64(amp, hg.SlmSpec.binary_phase(), 5, seed=3, adaptive=adaptive, gain=0.8)
    assert level_mismatches(run.set.levels, ref.levels).sum() <= 2
    assert np.max(np.abs(run.report.trace.values() - ref.cumulative_mse) / ref.cumulative_mse) < 1e-8
    assert np.max(np.abs(np.array(run.set.per_frame_mse) - ref.frame_mse) / ref.frame_mse) < 1e-8
    assert np.allclose(run.set.mean_intensity, ref.mean_intensity, rtol=1e-8, atol=1e-18)
