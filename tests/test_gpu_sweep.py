"""GPU: randomized parity sweep over small configurations (sizes 2..128 per
side, square or not; binary / multi-level / restricted / amplitude SLMs;
GS / WGS / LT; ROI and scale freedom; OSPR and adaptive OSPR) against the C
oracle.  Binary and restricted few-level SLMs are compared free-running;
multi-level runs compare the first iteration (chaotic afterwards, SURVEY
§0.5)."""
import numpy as np
import pytest

from helpers import level_mismatches

pytestmark = pytest.mark.gpu
hg = pytest.importorskip("paper_2008_12214_b200")

SIDES = [2, 4, 8, 16, 32, 64, 128]


def _slm(kind):
    if kind == "binary":
        return hg.SlmSpec.binary_phase(), 40
    if kind == "full16":
        return hg.SlmSpec.full_circle_phase(16), 1
    if kind == "restricted":
        return hg.SlmSpec.phase(4, 0.0, 0.75 * hg.TWO_PI), 1
    return hg.SlmSpec.amplitude(8, 0.0, 1.0), 1


@pytest.mark.parametrize("case", range(24))
def test_random_ifta_config_matches_oracle(oracle, case):
    r = np.random.default_rng(1000 + case)
    ny, nx = int(r.choice(SIDES[2:])), int(r.choice(SIDES[2:]))
    kind = ["binary", "full16", "restricted", "amplitude"][case % 4]
    slm, K = _slm(kind)
    variant = ["gs", "wgs", "lt"][case % 3]
    amp = r.uniform(0, 1, (ny, nx)) * (r.uniform(size=(ny, nx)) > 0.3)
    amp = hg.normalize_image(amp, hg.Normalization.UnitEnergy)
    roi = None
    if case % 5 == 0 or variant == "lt":
        roi = np.zeros((ny, nx), np.uint8)
        roi[ny // 4: ny // 4 + max(1, ny // 2), nx // 4: nx // 4 + max(1, nx // 2)] = 1
    scale = bool(case % 7 == 3)
    c = hg.IftaConfig(iterations=K, slm=slm, target=hg.TargetSpec(amp), seed=case,
                      variant={"gs": hg.IftaVariant.GS, "wgs": hg.IftaVariant.WeightedGS,
                               "lt": hg.IftaVariant.LiuTaghizadeh}[variant])
    c.target.roi = roi
    c.target.freedoms.scale = scale
    rep = hg.run_ifta(c)
    ref = oracle.ifta(amp, slm, K, seed=case, variant=variant, roi=roi, scale_freedom=scale)
    mism = level_mismatches(rep.levels, ref.levels).sum()
    assert mism <= max(2, nx * ny // 1000), (kind, variant, ny, nx, mism)
    rel = np.abs(rep.trace.values() - ref.trace) / np.maximum(ref.trace, 1e-30)
    assert np.max(rel) < 1e-3, (kind, variant, ny, nx, rel.max())


@pytest.mark.parametrize("case", range(8))
def test_random_ospr_config_matches_oracle(oracle, case):
    r = np.random.default_rng(2000 + case)
    ny, nx = int(r.choice(SIDES[1:])), int(r.choice(SIDES[1:]))
    adaptive = bool(case % 2)
    N = int(r.integers(1, 6))
    amp = hg.normalize_image(r.uniform(0, 1, (ny, nx)), hg.Normalization.UnitEnergy)
    cfg = hg.OsprConfig(variant=hg.OsprVariant.AdaptiveOspr if adaptive else hg.OsprVariant.Ospr, subframes=N,
                        slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=case, feedback_gain=0.6)
    run = hg.run_ospr_variant(cfg)
    ref = oracle.ospr(amp, hg.SlmSpec.binary_phase(), N, seed=case, adaptive=adaptive, gain=0.6)
    assert level_mismatches(run.set.levels, ref.levels).sum() <= N * max(1, nx * ny // 2000)
    assert np.max(np.abs(run.report.trace.values() - ref.cumulative_mse) / ref.cumulative_mse) < 1e-3
