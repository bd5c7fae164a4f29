"""GPU: plan shapes at the edges of the kernels' dispatch — extreme aspect
ratios (one quad row / one column pair), the smallest fields, non-square
TMA tiles (NY = 512 .. 4096 with narrow NX), odd batch sizes and the
L2-resident target grouping — against the oracle (binary, free-running)."""
import numpy as np
import pytest

from helpers import level_mismatches

pytestmark = pytest.mark.gpu
hg = pytest.importorskip("paper_2008_12214_b200")


@pytest.mark.parametrize("ny,nx", [(2, 2), (2, 4096), (4096, 2), (4, 8), (512, 16), (16, 512), (4096, 64),
                                   (64, 4096), (1024, 2048)])
def test_plan_shapes_match_oracle(oracle, ny, nx):
    r = np.random.default_rng(ny + 7 * nx)
    amp = hg.normalize_image(r.uniform(0, 1, (ny, nx)), hg.Normalization.UnitEnergy)
    slm = hg.SlmSpec.binary_phase()
    K = 6
    cfg = hg.IftaConfig(iterations=K, slm=slm, target=hg.TargetSpec(amp), seed=3)
    rep = hg.run_gs(cfg)
    ref = oracle.ifta(amp, slm, K, seed=3)
    assert level_mismatches(rep.levels, ref.levels).sum() <= max(2, nx * ny // 20000), (ny, nx)
    assert np.max(np.abs(rep.trace.values() - ref.trace) / ref.trace) < 1e-4


@pytest.mark.parametrize("batch,n", [(1, 256), (3, 256), (5, 1024), (17, 128)])
def test_batch_groups_match_single_runs(batch, n):
    """Batched plans (incl. L2-resident target groups at small sizes) equal
    independent single-target runs: identical levels; MSE traces equal up to
    the summation order (the launch's column width can differ, col_width_rt)."""
    amps = np.stack([np.roll(hg.patterns.bench_target(n), 11 * t, axis=1) for t in range(batch)])
    slm = hg.SlmSpec.full_circle_phase(8)
    cfg = hg.IftaConfig(iterations=4, slm=slm, target=hg.TargetSpec(amps[0]), seed=1)
    reps = hg.run_ifta_batch(cfg, amps, seeds=[1 + t for t in range(batch)])
    for t in (0, batch - 1):
        c = hg.IftaConfig(iterations=4, slm=slm, target=hg.TargetSpec(amps[t]), seed=1 + t)
        single = hg.run_gs(c)
        assert np.array_equal(reps[t].levels, single.levels)
        assert np.max(np.abs(reps[t].trace.values() - single.trace.values()) / single.trace.values()) < 1e-7


@pytest.mark.parametrize("ny,nx,N", [(2, 2, 3), (4096, 2, 2), (512, 64, 4)])
def test_ospr_shapes_match_oracle(oracle, ny, nx, N):
    r = np.random.default_rng(ny * 3 + nx)
    amp = hg.normalize_image(r.uniform(0, 1, (ny, nx)), hg.Normalization.UnitEnergy)
    cfg = hg.OsprConfig(subframes=N, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=5)
    run = hg.run_ospr(cfg)
    ref = oracle.ospr(amp, hg.SlmSpec.binary_phase(), N, seed=5)
    assert level_mismatches(run.set.levels, ref.levels).sum() <= N * max(1, nx * ny // 20000)
    assert np.max(np.abs(run.report.trace.values() - ref.cumulative_mse) / ref.cumulative_mse) < 1e-4


def test_staggered_halves_equal_single_graph(monkeypatch):
    """HG_STAGGER=1 (experiment: the batch's two halves on two graph branches,
    staggered by a pass) gives the same levels and traces bit for bit."""
    amp = hg.patterns.bench_target(1024)
    amps = np.stack([np.roll(amp, 37 * t, axis=1) for t in range(4)])
    cfg = hg.IftaConfig(iterations=5, slm=hg.SlmSpec.full_circle_phase(256), target=hg.TargetSpec(amp), seed=1)
    out = {}
    for m in ("0", "1"):
        monkeypatch.setenv("HG_STAGGER", m)
        reps = hg.run_ifta_batch(cfg, amps, seeds=[1, 2, 3, 4])
        out[m] = (np.stack([r.levels for r in reps]), np.stack([r.trace.values() for r in reps]))
    assert np.array_equal(out["0"][0], out["1"][0]) and np.array_equal(out["0"][1], out["1"][1])
