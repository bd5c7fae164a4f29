"""GPU parity of the rows-first OSPR subframe (csrc/ospr_rows.cuh): walk +
seed/row IFFT, column IFFT + quantiser + column FFT, row FFT + accumulation.

It is opt-in (measured slower than the column-first loop):
HG_OSPR_ROWS=2 selects it also for the few-job plans used here, and
HG_OSPR_ROWS=0 gives the column-first loop for comparison.  The seed stream is
the same bit-exact mt19937_64 (the walk only moves where each tile starts), so
levels differ from the oracle only near decision thresholds, exactly as for
the column-first loop (tests/test_gpu_ospr.py)."""
import numpy as np
import pytest

from helpers import level_mismatches, record, rel
from test_gpu_ospr import ocfg, ospr_frame_classes

pytestmark = pytest.mark.gpu
hg = pytest.importorskip("paper_2008_12214_b200")


def replay_mean_from_levels(levels: np.ndarray, L: int) -> np.ndarray:
    """sum_n |P(Q(levels_n))|^2 / N in double (ospr.hpp:134-156): the mean
    intensity the frames themselves imply.  (Against the oracle's own frames
    a single allowed near-threshold flip moves bright pixels by ~1e-3, so the
    run is checked for consistency with its own levels instead.)"""
    states = np.exp(2j * np.pi * np.arange(L) / L) if L > 2 else np.array([1.0, -1.0])
    acc = np.zeros(levels.shape[-2:])
    for lv in levels:
        acc += np.abs(np.fft.fft2(states[lv])) ** 2 / lv.size
    return acc / len(levels)


def assert_mean_consistent(run, L):
    want = replay_mean_from_levels(np.asarray(run.set.levels), L)
    assert np.allclose(run.set.mean_intensity, want, rtol=1e-4, atol=1e-6 * float(want.mean()))


@pytest.fixture
def rows(monkeypatch):
    monkeypatch.setenv("HG_OSPR_ROWS", "2")


@pytest.mark.parametrize("mode", ["2", "3"])  # 3: the walk stores every raw word
def test_rows_config3_matches_oracle(oracle, monkeypatch, mode):
    monkeypatch.setenv("HG_OSPR_ROWS", mode)
    amp = hg.patterns.bench_target(1024)
    run = hg.run_ospr(ocfg(amp, 24, 1))
    ref = oracle.ospr(amp, hg.SlmSpec.binary_phase(), 24, seed=1)
    cls = ospr_frame_classes(oracle, amp, 24, 1, run.set.levels, ref.levels, f"rows{mode}_config3_ospr_1024_binary_24")
    assert cls["bad"] == 0, cls
    assert np.max(np.abs(np.array(run.set.per_frame_mse) - ref.frame_mse) / ref.frame_mse) < 1e-4
    assert np.max(np.abs(run.report.trace.values() - ref.cumulative_mse) / ref.cumulative_mse) < 1e-4
    assert rel(hg.subframe_mse_statistic(run.set.per_frame_mse), oracle.subframe_mse_statistic(ref.frame_mse)) < 1e-4
    assert_mean_consistent(run, 2)


def _batch(monkeypatch, mode, amps, seeds, roi=None, N=5, slm=None):
    monkeypatch.setenv("HG_OSPR_ROWS", mode)
    tspec = hg.TargetSpec(amps[0], roi=roi)
    cfg = hg.OsprConfig(subframes=N, slm=slm or hg.SlmSpec.binary_phase(), target=tspec, seed=1)
    return hg.run_ospr_batch(cfg, seeds=seeds, amplitudes=amps, want_frames=False)


@pytest.mark.parametrize("levels", [2, 8])
def test_rows_equal_column_first_batches(monkeypatch, levels):
    """Per-job targets, an ROI, 3 jobs: rows-first vs column-first runs of the
    same plan differ only by float rounding of the transforms (levels within
    a few near-threshold pixels, traces within 1e-4)."""
    n = 1024
    base = hg.patterns.bench_target(n)
    amps = np.stack([np.roll(base, 97 * j, axis=0) for j in range(3)])
    roi = np.zeros((n, n), bool)
    roi[100:900, 50:1000] = True
    slm = hg.SlmSpec.binary_phase() if levels == 2 else hg.SlmSpec.full_circle_phase(levels)
    a = _batch(monkeypatch, "2", amps, [3, 4, 5], roi, slm=slm)
    b = _batch(monkeypatch, "0", amps, [3, 4, 5], roi, slm=slm)
    diff = 0
    for ra, rb in zip(a, b):
        diff += int(level_mismatches(ra.set.levels, rb.set.levels).sum())
        assert np.max(np.abs(np.array(ra.set.per_frame_mse) - rb.set.per_frame_mse) / rb.set.per_frame_mse) < 1e-4
        assert np.max(np.abs(ra.report.trace.values() - rb.report.trace.values()) / rb.report.trace.values()) < 1e-4
        assert_mean_consistent(ra, levels)
    record(f"rows_vs_column_first_{levels}level_3jobs_roi", {"mismatch": diff, "pixels": int(amps.size * 5)})
    assert diff <= amps.size * 5 * 2e-5, diff


def test_rows_profile_accounts_for_run(rows):
    amp = hg.patterns.bench_target(1024)
    run = hg.run_ospr(ocfg(amp, 4, 7))
    p = run.report.profile
    assert p.transform > 0 and p.constraint > 0 and p.metric > 0
    assert abs(p.total() - run.report.seconds) <= 1e-6 * max(1.0, run.report.seconds)


def test_rows_plan_reexecutes_identically(monkeypatch):
    """The walk restarts from the seeds on every execute (frame 1), so a
    re-executed plan reproduces its levels and traces bit for bit."""
    monkeypatch.setenv("HG_OSPR_ROWS", "2")
    amp = hg.patterns.bench_target(1024)
    cfg = ocfg(amp, 3, 11)
    p = hg.OsprPlan(cfg, 1024, 1024, 2)
    p.upload(amp, seeds=[11, 12])
    p.execute()
    a = p.download()
    p.execute()
    b = p.download()
    assert np.array_equal(a["levels"], b["levels"]) and np.array_equal(a["frame_mse"], b["frame_mse"])
    p.close()
