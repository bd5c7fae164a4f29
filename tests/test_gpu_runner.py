"""GPU: the batch executor.  Mixed jobs are grouped into
batched plans; every job's levels / trace / final_error must equal the
single-job run, and a bad job fails alone (cmd_batch, runner.cpp:387-405)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
hg = pytest.importorskip("paper_2008_12214_b200")
from paper_2008_12214_b200.runner import BatchJob, run_batch  # noqa: E402


def test_batch_groups_equal_single_runs_and_isolate_failures():
    n = 64
    amp = hg.patterns.bench_target(n)
    amp2 = np.roll(amp, 7, axis=1)
    slm = hg.SlmSpec.full_circle_phase(8)
    jobs = [BatchJob(f"gs{s}", hg.IftaConfig(iterations=5, slm=slm, target=hg.TargetSpec(a), seed=s))
            for s, a in ((1, amp), (2, amp2), (3, amp))]
    jobs.append(BatchJob("wgs", hg.IftaConfig(variant=hg.IftaVariant.WeightedGS, iterations=4, slm=slm,
                                              target=hg.TargetSpec(amp), seed=4)))
    bad = amp.copy()
    bad[3, 3] = np.nan
    jobs.append(BatchJob("bad", hg.IftaConfig(iterations=5, slm=slm, target=hg.TargetSpec(bad), seed=5)))
    jobs += [BatchJob(f"ospr{s}", hg.OsprConfig(subframes=3, slm=hg.SlmSpec.binary_phase(),
                                                target=hg.TargetSpec(amp), seed=s)) for s in (7, 8)]
    rows = run_batch(jobs)
    assert [r.ok for r in rows] == [True, True, True, True, False, True, True]
    assert "non-finite" in rows[4].message
    for r, j in zip(rows, jobs):
        if not r.ok:
            continue
        cfg = j.config
        if isinstance(cfg, hg.IftaConfig):
            ref = hg.run_ifta(cfg)
            assert np.array_equal(r.levels, ref.levels), r.job
            assert np.array_equal(r.trace, ref.trace.values()), r.job
            assert r.final_error == ref.final_error
        else:
            ref = hg.run_ospr(cfg)
            assert np.array_equal(r.levels, ref.set.levels), r.job
            assert np.allclose(r.trace, ref.report.trace.values(), rtol=0, atol=0), r.job
        assert r.seconds > 0
    table, csv = hg.runner.batch_summary(rows)
    assert "bad" in table and csv.count("\n") == len(rows) + 1


def test_thread_routing_policy_concurrent_runs():
    """hgc_set_device_policy(1): host threads (the runner's batch pool) bind
    round-robin to the GPUs; concurrent one-shot runs give the sequential
    results."""
    import threading
    from paper_2008_12214_b200 import _lib
    amp = hg.patterns.bench_target(64)
    cfgs = [hg.IftaConfig(iterations=4, slm=hg.SlmSpec.full_circle_phase(4), target=hg.TargetSpec(amp), seed=s)
            for s in range(1, 7)]
    want = [hg.run_gs(c) for c in cfgs]
    _lib.check(_lib.lib.hgc_set_device_policy(1))
    try:
        got = [None] * len(cfgs)

        def work(i):
            got[i] = hg.run_gs(cfgs[i])

        ts = [threading.Thread(target=work, args=(i,)) for i in range(len(cfgs))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    finally:
        _lib.check(_lib.lib.hgc_set_device_policy(0))
    for g, w in zip(got, want):
        assert np.array_equal(g.levels, w.levels) and g.final_error == w.final_error


@pytest.mark.parametrize("which", ["gs", "gs64", "ospr", "ospr64"])
def test_profile_accounts_for_the_whole_run(which):
    # test_ifta.cpp:270-280 ("profile accounts for the whole run"), bench.cpp:167-183
    amp = hg.normalize_image(hg.patterns.checkerboard(32, 32, 4), hg.Normalization.UnitEnergy)
    if which.startswith("gs"):
        cfg = hg.IftaConfig(iterations=10, slm=hg.SlmSpec.full_circle_phase(256), target=hg.TargetSpec(amp), seed=1)
        rep = hg.run_gs(cfg) if which == "gs" else hg.run_ifta_f64(cfg)
    else:
        cfg = hg.OsprConfig(subframes=6, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=1)
        rep = (hg.run_ospr(cfg) if which == "ospr" else hg.run_ospr_f64(cfg)).report
    p = rep.profile
    assert p.transform > 0 and p.constraint > 0 and p.metric > 0 and p.other >= 0
    assert rep.seconds > 0 and abs(p.total() - rep.seconds) <= 1e-9 * rep.seconds
