"""CPU: host logic of the batch executor — cmd_batch's
summary table / CSV (runner.cpp:423-447) and per-job validation failures."""
import numpy as np

import paper_2008_12214_b200 as hg
from paper_2008_12214_b200.runner import BatchJob, BatchRow, batch_summary, run_batch


def test_batch_summary_matches_cmd_batch_format():
    rows = [BatchRow("a.json", True, 0.0123456789, 1.5), BatchRow("b.json", False, message="bad, thing\nhere")]
    table, csv = batch_summary(rows)
    lines = table.splitlines()
    assert lines[0] == "%-32s %-8s %16s %10s" % ("job", "status", "final_error", "seconds")
    assert lines[1] == "%-32s %-8s %16s %10.3f" % ("a.json", "ok", "0.0123456789", 1.5)
    assert lines[2] == "%-32s %-8s %16s %10s" % ("b.json", "failed", "-", "-")
    assert csv.splitlines() == ["job,status,final_error,seconds,message", "a.json,ok,0.0123456789,1.50000000,",
                                "b.json,failed,-,-,bad; thing here"]


def test_invalid_configs_fail_per_job_without_a_device():
    amp = hg.patterns.bench_target(16)
    bad = hg.IftaConfig(iterations=0, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp))
    bad2 = hg.OsprConfig(subframes=0, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp))
    rows = run_batch([BatchJob("x", bad), BatchJob("y", bad2)])
    assert [r.ok for r in rows] == [False, False]
    assert "iterations" in rows[0].message and "subframes" in rows[1].message
