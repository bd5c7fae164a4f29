"""CPU: bench.py's launch plumbing (SURVEY §8 d/e) without a GPU.

* `--gpus 2` re-launches itself under torch.distributed.run; the dry run
  (gloo) shards BASELINE config 5's 64 targets and gathers every target's
  levels and trace to rank 0 in target order.
* The reference arm runs the reference's own CPU path (oracle/_ref) without
  importing the product package, on the same metric.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out: str) -> dict:
    for line in reversed(out.strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise AssertionError(out[-2000:])


@pytest.mark.parametrize("gpus", [2, 3])
def test_bench_gpus_flag_launches_ranks_and_gathers(gpus):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--dry-run"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _last_json(r.stdout)
    assert line["n_gpus"] == gpus and line["scaling"] == "strong"
    assert line["gathered_targets"] == 64 and line["gather_in_target_order"]
    assert sum(c for _, c in line["shards"]) == 64


def test_bench_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--dry-run"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode != 0


def test_reference_arm_does_not_import_the_product():
    from pyoracle import available
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n", "64",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _last_json(r.stdout)
    assert line["impl"] == "reference" and line["product_package_imported"] is False
    assert line["cpu_baseline"]["kind"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["single_core"]["seconds_per_iteration"] > 0
