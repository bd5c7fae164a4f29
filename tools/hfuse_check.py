"""Staggered-halves schedule (HG_HFUSE=1) vs the plain pass sequence:
levels and traces must be bit-identical.  python tools/hfuse_check.py [n] [batch] [K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2008_12214_b200 as hg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
K = int(sys.argv[3]) if len(sys.argv) > 3 else 3
amp = hg.patterns.bench_target(n)
slm = hg.SlmSpec.full_circle_phase(256)
out = {}
for hf in ("0", "1"):
    os.environ["HG_HFUSE"] = hf
    cfg = hg.IftaConfig(iterations=K, slm=slm, target=hg.TargetSpec(amp))
    reps = hg.run_ifta_batch(cfg, np.broadcast_to(amp, (B, n, n)), seeds=np.arange(1, B + 1))
    out[hf] = reps
for i in range(B):
    a, b = out["0"][i], out["1"][i]
    print(i, "levels equal", np.array_equal(a.levels, b.levels), "trace equal",
          np.array_equal(a.trace.values(), b.trace.values()), "replay equal", np.array_equal(a.replay, b.replay))
