"""Bit-exactness of a library switch read from the environment (e.g.
HG_ROW_PERSIST): run one batched GS plan and save levels / traces / replay,
then compare two saved runs.
  python tools/env_ab_check.py run out.npz [n] [batch] [K] [levels]
  python tools/env_ab_check.py cmp a.npz b.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        print(k, "identical" if np.array_equal(a[k], b[k]) else f"DIFFERENT ({np.count_nonzero(a[k] != b[k])})")
    sys.exit(0)
import paper_2008_12214_b200 as hg  # noqa: E402

out = sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
B = int(sys.argv[4]) if len(sys.argv) > 4 else 4
K = int(sys.argv[5]) if len(sys.argv) > 5 else 3
L = int(sys.argv[6]) if len(sys.argv) > 6 else 256
amp = hg.patterns.bench_target(n)
slm = hg.SlmSpec.full_circle_phase(L) if L > 2 else hg.SlmSpec.binary_phase()
cfg = hg.IftaConfig(iterations=K, slm=slm, target=hg.TargetSpec(amp))
reps = hg.run_ifta_batch(cfg, np.broadcast_to(amp, (B, n, n)), seeds=np.arange(1, B + 1))
np.savez(out, levels=np.stack([r.levels for r in reps]), trace=np.stack([r.trace.values() for r in reps]),
         replay=np.stack([r.replay for r in reps]))
print("saved", out)
