"""Small driver for ncu: one batched GS run (and optionally OSPR) so the
fused kernels can be captured in isolation.
  python tools/prof_gs.py [n] [batch] [iters] [levels] [--ospr]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2008_12214_b200 as hg  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = int(args[0]) if len(args) > 0 else 4096
B = int(args[1]) if len(args) > 1 else 2
K = int(args[2]) if len(args) > 2 else 2
L = int(args[3]) if len(args) > 3 else 256
if "--ospr" in sys.argv:
    amp = hg.patterns.bench_target(n)
    cfg = hg.OsprConfig(subframes=K, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp))
    p = hg.OsprPlan(cfg, n, n, B)
    p.upload(amp, seeds=np.arange(1, B + 1))
    p.execute()
    print(p.download()["cumulative_mse"][:, -1])
else:
    amp = hg.patterns.bench_target(n)
    slm = hg.SlmSpec.full_circle_phase(L) if L > 2 else hg.SlmSpec.binary_phase()
    cfg = hg.IftaConfig(iterations=K, slm=slm, target=hg.TargetSpec(amp))
    p = hg.IftaPlan(cfg, n, n, B)
    p.upload(np.broadcast_to(amp, (B, n, n)), seeds=np.arange(1, B + 1))
    p.execute()
    print(p.download().trace[:, -1])
