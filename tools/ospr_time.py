"""Device time of the config-3 OSPR stream (1024^2 binary, 24 subframes,
`jobs` jobs), CUDA events around whole plan executions; prints subframes/s and
a checksum of the levels/traces (for bit-exactness across library variants).
  python tools/ospr_time.py [jobs] [n] [subframes]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12214_b200 as hg  # noqa: E402

J = int(sys.argv[1]) if len(sys.argv) > 1 else 148
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
N = int(sys.argv[3]) if len(sys.argv) > 3 else 24
amp = hg.patterns.bench_target(n)
cfg = hg.OsprConfig(subframes=N, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp))
p = hg.OsprPlan(cfg, n, n, J)
p.upload(amp, seeds=np.arange(1, J + 1))
st = torch.cuda.Stream()
p.execute(st.cuda_stream)
torch.cuda.synchronize()
best = None
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    p.execute(st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    best = ms if best is None else min(best, ms)
out = p.download()
h = hashlib.sha1(np.ascontiguousarray(out["levels"]).tobytes() + out["cumulative_mse"].tobytes()).hexdigest()[:16]
print(f"ospr J={J} n={n} N={N}: {best:.2f} ms per step, {J * N / (best * 1e-3):.0f} subframes/s, digest {h}")
