"""Single-job OSPR (config 3) and seed_random_phase timing, for ncu launch lists.

    python tools/prof_ospr_single.py            # prints device ms per job
    ncu --metrics gpu__time_duration.sum --clock-control none python tools/prof_ospr_single.py --once
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2008_12214_b200 as hg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--once", action="store_true")
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--subframes", type=int, default=24)
a = ap.parse_args()
amp = hg.patterns.bench_target(a.n)
cfg = hg.OsprConfig(subframes=a.subframes, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=1)
p = hg.OsprBlockPlan(cfg, a.n, a.n, 0, a.subframes)
p.upload(amp)
st = torch.cuda.Stream()
reps = 1 if a.once else 10
for _ in range(1 if a.once else 3):
    p.execute(st.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(reps):
    p.execute(st.cuda_stream)
e1.record(st)
torch.cuda.synchronize()
print(f"ospr single job {a.n}^2 x {a.subframes}: {e0.elapsed_time(e1) / reps:.3f} ms/job, "
      f"launches {p.launches()}, profile {p.profile(3)}")
t = hg.patterns.bench_target(4096)
for k in range(2):
    torch.cuda.synchronize()
    e0.record()
    hg.seed_random_phase(t, 5)
    e1.record()
    torch.cuda.synchronize()
print(f"seed_random_phase 4096^2 (incl. H2D/D2H): {e0.elapsed_time(e1):.3f} ms")
