import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2008_12214_b200 as hg
J = 148; n = 1024
amp = hg.patterns.bench_target(n)
cfg = hg.OsprConfig(subframes=24, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp))
p = hg.OsprPlan(cfg, n, n, J)
p.upload(amp, seeds=np.arange(1, J + 1))
p.execute(); torch.cuda.synchronize()
print(os.environ.get("HG_OSPR_ROWS"), p.profile(reps=10))
