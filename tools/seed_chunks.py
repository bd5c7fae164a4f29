import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2008_12214_b200 as hg
n = int(sys.argv[1])
amp = hg.patterns.bench_target(n)
cfg = hg.IftaConfig(iterations=2, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=1)
p = hg.IftaPlan(cfg, n, n, 1)
p.upload(amp[None], seeds=[1])
p.execute(); p.download()
pr = p.profile(reps=20)
print(n, os.environ.get("HG_SEED_CHUNKS", "default"), f"seed {1e3*pr['seed']:.1f} us")
