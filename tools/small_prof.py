import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2008_12214_b200 as hg
for n, slm, K, var in ((512, hg.SlmSpec.binary_phase(), 100, hg.IftaVariant.GS), (1024, hg.SlmSpec.full_circle_phase(256), 200, hg.IftaVariant.WeightedGS), (2048, hg.SlmSpec.full_circle_phase(256), 100, hg.IftaVariant.GS)):
    amp = hg.patterns.bench_target(n)
    cfg = hg.IftaConfig(variant=var, iterations=K, slm=slm, target=hg.TargetSpec(amp), seed=1)
    p = hg.IftaPlan(cfg, n, n, 1)
    p.upload(amp[None], seeds=[1])
    st = torch.cuda.Stream()
    p.execute(st.cuda_stream); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5): p.execute(st.cuda_stream)
    e1.record(st); torch.cuda.synchronize()
    run = e0.elapsed_time(e1) / 5
    pr = p.profile(reps=50)
    print(n, f"run {run:.3f} ms = {1e3*run/K:.2f} us/iter; isolated row {1e3*pr['row']:.2f} us col {1e3*pr['col']:.2f} us seed {1e3*pr['seed']:.1f} us, launches {p.launches()}")
