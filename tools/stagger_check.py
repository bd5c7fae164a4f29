import os, sys, subprocess
sys.path.insert(0, os.getcwd())
code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2008_12214_b200 as hg
amp = hg.patterns.bench_target(1024)
amps = np.stack([np.roll(amp, 37 * t, axis=1) for t in range(4)])
cfg = hg.IftaConfig(iterations=5, slm=hg.SlmSpec.full_circle_phase(256), target=hg.TargetSpec(amp), seed=1)
reps = hg.run_ifta_batch(cfg, amps, seeds=[1, 2, 3, 4])
np.save(sys.argv[1], np.stack([r.levels for r in reps]))
np.save(sys.argv[1] + "_tr.npy", np.stack([r.trace.values() for r in reps]))
'''
for m in ("0", "1"):
    subprocess.run([sys.executable, "-c", code, f"/tmp/st{m}"], env=dict(os.environ, HG_STAGGER=m), check=True)
import numpy as np
a, b = np.load("/tmp/st0.npy"), np.load("/tmp/st1.npy")
print("levels equal", np.array_equal(a, b), "traces equal", np.array_equal(np.load("/tmp/st0_tr.npy"), np.load("/tmp/st1_tr.npy")))
