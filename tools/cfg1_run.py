"""Config 1 (GS 512^2 binary, K = 100) executed a few times: the workload for
an ncu launch list of the small-config passes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2008_12214_b200 as hg  # noqa: E402

n = int(os.environ.get("HG_N", "512"))
amp = hg.patterns.bench_target(n)
slm = hg.SlmSpec.binary_phase() if n == 512 else hg.SlmSpec.full_circle_phase(256)
cfg = hg.IftaConfig(iterations=int(os.environ.get("HG_K", "100")), slm=slm, target=hg.TargetSpec(amp), seed=1)
p = hg.IftaPlan(cfg, n, n, 1)
p.upload(amp[None], seeds=[1])
st = torch.cuda.Stream()
for _ in range(int(os.environ.get("HG_REPS", "2"))):
    p.execute(st.cuda_stream)
torch.cuda.synchronize()
print("done")
