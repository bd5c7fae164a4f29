"""In-graph per-iteration time of the batched GS plan: (t(K2) - t(K1)) / (K2 - K1)
with CUDA-event timing of whole plan executions (seed/finalize cancel out).
  python tools/iter_time.py [n] [batch] [levels]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12214_b200 as hg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
L = int(sys.argv[3]) if len(sys.argv) > 3 else 256
amp = hg.patterns.bench_target(n)
slm = hg.SlmSpec.full_circle_phase(L) if L > 2 else hg.SlmSpec.binary_phase()


st = torch.cuda.Stream()  # (stream 0 would mean: the plan's own stream)


def timed(K, reps=3):
    cfg = hg.IftaConfig(iterations=K, slm=slm, target=hg.TargetSpec(amp))
    p = hg.IftaPlan(cfg, n, n, B)
    p.upload(np.broadcast_to(amp, (B, n, n)), seeds=np.arange(1, B + 1))
    p.execute()
    p.download()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        p.execute(st.cuda_stream)
        e1.record(st)
        p.download()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    del p
    return min(ts)


t1, t2 = timed(5), timed(25)
it = (t2 - t1) / 20
print(f"n={n} B={B} L={L}: K=5 {t1:.2f} ms, K=25 {t2:.2f} ms, per iteration {it:.3f} ms, "
      f"{36 * n * n * B / it / 1e6:.0f} GB/s ({36 * n * n * B / it / 1e6 / 6550.1:.3f} of peak)")
