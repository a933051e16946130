"""Dev probe: K4r on a 5%-dense random n=4096 input, 1000 fixed passes; prints ms per call (CUDA events).
With a -DFRAM_DEV_RES_TIMING=1 variant of fram_api.cu (tools/build_variant.sh) the library also prints its
per-phase globaltimer breakdown (perturbs timing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.Generator(np.random.PCG64(0))
X = torch.tensor(rng.random((n, n)) * (rng.random((n, n)) < 0.05), dtype=torch.float32, device="cuda")
h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=1000))
for _ in range(2):
    fb.fram_sdsn(h, X, "fp32", want_gammas=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record()
    fb.fram_sdsn(h, X, "fp32", want_gammas=False)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"n={n} K4r 1000 passes: {min(ts):.3f} ms (min of 5), median {sorted(ts)[2]:.3f} ms")
