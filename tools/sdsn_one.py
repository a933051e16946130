"""Dev probe: one SDSN call (fixed passes) at n / precision from argv, repeated — for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb

n = int(sys.argv[1]); prec = sys.argv[2]; k = int(sys.argv[3]) if len(sys.argv) > 3 else 400
dt = torch.float64 if prec == "fp64" else torch.float32
rng = np.random.Generator(np.random.PCG64(n))
X = torch.tensor(rng.random((n, n)), dtype=dt, device="cuda")
h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=k))
for _ in range(3):
    fb.fram_sdsn(h, X, prec, want_gammas=False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); fb.fram_sdsn(h, X, prec, want_gammas=False); e1.record(); e1.synchronize()
print(f"n={n} {prec}: {e0.elapsed_time(e1) * 1e3 / k:.2f} us/pass")
