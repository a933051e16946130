"""Dev probe: one fram_sdsn call (fixed passes) for ncu: python tools/sdsn_prof.py n passes [fp32|fp64]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
k = int(sys.argv[2]) if len(sys.argv) > 2 else 200
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
dt = torch.float64 if prec == "fp64" else torch.float32
rng = np.random.Generator(np.random.PCG64(0))
X = torch.tensor(rng.random((n, n)) * (rng.random((n, n)) < 0.05), dtype=dt, device="cuda")
h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=k))
for _ in range(2):
    fb.fram_sdsn(h, X, prec, want_gammas=False)
torch.cuda.synchronize()
print("ok", n, k)
