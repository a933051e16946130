"""Dev probe: per-pass SDSN time at n (default 4096) from two fixed-pass fram_sdsn calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
dt = torch.float64 if prec == "fp64" else torch.float32
rng = np.random.Generator(np.random.PCG64(0))
X = torch.tensor(rng.random((n, n)) * (rng.random((n, n)) < 0.05), dtype=dt, device="cuda")
res = {}
for k in (100, 600):
    h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=k))
    fb.fram_sdsn(h, X, prec, want_gammas=False)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fb.fram_sdsn(h, X, prec, want_gammas=False); b.record(); b.synchronize()
    res[k] = a.elapsed_time(b)
us = (res[600] - res[100]) / 500 * 1e3
es = 8 if prec == "fp64" else 4
print(f"n={n} {prec}: {us:.2f} us/pass, algorithmic {2 * es * n * n / (us * 1e-6) / 1e9:.0f} GB/s")
