"""Dev probe: streaming SDSN (K4) per-pass time at n=4096 in FP64 (FP32 with a -DFRAM_DEV_FORCE_STREAM=1
variant of fram_api.cu, tools/build_variant.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
k = 200
dt = torch.float64 if prec == "fp64" else torch.float32
rng = np.random.Generator(np.random.PCG64(0))
X = torch.tensor(rng.random((n, n)) * (rng.random((n, n)) < 0.05), dtype=dt, device="cuda")
h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=k))
for _ in range(2):
    fb.fram_sdsn(h, X, prec, want_gammas=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record()
    fb.fram_sdsn(h, X, prec, want_gammas=False)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
us = min(ts) * 1e3 / k
esz = 8 if prec == "fp64" else 4
print(f"n={n} {prec} streaming SDSN: {us:.2f} us/pass, {2 * esz * n * n / us / 1e3:.0f} GB/s algorithmic")
