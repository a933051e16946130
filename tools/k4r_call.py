"""Dev probe: K4r per-call fixed cost at n = 4096 FP32 — time of a 10-pass call minus 10 × the per-pass time
(from 100- and 600-pass calls), on a sparse C4-like input."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.Generator(np.random.PCG64(0))
X = torch.tensor(rng.random((n, n)) * (rng.random((n, n)) < 0.05), dtype=torch.float32, device="cuda")
res = {}
for k in (10, 100, 600):
    h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=k))
    fb.fram_sdsn(h, X, "fp32", want_gammas=False)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fb.fram_sdsn(h, X, "fp32", want_gammas=False); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    res[k] = sorted(ts)[2]
us = (res[600] - res[100]) / 500 * 1e3
print(f"n={n}: {us:.3f} us/pass, 10-pass call {res[10] * 1e3:.1f} us -> fixed {res[10] * 1e3 - 10 * us:.1f} us/call")
