"""Dev probe: per-pass SDSN time on a real FRAM gradient (C4, bf16) vs a random sparse input."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb
from synth import config_c4

inst = config_c4(0)
n = inst.n
A = torch.tensor(inst.A, dtype=torch.float32, device="cuda")
B = torch.tensor(inst.B, dtype=torch.float32, device="cuda")
N0 = torch.full((n, n), 1.0 / n, dtype=torch.float64, device="cuda")
h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0))
G, _c = fb.fram_gradient(h, A, B, None, N0, "bf16")
rng = np.random.Generator(np.random.PCG64(0))
R = torch.tensor(rng.random((n, n)) * (rng.random((n, n)) < 0.05), dtype=torch.float32, device="cuda")
for name, X in (("fram-gradient", G), ("random-sparse", R), ("fram-gradient", G)):
    for k in (2, 100, 600):
        hh = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=k))
        fb.fram_sdsn(hh, X, "fp32", want_gammas=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fb.fram_sdsn(hh, X, "fp32", want_gammas=False)
        torch.cuda.synchronize()
        print(name, k, "passes:", (time.perf_counter() - t0) * 1e3, "ms", flush=True)
