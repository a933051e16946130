"""Dev probe: R17 LAP time on the C4 FRAM N (for A/B of LAP kernel variants with tools/ab.sh)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb
from synth import config_c4

path = "/tmp/c4_N.pt"
if os.path.exists(path):
    X = torch.load(path).cuda()
else:
    inst = config_c4(0)
    A = torch.tensor(inst.A, dtype=torch.float32, device="cuda")
    B = torch.tensor(inst.B, dtype=torch.float32, device="cuda")
    h = fb.fram_create(inst.n, schedule=fb.Schedule(theta=10.0))
    _, st, X, perm = fb.fram_solve(h, A, B, precision="bf16")
    torch.save(X.cpu(), path)
n = X.shape[0]
hh = fb.fram_create(n)
p = fb.fram_lap(hh, X)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    p = fb.fram_lap(hh, X)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"LAP on C4 N: {min(ts):.2f} ms  perm checksum {int((p.cpu().numpy().astype(np.int64) * np.arange(n)).sum())}")
