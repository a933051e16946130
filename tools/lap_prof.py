"""Dev probe: C4 bf16 solve, then two fram_lap calls on its N (for ncu -k regex:lap_kernel -s 2 -c 1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_00887_b200 as fb
from synth import config_c4

inst = config_c4(0)
A = torch.tensor(inst.A, dtype=torch.float32, device="cuda")
B = torch.tensor(inst.B, dtype=torch.float32, device="cuda")
h = fb.fram_create(inst.n, schedule=fb.Schedule(theta=10.0))
st, s, X, perm = fb.fram_solve(h, A, B, precision="bf16")
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = fb.fram_lap(h, X)
    torch.cuda.synchronize()
    print("lap ms", (time.perf_counter() - t0) * 1e3, "same", bool(torch.equal(p, perm)))
