"""Dev probe: fram_gradient (precondition + the two gradient GEMMs) at n / precision from argv; reports
ms per call and 4n³ flop / time (the precondition's ~0.5 ms included)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_00887_b200 as fb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.rand((n, n), device="cuda", generator=g, dtype=torch.float64) < 0.01).double()
A = torch.maximum(A, A.T)
N = torch.full((n, n), 1.0 / n, device="cuda", dtype=torch.float64)
h = fb.fram_create(n)
G, _ = fb.fram_gradient(h, A, A, None, N, prec)
for _ in range(2):
    fb.fram_gradient(h, A, A, None, N, prec, G_out=G)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    fb.fram_gradient(h, A, A, None, N, prec, G_out=G)
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"n={n} {prec}: {ms:.3f} ms per gradient, {4 * n ** 3 / (ms * 1e-3) / 1e12:.1f} TFLOP/s")
