"""Dev probe: R17 LAP time at n (default 16384) on a synthetic N (kind: twoperm | flat), for A/B of
LAP kernel variants with tools/ab.sh; prints the permutation checksum (variants must agree bit-exactly)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_00887_b200 as fb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
kind = sys.argv[2] if len(sys.argv) > 2 else "twoperm"
g = torch.Generator(device="cuda").manual_seed(5)
P1 = torch.randperm(n, generator=g, device="cuda")
P2 = torch.randperm(n, generator=g, device="cuda")
N = torch.rand((n, n), generator=g, dtype=torch.float64, device="cuda")
r = torch.arange(n, device="cuda")
if kind == "twoperm":
    N *= 0.05
    N[r, P1] += 0.5
    N[r, P2] += 0.45
else:                                                   # flat: a faint planted matching in noise
    N = N ** 8 * 0.02
    N[r, P1] += 0.01
h = fb.fram_create(n)
p = fb.fram_lap(h, N)
torch.cuda.synchronize()
t0 = time.perf_counter()
p = fb.fram_lap(h, N)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
w = torch.arange(1, n + 1, device="cuda", dtype=torch.int64)
print(f"LAP n={n} {kind}: {dt * 1e3:.1f} ms  checksum {int((p.long() * w).sum())}  planted {float((p == P1).double().mean()):.3f}")
