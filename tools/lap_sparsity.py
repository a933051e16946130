"""Dev probe: how sparse is the final C4 N as the LAP sees it?

In the R17 scan cur = (−N[i0][j] − u[i0]) − v[j] (FP64), an entry with N < ulp(|u[i0]|)/4 leaves
−N − u[i0] exactly equal to −u[i0], so such entries need not be loaded when u[i0] ≠ 0.  This probe
runs one C4 bf16 solve on the GPU, then (on the host, own instrumented copy of the R17 loop — not the
oracle) records |u[i0]| at every Dijkstra step and reports, per threshold τ, the fraction of N below τ,
the stored entries per row, and the fraction of steps whose u[i0] makes a τ-sparse row exact."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb
from synth import config_c4

inst = config_c4(0)
A = torch.tensor(inst.A, dtype=torch.float32, device="cuda")
B = torch.tensor(inst.B, dtype=torch.float32, device="cuda")
h = fb.fram_create(inst.n, schedule=fb.Schedule(theta=10.0))
st, s, X, perm = fb.fram_solve(h, A, B, precision="bf16")
N = X.cpu().numpy().astype(np.float64)
n = N.shape[0]
print(f"outer={s['outer_iters']} acc={(perm.cpu().numpy() == inst.perm_true).mean():.4f}", flush=True)
taus = [1e-12, 1e-16, 1e-18, 1e-20, 1e-22, 1e-25, 1e-30, 1e-40]
for tau in taus:
    keep = N >= tau
    per_row = keep.sum(1)
    print(f"tau={tau:.0e}: below {1 - keep.mean():.4f}; stored per row mean {per_row.mean():.1f} max {per_row.max()}; "
          f"min N {N.min():.3e}")

# instrumented R17 (same loop as the reading R17; here only to observe u[i0] per step)
t0 = time.time()
C = -N
u = np.zeros(n + 1); v = np.zeros(n + 1)
p = np.zeros(n + 1, dtype=np.int64); way = np.zeros(n + 1, dtype=np.int64)
uabs = []
for i in range(1, n + 1):
    p[0] = i; j0 = 0
    minv = np.full(n + 1, np.inf); used = np.zeros(n + 1, dtype=bool)
    while True:
        used[j0] = True
        i0 = p[j0]
        uabs.append(abs(u[i0]))
        free = ~used[1:]
        cur = (C[i0 - 1, :] - u[i0]) - v[1:]
        upd = free & (cur < minv[1:])
        minv[1:][upd] = cur[upd]; way[1:][upd] = j0
        masked = np.where(free, minv[1:], np.inf)
        j1 = int(np.argmin(masked)) + 1
        delta = masked[j1 - 1]
        uj = np.nonzero(used)[0]
        u[p[uj]] += delta; v[uj] -= delta; minv[~used] -= delta
        j0 = j1
        if p[j0] == 0:
            break
    while True:
        j1 = way[j0]; p[j0] = p[j1]; j0 = j1
        if j0 == 0:
            break
uabs = np.array(uabs)
pm = np.empty(n, dtype=np.int64)
for j in range(1, n + 1):
    pm[p[j] - 1] = j - 1
print(f"R17 steps {len(uabs)} ({time.time() - t0:.1f} s); same perm as the GPU: {np.array_equal(pm, perm.cpu().numpy())}")
print(f"|u[i0]| == 0 at {np.mean(uabs == 0):.4f} of steps; quantiles of |u[i0]| (nonzero):",
      np.quantile(uabs[uabs > 0], [0.001, 0.01, 0.1, 0.5]))
# exactness: N < ulp(|u|)/4 with ulp(x) = 2^(floor(log2 x) − 52)
ulp4 = np.where(uabs > 0, np.ldexp(1.0, (np.floor(np.log2(np.where(uabs > 0, uabs, 1.0))) - 54).astype(int)), 0.0)
for tau in taus:
    print(f"tau={tau:.0e}: steps whose u[i0] makes the tau-sparse row exact {np.mean(ulp4 > tau):.4f}")
