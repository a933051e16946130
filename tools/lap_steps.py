"""Dev probe: count R17-Hungarian Dijkstra steps per row on the N of a C4 GPU solve."""
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
N = X.cpu().numpy()
n = N.shape[0]
srt = np.sort(N, 1)
print("row max mean", srt[:, -1].mean(), "max/second", np.mean(srt[:, -1] / srt[:, -2]))
C = -N
INF = np.inf
u = np.zeros(n + 1); v = np.zeros(n + 1); p = np.zeros(n + 1, np.int64); way = np.zeros(n + 1, np.int64)
steps = np.zeros(n, np.int64)
t0 = time.time()
for i in range(1, n + 1):
    p[0] = i; j0 = 0; minv = np.full(n + 1, INF); used = np.zeros(n + 1, bool)
    while True:
        steps[i - 1] += 1
        used[j0] = True; i0 = p[j0]; free = ~used[1:]
        cur = (C[i0 - 1, :] - u[i0]) - v[1:]
        upd = free & (cur < minv[1:]); minv[1:][upd] = cur[upd]; way[1:][upd] = j0
        masked = np.where(free, minv[1:], INF); j1 = int(np.argmin(masked)) + 1; delta = masked[j1 - 1]
        uj = np.nonzero(used)[0]; u[p[uj]] += delta; v[uj] -= delta; minv[~used] -= delta
        j0 = j1
        if p[j0] == 0:
            break
    while True:
        j1 = way[j0]; p[j0] = p[j1]; j0 = j1
        if j0 == 0:
            break
print("time", time.time() - t0, "total steps", steps.sum(), "mean", steps.mean(), "max", steps.max())
print("hist", np.bincount(np.minimum(steps, 20)))
print("steps by row quartile", [steps[k * n // 4:(k + 1) * n // 4].mean() for k in range(4)])
