"""Dev probe: on the N of a C4 solve, how often is the next Dijkstra step's winner among the current
step's top-k (by minv) candidates?  (Guides speculative row prefetch in the GPU LAP.)"""
import os
import sys

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
C = -N
INF = np.inf
u = np.zeros(n + 1); v = np.zeros(n + 1); p = np.zeros(n + 1, np.int64); way = np.zeros(n + 1, np.int64)
hits = {1: 0, 2: 0, 4: 0, 8: 0}
rowhit = {2: 0, 4: 0, 8: 0}
steps = 0
for i in range(1, n + 1):
    p[0] = i; j0 = 0; minv = np.full(n + 1, INF); used = np.zeros(n + 1, bool)
    prev_top = None
    while True:
        used[j0] = True; i0 = p[j0]; free = ~used[1:]
        cur = (C[i0 - 1, :] - u[i0]) - v[1:]
        upd = free & (cur < minv[1:]); minv[1:][upd] = cur[upd]; way[1:][upd] = j0
        masked = np.where(free, minv[1:], INF)
        order = np.argsort(masked, kind="stable")[:8] + 1
        j1 = int(order[0]); delta = masked[j1 - 1]
        if prev_top is not None:
            steps += 1
            for k in hits:
                if j1 in prev_top[:k]:
                    hits[k] += 1
        # prev_top for the next step: candidates other than j1 (j1 becomes used)
        prev_top = [int(c) for c in order[1:9]]
        uj = np.nonzero(used)[0]; u[p[uj]] += delta; v[uj] -= delta; minv[~used] -= delta
        j0 = j1
        if p[j0] == 0:
            break
    while True:
        j1 = way[j0]; p[j0] = p[j1]; j0 = j1
        if j0 == 0:
            break
print("steps with a predecessor:", steps, {k: round(hits[k] / max(steps, 1), 3) for k in hits})
