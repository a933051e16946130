"""Dev probe: structure of the C4 FRAM N seen by the LAP (ties, row-maximum conflicts)."""
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
_, st, X, perm = fb.fram_solve(h, A, B, precision="bf16")
N = X.cpu().numpy()
n = N.shape[0]
perm = perm.cpu().numpy()
rmax = N.max(1)
am = N.argmax(1)
ties = (N == rmax[:, None]).sum(1)
print("rows with tied maxima:", int((ties > 1).sum()), " max tie multiplicity:", int(ties.max()))
u, cnt = np.unique(am, return_counts=True)
print("distinct argmax columns:", len(u), " rows in conflicts:", int(cnt[cnt > 1].sum()))
print("LAP perm == row argmax for", int((perm == am).sum()), "rows")
srt = np.sort(N, 1)
gap = srt[:, -1] - srt[:, -2]
print("row max: median", np.median(rmax), " gap(max-second): min", gap.min(), "median", np.median(gap),
      " rows with gap < 1e-12:", int((gap < 1e-12).sum()), " < 1e-7:", int((gap < 1e-7).sum()))
# duplicated rows / columns (automorphism-like symmetry)
_, ridx = np.unique(N, axis=0, return_inverse=True)
print("distinct rows:", ridx.max() + 1, "of", n)
_, cidx = np.unique(N.T, axis=0, return_inverse=True)
print("distinct columns:", cidx.max() + 1, "of", n)
