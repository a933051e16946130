"""C5 (n = 16384, BF16 storage, rows sharded) on ONE GPU through the virtual-shard group at W = 2/4/8:
the W-rank path of the sharded solve at full size (per rank n/W rows of A and G, K-blocked GEMM operand
over W gathered Uᵀ blocks, per-pass all-reduces, N all-gather + LAP), against the one-rank NCCL handle
with the same schedule (bounded: `max_outer` outer iterations).  Prints one JSON line per W."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb
from synth import config_c5

max_outer = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = config_c5(0)
n = inst.n
A = torch.tensor(inst.A, dtype=torch.bfloat16, device="cuda")
B = torch.tensor(inst.B, dtype=torch.bfloat16, device="cuda")
sch = fb.Schedule(theta=inst.theta, max_outer=max_outer, flags=fb.FLAG_TRACE | fb.FLAG_TIME_PHASES)
h1 = fb.fram_create_sharded(n, 1.0, sch, fb.fram_get_unique_id(), 0, 1)
t0 = time.time()
_, s1, X1, p1 = fb.fram_solve(h1, A, B, precision="bf16")
torch.cuda.synchronize()
base = dict(W=1, kind="nccl", wall_s=time.time() - t0, passes=s1["passes"], deltas=s1["deltas"],
            accuracy=float((p1.cpu().numpy() == inst.perm_true).mean()))
print(json.dumps(base), flush=True)
for W in (2, 4, 8):
    h = fb.fram_create_sharded_virtual(n, 1.0, sch, world=W)
    t0 = time.time()
    _, s, X, p = fb.fram_solve(h, A, B, precision="bf16")
    torch.cuda.synchronize()
    dX = float((X - X1).abs().max().item())
    print(json.dumps(dict(W=W, kind="virtual", wall_s=time.time() - t0, passes=s["passes"], deltas=s["deltas"],
                          max_abs_dN_vs_W1=dX, perm_equal_W1=bool(torch.equal(p, p1)),
                          accuracy=float((p.cpu().numpy() == inst.perm_true).mean()))), flush=True)
    del h, X, p
    torch.cuda.empty_cache()
