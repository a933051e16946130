"""Dev probe: per-pass time of the row-sharded SDSN (K4s) in a one-rank sharded solve at n (default
16384): two solves with max_outer=1 and 50 / 250 fixed SDSN passes; the difference of their SDSN
phase times over 200 passes.  FP32 SDSN (bf16 GEMM operands)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
mode = sys.argv[3] if len(sys.argv) > 3 else "nccl"      # "nccl": one-rank NCCL handle (graph-captured
W = int(mode.split(":")[1]) if mode.startswith("virtual") else 1   # pass chunks); "virtual:W": W virtual ranks
# A = Ã = 0 and K = I: G = λI, so N stays near the identity and the final LAP takes n steps (a dense
# graph's N after one outer iteration makes the n = 16384 LAP take minutes).  The SDSN passes stream
# every element regardless of the values, so the per-pass time is that of a real input.
Ad = torch.zeros((n, n), dtype=torch.bfloat16, device="cuda")
Kd = torch.eye(n, dtype=torch.bfloat16, device="cuda")
res = {}
for k in (50, 250):
    sch = fb.Schedule(theta=10.0, max_outer=1, sdsn_fixed=k, flags=fb.FLAG_TIME_PHASES)
    if W > 1 or mode.startswith("virtual"):
        h = fb.fram_create_sharded_virtual(n, 1.0, sch, world=W)
    else:
        h = fb.fram_create_sharded(n, 1.0, sch, fb.fram_get_unique_id(), 0, 1, device=0)
    X = torch.empty((n, n), dtype=torch.float64, device="cuda")
    perm = torch.empty((n,), dtype=torch.int32, device="cuda")
    ts = []
    for _ in range(2):
        _, s, _, _ = fb.fram_solve(h, Ad, Ad, Kd, precision=prec, X_out=X, perm_out=perm)
        ts.append(s["ms_sdsn"])
    res[k] = min(ts)
es = 8 if prec == "fp64" else 4
print(f"n={n} {prec} sharded SDSN ({mode}, W={W}): {(res[250] - res[50]) / 200 * 1e3:.1f} us/pass, "
      f"{2 * es * n * n / ((res[250] - res[50]) / 200 * 1e-3) / 1e12:.2f} TB/s algorithmic")
