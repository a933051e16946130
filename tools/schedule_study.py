"""NEXT-4 schedule study: FRAM under different SDSN schedules — the accuracy /
time-to-solution trade-off of reading R3 (γ_th, sdsn_max) and of θ.  One JSON line per
schedule.  `python tools/schedule_study.py [c4|c5]`: C4 (n=4096, bf16 GEMM / fp32 SDSN, single-GPU path)
or C5 (n=16384 weighted ER, BF16 storage, the row-sharded path at W = 1, one solve per schedule)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb
from synth import config_c4, config_c5

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
if which == "c5":
    inst = config_c5(0)
    A = torch.tensor(inst.A, dtype=torch.bfloat16, device="cuda")
    B = torch.tensor(inst.B, dtype=torch.bfloat16, device="cuda")
    grid = [dict(theta=10.0, gamma_th=1e-3, sdsn_max=m) for m in (100, 300, 1000)]
    grid += [dict(theta=10.0, gamma_th=g, sdsn_max=3000) for g in (0.1, 0.01)]
    grid += [dict(theta=th, gamma_th=1e-3, sdsn_max=1000) for th in (5.0, 20.0)]
else:
    inst = config_c4(0)
    A = torch.tensor(inst.A, dtype=torch.float32, device="cuda")
    B = torch.tensor(inst.B, dtype=torch.float32, device="cuda")
    grid = [dict(theta=10.0, gamma_th=1e-3, sdsn_max=m) for m in (30, 100, 300, 1000, 3000)]
    grid += [dict(theta=10.0, gamma_th=g, sdsn_max=20000) for g in (0.1, 0.03, 0.01)]
    grid += [dict(theta=th, gamma_th=1e-3, sdsn_max=1000) for th in (2.0, 5.0, 20.0)]
for cfg in grid:
    sch = fb.Schedule(theta=cfg["theta"], gamma_th=cfg["gamma_th"], sdsn_max=cfg["sdsn_max"], max_outer=100,
                      flags=fb.FLAG_TRACE | fb.FLAG_TIME_PHASES)
    if which == "c5":
        h = fb.fram_create_sharded(inst.n, 1.0, sch, fb.fram_get_unique_id(), 0, 1)
    else:
        h = fb.fram_create(inst.n, schedule=sch)
        fb.fram_solve(h, A, B, precision="bf16")                 # warm-up (workspace, clocks)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    st, s, X, perm = fb.fram_solve(h, A, B, precision="bf16")
    b.record()
    b.synchronize()
    acc = float((perm.cpu().numpy() == inst.perm_true).mean())
    print(json.dumps(dict(cfg, config=which, n=inst.n, time_to_solution_ms=a.elapsed_time(b), outer_iters=s["outer_iters"],
                          converged=bool(s["converged"]), total_passes=s["total_passes"],
                          mean_passes=s["total_passes"] / max(1, s["outer_iters"]), accuracy=acc,
                          ms_lap=s["ms_lap"])), flush=True)
