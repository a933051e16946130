"""Dev tool: time-to-solution and accuracy of one FRAM solve at the BASELINE configs C1, C2, C4 in each
precision mode (CUDA events around fram_solve, 1 warm-up + 3 timed solves, median), with the FP64
oracle's accuracy beside it for C1/C2 (oracle run with its own γ test).  Writes JSON lines to stdout."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2508_00887_b200 as fb
from synth import config_c1, config_c2, config_c4


def run(inst, prec, reps=3, with_oracle=False):
    n = inst.n
    dt = torch.float64 if prec == "fp64" else torch.float32
    A = torch.tensor(inst.A, dtype=dt, device="cuda")
    B = torch.tensor(inst.B, dtype=dt, device="cuda")
    h = fb.fram_create(n, schedule=fb.Schedule(theta=inst.theta))
    fb.fram_solve(h, A, B, precision=prec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        st, stats, X, perm = fb.fram_solve(h, A, B, precision=prec)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    p = perm.cpu().numpy()
    acc = float(np.mean(p == inst.perm_true))
    out = {"config": inst.name, "n": n, "precision": prec, "ms_to_solution": statistics.median(ts),
           "outer_iters": stats["outer_iters"], "total_passes": stats["total_passes"], "accuracy": acc,
           "converged": bool(stats["converged"])}
    if with_oracle:
        t0 = time.time()
        ref = oracle.fram(inst.A, inst.B, None, theta=inst.theta)
        out["oracle_accuracy"] = float(np.mean(np.asarray(ref["perm"]) == inst.perm_true))
        out["oracle_outer_iters"] = int(ref["outer_iters"]) if "outer_iters" in ref else None
        out["oracle_seconds"] = time.time() - t0
        phi = oracle.objective_perm(inst.A, inst.B, None, p)
        phi_o = oracle.objective_perm(inst.A, inst.B, None, np.asarray(ref["perm"]))
        out["objective_rel_diff_vs_oracle"] = abs(phi - phi_o) / max(abs(phi_o), 1e-300)
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c4"]
    if "c1" in which:
        for prec in ("fp64", "tf32", "bf16"):
            print(json.dumps(run(config_c1(0), prec, with_oracle=(prec == "fp64"))), flush=True)
    if "c2" in which:
        for prec in ("fp64", "tf32"):
            print(json.dumps(run(config_c2(0), prec, with_oracle=(prec == "fp64"))), flush=True)
    if "c4" in which:
        for prec in ("bf16", "tf32", "fp16", "fp64"):
            print(json.dumps(run(config_c4(0), prec, reps=2)), flush=True)
