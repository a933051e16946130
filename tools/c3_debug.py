import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2508_00887_b200 as fb, oracle
from synth import config_c3_batch
insts = config_c3_batch(8)
g = lambda x, dt=torch.float32: torch.tensor(np.ascontiguousarray(x), dtype=dt, device="cuda")
for b in range(3):
    inst = insts[b]
    for prec in ("fp64", "bf16"):
        h = fb.fram_create(64, schedule=fb.Schedule(theta=2.0, flags=fb.FLAG_TRACE))
        st, s, X, p = fb.fram_solve(h, g(inst.A), g(inst.B), g(inst.K), precision=prec)
        print(b, prec, "single: outer", s["outer_iters"], "passes", s["passes"][:12], "tot", s["total_passes"])
    for prec in ("fp64", "bf16"):
        hb = fb.fram_create(64, schedule=fb.Schedule(theta=2.0))
        st, s, X, p, sts = fb.fram_solve_batched(hb, g(inst.A[None]), g(inst.B[None]), g(inst.K[None]), precision=prec)
        print(b, prec, "batched: outer", s["outer_iters"], "tot", s["total_passes"])
ref = oracle.fram(insts[0].A, insts[0].B, insts[0].K, theta=2.0)
print("oracle inst0 outer", len(ref["passes"]), ref["passes"][:12], sum(ref["passes"]))
