import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2508_00887_b200 as fb
from synth import config_c1
inst = config_c1(0)
A = torch.tensor(inst.A, device="cuda"); B = torch.tensor(inst.B, device="cuda")
h = fb.fram_create(20, schedule=fb.Schedule(theta=10.0, max_outer=20))
st, s, X, p = fb.fram_solve(h, A, B, precision="fp64")
r = oracle.fram(inst.A, inst.B, None, theta=10.0, max_outer=20)
print("gpu passes", s["passes"]); print("orc passes", r["passes"])
print("gpu deltas", ["%.3e" % d for d in s["deltas"]]); print("orc deltas", ["%.3e" % d for d in r["deltas"]])
# first SDSN call directly
Ap, Bp, Kp, c = oracle.precondition(inst.A, inst.B, None)
G = oracle.gradient(Ap, np.full((20, 20), 0.05), Bp, Kp, 1.0)
h2 = fb.fram_create(20, schedule=fb.Schedule(theta=10.0))
D, k, gam = fb.fram_sdsn(h2, torch.tensor(G, device="cuda"), "fp64")
Do, ko, go = oracle.sdsn(G, 10.0, return_gammas=True)
print("sdsn k", k, ko, "maxdiff", np.abs(D.cpu().numpy() - Do).max())
print("gam gpu", gam[:5], gam[-3:]); print("gam orc", go[:5], go[-3:])
