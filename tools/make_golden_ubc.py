"""Write tests/golden/ubc2000_oracle.json: the FP64 oracle's attributed FRAM solve (oracle.fram_attributed,
Alg. 1 P:322-342 with K = F F̃ᵀ) of the NEXT-2 stand-in for the paper's ubc(2000) task
(synth.config_ubc(0), n = 2000, θ = 2, λ = 1, default schedule R3).  Calls only oracle/ and synth/."""
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from synth import config_ubc, SCHEDULES  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
out_path = os.path.join(ROOT, "tests", "golden", f"ubc{n}_oracle.json")
inst = config_ubc(0, n=n)
F, Ft = inst.meta["F"], inst.meta["Ft"]
sch = dict(SCHEDULES["default"])
t0 = time.time()
out = oracle.fram_attributed(inst.A, inst.B, F, Ft, n, lam=inst.lam, theta=inst.theta, alpha=sch["alpha"],
                             gamma_th=sch["gamma_th"], delta_th=sch["delta_th"], max_outer=sch["max_outer"],
                             sdsn_max=sch["sdsn_max"])
perm = out["perm_attr"]
K = oracle.unary_from_features(F, Ft)
res = {
    "source": "tools/make_golden_ubc.py (oracle/ only: fram_attributed, matching_error, objective_perm)",
    "config": f"synth.config_ubc(0, n={n}): fully connected Euclidean-distance keypoint graphs, d=128 features",
    "schedule": dict(sch, theta=inst.theta, lam=inst.lam),
    "outer_iters": out["outer_iters"], "converged": bool(out["converged"]), "passes": out["passes"],
    "deltas": out["deltas"], "perm": [int(x) for x in perm],
    "accuracy": oracle.node_accuracy(perm, inst.perm_true),
    "matching_error": oracle.matching_error(inst.A, inst.B, perm, F, Ft),
    "matching_error_true": oracle.matching_error(inst.A, inst.B, inst.perm_true, F, Ft),
    "phi_perm": oracle.objective_perm(inst.A, inst.B, K, perm, inst.lam),
    "host_seconds": time.time() - t0,
    "git": subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True, text=True).stdout.strip(),
}
with open(out_path, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps({k: v for k, v in res.items() if k not in ("perm", "passes", "deltas")}))
