"""Write tests/golden/c4_oracle.json: the FP64 oracle's FRAM solve of BASELINE config C4
(n = 4096 Barabási–Albert, seed 0, default schedule R3/R4: θ=10, α=0.95, λ=1, γ_th=1e-3,
δ_th=1e-4, max_outer=100, sdsn_max=1000, X0 = 11ᵀ/n).

Calls only `oracle/` (and the seeded generator `synth/`, which holds no method arithmetic).
Nothing here comes from the CUDA path.  The run takes ~2 h on one host core (the SDSN passes
are single-threaded NumPy), so it checkpoints N after every outer iteration under --ckpt and
resumes from there: the iteration is memoryless apart from t, so resuming with X0 = N_t
continues the same sequence (same arithmetic on the same N).

Usage:  python tools/make_golden_c4.py [--ckpt /tmp/golden_c4] [--out tests/golden/c4_oracle.json]
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import config_c4, SCHEDULES  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ckpt", default="/tmp/golden_c4")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c4_oracle.json"))
    ap.add_argument("--n", type=int, default=4096)
    args = ap.parse_args()
    os.makedirs(args.ckpt, exist_ok=True)
    inst = config_c4(0, n=args.n)
    sch = dict(SCHEDULES["default"])
    tr_path = os.path.join(args.ckpt, "trace.json")
    n_path = os.path.join(args.ckpt, "N.npy")
    trace = {"passes": [], "deltas": [], "secs": []}
    X0 = None
    if os.path.exists(tr_path) and os.path.exists(n_path):
        trace = json.load(open(tr_path))
        X0 = np.load(n_path)
        print(f"resuming after t={len(trace['passes'])}", flush=True)
    t_done = len(trace["passes"])
    last = [time.time()]

    def on_iter(t, N, k, delta):
        np.save(n_path + ".tmp.npy", N)
        os.replace(n_path + ".tmp.npy", n_path)
        trace["passes"].append(int(k))
        trace["deltas"].append(float(delta))
        trace["secs"].append(time.time() - last[0])
        last[0] = time.time()
        with open(tr_path + ".tmp", "w") as f:
            json.dump(trace, f)
        os.replace(tr_path + ".tmp", tr_path)
        print(f"t={t_done + t} k={k} delta={delta:.6e} {trace['secs'][-1]:.1f}s", flush=True)

    done = bool(trace["deltas"]) and trace["deltas"][-1] <= sch["delta_th"]
    if not done and t_done < sch["max_outer"]:
        out = oracle.fram(inst.A, inst.B, inst.K, lam=inst.lam, theta=inst.theta,
                          alpha=sch["alpha"], gamma_th=sch["gamma_th"], delta_th=sch["delta_th"],
                          max_outer=sch["max_outer"] - t_done, sdsn_max=sch["sdsn_max"],
                          X0=X0, on_iter=on_iter)
        N, perm = out["N"], out["perm"]
    else:
        N = np.load(n_path)
        perm = oracle.lap_max(N)
    T = len(trace["passes"])
    converged = trace["deltas"][-1] <= sch["delta_th"]
    res = {
        "source": "tools/make_golden_c4.py (oracle/ only; FP64 Alg.1 P:322-342 + Alg.2 P:344-361 "
                  "+ R17 LAP P:337)",
        "config": "C4 n=%d BA(m=5), 5%% rewiring, seed 0, K=0" % args.n,
        "schedule": dict(sch, theta=inst.theta, lam=inst.lam, X0="uniform 1/n"),
        "outer_iters": T,
        "converged": bool(converged),
        "passes": trace["passes"],
        "deltas": trace["deltas"],
        "total_passes": int(sum(trace["passes"])),
        "perm": [int(x) for x in perm],
        "phi_perm": oracle.objective_perm(inst.A, inst.B, inst.K, perm, inst.lam),
        "phi_true": oracle.objective_perm(inst.A, inst.B, inst.K, inst.perm_true, inst.lam),
        "phi_N": oracle.objective(inst.A, inst.B, inst.K, N, inst.lam),
        "accuracy": oracle.node_accuracy(perm, inst.perm_true),
        "matching_error": oracle.matching_error(inst.A, inst.B, perm),
        "N_sum": float(N.sum()),
        "N_fro": float(np.linalg.norm(N)),
        "host_seconds": float(sum(trace["secs"])),
        "git": subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                              capture_output=True, text=True).stdout.strip(),
    }
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k not in ("perm", "deltas", "passes")}))


if __name__ == "__main__":
    main()
