import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2508_00887_b200 as fb
import oracle
for n in (4096, 2048, 3000, 1500):
    rng = np.random.Generator(np.random.PCG64(n))
    X = (rng.random((n, n)) * (rng.random((n, n)) < 0.1)).astype(np.float32)
    X[0, 0] = max(X[0, 0], 0.5)
    k = 12
    h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=k))
    D, kk, gam = fb.fram_sdsn(h, torch.tensor(X, device="cuda"), "fp32")
    D32, _, g32 = oracle.sdsn_fp32(X.astype(np.float64), 10.0, sdsn_fixed=k, return_gammas=True)
    e = np.max(np.abs(D.cpu().numpy().astype(np.float64) - D32)) * n
    print(n, kk, "err*n", e, "gamma err", np.max(np.abs(np.array(gam) - np.array(g32))), flush=True)
