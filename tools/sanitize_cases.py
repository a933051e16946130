"""compute-sanitizer driver: runs ONE small case of a libfram kernel per invocation, so that
memcheck / racecheck / synccheck can be applied kernel by kernel (tools/sanitize.sh).
Cases: k4r<n> (FP32 on-chip SDSN), k4c<n> (one-cluster SDSN, FP64 or FP32 small n), k4<n> (streaming
FP64 SDSN), k7<n> / k7c<n> (single-CTA / cluster LAP), k8 (batched n=64), gemm<n> (tcgen05 GEMMs),
k4s<n> (row-sharded SDSN, one rank), fram<n> (a full bf16 solve, max_outer 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb
from synth import config_c3_batch, random_nonneg, random_perm_matrix

kind = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
case = f"{kind}:{n}"
rng = np.random.Generator(np.random.PCG64(n))
dev = "cuda"
if kind in ("k4r", "k4c32"):              # FP32 (K4c for n ≤ 160, K4r above)
    X = torch.tensor(random_nonneg(rng, n, "sparse") + np.eye(n), dtype=torch.float32, device=dev)
    h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=3))
    D, k, _ = fb.fram_sdsn(h, X, "fp32")
elif kind in ("k4c", "k4"):
    X = torch.tensor(random_nonneg(rng, n, "sparse") + np.eye(n), dtype=torch.float64, device=dev)
    h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=3))
    D, k, _ = fb.fram_sdsn(h, X, "fp64")
elif kind in ("k7", "k7c"):
    N = 0.8 * random_perm_matrix(rng, n) + 0.2 * rng.random((n, n)) / n
    h = fb.fram_create(n)
    p = fb.fram_lap(h, torch.tensor(N, device=dev))
elif kind == "k8":
    insts = config_c3_batch(8)
    st = lambda a: torch.tensor(np.stack([getattr(i, a) for i in insts]), dtype=torch.float32, device=dev)
    h = fb.fram_create(64, schedule=fb.Schedule(theta=2.0, max_outer=3))
    fb.fram_solve_batched(h, st("A"), st("B"), st("K"), precision="bf16")
elif kind == "gemm":
    A = torch.tensor(rng.random((n, n)), dtype=torch.float64, device=dev)
    A = A + A.T
    N = torch.full((n, n), 1.0 / n, dtype=torch.float64, device=dev)
    h = fb.fram_create(n)
    fb.fram_gradient(h, A, A, None, N, "bf16")
elif kind == "k4s":
    A = rng.random((n, n))
    A = torch.tensor(A + A.T, dtype=torch.float64, device=dev)
    h = fb.fram_create_sharded(n, 1.0, fb.Schedule(theta=10.0, max_outer=1, sdsn_fixed=3), fb.fram_get_unique_id(), 0, 1)
    fb.fram_solve(h, A, A, precision="fp64")
elif kind == "fram":
    A = rng.random((n, n)) * (rng.random((n, n)) < 0.1)
    A = torch.tensor(A + A.T, dtype=torch.float32, device=dev)
    h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, max_outer=2, sdsn_max=5))
    fb.fram_solve(h, A, A, precision="bf16")
else:
    raise SystemExit(f"unknown case {case}")
torch.cuda.synchronize()
print("ok", case)
