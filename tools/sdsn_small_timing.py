"""Dev probe: SDSN time per pass at small n for the kernel the library picks (compare K4r / K4 with
variant libraries: bash tools/build_variant.sh <name> fram_api.cu -DFRAM_DEV_NOCLUSTER=1 or
-DFRAM_DEV_FORCE_STREAM=1, then bash tools/ab.sh python tools/sdsn_small_timing.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_00887_b200 as fb

k = 400
tag = os.environ.get("TAG", "default")
for n in (20, 64, 128, 256, 384, 500, 600, 800):
    for prec, dt in (("fp32", torch.float32), ("fp64", torch.float64)):
        rng = np.random.Generator(np.random.PCG64(n))
        X = torch.tensor(rng.random((n, n)), dtype=dt, device="cuda")
        h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0, sdsn_fixed=k))
        try:
            fb.fram_sdsn(h, X, prec, want_gammas=False)
        except Exception as e:
            print(tag, n, prec, "error", e)
            continue
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(3):
            e0.record()
            fb.fram_sdsn(h, X, prec, want_gammas=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{tag} n={n} {prec}: {min(ts) * 1e3 / k:.2f} us/pass", flush=True)
