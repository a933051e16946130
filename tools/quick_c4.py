"""Dev probe: one C4 (n=4096) bf16 solve with phase timing (not the bench)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_00887_b200 as fb
from synth import config_c4
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
t0 = time.time(); inst = config_c4(0); print("gen", time.time() - t0, flush=True)
A = torch.tensor(inst.A, dtype=torch.float32, device="cuda"); B = torch.tensor(inst.B, dtype=torch.float32, device="cuda")
h = fb.fram_create(inst.n, schedule=fb.Schedule(theta=10.0, flags=fb.FLAG_TRACE | fb.FLAG_CHECK_SYMMETRY | fb.FLAG_TIME_PHASES))
for rep in range(2):
    t0 = time.time()
    st, s, X, perm = fb.fram_solve(h, A, B, precision=prec)
    torch.cuda.synchronize()
    wall = time.time() - t0
    acc = float((perm.cpu().numpy() == inst.perm_true).mean())
    n = inst.n
    print(f"status={st} wall={wall:.3f}s outer={s['outer_iters']} passes={s['total_passes']} acc={acc:.4f}")
    print({k: round(v, 3) for k, v in s.items() if k.startswith("ms_")}, "launches", s["kernel_launches"])
    gbs = 8.0 * n * n * s["total_passes"] / (s["ms_sdsn"] * 1e-3) / 1e9
    tf = 4.0 * n**3 * s["outer_iters"] / (s["ms_gemm"] * 1e-3) / 1e12
    print(f"SDSN algorithmic GB/s={gbs:.1f}  GEMM TFLOP/s={tf:.1f}  us/pass={s['ms_sdsn']*1e3/s['total_passes']:.2f}")
    print("passes per iter", s["passes"][:10], "...", s["passes"][-3:])
