"""Dev probe: where the end-to-end (host-buffer) C4 solve spends its extra time — median solve time with
device or pinned-host inputs (A, B) and output (X_out)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_00887_b200 as fb
from synth import config_c4

inst = config_c4(0)
n = inst.n
Ad = torch.tensor(inst.A, dtype=torch.float32, device="cuda"); Bd = torch.tensor(inst.B, dtype=torch.float32, device="cuda")
Ah, Bh = Ad.cpu().pin_memory(), Bd.cpu().pin_memory()
Xd = torch.empty((n, n), dtype=torch.float64, device="cuda"); Xh = torch.empty((n, n), dtype=torch.float64).pin_memory()
pd = torch.empty((n,), dtype=torch.int32, device="cuda"); ph = torch.empty((n,), dtype=torch.int32).pin_memory()
h = fb.fram_create(n, schedule=fb.Schedule(theta=10.0))
st = torch.cuda.current_stream()
for name, A, B, X, p in (("dev in / dev out", Ad, Bd, Xd, pd), ("host in / dev out", Ah, Bh, Xd, pd),
                         ("dev in / host out", Ad, Bd, Xh, ph), ("host in / host out", Ah, Bh, Xh, ph)):
    fb.fram_solve(h, A, B, precision="bf16", X_out=X, perm_out=p, stream=st)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fb.fram_solve(h, A, B, precision="bf16", X_out=X, perm_out=p, stream=st); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{name:20s} {sorted(ts)[2]:8.2f} ms")
