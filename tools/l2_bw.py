"""Dev probe: L2-resident streaming bandwidth on B200 (copy of buffers that fit in L2)."""
import torch
for mib in (16, 32, 48, 64, 96, 256, 1024):
    n = mib * 1024 * 1024 // 4
    a = torch.rand(n, device="cuda"); b = torch.empty_like(a)
    for _ in range(3): b.copy_(a)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    s.record()
    for _ in range(reps): b.copy_(a)
    e.record(); e.synchronize()
    t = s.elapsed_time(e) / reps
    print(f"copy {mib:5d} MiB src+dst {2*mib} MiB: {2 * n * 4 / t / 1e6:.0f} GB/s ({t*1e3:.1f} us)")
