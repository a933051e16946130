"""Measure the peaks MEASURED_PEAKS.json does not carry, the same way it measures BF16 (torch.matmul
8192³, 2·N³ flop, best of 10 = burst; back to back for 4 s = sustained; CUDA events): TF32 (the
paper's step-5 precision), FP16, and FP64 (cuBLAS DGEMM = the DMMA tensor-core path, the
paper's "GPU-FP64" comparison); plus the L2-resident copy bandwidth (read + write bytes of a
buffer pair that fits in the 126 MB L2) as the ceiling for streaming kernels whose iterate stays in L2.
Writes profiles/measured_peaks_extra.json."""
import json
import os
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gemm_rate(dtype, n=8192, tf32=False):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = torch.empty(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    burst = 2 * n ** 3 / (best / 1e3) / 1e12
    reps, t0 = 0, time.time()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b, out=c)
        reps += 1
        if reps % 8 == 0:
            torch.cuda.synchronize()
    e.record()
    e.synchronize()
    sust = 2 * n ** 3 * reps / (s.elapsed_time(e) / 1e3) / 1e12
    torch.backends.cuda.matmul.allow_tf32 = False
    return burst, sust


def l2_copy_gbs(mib=32, reps=200):
    n = mib * 1024 * 1024 // 4
    a = torch.rand(n, device="cuda")
    b = torch.empty_like(a)
    for _ in range(5):
        b.copy_(a)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        b.copy_(a)
    e.record()
    e.synchronize()
    return 2 * n * 4 * reps / (s.elapsed_time(e) / 1e3) / 1e9


def main():
    out = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "how": __doc__.split("\n")[0] + " (tools/measure_peaks.py)"}
    for name, dt, tf in (("tf32", torch.float32, True), ("fp16", torch.float16, False), ("fp64", torch.float64, False)):
        b, s = gemm_rate(dt, tf32=tf)
        out[f"{name}_tflops"] = b
        out[f"{name}_tflops_sustained"] = s
    out["l2_copy_gbs_32mib"] = l2_copy_gbs(32)
    out["l2_copy_gbs_48mib"] = l2_copy_gbs(48)
    path = os.path.join(ROOT, "profiles", "measured_peaks_extra.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
