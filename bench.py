#!/usr/bin/env python
"""bench.py — FRAM iterations/s and time-to-solution at n=4096 (BASELINE.json `metric`, config C4).

One *step* = one complete fram_solve (Alg. 1: preconditioning, the outer loop of
tcgen05 gradient GEMMs + SDSN passes + FP64 update/δ, and the final GPU Hungarian) on the C4
workload: Barabási–Albert n=4096 (m=5), Ã = P·A·Pᵀ with 5% edge rewiring, X0 = 11ᵀ/n,
bf16-GEMM / fp32-SDSN, θ=10, α=0.95, λ=1, γ_th=1e-3, δ_th=1e-4, sdsn_max=1000, max_outer=100.
`value` = outer iterations of all ranks ÷ max-over-ranks device time of the K timed steps.

Multi-GPU (--gpus N, torchrun): C4 does not shard: each rank solves an independent
replica (seed = rank), no data-path collective ("scaling": "weak").

--impl reference: the FP64 CPU oracle (oracle/) as it stands, on a bounded sample of the same
workload (one gradient + a few SDSN passes + one update per step, extrapolated to iterations/s).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

# stdout carries exactly one JSON line per run.  Native libraries print to fd 1 on their own (NCCL
# prints its "NCCL version" banner under NCCL_DEBUG=VERSION straight to stdout), so while the bench runs
# fd 1 points at stderr and the JSON line is written to the saved original stdout (emit()).
_JSON_FD = None


def _claim_stdout():
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line):
    """Write the run's JSON line to the real stdout."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FRAM iters/s & time-to-solution at n=4096; GEMM TC util %, SDSN HBM GB/s"
UNIT = "outer iterations/s"
def workload(prec):
    sd = "fp64-SDSN" if prec == "fp64" else "fp32-SDSN"
    return f"C4: BA(m=5) n=4096, 5% rewiring, X0=11^T/n, {prec}-GEMM/{sd}, theta=10"


def dtype_label(prec):
    return "f64" if prec == "fp64" else f"{prec}-gemm/f32-sdsn/f64-update"
SCHEDULE = dict(theta=10.0, alpha=0.95, lam=1.0, gamma_th=1e-3, delta_th=1e-4, sdsn_max=1000, max_outer=100)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--precision", default="bf16", choices=["bf16", "tf32", "fp16", "fp64"])
    p.add_argument("--n", "--problem-size", dest="n", type=int, default=4096,
                   help="dev override (the metric is quoted at 4096); use --problem-size under torchrun")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-extra-precisions", action="store_true",
                   help="skip the TF32 (the paper's step-5 precision) and FP64 C4 solves reported beside the main line")
    p.add_argument("--workload", default="c4", choices=["c4", "c3", "c5", "ubc"],
                   help="c4: the metric's config (n=4096, replicas across ranks); c3: 4096 keypoint instances "
                        "(n=64) split across the ranks, one CTA per instance; c5: n=16384 row-sharded across "
                        "the ranks (NCCL); ubc: NEXT-2, the paper's ubc(2000) regime (n=2000 fully connected "
                        "keypoint graphs with 128-d features, theta=2), mixed vs FP64.  c3/c5/ubc are not part of "
                        "the default run")
    p.add_argument("--max-outer", type=int, default=None, help="c5: cap on outer iterations per solve (bounded runs)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), \
            "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


# B200 nominal dense tensor rates relative to BF16 (2.25 PFLOP/s): TF32 1/2, FP16 1, FP64 40 TF/s (DMMA)
NOMINAL_RATIO = {"bf16": 1.0, "fp16": 1.0, "tf32": 0.5, "fp64": 40.0 / 2250.0}


def gemm_peak(prec):
    """Sustained dense GEMM peak for the operand format: measured (profiles/measured_peaks_extra.json,
    tools/measure_peaks.py, the same recipe as MEASURED_PEAKS.json's BF16) when present, else the BF16
    measured sustained peak × the nominal ratio."""
    _, _, bf16s, src = peaks()
    if prec == "bf16":
        return bf16s, f"{src} bf16_tflops_sustained"
    try:
        with open(os.path.join(ROOT, "profiles", "measured_peaks_extra.json")) as f:
            d = json.load(f)
        return float(d[f"{prec}_tflops_sustained"]), f"profiles/measured_peaks_extra.json {prec}_tflops_sustained"
    except Exception:
        return bf16s * NOMINAL_RATIO[prec], f"{src} bf16 sustained x nominal {prec}/bf16 ratio {NOMINAL_RATIO[prec]:.4g}"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"] or [1])
    except Exception:
        return 1


def oracle_sample(inst, passes_per_iter, budget_s=12.0):
    """Time the FP64 oracle (as it stands) on a bounded sample of one outer iteration of the workload:
    precondition, one gradient (two BLAS GEMMs), a few SDSN passes, one update; extrapolate one outer
    iteration to `passes_per_iter` SDSN passes.  Returns (iters_per_s, seconds_used, description)."""
    import numpy as np
    import oracle

    t0 = time.perf_counter()
    Ap, Bp, Kp, c = oracle.precondition(inst.A, inst.B, inst.K)
    n = inst.n
    N = np.full((n, n), 1.0 / n)
    tg = time.perf_counter()
    G = oracle.gradient(Ap, N, Bp, Kp, 1.0)
    t_grad = time.perf_counter() - tg
    ts = time.perf_counter()
    oracle.sdsn(G, inst.theta, sdsn_fixed=2, check_nonneg=False)
    t2 = (time.perf_counter() - ts) / 2
    k = int(max(2, min(200, (budget_s - (time.perf_counter() - t0)) / max(t2, 1e-6))))
    ts = time.perf_counter()
    D, _ = oracle.sdsn(G, inst.theta, sdsn_fixed=k, check_nonneg=False)
    t_pass = (time.perf_counter() - ts) / k
    tu = time.perf_counter()
    N_new = (1.0 - 0.95) * N + 0.95 * D
    float(np.linalg.norm(N_new - N) / np.linalg.norm(N_new))
    t_upd = time.perf_counter() - tu
    it = t_grad + passes_per_iter * t_pass + t_upd
    desc = (f"FP64 NumPy oracle on the {inst.name} n={n} input: 1 gradient (2 BLAS GEMMs, {blas_threads()} BLAS "
            f"threads) {t_grad:.2f}s + {k} SDSN passes at {t_pass * 1e3:.1f} ms/pass (NumPy, one core) + 1 update "
            f"{t_upd:.2f}s, timed; one outer iteration extrapolated to {passes_per_iter:.0f} passes/iteration")
    return 1.0 / it, time.perf_counter() - t0, desc, t_pass, t_grad


def _oracle_worker(args):
    n, ppi, budget = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from synth import config_c4
    return oracle_sample(config_c4(0, n=n), ppi, budget_s=budget)[0]


def oracle_all_cores(n, ppi, budget_s=10.0):
    """The oracle's SDSN pass is single-threaded NumPy, so the host's full capacity is measured the way
    a multi-core user would get it: P = os.cpu_count() independent oracle samples in P processes at
    once (one BLAS thread each); aggregate iterations/s = Σ of the per-process rates."""
    import concurrent.futures as cf
    import multiprocessing as mp
    P = os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    with cf.ProcessPoolExecutor(max_workers=P, mp_context=ctx) as ex:
        rates = list(ex.map(_oracle_worker, [(n, ppi, budget_s)] * P))
    return sum(rates), P


def cpu_baseline_entry(inst, ppi, budget_s, all_cores=True):
    v, secs, desc, t_pass, _ = oracle_sample(inst, ppi, budget_s=budget_s)
    out = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": desc + " (cores = 1: the SDSN passes, >99% of the oracle's time, use one core)"}
    if all_cores:
        agg, P = oracle_all_cores(inst.n, ppi, budget_s=min(budget_s, 8.0))
        out["all_cores"] = {"value": agg, "unit": UNIT, "cores": P,
                            "sample": f"{P} independent oracle samples of the same workload run concurrently in "
                                      f"{P} processes (1 BLAS thread each); aggregate outer iterations/s"}
    return out


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    from synth import config_c4
    inst = config_c4(0, n=args.n)
    ppi = float(SCHEDULE["sdsn_max"])    # at C4 the 1000-pass cap binds on every call (R3, [M16], golden)
    for _ in range(args.warmup):
        oracle_sample(inst, ppi, budget_s=4.0)
    vals, secs = [], []
    desc = ""
    for _ in range(args.steps):
        v, s_, desc, _, _ = oracle_sample(inst, ppi, budget_s=8.0)
        vals.append(v)
        secs.append(s_)
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(secs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded C4 generator; SNAP Facebook-ego stand-in)",
            "config": {"workload": workload(args.precision), "n": args.n, "schedule": SCHEDULE, "seed": 0},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2508_00887_b200 as fb
    from synth import config_c4

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    inst = config_c4(seed=rank, n=args.n)
    n = inst.n
    A = torch.tensor(inst.A, dtype=torch.float32, device=dev)
    B = torch.tensor(inst.B, dtype=torch.float32, device=dev)
    flags = fb.FLAG_TRACE | fb.FLAG_CHECK_SYMMETRY | fb.FLAG_TIME_PHASES
    sch = fb.Schedule(theta=inst.theta, alpha=SCHEDULE["alpha"], gamma_th=SCHEDULE["gamma_th"],
                      delta_th=SCHEDULE["delta_th"], max_outer=SCHEDULE["max_outer"],
                      sdsn_max=SCHEDULE["sdsn_max"], flags=flags)
    h = fb.fram_create(n, lam=SCHEDULE["lam"], schedule=sch, device=local)
    X = torch.empty((n, n), dtype=torch.float64, device=dev)
    perm = torch.empty((n,), dtype=torch.int32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)     # 256 MiB > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()

    def timed(prec, steps, warmup, sampler=None):
        """`steps` device-timed solves (CUDA events on the current stream, L2 flushed before each)."""
        for _ in range(warmup):
            fb.fram_solve(h, A, B, precision=prec, X_out=X, perm_out=perm)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.start()
        stats = []
        for k in range(steps):
            flush.fill_(float(k))                                         # L2 flush, outside the events
            ev[k][0].record()
            st, s_, _, _ = fb.fram_solve(h, A, B, precision=prec, X_out=X, perm_out=perm)
            ev[k][1].record()
            stats.append(s_)
        torch.cuda.synchronize()
        barrier()
        clocks = sampler.stop() if sampler else None
        return [a.elapsed_time(b) for a, b in ev], stats, clocks

    def allmax(v):
        if world == 1:
            return float(v)
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(v):
        if world == 1:
            return float(v)
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    step_ms, stats, clocks = timed(args.precision, args.steps, args.warmup, ClockSampler(local))
    tot_ms = sum(step_ms)
    iters = sum(s_["outer_iters"] for s_ in stats)
    passes = sum(s_["total_passes"] for s_ in stats)
    launches = sum(s_["kernel_launches"] for s_ in stats)
    ms_sdsn = sum(s_["ms_sdsn"] for s_ in stats)
    ms_gemm = sum(s_["ms_gemm"] for s_ in stats)
    ms_lap = sum(s_["ms_lap"] for s_ in stats)
    acc = float((perm.cpu().numpy() == inst.perm_true).mean())
    tot_ms_all, iters_all = allmax(tot_ms), allsum(iters)
    value = iters_all / (tot_ms_all / 1e3)

    # ---- e2e: same solve through the C ABI with pinned HOST buffers (H2D/D2H inside the region)
    e2e = None
    if not args.no_e2e:
        Ah = A.cpu().pin_memory()
        Bh = B.cpu().pin_memory()
        Xh = torch.empty((n, n), dtype=torch.float64).pin_memory()
        ph = torch.empty((n,), dtype=torch.int32).pin_memory()
        fb.fram_solve(h, Ah, Bh, precision=args.precision, X_out=Xh, perm_out=ph,
                      stream=torch.cuda.current_stream(dev))
        barrier()
        torch.cuda.synchronize()
        e_ms, e_it = 0.0, 0
        for k in range(args.steps):
            flush.fill_(float(k))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _, s_, _, _ = fb.fram_solve(h, Ah, Bh, precision=args.precision, X_out=Xh, perm_out=ph,
                                        stream=torch.cuda.current_stream(dev))
            b.record()
            b.synchronize()
            e_ms += a.elapsed_time(b)
            e_it += s_["outer_iters"]
        e_ms, e_it = allmax(e_ms), allsum(e_it)
        e2e = {"value": e_it / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(Ah.nbytes + Bh.nbytes),
               "d2h_bytes_per_step": int(Xh.nbytes + ph.nbytes)}

    hbm, bf16, bf16s, psrc = peaks()
    sdsn_launches = iters                                     # one persistent SDSN launch per outer iteration
    resident = stats[0].get("sdsn_kernel", 1) == 2
    avg_launch_s = ms_sdsn / 1e3 / sdsn_launches
    passes_per_launch = passes / sdsn_launches
    esz = 8.0 if args.precision == "fp64" else 4.0            # SDSN iterate: FP64 in FP64 mode, else FP32
    bytes_per_launch = 2.0 * esz * n * n * passes_per_launch  # algorithmic: Y read + write per pass
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "sdsn_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f).get("resident" if resident else
                                      ("streaming_fp64" if args.precision == "fp64" else "streaming"), {})
            if int(tj.get("n", 0)) == n:
                traffic = float(tj["dram_bytes_per_launch"]) if resident else \
                    float(tj["dram_bytes_per_pass"]) * passes_per_launch
        except Exception:
            traffic = None
    if resident:
        # K4r keeps Y on chip (TMEM + shared memory): HBM is touched only to load G and store D once per
        # launch, so the pass loop is bound by the SM datapath.  Roofline: 5 FP32 ops per
        # element per pass (x+a, +b, max, column and row accumulation).  The four adds run on the FP32
        # lanes (128 per SM per cycle; a paired FADD2 issues in 2 cycles, measured by tools/pipe_probe.cu)
        # while the max overlaps on the ALU pipe, so the element rate is 148 x 128 x f_max / 4 and the
        # op peak is 5/4 of the FP32 lane rate: 46.5 TFLOP/s at 1.965 GHz.
        f_max = 1.965e9
        alu_peak = 148 * 128 * f_max * 5.0 / 4.0 / 1e12
        achieved = 5.0 * n * n * passes_per_launch / avg_launch_s / 1e12
        roof = {"kernel": "sdsn_res_kernel<32> (K4r, on-chip resident; one persistent launch per SDSN call)",
                "bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "TFLOP/s",
                "frac": achieved / alu_peak, "traffic": traffic,
                "peak_source": "derived: 148 SM x 128 FP32 lanes x 1.965 GHz x 5/4 (4 FP32 adds per element on the "
                               "FP32 lanes, the max overlapped on the ALU pipe; B200_PROFILING.md unit counts, "
                               "FADD2 rate measured by tools/pipe_probe.cu)",
                "algorithmic_flops_per_launch": 5.0 * n * n * passes_per_launch,
                "hbm_note": "the iterate never leaves the chip, so the north star's >=70%-of-HBM SDSN target does "
                            "not apply to K4r: its DRAM traffic is the one G load + D store per launch",
                "dram": {"bytes_per_launch": traffic,
                         "achieved_gbs": (traffic / avg_launch_s / 1e9) if traffic else None,
                         "frac_of_hbm": (traffic / avg_launch_s / 1e9 / hbm) if traffic else None,
                         "source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                   "(profiles/sdsn_traffic.json) over the live launch time"}}
    else:
        hbm_equiv = bytes_per_launch / avg_launch_s / 1e9
        roof = {"kernel": f"sdsn_kernel<{'double' if esz == 8 else 'float'}> (K4, streaming through L2/HBM)",
                "bound": "hbm", "achieved": hbm_equiv,
                "peak": hbm, "unit": "GB/s", "frac": hbm_equiv / hbm, "traffic": traffic, "peak_source": psrc,
                "algorithmic_bytes_per_launch": bytes_per_launch}
        if traffic:
            # snake row order keeps part of the iterate in L2, so DRAM moves less than the algorithmic
            # bytes and the algorithmic rate can exceed the HBM peak; the DRAM rate is reported beside it
            roof["dram"] = {"achieved_gbs": traffic / avg_launch_s / 1e9, "frac": traffic / avg_launch_s / 1e9 / hbm,
                            "note": "ncu DRAM bytes per launch (profiles/sdsn_traffic.json) over the launch time"}
    roof.update({"passes_per_launch": passes_per_launch, "ms_per_launch": avg_launch_s * 1e3,
                 "us_per_pass": avg_launch_s * 1e6 / passes_per_launch, "share_of_step": ms_sdsn / tot_ms})

    def gemm_entry(prec, ms_gemm_, iters_, steps_):
        tfl = 4.0 * n ** 3 * iters_ / (ms_gemm_ / 1e3) / 1e12 if ms_gemm_ > 0 else None
        pk, src = gemm_peak(prec)
        out = {"tflops": tfl, "peak_tflops": pk, "peak_source": src, "frac_of_sustained": (tfl or 0) / pk,
               "ms_per_step": ms_gemm_ / steps_, "operand_format": prec}
        if prec == "bf16":
            # the metric's "GEMM TC util %": ncu sm__pipe_tensor_cycles_active of the two GEMMs at C4 (a profiler
            # number, from the committed capture, not measured in this run)
            out["tensor_pipe_active_pct_ncu"] = {"gemm1": 82.6, "gemm2": 73.4,
                                                 "source": "profiles/r02/ncu_prof_gemm_r02_raw.csv"}
        return out

    # ---- the paper's precisions beside the headline (TF32 = step 5 of Alg.1; FP64 = "GPU-FP64")
    extra = {}
    if not args.no_extra_precisions:
        for prec in ("tf32", "fp64"):
            if prec == args.precision:
                continue
            sm_, st_, _ = timed(prec, 2, 1)
            it_ = sum(x["outer_iters"] for x in st_)
            ms_ = allmax(sum(sm_))
            ms_s = sum(x["ms_sdsn"] for x in st_)
            ps_ = sum(x["total_passes"] for x in st_)
            extra[prec] = {"value": allsum(it_) / (ms_ / 1e3), "unit": UNIT, "time_to_solution_ms": statistics.median(sm_),
                           "outer_iters_per_solve": it_ / 2, "mean_passes_per_iter": ps_ / it_,
                           "accuracy": float((perm.cpu().numpy() == inst.perm_true).mean()),
                           "sdsn_us_per_pass": 1e3 * ms_s / ps_, "dtype": dtype_label(prec),
                           "gemm": gemm_entry(prec, sum(x["ms_gemm"] for x in st_), it_, 2),
                           "lap_ms_per_step": sum(x["ms_lap"] for x in st_) / 2,
                           "steps": 2, "warmup": 1}
            if prec == "fp64":
                # the streaming FP64 SDSN (K4) against the HBM copy peak: algorithmic 16n^2 B per pass
                extra[prec]["sdsn_algorithmic_gbs"] = 16.0 * n * n * ps_ / (ms_s / 1e3) / 1e9
                extra[prec]["sdsn_algorithmic_frac_of_hbm"] = extra[prec]["sdsn_algorithmic_gbs"] / hbm
        if "fp64" in extra:
            extra["mixed_vs_fp64_time_to_solution"] = extra["fp64"]["time_to_solution_ms"] / statistics.median(step_ms)

    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": tot_ms_all / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": dtype_label(args.precision),
                "data": "synthetic (seeded C4 generator; SNAP Facebook-ego stand-in)",
                "config": {"workload": workload(args.precision), "n": n, "precision": args.precision,
                           "schedule": SCHEDULE, "seed": "rank", "replicas": world,
                           "l2": "flushed between steps (256 MiB write)",
                           "parallelism": f"{world} independent replicas (C4 does not shard, SURVEY 8(e))"},
                "time_to_solution_ms": statistics.median(step_ms),
                "outer_iters_per_solve": iters / args.steps, "mean_passes_per_iter": passes / iters,
                "accuracy": acc,
                "roofline": roof,
                "gemm": gemm_entry(args.precision, ms_gemm, iters, args.steps),
                "lap_ms_per_step": ms_lap / args.steps,
                "e2e": e2e, "gpu_launches": launches, "clocks": clocks}
        if extra:
            line["precisions"] = extra
    if world > 1:
        dist.barrier()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_entry(inst, passes / iters, budget_s=15.0)
    if rank == 0:
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_c5(args):
    """C5 (BASELINE configs[4]): weighted ER n=16384, rows of A, G and N sharded across the ranks
    (fram_create_sharded; NCCL all-gather of the Uᵀ blocks per outer iteration and an all-reduce of
    the column sums per SDSN pass).  `value` = outer iterations of the one sharded solve ÷ max-over-ranks
    device time ("scaling": "strong": the problem is fixed as the rank count grows)."""
    import torch
    import torch.distributed as dist

    import paper_2508_00887_b200 as fb
    from synth import config_c5

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = 16384 if args.n == 4096 else args.n
    inst = config_c5(0, n=n)
    r0, r1 = fb.shard_rows(n, rank, world)
    A = torch.tensor(inst.A[r0:r1], dtype=torch.bfloat16, device=dev)      # C5 is stored dense BF16
    B = torch.tensor(inst.B, dtype=torch.bfloat16, device=dev)
    flags = fb.FLAG_TRACE | fb.FLAG_TIME_PHASES
    sch = fb.Schedule(theta=inst.theta, alpha=SCHEDULE["alpha"], gamma_th=SCHEDULE["gamma_th"],
                      delta_th=SCHEDULE["delta_th"], max_outer=args.max_outer or SCHEDULE["max_outer"],
                      sdsn_max=SCHEDULE["sdsn_max"], flags=flags)
    if world > 1:
        h = fb.create_sharded_dist(n, lam=SCHEDULE["lam"], schedule=sch)
    else:
        h = fb.fram_create_sharded(n, SCHEDULE["lam"], sch, fb.fram_get_unique_id(), 0, 1, device=local)
    X = torch.empty((r1 - r0, n), dtype=torch.float64, device=dev)
    perm = torch.empty((n,), dtype=torch.int32, device=dev)
    for _ in range(args.warmup):
        fb.fram_solve(h, A, B, precision=args.precision, X_out=X, perm_out=perm)
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    tot_ms, stats = 0.0, []
    for k in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _, s, _, _ = fb.fram_solve(h, A, B, precision=args.precision, X_out=X, perm_out=perm)
        b.record()
        b.synchronize()
        tot_ms += a.elapsed_time(b)
        stats.append(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    clocks = sampler.stop()
    iters = sum(s["outer_iters"] for s in stats)
    passes = sum(s["total_passes"] for s in stats)
    if rank == 0:
        acc = float((perm.cpu().numpy() == inst.perm_true).mean())
        line = {"metric": METRIC, "value": iters / (tot_ms / 1e3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": dtype_label(args.precision), "data": "synthetic (seeded C5 generator)",
                "config": {"workload": "C5: weighted ER(p=0.01) n=16384, BF16 storage, 5% rewiring, rows sharded",
                           "n": n, "precision": args.precision, "schedule": dict(SCHEDULE, max_outer=sch.max_outer),
                           "parallelism": f"row-sharded over {world} rank(s) (NCCL)"},
                "outer_iters_per_solve": iters / args.steps, "mean_passes_per_iter": passes / max(iters, 1),
                "accuracy": acc, "sdsn_us_per_pass": 1e3 * sum(s["ms_sdsn"] for s in stats) / max(passes, 1),
                "gemm_ms_per_iter": sum(s["ms_gemm"] for s in stats) / max(iters, 1),
                "lap_ms_per_step": sum(s["ms_lap"] for s in stats) / args.steps,
                "gpu_launches": sum(s["kernel_launches"] for s in stats), "clocks": clocks}
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_c3(args):
    """C3 (BASELINE configs[2]): 4096 keypoint-style instances (n=64, θ=2, unary term), bf16 GEMM /
    fp32 SDSN, instances split evenly across the ranks (no collective in the data path: "weak" in the
    per-rank sense is not applicable, the batch is fixed → "strong").  One step = fram_solve_batched
    over this rank's instances.  `value` = instances solved per second over the job."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2508_00887_b200 as fb
    from synth import config_c3_batch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    total = 4096
    per = total // world
    insts = config_c3_batch(per, start=rank * per)
    st = lambda a: torch.tensor(np.ascontiguousarray(np.stack([getattr(i, a) for i in insts])), dtype=torch.float32,
                                device=dev)
    A, B, K = st("A"), st("B"), st("K")
    sch = fb.Schedule(theta=2.0, alpha=SCHEDULE["alpha"], gamma_th=SCHEDULE["gamma_th"], delta_th=SCHEDULE["delta_th"],
                      max_outer=SCHEDULE["max_outer"], sdsn_max=SCHEDULE["sdsn_max"])
    h = fb.fram_create(64, lam=SCHEDULE["lam"], schedule=sch, device=local)
    for _ in range(args.warmup):
        fb.fram_solve_batched(h, A, B, K, precision=args.precision)
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    tot_ms, res = 0.0, None
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        res = fb.fram_solve_batched(h, A, B, K, precision=args.precision)
        b.record()
        b.synchronize()
        tot_ms += a.elapsed_time(b)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    clocks = sampler.stop()
    _, stats, X, perm, sts = res
    perm = perm.cpu().numpy()
    acc = float(np.mean([(perm[b] == inst.perm_true)[inst.inlier_mask].mean() for b, inst in enumerate(insts)]))
    if rank == 0:
        line = {"metric": "FRAM batched instances/s (C3)", "value": total * args.steps / (tot_ms / 1e3),
                "unit": "instances/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": dtype_label(args.precision),
                "data": "synthetic (seeded C3 keypoint generator)",
                "config": {"workload": "C3: 4096 x n=64 keypoint graphs, unary K, theta=2", "batch": total,
                           "precision": args.precision, "parallelism": f"instances split over {world} rank(s)"},
                "outer_iters_max": stats["outer_iters"], "total_passes_rank0": stats["total_passes"],
                # K8 keeps each instance's iterate in shared memory: per SDSN pass it reads and writes the
                # 64x64 FP32 Y once (32 KB), so its ceiling is the SMEM bandwidth, 128 B/clk/SM (B200_PROFILING.md)
                "roofline": {"kernel": "batched_kernel (K8, one CTA per instance)", "bound": "smem",
                             "achieved": 2.0 * 4 * 64 * 64 * stats["total_passes"] * args.steps / (tot_ms / 1e3) / 1e9,
                             "peak": 148 * 128 * 1.965e9 / 1e9, "unit": "GB/s",
                             "frac": 2.0 * 4 * 64 * 64 * stats["total_passes"] * args.steps / (tot_ms / 1e3) / 1e9
                             / (148 * 128 * 1.965e9 / 1e9),
                             "traffic": None,
                             "note": "SDSN-pass shared-memory bytes only (GEMMs, update, LAP excluded); the kernel is "
                                     "latency / barrier bound at 2 CTAs per SM (DESIGN.md section 10)"},
                "inlier_accuracy_rank0": acc, "gpu_launches": args.steps, "clocks": clocks}
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_ubc(args):
    """NEXT-2: the attributed, fully connected keypoint-graph regime of the paper's mixed-precision
    headline, ubc(2000) (graphs from images P:1047), on the synthetic stand-in synth.config_ubc
    (UBC images are not available).  One step = fram_solve_attributed (K = F F̃ᵀ on the device, Alg. 1) at
    n = 2000, θ = 2; the same solve in FP64 mode is timed beside it, giving the analogue of the paper's
    12.7× mixed-vs-GPU-FP64 ratio.  Quality: matching error and Φ(M) on the device (fram_evaluate)."""
    import numpy as np
    import torch

    import paper_2508_00887_b200 as fb
    from synth import config_ubc

    rank, world, local = dist_env()
    if rank != 0:
        return 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n = 2000 if args.n == 4096 else args.n
    inst = config_ubc(0, n=n)
    A = torch.tensor(inst.A, dtype=torch.float64, device=dev)
    B = torch.tensor(inst.B, dtype=torch.float64, device=dev)
    F = torch.tensor(inst.meta["F"], dtype=torch.float64, device=dev)
    Ft = torch.tensor(inst.meta["Ft"], dtype=torch.float64, device=dev)
    sch = fb.Schedule(theta=inst.theta, alpha=SCHEDULE["alpha"], gamma_th=SCHEDULE["gamma_th"],
                      delta_th=SCHEDULE["delta_th"], max_outer=SCHEDULE["max_outer"], sdsn_max=SCHEDULE["sdsn_max"],
                      flags=fb.FLAG_TRACE | fb.FLAG_CHECK_SYMMETRY | fb.FLAG_TIME_PHASES)
    h = fb.fram_create(n, lam=SCHEDULE["lam"], schedule=sch, device=local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    res = {}
    sampler = ClockSampler(local)
    for prec in (args.precision, "fp64"):
        for _ in range(args.warmup):
            fb.fram_solve_attributed(h, A, B, F, Ft, precision=prec)
        torch.cuda.synchronize()
        if prec == args.precision:
            sampler.start()
        ms, its, stats = [], 0, None
        for k in range(args.steps):
            flush.fill_(float(k))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _, stats, X, perm = fb.fram_solve_attributed(h, A, B, F, Ft, precision=prec)
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
            its += stats["outer_iters"]
        clocks = sampler.stop() if prec == args.precision else None
        p = perm.cpu().numpy()
        ev = fb.fram_evaluate(h, A, B, torch.tensor(p, dtype=torch.int32, device=dev), F, Ft)
        res[prec] = {"time_to_solution_ms": statistics.median(ms), "iters_per_s": its / (sum(ms) / 1e3),
                     "outer_iters_per_solve": its / args.steps, "mean_passes_per_iter": stats["total_passes"] /
                     max(1, stats["outer_iters"]), "accuracy": float((p == inst.perm_true).mean()),
                     "matching_error": ev["matching_error"], "phi": ev["phi"], "ms_sdsn": stats["ms_sdsn"],
                     "ms_gemm": stats["ms_gemm"], "ms_lap": stats["ms_lap"], "clocks": clocks}
    main = res[args.precision]
    line = {"metric": "ubc(2000)-regime time to solution (NEXT-2)", "value": main["time_to_solution_ms"], "unit": "ms",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": False,
            "dtype": dtype_label(args.precision), "data": "synthetic (synth.config_ubc: UBC ubc(2000) stand-in)",
            "config": {"workload": "UBC stand-in: n=2000 fully connected Euclidean-distance graphs, d=128 features, "
                                   "theta=2, lambda=1", "n": n, "precision": args.precision,
                       "schedule": dict(SCHEDULE, theta=inst.theta)},
            "mixed": main, "fp64": res["fp64"],
            "fp64_over_mixed_time_to_solution": res["fp64"]["time_to_solution_ms"] / main["time_to_solution_ms"],
            "paper_context": "12.7x mixed over GPU-FP64 on an RTX 4080 SUPER (P:551), whose FP64 rate is 1/64 of FP32"}
    emit(line)
    return 0


def main():
    args = parse()
    _claim_stdout()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "c5":
        return run_c5(args)
    if args.workload == "c3":
        return run_c3(args)
    if args.workload == "ubc":
        return run_ubc(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
