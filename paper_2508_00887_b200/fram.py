"""Thin ctypes binding of libfram.so (include/fram.h) — argument marshalling only.

Every arithmetic step of FRAM runs in the library's CUDA kernels; this module only converts
torch tensors / numpy arrays to pointers, builds the C structs and raises on error statuses.
There is no CPU fallback: if libfram.so is missing or no sm_100 device is present, calls fail
loudly.  Function names follow the C ABI.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libfram.so")

FRAM_OK, FRAM_ERR_USAGE, FRAM_ERR_DATA, FRAM_NOT_CONVERGED, FRAM_ERR_CUDA, FRAM_ERR_NCCL, FRAM_ERR_OOM = range(7)
STATUS_NAMES = ["OK", "ERR_USAGE", "ERR_DATA", "NOT_CONVERGED", "ERR_CUDA", "ERR_NCCL", "ERR_OOM"]
PREC = {"fp64": 0, "tf32": 1, "bf16": 2, "fp16": 3}
DT = {"f64": 0, "f32": 1, "bf16": 2}
FLAG_TRACE, FLAG_CHECK_SYMMETRY, FLAG_NO_THETA_SCALE, FLAG_TIME_PHASES = 1, 2, 4, 8

EXPORTED = ["fram_create", "fram_set_schedule", "fram_solve", "fram_solve_batched", "fram_destroy",
            "fram_last_error", "fram_get_unique_id", "fram_create_sharded", "fram_sdsn", "fram_gradient",
            "fram_lap", "fram_abi_version", "fram_build_info", "fram_solve_attributed", "fram_create_sharded_virtual",
            "fram_evaluate"]


class FramError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 7 else status}: {msg}")
        self.status = status


class _Schedule(C.Structure):
    _fields_ = [("theta", C.c_double), ("alpha", C.c_double), ("gamma_th", C.c_double), ("delta_th", C.c_double),
                ("max_outer", C.c_int32), ("sdsn_max", C.c_int32), ("sdsn_fixed", C.c_int32), ("flags", C.c_int32),
                ("replay_passes", C.POINTER(C.c_int32)), ("replay_len", C.c_int32)]


class _Stats(C.Structure):
    _fields_ = [("outer_iters", C.c_int32), ("converged", C.c_int32), ("sdsn_capped_calls", C.c_int32),
                ("sdsn_kernel", C.c_int32), ("total_passes", C.c_int64), ("passes_per_iter", C.POINTER(C.c_int32)),
                ("delta_trace", C.POINTER(C.c_double)), ("gamma_last", C.POINTER(C.c_double)),
                ("ms_precond", C.c_double), ("ms_gemm", C.c_double), ("ms_sdsn", C.c_double),
                ("ms_update", C.c_double), ("ms_lap", C.c_double), ("ms_total", C.c_double),
                ("kernel_launches", C.c_int64)]


@dataclass
class Schedule:
    """fram_schedule (include/fram.h); defaults = SURVEY §8(d) / P:374."""
    theta: float = 10.0
    alpha: float = 0.95
    gamma_th: float = 1e-3
    delta_th: float = 1e-4
    max_outer: int = 100
    sdsn_max: int = 1000
    sdsn_fixed: int = 0
    flags: int = FLAG_CHECK_SYMMETRY | FLAG_TRACE
    replay: list | None = None

    def to_c(self):
        s = _Schedule(self.theta, self.alpha, self.gamma_th, self.delta_th, self.max_outer, self.sdsn_max,
                      self.sdsn_fixed, self.flags, None, 0)
        keep = None
        if self.replay:
            keep = (C.c_int32 * len(self.replay))(*[int(x) for x in self.replay])
            s.replay_passes = C.cast(keep, C.POINTER(C.c_int32))
            s.replay_len = len(self.replay)
        return s, keep


_lib_handle = None


def lib():
    """Load libfram.so (fails loudly if it has not been built)."""
    global _lib_handle
    if _lib_handle is not None:
        return _lib_handle
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2508_00887_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    L.fram_create.argtypes = [i64, dbl, C.POINTER(_Schedule), C.c_int, C.POINTER(vp)]
    L.fram_set_schedule.argtypes = [vp, C.POINTER(_Schedule)]
    L.fram_solve.argtypes = [vp, C.c_int, vp, vp, vp, vp, C.c_int, vp, vp, vp, C.POINTER(_Stats)]
    L.fram_solve_batched.argtypes = [vp, i64, C.c_int, vp, vp, vp, vp, C.c_int, vp, vp, vp, vp, C.POINTER(_Stats)]
    L.fram_destroy.argtypes = [vp]
    L.fram_destroy.restype = None
    L.fram_last_error.restype = C.c_char_p
    L.fram_get_unique_id.argtypes = [C.c_char_p]
    L.fram_create_sharded.argtypes = [i64, dbl, C.POINTER(_Schedule), C.c_char_p, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(vp)]
    L.fram_evaluate.argtypes = [vp, C.c_int, vp, vp, vp, vp, i64, vp, vp, C.POINTER(dbl)]
    L.fram_create_sharded_virtual.argtypes = [i64, dbl, C.POINTER(_Schedule), C.c_int, C.c_int, C.POINTER(vp)]
    L.fram_sdsn.argtypes = [vp, C.c_int, vp, vp, C.POINTER(i32), vp, vp]
    L.fram_gradient.argtypes = [vp, C.c_int, vp, vp, vp, vp, C.c_int, vp, vp, C.POINTER(dbl)]
    L.fram_lap.argtypes = [vp, vp, vp, vp]
    L.fram_build_info.restype = C.c_char_p
    L.fram_solve_attributed.argtypes = [vp, C.c_int, C.c_int64, C.c_int64, C.c_int64, vp, vp, vp, vp, C.c_int, vp, vp,
                                        vp, C.POINTER(_Stats)]
    for f in ("fram_create", "fram_set_schedule", "fram_solve", "fram_solve_batched", "fram_get_unique_id",
              "fram_solve_attributed",
              "fram_create_sharded", "fram_create_sharded_virtual", "fram_sdsn", "fram_gradient", "fram_lap",
              "fram_evaluate"):
        getattr(L, f).restype = C.c_int
    _lib_handle = L
    return L


def _err(status):
    return FramError(status, lib().fram_last_error().decode(errors="replace"))


def _check(status, allow_nc=False):
    if status == FRAM_OK or (allow_nc and status == FRAM_NOT_CONVERGED):
        return status
    raise _err(status)


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(x.data_ptr())
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return C.c_void_p(x.ctypes.data)
    raise TypeError(f"unsupported buffer type {type(x)}")


def _dt_of(x):
    if _is_torch(x):
        import torch
        return {torch.float64: 0, torch.float32: 1, torch.bfloat16: 2}[x.dtype]
    return {np.dtype(np.float64): 0, np.dtype(np.float32): 1}[x.dtype]


def _stream(stream, *bufs):
    if stream is not None:
        return C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
    for b in bufs:
        if b is not None and _is_torch(b) and b.is_cuda:
            import torch
            return C.c_void_p(torch.cuda.current_stream(b.device).cuda_stream)
    return None


def _like(ref, shape, kind):
    """Allocate an output on the same side (device/host) as `ref`."""
    if _is_torch(ref):
        import torch
        dt = torch.float64 if kind == "f64" else torch.int32
        return torch.empty(shape, dtype=dt, device=ref.device)
    return np.empty(shape, dtype=np.float64 if kind == "f64" else np.int32)


class Handle:
    """Owns a fram_handle (fram_create / fram_destroy).  `rows` = n, or n/W for a sharded handle."""

    def __init__(self, ptr, n, rows=None, rank=0, world=1, schedule=None):
        self.ptr = ptr
        self.n = n
        self.schedule = schedule or Schedule()     # sizes the stats trace arrays (max_outer entries)
        self.rows = n if rows is None else rows
        self.rank = rank
        self.world = world

    def __del__(self):
        try:
            if self.ptr:
                lib().fram_destroy(self.ptr)
        except Exception:
            pass
        self.ptr = None

    @property
    def _as_arg(self):
        return self.ptr


def fram_create(n, lam=1.0, schedule: Schedule | None = None, device=0) -> Handle:
    s, keep = (schedule or Schedule()).to_c()
    out = C.c_void_p()
    _check(lib().fram_create(int(n), float(lam), C.byref(s), int(device), C.byref(out)))
    del keep
    return Handle(out, int(n), schedule=schedule)


def fram_set_schedule(h: Handle, schedule: Schedule):
    s, keep = schedule.to_c()
    _check(lib().fram_set_schedule(h.ptr, C.byref(s)))
    del keep
    h.schedule = schedule


def _stats_dict(st, nout, arrays):
    d = dict(outer_iters=st.outer_iters, converged=bool(st.converged), sdsn_capped_calls=st.sdsn_capped_calls,
             total_passes=int(st.total_passes), ms_precond=st.ms_precond, ms_gemm=st.ms_gemm,
             ms_sdsn=st.ms_sdsn, ms_update=st.ms_update, ms_lap=st.ms_lap, ms_total=st.ms_total,
             kernel_launches=int(st.kernel_launches), sdsn_kernel=int(st.sdsn_kernel))
    if arrays is not None:
        t = st.outer_iters
        d["passes"] = [int(x) for x in arrays[0][:t]]
        d["deltas"] = [float(x) for x in arrays[1][:t]]
        d["gamma_last"] = [float(x) for x in arrays[2][:t]]
    return d


def _trace_arrays(h: Handle):
    """Host trace arrays of fram_stats, sized from the handle's schedule (the C side writes at most
    max_outer entries; a replay longer than max_outer is rejected by check_schedule)."""
    cap = max(1, int(h.schedule.max_outer), len(h.schedule.replay or []))
    arrays = ((C.c_int32 * cap)(), (C.c_double * cap)(), (C.c_double * cap)())
    st = _Stats()
    st.passes_per_iter = C.cast(arrays[0], C.POINTER(C.c_int32))
    st.delta_trace = C.cast(arrays[1], C.POINTER(C.c_double))
    st.gamma_last = C.cast(arrays[2], C.POINTER(C.c_double))
    return st, arrays


def fram_solve(h: Handle, A, B, K=None, X0=None, precision="bf16", stream=None, X_out=None, perm_out=None):
    """Alg. 1 end to end.  Returns (status, stats, X_out, perm_out); raises FramError on errors."""
    n = h.n
    X_out = _like(A, (h.rows, n), "f64") if X_out is None else X_out
    perm_out = _like(A, (n,), "i32") if perm_out is None else perm_out
    st, arrays = _trace_arrays(h)
    status = lib().fram_solve(h.ptr, _dt_of(A), _ptr(A), _ptr(B), _ptr(K), _ptr(X0), PREC[precision],
                              _stream(stream, A), _ptr(X_out), _ptr(perm_out), C.byref(st))
    _check(status, allow_nc=True)
    return status, _stats_dict(st, n, arrays), X_out, perm_out


def fram_solve_attributed(h: Handle, A, B, F=None, Ft=None, precision="bf16", stream=None, X_out=None,
                          perm_out=None):
    """Attributed graphs of possibly unequal size (R30): A n1×n1, B n2×n2, F n1×d, F̃ n2×d; padded to
    the handle's n; K = F F̃ᵀ on the device.  Returns (status, stats, X_out (n×n), perm_out (n1; −1 =
    matched to a padding node))."""
    n = h.n
    n1, n2 = A.shape[0], B.shape[0]
    d = 0 if F is None else F.shape[1]
    X_out = _like(A, (n, n), "f64") if X_out is None else X_out
    perm_out = _like(A, (n1,), "i32") if perm_out is None else perm_out
    st, arrays = _trace_arrays(h)
    status = lib().fram_solve_attributed(h.ptr, _dt_of(A), int(n1), int(n2), int(d), _ptr(A), _ptr(B), _ptr(F),
                                         _ptr(Ft), PREC[precision], _stream(stream, A), _ptr(X_out),
                                         _ptr(perm_out), C.byref(st))
    _check(status, allow_nc=True)
    return status, _stats_dict(st, n, arrays), X_out, perm_out


def fram_solve_batched(h: Handle, A, B, K=None, X0=None, precision="bf16", stream=None, X_out=None,
                       perm_out=None, status_out=None):
    """`batch` independent solves (A, B, K: batch×n×n).  Returns (status, stats, X_out, perm_out, status_out)."""
    n = h.n
    batch = A.shape[0]
    X_out = _like(A, (batch, n, n), "f64") if X_out is None else X_out
    perm_out = _like(A, (batch, n), "i32") if perm_out is None else perm_out
    status_out = np.zeros(batch, dtype=np.int32) if status_out is None else status_out
    st = _Stats()
    status = lib().fram_solve_batched(h.ptr, int(batch), _dt_of(A), _ptr(A), _ptr(B), _ptr(K), _ptr(X0),
                                      PREC[precision], _stream(stream, A), _ptr(X_out), _ptr(perm_out),
                                      _ptr(status_out), C.byref(st))
    if status not in (FRAM_OK, FRAM_NOT_CONVERGED, FRAM_ERR_DATA):
        raise _err(status)
    return status, _stats_dict(st, n, None), X_out, perm_out, status_out


def fram_sdsn(h: Handle, X, precision="fp32", D_out=None, stream=None, want_gammas=True, cap=None):
    """One SDSN call (Alg. 2).  precision 'fp64' (X float64) or anything else (X float32).
    Returns (D, passes, gammas)."""
    p = 0 if precision == "fp64" else 2
    if D_out is None:
        if _is_torch(X):
            import torch
            D_out = torch.empty_like(X)
        else:
            D_out = np.empty_like(X)
    passes = C.c_int32(0)
    sch = h.schedule
    cap = cap or max(1, int(sch.sdsn_max), int(sch.sdsn_fixed))    # fram.h: double[max(sdsn_max, sdsn_fixed)]
    gh = (C.c_double * cap)() if want_gammas else None
    _check(lib().fram_sdsn(h.ptr, p, _ptr(X), _ptr(D_out), C.byref(passes),
                           C.cast(gh, C.c_void_p) if gh is not None else None, _stream(stream, X)))
    k = passes.value
    gam = [float(gh[i]) for i in range(k)] if gh is not None else None
    return D_out, k, gam


def fram_gradient(h: Handle, A, B, K, N, precision="bf16", stream=None, G_out=None):
    """Preconditioning + G = A'·N·Ã' + λK'.  Returns (G, c)."""
    n = h.n
    if G_out is None:
        if _is_torch(A):
            import torch
            G_out = torch.empty((n, n), dtype=torch.float64 if precision == "fp64" else torch.float32,
                                device=A.device)
        else:
            G_out = np.empty((n, n), dtype=np.float64 if precision == "fp64" else np.float32)
    c = C.c_double(0)
    _check(lib().fram_gradient(h.ptr, _dt_of(A), _ptr(A), _ptr(B), _ptr(K), _ptr(N), PREC[precision],
                               _stream(stream, A), _ptr(G_out), C.byref(c)))
    return G_out, c.value


def fram_lap(h: Handle, N, perm_out=None, stream=None):
    """Deterministic Hungarian (R17) on FP64 N.  Returns perm (int32)."""
    perm_out = _like(N, (h.n,), "i32") if perm_out is None else perm_out
    _check(lib().fram_lap(h.ptr, _ptr(N), _ptr(perm_out), _stream(stream, N)))
    return perm_out


def fram_evaluate(h: Handle, A, B, perm, F=None, Ft=None, stream=None):
    """Matching quality on the device (K9; Eq.(1)).  Returns dict(matching_error, edge_error,
    feature_error, phi) for M[i, perm[i]] = 1 (perm int32, device or host)."""
    out = (C.c_double * 4)()
    d = 0 if F is None else int(F.shape[1])
    _check(lib().fram_evaluate(h.ptr, _dt_of(A), _ptr(A), _ptr(B), _ptr(F), _ptr(Ft), d, _ptr(perm),
                               _stream(stream, A), out))
    return dict(matching_error=out[0], edge_error=out[1], feature_error=out[2], phi=out[3])


def fram_get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().fram_get_unique_id(buf))
    return buf.raw


def fram_create_sharded(n, lam, schedule: Schedule | None, uid: bytes, rank, world, device=0) -> Handle:
    """Row-sharded handle (rank owns rows [rank·n/W, (rank+1)·n/W)); `uid` from fram_get_unique_id on one
    rank, shared with all (see create_sharded_dist)."""
    s, keep = (schedule or Schedule()).to_c()
    out = C.c_void_p()
    _check(lib().fram_create_sharded(int(n), float(lam), C.byref(s), uid, int(rank), int(world), int(device),
                                     C.byref(out)))
    del keep
    return Handle(out, int(n), rows=int(n) // int(world), rank=int(rank), world=int(world), schedule=schedule)


def fram_create_sharded_virtual(n, lam=1.0, schedule: Schedule | None = None, world=2, device=0) -> Handle:
    """Virtual-shard group on ONE GPU (include/fram.h): `world` ranks of the row-sharded solve, collectives
    as fixed-order device sums/copies.  fram_solve on it takes and returns full n×n matrices."""
    s, keep = (schedule or Schedule()).to_c()
    out = C.c_void_p()
    _check(lib().fram_create_sharded_virtual(int(n), float(lam), C.byref(s), int(world), int(device), C.byref(out)))
    del keep
    return Handle(out, int(n), rows=int(n), rank=0, world=int(world), schedule=schedule)


def shard_rows(n, rank, world):
    """Row range [r0, r1) owned by `rank` in a sharded solve (n % world == 0)."""
    if n % world:
        raise ValueError("n must be divisible by the number of ranks")
    m = n // world
    return rank * m, (rank + 1) * m


def broadcast_unique_id(make_id, group=None, src=0):
    """Rank `src` calls make_id() (fram_get_unique_id for real runs), the 128 bytes are broadcast over
    torch.distributed (CPU tensor: works for gloo and nccl process groups).  Returns bytes."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == src:
        raw = make_id()
        if len(raw) != 128:
            raise ValueError("unique id must be 128 bytes")
        buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
        g = buf.to(dev)
        dist.broadcast(g, src, group=group)
        buf = g.cpu()
    else:
        dist.broadcast(buf, src, group=group)
    return bytes(buf.numpy().tobytes())


def create_sharded_dist(n, lam=1.0, schedule: Schedule | None = None, group=None, device=None) -> Handle:
    """fram_create_sharded for the calling torch.distributed rank (one process per GPU)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device() if device is None else device
    uid = broadcast_unique_id(fram_get_unique_id, group=group)
    return fram_create_sharded(n, lam, schedule, uid, rank, world, device=dev)


def fram_build_info() -> str:
    return lib().fram_build_info().decode()
