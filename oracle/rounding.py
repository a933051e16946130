"""Round-to-nearest-even helpers for the emulated-rounding *diagnostic* oracle.
TEST INFRASTRUCTURE ONLY.  Operate on the FP32 bit pattern of the input (values are first
rounded to FP32, as an FP32-accumulating tensor-core GEMM would see them)."""
from __future__ import annotations

import numpy as np


def _rne_keep(x, drop_bits):
    f = np.asarray(x, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    half = np.uint64((1 << (drop_bits - 1)) - 1)
    lsb = (b >> np.uint64(drop_bits)) & np.uint64(1)
    b = (b + half + lsb) & ~np.uint64((1 << drop_bits) - 1)
    return (b.astype(np.uint32)).view(np.float32).astype(np.float64)


def round_bf16(x):
    """BF16: 8-bit significand (drop 16 of FP32's 23 fraction bits), RNE."""
    return _rne_keep(x, 16)


def round_tf32(x):
    """TF32: 11-bit significand (drop 13 fraction bits), FP32 range, RNE.  S:418: 1+2⁻¹¹ → 1.0."""
    return _rne_keep(x, 13)


def round_fp16(x):
    """FP16 (11-bit significand, FP16 range) via numpy's IEEE half conversion (RNE)."""
    return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float64)
