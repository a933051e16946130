"""Pins for oracle/rounding.py (RNE to BF16 / FP16 / TF32) — ties, overflow, and an
independent converter (torch's CPU casts; numpy's IEEE half for TF32 in the FP16 normal range)."""
import numpy as np
import pytest
import torch

from oracle.rounding import round_bf16, round_fp16, round_tf32


def test_tf32_tie_examples():
    # 1 + 2⁻¹¹ is the midpoint of 1 and 1 + 2⁻¹⁰ → ties to even → 1.0
    assert round_tf32(1.0 + 2.0 ** -11) == 1.0
    # 1 + 3·2⁻¹¹ is the midpoint of 1 + 2⁻¹⁰ (odd) and 1 + 2⁻⁹ (even) → 1 + 2⁻⁹
    assert round_tf32(1.0 + 3 * 2.0 ** -11) == 1.0 + 2.0 ** -9
    assert round_tf32(1.0 + 2.0 ** -11 + 2.0 ** -20) == 1.0 + 2.0 ** -10     # above the midpoint
    assert round_tf32(3.0e38) == pytest.approx(3.0e38, rel=2.0 ** -11)       # FP32 range kept (no FP16 overflow)


def test_bf16_ties_and_overflow():
    assert round_bf16(1.0 + 2.0 ** -8) == 1.0                                # midpoint → even
    assert round_bf16(1.0 + 3 * 2.0 ** -8) == 1.0 + 2.0 ** -6                # midpoint → even (up)
    big = float(np.finfo(np.float32).max)
    assert np.isinf(round_bf16(big))                                         # rounds past BF16 max → inf


def test_fp16_ties_and_overflow():
    assert round_fp16(1.0 + 2.0 ** -11) == 1.0
    assert round_fp16(65504.0) == 65504.0
    assert np.isinf(round_fp16(65520.0))                                     # midpoint of max and 2¹⁶ → inf


@pytest.mark.parametrize("scale", [1e-6, 1.0, 1e3])
def test_against_independent_converters(rng, scale):
    x = (rng.standard_normal(20000) * scale).astype(np.float32)
    t = torch.from_numpy(x)
    assert np.array_equal(round_bf16(x), t.to(torch.bfloat16).to(torch.float64).numpy())
    assert np.array_equal(round_fp16(x), t.to(torch.float16).to(torch.float64).numpy())
    # TF32 has FP16's 10-bit fraction: inside FP16's normal range the two roundings coincide.  A power-of-
    # two rescaling (exact in FP32) brings the sample into that range and commutes with the rounding.
    e = int(round(-np.log2(scale)))
    xs = (x * np.float32(2.0 ** e)).astype(np.float32)
    sel = (np.abs(xs) >= 2.0 ** -14) & (np.abs(xs) <= 60000.0)
    assert sel.sum() > 1000
    assert np.array_equal(round_tf32(x[sel]) * 2.0 ** e, xs[sel].astype(np.float16).astype(np.float64))
