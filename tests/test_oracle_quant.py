"""Pins of the oracle's quantizer, wire format and bf16 helpers against what the
paper, SPEC and mathematics fix (no GPU).  Each test names the passage it pins.
"""
import numpy as np
import pytest
import torch

from oracle import (F32, TINY, bf16_round, bf16_widen, comm_bits_per_param, dequantize, pack_codes,
                    q_levels, quantize, unpack_codes, wire_unit, wire_unit_bytes, wire_unit_decode)
from synth import edge_case_groups, spiky_numpy
from tests.conftest import golden


def test_q_levels_closed_form():
    # 2^(k-1) - 1
    assert [q_levels(k) for k in (2, 4, 8)] == [1, 7, 127]


def test_spec_quantize_examples():
    g = golden("quantize_examples.json")
    for case in g["quantize"]:
        codes, scales = quantize(np.array(case["x"], F32), case["k"], case["G"])
        assert codes.tolist() == case["codes"], case["cite"]
        assert scales.tolist() == case["scales"], case["cite"]
        if "dequantized" in case:
            assert dequantize(codes, scales, case["k"], case["G"]).tolist() == case["dequantized"]


def test_spec_dequantize_examples():
    g = golden("quantize_examples.json")
    for case in g["dequantize"]:
        x = dequantize(np.array(case["codes"]), np.array(case["scales"], F32), case["k"], case["G"])
        np.testing.assert_allclose(x, case["x"], rtol=case.get("rtol", 0), atol=0, err_msg=case["cite"])
    # rn(1/7)*7 == 1 exactly, so the code q_k dequantizes to exactly s
    assert F32(7) * (F32(1) / F32(7)) == F32(1)


@pytest.mark.parametrize("k", [4, 8])
@pytest.mark.parametrize("G", [32, 128, 2048])
def test_half_step_bound(k, G):
    # |x - x_hat| <= s / (2 q_k); slack for the two fp32 roundings
    # of inv = rn(q/s) and ds = rn(s/q) (each < 2^-24 relative) and of the products.
    x = spiky_numpy(G * 64, seed=11 + k + G)
    codes, s = quantize(x, k, G)
    xh = dequantize(codes, s, k, G)
    q = q_levels(k)
    err = np.abs(x.astype(np.float64) - xh.astype(np.float64)).reshape(-1, G)
    bound = s.astype(np.float64) / (2 * q) + s.astype(np.float64) * 4 * 2.0 ** -24
    assert np.all(err <= bound[:, None])
    assert np.abs(codes).max() <= q


def test_signed_max_would_overflow_abs_max_does_not():
    # R2 reading of P:281 "s = max(x)": a negative-heavy group must not overflow the code range.
    x = np.array([-4.0, -2.0, 1.0, 0.5], F32)
    codes, s = quantize(x, 4, 4)
    assert s[0] == 4.0 and codes.tolist() == [-7, -4, 2, 1]   # -3.5 -> -4 (RNE), 1.75 -> 2, 0.875 -> 1


def test_rne_ties():
    # R3: round = round-half-to-even (one cvt.rni); exact .5 ties with s = q_k.
    x = np.array([7.0, 0.5, 1.5, 2.5, -0.5, -1.5, -2.5, 3.5], F32)
    codes, s = quantize(x, 4, 8)
    assert codes.tolist() == [7, 0, 2, 2, 0, -2, -2, 4]


def test_contraction_and_sign_oddness():
    # S:112 contraction ||x_hat - x|| <= ||x||;  S:212 sign-oddness q(-x) = -q(x)
    for seed in range(20):
        x = spiky_numpy(128 * 8, seed=seed)
        for k in (2, 4, 8):
            c, s = quantize(x, k, 128)
            xh = dequantize(c, s, k, 128)
            assert np.linalg.norm(xh.astype(np.float64) - x) <= np.linalg.norm(x.astype(np.float64))
            c2, s2 = quantize(-x, k, 128)
            assert np.array_equal(c2, -c) and np.array_equal(s2, s)


def test_scale_covariance_power_of_two():
    # quantize(2^e x) has identical codes and scales 2^e s (bit-exact).
    x = spiky_numpy(128 * 16, seed=3)
    c0, s0 = quantize(x, 4, 128)
    for e in (-20, -3, 1, 7, 30):
        a = F32(2.0 ** e)
        c1, s1 = quantize((x * a).astype(F32), 4, 128)
        assert np.array_equal(c0, c1)
        assert np.array_equal(s1, (s0 * a).astype(F32))


@pytest.mark.parametrize("k", [4, 8])
def test_lattice_points_roundtrip_exactly(k):
    # x on the lattice {j s / q_k} round-trips exactly.  With s = q_k the
    # lattice is the integers, and x = j exactly.
    q = q_levels(k)
    rng = np.random.default_rng(5)
    x = rng.integers(-q, q + 1, size=(50, 64)).astype(F32)
    x[:, 0] = q
    c, s = quantize(x.reshape(-1), k, 64)
    assert np.array_equal(dequantize(c, s, k, 64), x.reshape(-1))
    assert np.array_equal(c, x.reshape(-1).astype(np.int32))


def test_edge_groups():
    # R2/R5: zero group -> scale 0; tiny scale (< 2^-120) -> zero group; NaN/Inf -> codes 0 and the
    # group dequantizes to NaN (poison); subnormal-but-not-tiny values stay representable.
    G = 64
    x = edge_case_groups(G).numpy()
    c, s = quantize(x, 8, G)
    xh = dequantize(c, s, 8, G).reshape(-1, G)
    c = c.reshape(-1, G)
    assert s[0] == 0 and not c[0].any() and not xh[0].any()
    assert s[7] == 0 and not c[7].any()              # 2^-125 < TINY
    for row in (8, 9, 10):                           # NaN, +Inf, -Inf groups
        assert not c[row].any() and np.all(np.isnan(xh[row]))
    assert np.isnan(s[8]) and s[9] == np.inf and s[10] == np.inf
    assert s[5] > TINY and np.abs(c[5]).max() == 127  # tiny-but-normal group is quantized normally
    assert np.all(np.isfinite(xh[11]))               # 1e30-scale group


def test_bf16_round_matches_torch():
    # bf16 RNE narrowing (R11) pinned against the library conversion of torch (CPU).
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(100000).astype(F32) * F32(3.0),
        np.array([0.0, -0.0, 1.0, -1.0, 3.4e38, -3.4e38, np.inf, -np.inf, 1e-40, -1e-45,
                  1.00390625, 1.01171875, 1.0078125], F32),    # exact ties 1+2^-8 (even), 1+3*2^-8 (odd)
    ])
    ours = bf16_round(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    assert np.array_equal(bf16_widen(ours), torch.from_numpy(ref.view(np.int16)).view(torch.bfloat16).float().numpy())
    assert np.isnan(bf16_widen(bf16_round(np.array([np.nan], F32))))[0]


def test_pack_unpack_and_wire_sizes():
    g = golden("wire_sizes.json")
    for p in g["payload"]:
        assert wire_unit_bytes(p["n"], p["k"], p["G"]) == p["bytes"], p["cite"]
    for b in g["bits_per_param"]:
        assert comm_bits_per_param(b["k"], b["G"], b["scale_bits"]) == b["bits"], b["cite"]
    # nibble order: element 2j in the low nibble, two's complement
    assert pack_codes(np.array([1, -1, -7, 7]), 4).tolist() == [0xF1, 0x79]
    assert unpack_codes(np.array([0xF1, 0x79], np.uint8), 4, 4).tolist() == [1, -1, -7, 7]
    rng = np.random.default_rng(1)
    for k, q in ((4, 7), (8, 127)):
        codes = rng.integers(-q, q + 1, 4096)
        scales = rng.random(4096 // 128).astype(F32)
        w = wire_unit(codes, scales, k, 128)
        assert len(w) % 256 == 0
        c2, s2 = wire_unit_decode(w, 4096, k, 128)
        assert np.array_equal(c2, codes) and np.array_equal(s2, scales)


def test_codes_are_single_rounding_of_exact_product():
    # R3 (P:281 has one round()): code = RNE(x * inv) of the EXACT product, inv = rn(q/s).
    # Pinned against exact rational arithmetic (fractions; Python's round() is half-to-even) on
    # groups built so that rn(x * inv) lands on a .5 tie while the exact product does not: there
    # the single-rounding and the double-rounding readings give different codes.
    from fractions import Fraction
    rng = np.random.default_rng(42)
    k, q = 4, q_levels(4)
    found = 0
    for trial in range(400):
        s_ = F32(rng.uniform(1.0, 2.0))
        inv = F32(F32(q) / s_)
        t = float(rng.integers(0, q)) + 0.5
        x0 = np.float32(t / float(inv))
        for x in (np.nextafter(x0, np.float32(0)), x0, np.nextafter(x0, np.float32(10))):
            x = F32(x)
            if not (0 < x < s_):
                continue
            exact = Fraction(float(x)) * Fraction(float(inv))
            if exact == t or F32(x * inv) != F32(t):
                continue
            codes, sc = quantize(np.array([s_, x], F32), k, 2)
            assert sc[0] == s_ and codes[0] == q
            assert codes[1] == round(exact)
            found += round(exact) != round(Fraction(t))      # double rounding would give round(t)
    assert found >= 10
