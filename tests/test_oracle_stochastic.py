"""Pins of the oracle's stochastic rounding mode (NEXT-2, reading R14): unbiasedness (Def. 1,
P:444-445 -- the gradient compressor U_g must satisfy E[U(v)] = v), bounded error,
exactness on the lattice, determinism, and the hash's uniformity."""
import numpy as np
import pytest

from oracle import (F32, STAGE_INTRA, Topology, dequantize, exact_reduce_scatter_f64, mix32, q_levels, quantize,
                    sr_key, sr_uniform, tlq_hs_reduce_scatter)
from synth import spiky_numpy


def py_mix32(x):
    # independent scalar reimplementation with Python integers
    x &= 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x7FEB352D) & 0xFFFFFFFF
    x ^= x >> 15
    x = (x * 0x846CA68B) & 0xFFFFFFFF
    x ^= x >> 16
    return x


def test_mix32_matches_scalar_and_is_a_bijection():
    xs = np.arange(0, 1 << 20, dtype=np.uint64) * 4099 + 7
    got = mix32(xs)
    for v in list(xs[:50]) + [0, 1, 0xFFFFFFFF, 0x80000000]:
        assert int(mix32(np.uint64(v))) == py_mix32(int(v))
    assert len(np.unique(got)) == len(xs)      # xorshift and odd multiplies are invertible mod 2^32
    assert int(mix32(np.uint64(0))) == 0


def test_uniform_draws_are_uniform():
    u = sr_uniform(np.arange(1 << 20, dtype=np.uint64), sr_key(2410, STAGE_INTRA, 3)).astype(np.float64)
    assert u.min() >= 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 3 * (1 / np.sqrt(12)) / np.sqrt(len(u))
    hist = np.bincount((u * 64).astype(int), minlength=64)
    chi2 = ((hist - len(u) / 64) ** 2 / (len(u) / 64)).sum()
    assert chi2 < 120       # 63 dof: p ~ 1e-5
    # different stages / ranks / seeds give different streams
    u2 = sr_uniform(np.arange(1024, dtype=np.uint64), sr_key(2410, STAGE_INTRA, 4))
    assert not np.array_equal(u[:1024].astype(F32), u2)


@pytest.mark.parametrize("k", [4, 8])
def test_stochastic_rounding_is_unbiased(k):
    # Def. 1: E[U(v)] = v.  Mean over 4000 seeds of the dequantized values vs x, per
    # element, within 5 standard errors (each draw's error is < one step).
    G = 128
    x = spiky_numpy(G * 4, seed=k)
    q = q_levels(k)
    _, s = quantize(x, k, G)
    step = np.repeat(s.astype(np.float64) / q, G)
    acc = np.zeros(len(x))
    T = 4000
    for seed in range(T):
        c, sc = quantize(x, k, G, sr=(0, sr_key(seed, STAGE_INTRA, 0)))
        xh = dequantize(c, sc, k, G).astype(np.float64)
        assert np.all(np.abs(xh - x) <= step * (1 + 1e-5))          # within one step, always
        acc += xh
    mean = acc / T
    se = step / 2 / np.sqrt(T)
    assert np.max(np.abs(mean - x) / se) < 5.5


def test_stochastic_rounding_exact_on_lattice_and_deterministic():
    q = q_levels(4)
    rng = np.random.default_rng(0)
    x = rng.integers(-q, q + 1, size=(64, 32)).astype(F32)
    x[:, 0] = q
    c, s = quantize(x.reshape(-1), 4, 32, sr=(0, sr_key(1, STAGE_INTRA, 0)))
    assert np.array_equal(c, x.reshape(-1).astype(np.int32))       # fr = 0: no randomness
    y = spiky_numpy(32 * 64, seed=9)
    a = quantize(y, 4, 32, sr=(5, sr_key(7, 2, 1)))[0]
    b = quantize(y, 4, 32, sr=(5, sr_key(7, 2, 1)))[0]
    d = quantize(y, 4, 32, sr=(5, sr_key(8, 2, 1)))[0]
    assert np.array_equal(a, b) and not np.array_equal(a, d)


def test_tlq_hs_with_stochastic_rounding_is_unbiased():
    # the whole two-level reduce-scatter becomes an unbiased estimator of the mean
    topo = Topology(2, 2)
    P, G, b = 4, 128, 64
    D = P * G * 2
    grads = [spiky_numpy(D, seed=40 + r) for r in range(P)]
    exact = np.concatenate(exact_reduce_scatter_f64(grads, P))
    T = 300
    acc = np.zeros(D)
    for seed in range(T):
        acc += np.concatenate(tlq_hs_reduce_scatter(grads, topo, G, b, 8, 4, True, seed=seed).out)
    mean = acc / T
    rne = np.concatenate(tlq_hs_reduce_scatter(grads, topo, G, b, 8, 4, True).out)
    # the seed-averaged error is far below the deterministic (nearest) error
    assert np.linalg.norm(mean - exact) < 0.25 * np.linalg.norm(rne - exact)
