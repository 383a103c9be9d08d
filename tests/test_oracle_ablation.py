"""Pins of the oracle's ablation codecs: direct weight quantization qW
(Alg. 1; Counterexample 1), the int2 (ternary) wire codec (R4), and
the ring reduce-scatter with per-hop quantization (sec. 2.3)."""
import numpy as np
import pytest

from oracle import (F32, Topology, bf16_round, dequantize, exact_reduce_scatter_f64, pack_codes, q_levels, quantize,
                    qw_step, qwd_step, ring_reduce_scatter, tlq_hs_reduce_scatter, unfused_tlq_hs_reduce_scatter,
                    unpack_codes, wire_unit, wire_unit_decode)
from synth import main_weights, model_weights, spiky_numpy
from tests.conftest import golden


# ------------------------------------------------------------------------------ int2 codec
def test_int2_packing_golden():
    for ex in golden("int2_packing.json")["examples"]:
        assert pack_codes(np.array(ex["codes"]), 2).tolist() == ex["bytes"]
        assert unpack_codes(np.array(ex["bytes"], np.uint8), 2, len(ex["codes"])).tolist() == ex["codes"]


def test_int2_wire_roundtrip():
    rng = np.random.default_rng(3)
    c = rng.integers(-1, 2, size=4096)
    s = rng.random(4096 // 64).astype(F32)
    c2, s2 = wire_unit_decode(wire_unit(c, s, 2, 64), 4096, 2, 64)
    assert np.array_equal(c2, c) and np.array_equal(s2, s)
    assert q_levels(2) == 1        # ternary {-1, 0, 1}


# ----------------------------------------------------------------------------------- qW
def _counterexample_padded(w, G=64):
    # the 2-element problem embedded in one 64-element group: zeros quantize to 0 and do not
    # change s = max|w|, so the codec sees exactly the paper's ternary quantizer
    x = np.zeros(G, F32)
    x[:2] = w
    return x


def test_qw_counterexample_stuck_on_both_branches():
    g = golden("counterexample1.json")
    eta = F32(g["eta"])
    w0 = np.array(g["w_init"], F32)
    for branch in (np.array([4 * w0[0], 0], F32), np.array([0, 4 * w0[1]], F32)):
        w_main = (w0 - eta * branch).astype(F32)
        _, new = qw_step([_counterexample_padded(w_main)], 2, 64, model_bf16=False)
        assert new[:2].tolist() == g["qW_after"] and not new[2:].any()      # stuck at (1, -1)


def test_qwd_int2_counterexample_step():
    g = golden("counterexample1.json")
    w0 = _counterexample_padded(np.array(g["w_init"], F32))
    w_main = _counterexample_padded(np.array(g["w_main_after"], F32))
    units, new = qwd_step([w_main], w0, 2, 64, model_bf16=False)
    np.testing.assert_allclose(dequantize(*units[0], 2, 64)[:2], g["d_tilde"], rtol=1e-6)
    np.testing.assert_allclose(new[:2], g["w_model_after"], rtol=1e-6)


def test_qw_identity_codec_is_bf16_of_main():
    w = main_weights(model_weights(4096, seed=4), seed=5).numpy()
    _, new = qw_step([w[:2048], w[2048:]], 32, 128, model_bf16=True)
    assert np.array_equal(new, bf16_round(w))


@pytest.mark.parametrize("k", [2, 4, 8])
def test_qw_half_step_bound(k):
    G = 128
    w = spiky_numpy(G * 16, seed=k)
    units, new = qw_step([w[: G * 8], w[G * 8:]], k, G, model_bf16=False)
    s = np.concatenate([u[1] for u in units]).astype(np.float64)
    step = np.repeat(s / q_levels(k), G)
    assert np.all(np.abs(new.astype(np.float64) - w) <= step / 2 * (1 + 1e-6) + 1e-30)


# --------------------------------------------------------------------------- ring
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_ring_identity_codec_equals_exact_sum(P):
    # integer-valued inputs: every fp32 partial sum is exact, so the ring (any order) must
    # equal the brute-force sum -- a wrong chunk index or a dropped hop fails
    rng = np.random.default_rng(P)
    D = P * 64 * 3
    grads = [rng.integers(-1000, 1000, size=D).astype(F32) for _ in range(P)]
    tr = ring_reduce_scatter(grads, 32, 64, average=False)
    ex = exact_reduce_scatter_f64(grads, P, average=False)
    for r in range(P):
        assert np.array_equal(tr.out[r].astype(np.float64), ex[r])


def test_ring_golden_example():
    g = golden("reduce_scatter_example.json")
    tr = ring_reduce_scatter([np.array(x, F32) for x in g["grads"]], 32, 1, average=True)
    assert [o.tolist() for o in tr.out] == g["shards"]


def test_ring_message_routing():
    # hop t: rank r forwards chunk (r - t - 1) mod P; with the identity codec its payload is the
    # running sum of g_{c+1} .. g_r over that chunk (tagging payloads)
    P, S = 4, 64
    grads = [np.full(P * S, F32(10 ** r)) for r in range(P)]      # rank r tagged by 10^r
    tr = ring_reduce_scatter(grads, 32, 64, average=False)
    for t in range(P - 1):
        for r in range(P):
            c = (r - t - 1) % P
            want = sum(10 ** ((c + 1 + i) % P) for i in range(t + 1))
            assert np.all(tr.send[t][r][0] == want), (t, r)


def test_ring_error_bound_from_messages():
    # each hop adds at most half a quantization step of its message; /P at the end (R8)
    P, G, k = 4, 128, 4
    D = P * G * 4
    grads = [spiky_numpy(D, seed=60 + r) for r in range(P)]
    tr = ring_reduce_scatter(grads, k, G, True)
    ex = np.concatenate(exact_reduce_scatter_f64(grads, P))
    S = D // P
    bound = np.zeros(D)
    for t in range(P - 1):
        for r in range(P):
            c = (r - t - 1) % P
            bound[c * S:(c + 1) * S] += np.repeat(tr.send[t][r][1].astype(np.float64) / q_levels(k), G) / 2
    bound = bound / P + 1e-6 * np.abs(ex) + 1e-12
    assert np.all(np.abs(np.concatenate(tr.out) - ex) <= bound)


def test_ring_error_grows_with_P():
    # "P-1 rounds of quantization and dequantization, potentially leading to error
    # propagation": the median relative error at P = 16 exceeds P = 4 on the same
    # total data (relative to the exact mean, whose norm itself shrinks with P)
    G, D = 128, 16 * 128 * 2

    def err(P, seed):
        grads = [spiky_numpy(D, seed=seed * 100 + r) for r in range(P)]
        out = np.concatenate(ring_reduce_scatter(grads, 4, G, True).out)
        ex = np.concatenate(exact_reduce_scatter_f64(grads, P))
        return np.linalg.norm(out - ex) / np.linalg.norm(ex)
    e4 = np.median([err(4, s) for s in range(12)])
    e16 = np.median([err(16, s) for s in range(12)])
    assert e16 > e4


# ------------------------------------------------------- unfused Hadamard (KP4)
@pytest.mark.parametrize("b", [4, 64, 256])
def test_unfused_identity_codec_recovers_the_mean(b):
    # H (mean of H g) = mean of g (H H = I, linearity): with lossless codecs the
    # unfused passes reproduce the exact reduce-scatter up to fp32 rounding
    P, G = 4, 256
    D = P * G * 4
    grads = [spiky_numpy(D, seed=80 + r) for r in range(P)]
    out = np.concatenate(unfused_tlq_hs_reduce_scatter(grads, Topology(2, 2), G, b, 32, 32, True))
    ex = np.concatenate(exact_reduce_scatter_f64(grads, P))
    assert np.max(np.abs(out - ex)) <= 1e-5 * np.max(np.abs(ex))


def test_unfused_and_fused_agree_within_quantization_error():
    # the fused (pruned, R6-R8) and the unfused paths differ only by rounding placement: both
    # are within the same few quantization steps of the exact mean, and close to each other
    P, G, b = 4, 128, 64
    D = P * G * 8
    grads = [spiky_numpy(D, seed=90 + r) for r in range(P)]
    fused = np.concatenate(tlq_hs_reduce_scatter(grads, Topology(2, 2), G, b, 8, 4, True).out)
    unf = np.concatenate(unfused_tlq_hs_reduce_scatter(grads, Topology(2, 2), G, b, 8, 4, True))
    ex = np.concatenate(exact_reduce_scatter_f64(grads, P))
    ef, eu = np.linalg.norm(fused - ex), np.linalg.norm(unf - ex)
    assert abs(ef - eu) < 0.1 * ef
    assert np.linalg.norm(fused - unf) < 0.5 * ef
