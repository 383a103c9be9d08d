"""Pins of the oracle's qWD path (sec. 3.1, Alg. 2 l.2-5 P:259-262,
Counterexample 1 P:412-416, Alg. 4)."""
import numpy as np
import pytest
import torch

from oracle import (F32, bf16_round, bf16_widen, dequantize, q_levels, quantize, qwd_allgather_apply,
                    qwd_quantize, qwd_step)
from synth import bf16_bits, main_weights, model_weights
from tests.conftest import golden


def test_counterexample_one_step():
    # P:413-415 / S:333: w=(1,-1), eta=0.1, gradient branch (4 w1, 0), ternary weight-diff codec.
    g = golden("counterexample1.json")
    w_model = np.array(g["w_init"], F32)
    w_main = (w_model - F32(g["eta"]) * np.array([4 * w_model[0], 0.0], F32)).astype(F32)
    np.testing.assert_allclose(w_main, g["w_main_after"], rtol=1e-7)
    codes, s, d = qwd_quantize(w_main, w_model, k=g["ternary_k"], G=2)
    np.testing.assert_allclose(d, g["d"], rtol=1e-6)
    np.testing.assert_allclose(s, [g["s"]], rtol=1e-6)
    assert codes.tolist() == g["codes"]
    d_tilde = dequantize(codes, s, 2, 2)
    np.testing.assert_allclose(d_tilde, g["d_tilde"], rtol=1e-6)
    w_new = qwd_allgather_apply([(codes, s)], w_model, 2, 2, model_bf16=False)
    np.testing.assert_allclose(w_new, g["w_model_after"], rtol=1e-6)
    # direct weight quantization qW: q(w_main) = (1, -1) -- stuck
    c, sw = quantize(w_main, 2, 2)
    assert dequantize(c, sw, 2, 2).tolist() == g["qW_after"]


def _run_counterexample(mode, eta=0.1, T=1000, seed=7):
    """Alg. 4 on Counterexample 1's least-squares problem with
    identity gradient compressor and a ternary (k = 2) weight compressor."""
    rng = np.random.default_rng(seed)
    w = np.array([1.0, -1.0], F32)       # main weights w_t
    wt = w.copy()                        # compressed weights w~_t
    for _ in range(T):
        g = np.array([4 * wt[0], 0.0], F32) if rng.random() < 0.5 else np.array([0.0, 4 * wt[1]], F32)
        w = (w - F32(eta) * g).astype(F32)
        if mode == "none":
            wt = w.copy()
        elif mode == "qW":
            c, s = quantize(w, 2, 2)
            wt = dequantize(c, s, 2, 2)
            w = wt.copy()                # QSDP/ZeRO++: the quantized weights are the weights
        elif mode == "qWD":
            c, s, _ = qwd_quantize(w, wt, 2, 2)
            wt = qwd_allgather_apply([(c, s)], wt, 2, 2, model_bf16=False)
    return w, wt


def test_counterexample_qw_stuck_qwd_converges():
    # qW stays at (1,-1); plain SGD and qWD converge to w* = 0.
    _, wt = _run_counterexample("qW")
    assert wt.tolist() == [1.0, -1.0]
    _, wt = _run_counterexample("none")
    assert np.linalg.norm(wt) < 1e-3
    _, wt = _run_counterexample("qWD")
    assert np.linalg.norm(wt) < 1e-2


@pytest.mark.parametrize("G", [128, 2048])
def test_qwd_half_step_and_apply(G):
    # Alg. 2 l.2-5 with 4 bits: |d~ - d| <= s/(2*7) per group; the applied replica is
    # bf16_rn(w_model + d~), pinned against torch's own fp32 add + bf16 conversion.
    P, S = 4, G * 16
    w_model = model_weights(P * S, seed=1)
    wm32 = w_model.float()
    shards = [main_weights(wm32[r * S:(r + 1) * S].to(torch.bfloat16), seed=100 + r).numpy() for r in range(P)]
    units, new = qwd_step(shards, bf16_bits(w_model), 4, G, model_bf16=True)
    d_hat_all = []
    for r, (c, s) in enumerate(units):
        d = (shards[r] - wm32[r * S:(r + 1) * S].numpy()).astype(F32)
        dh = dequantize(c, s, 4, G)
        err = np.abs(dh.astype(np.float64) - d).reshape(-1, G)
        assert np.all(err <= s[:, None].astype(np.float64) / 14 * (1 + 1e-5))
        d_hat_all.append(dh)
    ref = (wm32 + torch.from_numpy(np.concatenate(d_hat_all))).to(torch.bfloat16)
    assert np.array_equal(new, bf16_bits(ref))


def test_qwd_identity_codec_collapse():
    # with lossless compressors w_model + (w_main - w_model) = w_main; bit-exact where
    # Sterbenz holds (w_main in [w_model/2, 2 w_model]) and within 1 ulp elsewhere (fp32 model).
    rng = np.random.default_rng(3)
    wm = rng.standard_normal(4096).astype(F32)
    wmain = (wm + rng.uniform(-1e-3, 1e-3, 4096).astype(F32)).astype(F32)
    units, new = qwd_step([wmain[:2048], wmain[2048:]], wm, 32, 128, model_bf16=False)
    ster = (np.sign(wm) == np.sign(wmain)) & (np.abs(wmain) >= np.abs(wm) / 2) & (np.abs(wmain) <= 2 * np.abs(wm))
    assert np.array_equal(new[ster], wmain[ster])
    assert np.all(np.abs(new - wmain) <= np.spacing(np.abs(wmain)))


def test_qwd_smaller_error_than_qw():
    # sec. 3.1 P:330-333 "weight differences are easier to quantize": relative-to-w error of
    # 4-bit qWD is far below that of direct 4-bit qW (desk analog of S:473), G = 2048.
    n, G = 2048 * 32, 2048
    w_model = model_weights(n, seed=9)
    wmain = main_weights(w_model, seed=10).numpy()
    c, s, d = qwd_quantize(wmain, w_model.float().numpy(), 4, G)
    err_qwd = np.linalg.norm(dequantize(c, s, 4, G) - d) / np.linalg.norm(wmain)
    cw, sw = quantize(wmain, 4, G)
    err_qw = np.linalg.norm(dequantize(cw, sw, 4, G) - wmain) / np.linalg.norm(wmain)
    assert err_qwd < 0.05 * err_qw


def test_bf16_widen_roundtrip_is_identity():
    bits = np.arange(0, 65536, dtype=np.uint32).astype(np.uint16)
    w = bf16_widen(bits)
    fin = np.isfinite(w)
    assert np.array_equal(bf16_round(w[fin]), bits[fin])
    assert q_levels(4) == 7
