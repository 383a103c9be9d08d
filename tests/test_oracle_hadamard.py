"""Pins of the oracle's blockwise Hadamard (sec. 3.2.2, sec. 3.3)."""
import numpy as np
import pytest
import scipy.linalg

from oracle import F32, fwht_unnormalized, hadamard_c, hadamard_normalized
from synth import spiky_numpy
from tests.conftest import golden

BLOCKS = [2, 4, 8, 16, 32, 64, 128, 256]


def test_spec_b2_examples():
    for c in golden("hadamard_b2.json")["cases"]:
        np.testing.assert_allclose(hadamard_normalized(np.array(c["x"], F32), c["b"]), c["Hx"],
                                   rtol=1e-6, atol=1e-7, err_msg=c["cite"])


@pytest.mark.parametrize("b", BLOCKS)
def test_butterfly_equals_dense_sylvester_exactly_on_integers(b):
    # The butterfly is the Sylvester-order matrix (scipy.linalg.hadamard, a library routine):
    # on small integers every fp32 operation is exact, so the results must be identical.
    rng = np.random.default_rng(b)
    x = rng.integers(-50, 51, size=(40, b)).astype(F32)
    H = scipy.linalg.hadamard(b).astype(np.float64)
    ref = x.astype(np.float64) @ H.T
    assert np.array_equal(fwht_unnormalized(x.reshape(-1), b).reshape(-1, b), ref.astype(F32))


@pytest.mark.parametrize("b", BLOCKS)
def test_butterfly_matches_dense_fp64_on_floats(b):
    # within 1e-5 * max|x| per block against a dense fp64 product.
    x = spiky_numpy(b * 200, seed=b)
    H = scipy.linalg.hadamard(b).astype(np.float64) / np.sqrt(b)
    ref = x.reshape(-1, b).astype(np.float64) @ H.T
    got = hadamard_normalized(x, b).reshape(-1, b).astype(np.float64)
    tol = 1e-5 * np.abs(x.reshape(-1, b)).max(axis=1, keepdims=True)
    assert np.all(np.abs(got - ref) <= tol)


@pytest.mark.parametrize("b", BLOCKS)
def test_orthonormal_involution_and_norm(b):
    # P:353 H = H^T, H H^T = I  =>  H(H x) = x and ||H x|| = ||x||, within 1e-5.
    x = spiky_numpy(b * 100, seed=100 + b)
    y = hadamard_normalized(hadamard_normalized(x, b), b)
    assert np.max(np.abs(y - x)) <= 1e-5 * np.abs(x).max()
    n0 = np.linalg.norm(x.reshape(-1, b).astype(np.float64), axis=1)
    n1 = np.linalg.norm(hadamard_normalized(x, b).reshape(-1, b).astype(np.float64), axis=1)
    assert np.all(np.abs(n1 - n0) <= 1e-5 * n0 + 1e-30)


def test_c_b_closed_form():
    # c_b^2 = 1/b (orthonormality); for b = 4^j c_b is a power of two, exact
    for b in BLOCKS:
        assert abs(float(hadamard_c(b)) ** 2 * b - 1) < 2e-7
    for b in (4, 16, 64, 256):
        assert float(hadamard_c(b)) == 2.0 ** (-np.log2(b) / 2)


def test_linearity_distributive():
    # P:390 "sum_i H g_i = H sum_i g_i": within 1e-4 over 16-term sums.
    b = 32
    gs = [spiky_numpy(b * 64, seed=200 + i) for i in range(16)]
    lhs = np.zeros_like(gs[0])
    for g in gs:
        lhs = (lhs + hadamard_normalized(g, b)).astype(F32)
    tot = np.zeros_like(gs[0])
    for g in gs:
        tot = (tot + g).astype(F32)
    rhs = hadamard_normalized(tot, b)
    assert np.max(np.abs(lhs - rhs)) <= 1e-4 * max(1.0, np.abs(rhs).max())


def test_smoothing_spiky_inputs():
    # S:155 / P:352 "distributing outlier information across nearby elements" (Fig. 6):
    # max/rms over the vector drops after the transform in >= 95% of 200 seeded spiky trials
    # (trials whose draw contains no outlier, |x| > 10 sigma, are redrawn: they are not spiky).
    b = 32
    better, t, trials = 0, 0, 0
    while trials < 200:
        x = spiky_numpy(b * 8, seed=1000 + t, spike_prob=0.01, spike_scale=50.0).reshape(-1, b)
        t += 1
        if np.abs(x).max() <= 10:
            continue
        trials += 1
        y = hadamard_normalized(x.reshape(-1), b).reshape(-1, b)

        def ratio(v):
            return np.max(np.abs(v)) / np.sqrt(np.mean(v.astype(np.float64) ** 2))
        better += ratio(y) < ratio(x)
    assert better >= 190
