"""Pins of the oracle's TLq-HS reduce-scatter (Alg. 3, sec. 3.2 P:341-353,
sec. 3.3) against closed forms, brute-force sums and error bounds."""
import numpy as np
import pytest

from oracle import (F32, Topology, dequantize, exact_reduce_scatter_f64, hadamard_c,
                    naive_tlq_hs_reduce_scatter, q_levels, tlq_hs_reduce_scatter)
from synth import spiky_numpy, uniform_ints
from tests.conftest import golden

TOPOS = [(1, 1), (1, 2), (2, 1), (2, 2), (1, 4), (4, 1), (2, 4), (4, 2), (1, 8), (8, 1)]


def test_spec_reduce_scatter_example():
    # S:249 with S:267: identity quantizers, no Hadamard, average -> exact mean per shard.
    g = golden("reduce_scatter_example.json")
    P, N = g["P"], g["N"]
    grads = [np.array(r, F32) for r in g["grads"]]
    tr = tlq_hs_reduce_scatter(grads, Topology(P // N, N), G=1, b=0, k_intra=32, k_inter=32, average=True)
    assert [o.tolist() for o in tr.out] == g["shards"]


@pytest.mark.parametrize("M,N", TOPOS)
def test_identity_codec_equals_brute_force_sum_on_integers(M, N):
    # North star: "brute-force all-reduce equivalence on tiny buffers with bits set to 32".
    # Small-integer inputs make every fp32 partial sum exact, so the two-level order must
    # reproduce the fp64 brute-force reduce-scatter bit-exactly; a routing error (a shard
    # landing on the wrong rank, a wrong sub-block) changes the sums.
    P = M * N
    D = P * 64 * 3
    grads = [uniform_ints(D, seed=7 * r + 1).numpy() for r in range(P)]
    tr = tlq_hs_reduce_scatter(grads, Topology(M, N), G=64, b=0, k_intra=32, k_inter=32, average=False)
    ref = exact_reduce_scatter_f64(grads, P, average=False)
    for r in range(P):
        assert np.array_equal(tr.out[r].astype(np.float64), ref[r])


@pytest.mark.parametrize("M,N", [(2, 4), (4, 2), (1, 8)])
@pytest.mark.parametrize("b", [2, 16, 32, 64, 256])
def test_identity_codec_with_hadamard_within_rounding(M, N, b):
    # with identity quantizers and the Hadamard on, out = mean within rounding.
    # fp32 summation bound plus log2(b) butterfly roundings per transform.
    P = M * N
    D = P * 256 * 2
    grads = [spiky_numpy(D, seed=31 * r + b) for r in range(P)]
    tr = tlq_hs_reduce_scatter(grads, Topology(M, N), G=256, b=b, k_intra=32, k_inter=32, average=True)
    ref = exact_reduce_scatter_f64(grads, P, average=True)
    absum = np.zeros(D)
    for g in grads:
        absum += np.abs(g)
    S = D // P
    for r in range(P):
        blk = absum[r * S:(r + 1) * S].reshape(-1, b).max(axis=1, keepdims=True) / P
        tol = (P + 4 * np.log2(b) + 4) * 2.0 ** -24 * np.sqrt(b) * blk
        err = np.abs(tr.out[r].astype(np.float64) - ref[r]).reshape(-1, b)
        assert np.all(err <= tol)


def _error_bound_per_block(tr, topo, G, b, k_intra, k_inter, S):
    """Per output block, the norm bound implied by half-step quantization errors
     of every message on the path, carried through the orthonormal H:
    ||out - exact||_2 <= (1/P) (sum over intra messages ||e8|| + sum over inter ||e4||)."""
    M, N, P = topo.M, topo.N, topo.P
    bb = b if b else G
    qi, qe = q_levels(k_intra), q_levels(k_inter)
    bounds = []
    for r in range(P):
        m, l = topo.coords(r)
        tot = np.zeros(S // bb)
        for mpp in range(M):                          # inter messages into rank r
            _, s4 = tr.inter_send[topo.rank(mpp, l)][m]
            step = np.repeat(s4.astype(np.float64) / qe, G // bb) if G >= bb else s4 / qe
            tot += np.sqrt(bb) * step / 2
            src = topo.rank(mpp, l)
            ms, ls = topo.coords(src)
            for lpp in range(N):                      # intra messages into that source
                _, s8 = tr.intra_send[topo.rank(ms, lpp)][ls][m]
                step8 = np.repeat(s8.astype(np.float64) / qi, G // bb)
                tot += np.sqrt(bb) * step8 / 2
        bounds.append(tot / P * (1 + 1e-5) + 1e-30)
    return bounds


@pytest.mark.parametrize("M,N", [(1, 1), (2, 4), (4, 2), (8, 1), (1, 8)])
@pytest.mark.parametrize("mode", ["TLq-HS", "TLq", "ULq"])
def test_quantized_path_within_half_step_error_bound(M, N, mode):
    # The exact mean is reached up to the quantization errors the method introduces.
    k_intra, k_inter, b = {"TLq-HS": (8, 4, 64), "TLq": (8, 4, 0), "ULq": (4, 4, 0)}[mode]
    topo = Topology(M, N)
    P, G = topo.P, 128
    D = P * G * 6
    grads = [spiky_numpy(D, seed=97 * r + M) for r in range(P)]
    tr = tlq_hs_reduce_scatter(grads, topo, G=G, b=b, k_intra=k_intra, k_inter=k_inter, average=True)
    ref = exact_reduce_scatter_f64(grads, P, average=True)
    S = D // P
    bb = b if b else G
    bounds = _error_bound_per_block(tr, topo, G, b, k_intra, k_inter, S)
    for r in range(P):
        err = np.linalg.norm((tr.out[r].astype(np.float64) - ref[r]).reshape(-1, bb), axis=1)
        assert np.all(err <= bounds[r] * 1.0001 + 1e-6 * np.abs(ref[r]).max())


def test_pruned_equals_naive_within_one_step():
    # sec. 3.3: pruning is exact in exact arithmetic; in fp32 a few
    # 4-bit codes may flip by one step (DESIGN.md reading); everything else within 1e-4.
    topo = Topology(4, 4)
    P, G, b = 16, 128, 32
    D = P * G * 4
    worst_frac = 0.0
    for trial in range(5):
        grads = [spiky_numpy(D, seed=5000 + 100 * trial + r) for r in range(P)]
        tr = tlq_hs_reduce_scatter(grads, topo, G, b, 8, 4, True)
        naive = naive_tlq_hs_reduce_scatter(grads, topo, G, b, 8, 4, True)
        for r in range(P):
            m, l = topo.coords(r)
            step = max(float(np.max(tr.inter_send[topo.rank(mm, l)][m][1])) for mm in range(topo.M)) / 7 / P
            d = np.abs(tr.out[r] - naive[r])
            big = d > 1e-4 * max(1.0, float(np.abs(naive[r]).max()))
            worst_frac = max(worst_frac, big.mean())
            assert np.all(d <= 1.01 * step * np.sqrt(b) + 1e-4)
    assert worst_frac <= 0.02


def test_error_ordering_tlqhs_tlq_ulq():
    # S:269/S:471, desk analog of Fig. 5 and P:350: on spiky gradients the median
    # reduce-scatter error orders TLq-HS < TLq < ULq.
    topo = Topology(4, 4)
    P, G = 16, 128
    D = P * G * 2
    errs = {"TLq-HS": [], "TLq": [], "ULq": []}
    for t in range(30):
        grads = [spiky_numpy(D, seed=20000 + 50 * t + r, spike_prob=0.01, spike_scale=50.0) for r in range(P)]
        ref = np.concatenate(exact_reduce_scatter_f64(grads, P))
        for mode, (ki, ke, b) in {"TLq-HS": (8, 4, 32), "TLq": (8, 4, 0), "ULq": (4, 4, 0)}.items():
            out = np.concatenate(tlq_hs_reduce_scatter(grads, topo, G, b, ki, ke, True).out)
            errs[mode].append(np.linalg.norm(out - ref))
    med = {k: np.median(v) for k, v in errs.items()}
    assert med["TLq-HS"] < med["TLq"] < med["ULq"]


def test_stage_messages_are_quantizer_outputs():
    # Alg. 3 l.2-3: the intra message for shard j is Quantize8(H g_r)[shard j] with the scale
    # carrying c_b (R6).  Check against the definition H = c_b H_unnorm applied explicitly:
    # dequantized messages approximate H g within half a step.
    topo = Topology(2, 2)
    G, b = 128, 64
    D = 4 * G * 2
    grads = [spiky_numpy(D, seed=300 + r) for r in range(4)]
    tr = tlq_hs_reduce_scatter(grads, topo, G, b, 8, 4, True)
    import scipy.linalg
    H = scipy.linalg.hadamard(b) / np.sqrt(b)
    S = D // 4
    for r in range(4):
        Hg = (grads[r].reshape(-1, b).astype(np.float64) @ H.T).reshape(-1)
        for lp in range(2):
            for mp in range(2):
                j = mp * 2 + lp
                c, s = tr.intra_send[r][lp][mp]
                xh = dequantize(c, s, 8, G).astype(np.float64)
                err = np.abs(xh - Hg[j * S:(j + 1) * S]).reshape(-1, G)
                assert np.all(err <= (s[:, None] / 254) * (1 + 1e-5) + 1e-12)
    assert hadamard_c(64) == F32(0.125)
