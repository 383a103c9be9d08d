"""GPU parity of the ablation baselines and the Alg. 4 training harness on
Counterexample 1 (NEXT-4), through the C ABI, against the oracle.

* qW (Alg. 1): K1 without the replica read, K2 assigning instead of adding.
* int2 weight codec (ternary; R4) for both qW and qWD.
* ring reduce-scatter with per-hop quantization: P = 1 here (K6 first+last hop);
  P > 1 through tests/dist_parity.py.
* Counterexample 1 run as Alg. 4 on the GPU: identity gradient
  compressor, ternary weight codec; the compressed weights w~ follow the oracle's
  trajectory bit for bit, qW stays stuck at (1, -1), qWD converges to w* = 0."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2410_15526_b200 import Comm, tlq_stage_final, tlq_stage_quantize
from tests.test_gpu_parity import assert_unit_equal, bf16_equal, f32_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = Comm()
    yield c
    c.close()


@pytest.mark.parametrize("model_dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("bits,G", [(2, 64), (4, 128), (4, 2048), (8, 32), (32, 128)])
def test_qw_parity(comm, model_dtype, bits, G):
    D = max(G, 64) * 41
    w_main = synth.main_weights(synth.model_weights(D, seed=21, dtype=model_dtype), seed=22)
    ws = torch.zeros(comm.qwd_workspace_bytes(D, bits, G), dtype=torch.uint8, device="cuda")
    wm = torch.full((D,), 7.0, dtype=model_dtype, device="cuda")        # overwritten, never read
    comm.qw_quantize(w_main.cuda(), D, ws, bits, G)
    torch.cuda.synchronize()
    unit = ws.cpu().numpy().copy()
    comm.qw_allgather_apply(ws, wm, bits, G)
    torch.cuda.synchronize()
    bf = model_dtype == torch.bfloat16
    units, want = oracle.qw_step([w_main.numpy()], bits, G, model_bf16=bf)
    assert_unit_equal(unit, *units[0], bits, G, D, "qW unit")
    if bf:
        assert bf16_equal(synth.bf16_bits(wm.cpu()), want)
    else:
        assert f32_equal(wm.cpu().numpy(), want)


@pytest.mark.parametrize("G", [64, 256])
def test_qwd_int2_parity(comm, G):
    D = G * 37
    w_model = synth.model_weights(D, seed=23)
    w_main = synth.main_weights(w_model, seed=24)
    ws = torch.zeros(comm.qwd_workspace_bytes(D, 2, G), dtype=torch.uint8, device="cuda")
    wm = w_model.cuda()
    comm.qwd_quantize(w_main.cuda(), wm, ws, 2, G)
    torch.cuda.synchronize()
    unit = ws.cpu().numpy().copy()
    comm.qwd_allgather_apply(ws, wm, 2, G)
    torch.cuda.synchronize()
    units, want = oracle.qwd_step([w_main.numpy()], synth.bf16_bits(w_model), 2, G, model_bf16=True)
    assert_unit_equal(unit, *units[0], 2, G, D, "qWD int2 unit")
    assert bf16_equal(synth.bf16_bits(wm.cpu()), want)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("bits", [4, 8, 32])
def test_ring_single_rank(comm, dtype, bits):
    D = 2048 * 9 + 128 * 3
    g = synth.gradient(D, seed=25, dtype=dtype)
    ws = torch.zeros(comm.ring_workspace_bytes(D, bits, 128), dtype=torch.uint8, device="cuda")
    out = torch.empty(D, dtype=torch.float32, device="cuda")
    comm.ring_reduce_scatter(g.cuda(), out, ws, bits, 128, True)
    torch.cuda.synchronize()
    assert f32_equal(out.cpu().numpy(), oracle.ring_reduce_scatter([g.float().numpy()], bits, 128, True).out[0])


# ------------------------------------------------- Alg. 4 on Counterexample 1 (NEXT-4)
def _branches(T, seed):
    rng = np.random.default_rng(seed)
    return [int(rng.random() >= 0.5) for _ in range(T)]


def _oracle_run(mode, branches, eta, G=64):
    """Alg. 4 with the oracle's codec: w_t = w_{t-1} - eta*g(w~_{t-1}); qWD:
    w~_t = w~_{t-1} + C(w_t - w~_{t-1}); qW: w~_t = C(w_t) (and the main weights follow it,
    as in QSDP / ZeRO++ where the quantized weights are the weights)."""
    w = np.zeros(G, np.float32)
    w[:2] = (1.0, -1.0)
    wt = w.copy()
    traj = []
    for br in branches:
        g = np.zeros(G, np.float32)
        g[br] = np.float32(4.0) * wt[br]
        w = (w - (np.float32(eta) * g).astype(np.float32)).astype(np.float32)
        if mode == "qWD":
            _, wt = oracle.qwd_step([w], wt, 2, G, model_bf16=False)
        else:
            _, wt = oracle.qw_step([w], 2, G, model_bf16=False)
            w = wt.copy()
        traj.append(wt[:2].copy())
    return np.array(traj)


def _gpu_run(comm, mode, branches, eta, G=64):
    """The same loop on the GPU: the gradient and the SGD step in torch (two separately
    rounded fp32 ops, as the oracle), the weight communication through libsdp4."""
    dev = "cuda"
    w = torch.zeros(G, dtype=torch.float32, device=dev)
    w[:2] = torch.tensor([1.0, -1.0])
    wt = w.clone()
    ws = torch.zeros(comm.qwd_workspace_bytes(G, 2, G), dtype=torch.uint8, device=dev)
    eta_t = torch.tensor(eta, dtype=torch.float32, device=dev)
    traj = []
    for br in branches:
        g = torch.zeros(G, dtype=torch.float32, device=dev)
        g[br] = 4.0 * wt[br]
        w = w - eta_t * g
        if mode == "qWD":
            comm.qwd_quantize(w, wt, ws, 2, G)
            comm.qwd_allgather_apply(ws, wt, 2, G)
        else:
            comm.qw_quantize(w, G, ws, 2, G)
            comm.qw_allgather_apply(ws, wt, 2, G)
            w = wt.clone()
        traj.append(wt[:2].clone())
    return torch.stack(traj).cpu().numpy()


def test_counterexample_alg4_on_gpu(comm):
    T, eta = 300, 0.1
    br = _branches(T, seed=7)
    for mode in ("qW", "qWD"):
        want = _oracle_run(mode, br, eta)
        got = _gpu_run(comm, mode, br, eta)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"{mode} trajectory differs"
    assert np.all(got[-1] == got[-1])
    qw = _gpu_run(comm, "qW", br, eta)
    assert np.all(qw == np.array([1.0, -1.0], np.float32))                 # stuck for every t
    qwd = _gpu_run(comm, "qWD", br, eta)
    assert np.linalg.norm(qwd[-1]) < 1e-2                                  # converges to w* = 0


# ------------------------------------------- unfused Hadamard comparator (NEXT-3)
def unfused_on_gpu(comm, grad, G, b, bi=8, be=4):
    """Separate Hadamard passes around the b = 0 reduce-scatter, from the library's own
    kernels: K3 with the identity codec writes rn(H_unnorm(g) * c_b) (R12), the TLq
    reduce-scatter runs with b = 0, and K5 with the identity codec, M = 1 and no averaging
    applies rn(H_unnorm(x) * c_b) to the reduced shard."""
    D = grad.numel()
    S = D // comm.world
    h = torch.empty(D, dtype=torch.float32, device="cuda")
    tlq_stage_quantize(grad, h.view(torch.uint8), 1, 1, 32, G, b)
    red = torch.empty(S, dtype=torch.float32, device="cuda")
    ws = torch.zeros(comm.tlq_workspace_bytes(D, bi, be, G), dtype=torch.uint8, device="cuda")
    comm.tlq_hs_reduce_scatter(h, red, ws, bi, be, G, 0, True)
    out = torch.empty(S, dtype=torch.float32, device="cuda")
    tlq_stage_final(red.view(torch.uint8), out, S, 1, 1, 32, G, b, False)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("G,b", [(128, 64), (256, 256), (64, 16)])
def test_unfused_hadamard_comparator(comm, G, b):
    D = 16384 * 2 + max(G, 64) * 5
    g = synth.gradient(D, seed=41 + b, dtype=torch.bfloat16)
    got = unfused_on_gpu(comm, g.cuda(), G, b)
    want = oracle.unfused_tlq_hs_reduce_scatter([g.float().numpy()], oracle.Topology(1, 1), G, b)[0]
    assert f32_equal(got, want)
