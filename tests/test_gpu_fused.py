"""Parity of the one-launch small-message kernels (k_fused.cu) on ONE GPU.

The P2P transport runs sdp4_qwd_step and sdp4_tlq_hs_reduce_scatter on small buffers as one
kernel per rank, its exchanges (the qWD all-gather, Alg. 2 l.4 P:261; the intra / inter
all-to-alls, Alg. 3 l.4 and l.10) done by peer loads / stores and in-kernel flag
waits.  sdp4_emu_* runs those same kernels for EVERY rank of an emulated M x N job in one
launch on this device, so the exchange logic -- which rank's region each phase writes, which
flags it waits for and raises, the flag resets between calls -- is checked bit for bit against
the oracle here, on any one-GPU box.  Several consecutive calls per case (fresh=False after the
first) exercise the flag handshake across calls; tiles span several warp / CTA tasks and a
ragged tail; edge-case groups (zero, tiny, NaN, Inf, ties) ride in the buffers."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _bits_equal(a, b):
    """Bit-identical fp32 arrays or bf16 bit patterns, NaN equal to NaN (payloads may differ)."""
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype == np.float32:
        return bool(np.all((a.view(np.uint32) == b.astype(np.float32).view(np.uint32)) | (np.isnan(a) & np.isnan(b))))
    fa, fb = oracle.bf16_widen(a), oracle.bf16_widen(b)
    return bool(np.all((a == b) | (np.isnan(fa) & np.isnan(fb))))


def _shard_len(G, tiles=3):
    """Several 2048-element tasks plus a ragged tail, a multiple of lcm(G, 64)."""
    g = max(G, 64)
    return 2048 * tiles + (5 * g if g < 2048 else 0)


QWD_CASES = [  # P, bits, G, model dtype, stochastic seed
    (2, 4, 128, torch.bfloat16, None),
    (3, 4, 128, torch.bfloat16, None),
    (4, 8, 32, torch.float32, None),
    (8, 4, 128, torch.bfloat16, None),
    (2, 2, 64, torch.bfloat16, None),
    (4, 32, 128, torch.float32, None),
    (2, 4, 2048, torch.bfloat16, None),
    (4, 4, 256, torch.bfloat16, 7),
    (8, 8, 128, torch.float32, 3),
]


@pytest.mark.parametrize("P,bits,G,dt,seed", QWD_CASES)
def test_emu_qwd_step(P, bits, G, dt, seed):
    _need_gpu()
    from paper_2410_15526_b200 import emu_qwd_step, emu_qwd_workspace_bytes
    S = _shard_len(G)
    D = P * S
    ws = torch.empty(emu_qwd_workspace_bytes(P, D, bits, G), dtype=torch.uint8, device="cuda")
    w0 = synth.model_weights(D, seed=1, dtype=dt)
    state = synth.bf16_bits(w0) if dt == torch.bfloat16 else w0.numpy().copy()
    replicas = [w0.clone().cuda() for _ in range(P)]
    for call in range(3):
        cur = replicas[0].cpu()
        mains = [synth.main_weights(cur[p * S:(p + 1) * S], seed=100 * call + p) for p in range(P)]
        if call == 1:  # edge-case groups in rank 0's weight difference
            e = synth.edge_case_groups(G)[:S]
            mains[0][:e.numel()] = cur[:e.numel()].float() + e
        emu_qwd_step([m.cuda() for m in mains], replicas, ws, bits, G, seed=seed, fresh=(call == 0))
        torch.cuda.synchronize()
        _, want = oracle.qwd_step([m.numpy() for m in mains], state, bits, G, model_bf16=dt == torch.bfloat16,
                                  seed=seed)
        for p in range(P):
            got = synth.bf16_bits(replicas[p].cpu()) if dt == torch.bfloat16 else replicas[p].cpu().numpy()
            assert _bits_equal(got, want), f"call {call}: rank {p}'s replica differs from the oracle"
        state = want


TLQ_CASES = [  # M, N, bits_intra, bits_inter, G, b, grad dtype, seed, average
    (1, 2, 8, 4, 128, 64, torch.bfloat16, None, True),
    (2, 1, 8, 4, 128, 64, torch.bfloat16, None, True),
    (2, 2, 8, 4, 128, 64, torch.bfloat16, None, True),
    (2, 4, 8, 4, 128, 64, torch.bfloat16, None, True),
    (4, 2, 8, 4, 128, 64, torch.float32, None, True),
    (1, 8, 8, 4, 128, 64, torch.float32, None, True),
    (8, 1, 8, 4, 128, 64, torch.bfloat16, None, True),
    (2, 2, 4, 4, 128, 0, torch.float32, None, True),      # ULq
    (2, 2, 8, 8, 32, 32, torch.bfloat16, None, True),
    (2, 2, 8, 4, 256, 256, torch.float32, None, True),
    (3, 2, 8, 4, 64, 2, torch.float32, None, False),
    (2, 3, 4, 8, 2048, 128, torch.bfloat16, None, True),
    (2, 2, 8, 4, 128, 64, torch.bfloat16, 11, True),      # stochastic rounding (R14)
    (2, 4, 8, 4, 64, 16, torch.float32, 5, True),
]


@pytest.mark.parametrize("M,N,bi,be,G,b,dt,seed,avg", TLQ_CASES)
def test_emu_tlq_hs(M, N, bi, be, G, b, dt, seed, avg):
    _need_gpu()
    from paper_2410_15526_b200 import emu_tlq_hs_reduce_scatter, emu_tlq_workspace_bytes
    P = M * N
    S = _shard_len(G, tiles=2)
    D = P * S
    ws = torch.empty(emu_tlq_workspace_bytes(M, N, D, bi, be, G), dtype=torch.uint8, device="cuda")
    outs = [torch.empty(S, dtype=torch.float32, device="cuda") for _ in range(P)]
    for call in range(3):
        grads = [synth.gradient(D, seed=1000 * call + 20 + r, dtype=dt) for r in range(P)]
        if call == 1:  # edge-case groups in rank 1's gradient
            e = synth.edge_case_groups(G)[:S].to(dt)
            grads[1 % P][:e.numel()] = e
        emu_tlq_hs_reduce_scatter(M, N, [g.cuda() for g in grads], outs, ws, bi, be, G, b, avg, seed=seed,
                                  fresh=(call == 0))
        torch.cuda.synchronize()
        tr = oracle.tlq_hs_reduce_scatter([g.float().numpy() for g in grads], oracle.Topology(M, N), G, b, bi, be,
                                          avg, seed=seed)
        for r in range(P):
            assert _bits_equal(outs[r].cpu().numpy(), tr.out[r]), f"call {call}: rank {r}'s shard differs"


def test_emu_rejects_unsupported():
    """The one-launch TLq-HS takes 4/8-bit codes only (the identity codec stays multi-launch)."""
    _need_gpu()
    from paper_2410_15526_b200 import SDP4Error, emu_tlq_hs_reduce_scatter, emu_tlq_workspace_bytes
    S, M, N = 2048, 1, 2
    ws = torch.empty(emu_tlq_workspace_bytes(M, N, 2 * S, 32, 4, 128), dtype=torch.uint8, device="cuda")
    g = [torch.zeros(2 * S, device="cuda") for _ in range(2)]
    o = [torch.empty(S, device="cuda") for _ in range(2)]
    with pytest.raises(SDP4Error):
        emu_tlq_hs_reduce_scatter(M, N, g, o, ws, 32, 4, 128, 64)
