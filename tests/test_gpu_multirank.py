"""Multi-rank TLq-HS parity on ONE GPU: P = M x N ranks emulated through the stage entry
points (sdp4_tlq_stage_quantize / _reduce / _final).  The two all-to-alls of Alg. 3
 are done here by slicing the documented workspace layouts (R9, R15), so
K3/K4/K5 run with real M, N > 1 (multi-source fp32 reductions, per-shard routing) and are
compared with the oracle message by message.  The NCCL path itself is covered by
tests/dist_parity.py (multi-GPU)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2410_15526_b200 import tlq_stage_final, tlq_stage_quantize, tlq_stage_reduce, wire_unit_bytes
from tests.test_gpu_parity import assert_unit_equal, f32_equal

pytestmark = pytest.mark.gpu


def emulate(grads, M, N, bi, be, G, b, average=True, seed=None):
    P = M * N
    D = grads[0].numel()
    S = D // P
    w8, w4 = wire_unit_bytes(S, bi, G), wire_unit_bytes(S, be, G)
    dev = "cuda"
    intra_send = []
    for r in range(P):
        buf = torch.zeros(N * M * w8, dtype=torch.uint8, device=dev)
        tlq_stage_quantize(grads[r].to(dev), buf, M, N, bi, G, b, seed=seed, rank=r)
        intra_send.append(buf)
    inter_send = []
    for r in range(P):
        m, l = divmod(r, N)
        recv = torch.cat([intra_send[m * N + lpp][l * M * w8:(l + 1) * M * w8] for lpp in range(N)])
        buf = torch.zeros(M * w4, dtype=torch.uint8, device=dev)
        tlq_stage_reduce(recv, buf, D, M, N, bi, be, G, seed=seed, rank=r)
        inter_send.append(buf)
    outs = []
    for r in range(P):
        m, l = divmod(r, N)
        recv = torch.cat([inter_send[mpp * N + l][m * w4:(m + 1) * w4] for mpp in range(M)])
        out = torch.empty(S, dtype=torch.float32, device=dev)
        tlq_stage_final(recv, out, D, M, N, be, G, b, average)
        outs.append(out)
    torch.cuda.synchronize()
    return ([x.cpu().numpy() for x in intra_send], [x.cpu().numpy() for x in inter_send],
            [x.cpu().numpy() for x in outs], w8, w4, S)


CASES = [  # (M, N, bits_intra, bits_inter, G, b, dtype, seed)
    (2, 4, 8, 4, 128, 64, torch.bfloat16, None),
    (4, 2, 8, 4, 128, 64, torch.bfloat16, None),
    (2, 4, 8, 4, 128, 32, torch.float32, None),
    (1, 8, 8, 4, 128, 64, torch.bfloat16, None),
    (8, 1, 8, 4, 128, 64, torch.bfloat16, None),
    (2, 2, 4, 4, 128, 0, torch.float32, None),      # ULq
    (3, 2, 8, 4, 64, 16, torch.float32, None),      # P = 6: kappa = rn(c_b / 6)
    (2, 4, 8, 4, 256, 256, torch.bfloat16, None),   # cross-lane Hadamard stages
    (2, 2, 8, 4, 32, 32, torch.bfloat16, None),     # two groups per row
    (2, 2, 32, 32, 128, 64, torch.float32, None),   # identity codec (R12)
    (4, 2, 8, 8, 2048, 128, torch.bfloat16, None),  # large groups (cross-warp K4 group max)
    (2, 4, 8, 4, 128, 64, torch.bfloat16, 2410),    # stochastic rounding (R14): per-rank keys
    (4, 2, 4, 4, 32, 0, torch.float32, 2 ** 36 + 1),
]


@pytest.mark.parametrize("M,N,bi,be,G,b,dtype,seed", CASES)
def test_tlq_multirank_emulated(M, N, bi, be, G, b, dtype, seed):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    P = M * N
    align = P * max(G, 64)
    D = ((16384 * P * 2 + 64 * 37 * P) // align + 1) * align     # > 2 tiles per shard + ragged tail
    grads = [synth.gradient(D, seed=synth.seed_for(r, 3), dtype=dtype) for r in range(P)]
    intra, inter, outs, w8, w4, S = emulate(grads, M, N, bi, be, G, b, seed=seed)
    tr = oracle.tlq_hs_reduce_scatter([g.float().numpy() for g in grads], oracle.Topology(M, N), G, b, bi, be, True,
                                      seed=seed)
    for r in range(P):
        for lp in range(N):
            for mp in range(M):
                off = (lp * M + mp) * w8
                c, s = tr.intra_send[r][lp][mp]
                assert_unit_equal(intra[r][off:off + w8], c, s, bi, G, S, f"rank {r} intra block {lp} unit {mp}")
        for mp in range(M):
            c, s = tr.inter_send[r][mp]
            assert_unit_equal(inter[r][mp * w4:(mp + 1) * w4], c, s, be, G, S, f"rank {r} inter unit {mp}")
        assert f32_equal(outs[r], tr.out[r]), f"rank {r} output shard differs"


def test_multirank_matches_exact_mean_within_quantization_error():
    # end to end sanity at 2 x 4: the emulated outputs approach the exact mean
    M, N, G, b = 2, 4, 128, 64
    P = M * N
    D = P * 16384
    grads = [synth.gradient(D, seed=100 + r) for r in range(P)]
    _, _, outs, _, _, S = emulate(grads, M, N, 8, 4, G, b)
    exact = oracle.exact_reduce_scatter_f64([g.numpy() for g in grads], P)
    rel = np.linalg.norm(np.concatenate(outs) - np.concatenate(exact)) / np.linalg.norm(np.concatenate(exact))
    assert rel < 0.2


K34_CASES = [  # (M, G, b, dtype, seed): one GPU per group (N = 1), K3 + K4 fused
    (2, 128, 64, torch.bfloat16, None),
    (3, 64, 16, torch.float32, None),
    (4, 32, 32, torch.bfloat16, None),
    (8, 2048, 256, torch.bfloat16, None),
    (2, 256, 0, torch.float32, None),
    (4, 128, 64, torch.bfloat16, 2410),
]


@pytest.mark.parametrize("M,G,b,dtype,seed", K34_CASES)
def test_k34_units_emulated(M, G, b, dtype, seed):
    """K34 (sdp4_tlq_stage_quantize_reduce) on every node of an emulated M x 1 job: its 4-bit
    inter units equal the oracle's messages of Alg. 3 l.10 bit for bit (the 8-bit intra units
    it dequantizes in registers are the oracle's intra messages by construction)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_15526_b200 import tlq_stage_quantize_reduce
    P = M
    align = P * max(G, 64)
    D = ((16384 * P * 2 + 64 * 37 * P) // align + 1) * align
    grads = [synth.gradient(D, seed=synth.seed_for(r, 5), dtype=dtype) for r in range(P)]
    e = synth.edge_case_groups(G)[:D // P].to(dtype)
    grads[0][:e.numel()] = e
    S = D // P
    w4 = wire_unit_bytes(S, 4, G)
    tr = oracle.tlq_hs_reduce_scatter([g.float().numpy() for g in grads], oracle.Topology(M, 1), G, b, 8, 4, True,
                                      seed=seed)
    for r in range(P):
        buf = torch.zeros(M * w4, dtype=torch.uint8, device="cuda")
        tlq_stage_quantize_reduce(grads[r].cuda(), buf, M, G, b, seed=seed, rank=r)
        torch.cuda.synchronize()
        got = buf.cpu().numpy()
        for mp in range(M):
            c, s = tr.inter_send[r][mp]
            assert_unit_equal(got[mp * w4:(mp + 1) * w4], c, s, 4, G, S, f"K34 rank {r} inter unit {mp}")


@pytest.mark.parametrize("M,G,b,dtype", [(2, 128, 64, torch.bfloat16), (3, 32, 0, torch.float32),
                                          (2, 256, 16, torch.float32), (4, 64, 64, torch.bfloat16)])
def test_k34_code_map_tiny_inter_groups(M, G, b, dtype):
    """K34's shortcut for ok 8-bit groups (the 4-bit group max taken as rn(127 * d8) instead
    of a pass over the row, k_local34.cu) on groups whose 8-bit scale is ok but whose 4-bit max
    lands at or below 2^-120 (a zero group at 4 bits, R2): every third group of every rank is scaled
    to a max in [2^-120, 2^-116] (incl. 2^-120 and one ulp above), all other groups are plain gaussian, so whole warps take the
    shortcut.  Inter units bit-exact against the oracle (R2, R3, R5)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_15526_b200 import tlq_stage_quantize_reduce
    P = M
    align = P * max(G, 64)
    D = ((16384 * P * 2 + 64 * 37 * P) // align + 1) * align
    grads = []
    for r in range(P):
        g = synth.gradient(D, seed=synth.seed_for(r, 6), dtype=torch.float32).view(-1, G).clone()
        gen = torch.Generator().manual_seed(100 + r)
        sel = torch.arange(0, g.shape[0], 3)
        tgt = torch.exp2(torch.empty(sel.numel()).uniform_(-120.0, -116.0, generator=gen))
        tgt[::7] = 2.0 ** -120                      # the R2 boundary itself, and one ulp above
        tgt[1::7] = 2.0 ** -120 * (1 + 2.0 ** -23)
        g[sel] = g[sel] / g[sel].abs().amax(dim=1, keepdim=True) * tgt[:, None]
        grads.append(g.reshape(-1).to(dtype))
    S = D // P
    w4 = wire_unit_bytes(S, 4, G)
    tr = oracle.tlq_hs_reduce_scatter([g.float().numpy() for g in grads], oracle.Topology(M, 1), G, b, 8, 4, True)
    for r in range(P):
        buf = torch.zeros(M * w4, dtype=torch.uint8, device="cuda")
        tlq_stage_quantize_reduce(grads[r].cuda(), buf, M, G, b, rank=r)
        torch.cuda.synchronize()
        got = buf.cpu().numpy()
        for mp in range(M):
            c, s = tr.inter_send[r][mp]
            assert_unit_equal(got[mp * w4:(mp + 1) * w4], c, s, 4, G, S, f"K34 rank {r} inter unit {mp}")
