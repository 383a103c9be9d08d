"""Guard-band bounds checks (compute-sanitizer is closed on this GPU pool, so out-of-bounds
accesses are caught with canaries of our own): every caller-visible buffer of every entry
point -- inputs, outputs, workspaces -- is carved out of a larger allocation between 64 KB
guard zones filled with a byte pattern (0xA5, i.e. a NaN-free float pattern the kernels never
produce).  After each call the guard zones must be untouched (no out-of-bounds WRITE) and
the results must equal the oracle bit for bit (an out-of-bounds READ of a guard would pull
the pattern into some output).  Sizes span several tiles of every kernel and a ragged tail;
the stage entry points run an emulated 2 x 2 topology (multi-source K4 / K5)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

GUARD = 64 * 1024
PAT = 0xA5


class Arena:
    """One device allocation; carve() hands out 256-byte-aligned views separated by guards."""

    def __init__(self, nbytes):
        self.buf = torch.full((nbytes,), PAT, dtype=torch.uint8, device="cuda")
        self.off = GUARD
        self.spans = []

    def carve(self, numel, dtype):
        esz = torch.tensor([], dtype=dtype).element_size()
        nb = numel * esz
        start = (self.off + 255) // 256 * 256
        view = self.buf[start:start + nb].view(dtype)
        self.spans.append((start, start + nb))
        self.off = start + nb + GUARD
        assert self.off <= self.buf.numel(), "arena too small"
        return view

    def guards_intact(self):
        b = self.buf.cpu().numpy()
        prev = 0
        for s, e in self.spans:
            if not np.all(b[prev:s] == PAT):
                return False, (prev, s)
            prev = e
        return bool(np.all(b[prev:self.off] == PAT)), (prev, self.off)


@pytest.fixture(scope="module")
def comm():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2410_15526_b200 import Comm
    c = Comm()
    yield c
    c.close()


def _same(a, b):
    """Bit-identical fp32 arrays (NaN equals NaN)."""
    a, b = np.asarray(a, dtype=np.float32), np.asarray(b, dtype=np.float32)
    return bool(np.all((a.view(np.uint32) == b.view(np.uint32)) | (np.isnan(a) & np.isnan(b))))


D = 16384 * 3 + 128 * 5    # several K1..K5 tiles and a ragged tail
G = 128


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_guard_qwd_and_qw(comm, bits):
    ar = Arena(D * 32 + 16 * GUARD)
    wm0 = synth.model_weights(D, seed=1)
    main = synth.main_weights(wm0, seed=2)
    wm = ar.carve(D, torch.bfloat16)
    wm.copy_(wm0)
    wmain = ar.carve(D, torch.float32)
    wmain.copy_(main)
    ws = ar.carve(comm.qwd_workspace_bytes(D, bits, G), torch.uint8)
    comm.qwd_step(wmain, wm, ws, bits, G)
    torch.cuda.synchronize()
    ok, where = ar.guards_intact()
    assert ok, f"qwd_step wrote outside its buffers near bytes {where}"
    _, want = oracle.qwd_step([main.numpy()], synth.bf16_bits(wm0), bits, G, model_bf16=True)
    assert np.array_equal(synth.bf16_bits(wm.cpu()), want)
    wq = ar.carve(D, torch.bfloat16)
    comm.qw_quantize(wmain, D, ws, bits, G)
    comm.qw_allgather_apply(ws, wq, bits, G)
    torch.cuda.synchronize()
    ok, where = ar.guards_intact()
    assert ok, f"qW wrote outside its buffers near bytes {where}"
    _, want = oracle.qw_step([main.numpy()], bits, G, model_bf16=True)
    assert np.array_equal(synth.bf16_bits(wq.cpu()), want)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("bi,be,b,seed", [(8, 4, 64, None), (8, 4, 0, None), (4, 4, 128, None), (8, 4, 64, 11),
                                          (32, 32, 64, None), (8, 8, 32, None)])
def test_guard_tlq_and_ring(comm, dtype, bi, be, b, seed):
    ar = Arena(D * 24 + comm.tlq_workspace_bytes(D, bi, be, G) + 16 * GUARD)
    g0 = synth.gradient(D, seed=3, dtype=dtype)
    grad = ar.carve(D, dtype)
    grad.copy_(g0)
    out = ar.carve(D, torch.float32)
    tws = ar.carve(comm.tlq_workspace_bytes(D, bi, be, G), torch.uint8)
    comm.tlq_hs_reduce_scatter(grad, out, tws, bi, be, G, b, True, seed=seed)
    torch.cuda.synchronize()
    ok, where = ar.guards_intact()
    assert ok, f"TLq-HS wrote outside its buffers near bytes {where}"
    want = oracle.tlq_hs_reduce_scatter([g0.float().numpy()], oracle.Topology(1, 1), G, b, bi, be, True,
                                        seed=seed).out[0]
    assert _same(out.cpu().numpy(), want)
    if seed is None and bi == 8 and b == 64:
        rws = ar.carve(comm.ring_workspace_bytes(D, 4, G), torch.uint8)
        comm.ring_reduce_scatter(grad, out, rws, 4, G, True)
        torch.cuda.synchronize()
        ok, where = ar.guards_intact()
        assert ok, f"ring wrote outside its buffers near bytes {where}"


def test_guard_stages_emulated_2x2():
    """K3 / K4 / K5 through the stage entry points on an emulated 2 x 2 topology (rank 0's
    view), every buffer guarded; codes, scales and the output shard equal the oracle's."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2410_15526_b200 import (tlq_stage_final, tlq_stage_quantize, tlq_stage_reduce,
                                       tlq_workspace_bytes, tlq_workspace_offset)
    M, N, P = 2, 2, 4
    D2 = P * (16384 + 128 * 3)
    S = D2 // P
    nbytes = tlq_workspace_bytes(M, N, D2, 8, 4, G)
    off = [tlq_workspace_offset(M, N, D2, 8, 4, G, r) for r in range(4)]
    ar = Arena(P * (D2 * 2 + nbytes) + S * 4 + 32 * GUARD)
    g0 = [synth.gradient(D2, seed=20 + r, dtype=torch.bfloat16) for r in range(P)]
    grads, wss = [], []
    for r in range(P):
        g = ar.carve(D2, torch.bfloat16)
        g.copy_(g0[r])
        grads.append(g)
        wss.append(ar.carve(nbytes, torch.uint8))
    for r in range(P):
        tlq_stage_quantize(grads[r], wss[r][off[0]:], M, N, 8, G, 64, rank=r)
    w8 = (off[1] - off[0]) // (N * M)
    for lp in range(N):   # rank 0 = (m 0, l 0) receives block 0 of local ranks 0 and 1
        wss[0][off[1] + lp * M * w8:off[1] + (lp + 1) * M * w8].copy_(wss[lp][off[0]:off[0] + M * w8])
    tlq_stage_reduce(wss[0][off[1]:], wss[0][off[2]:], D2, M, N, 8, 4, G, rank=0)
    # rank 2 = (m 1, l 0) does the same for its group; rank 0 receives unit 0 of both nodes
    for lp in range(N):
        wss[2][off[1] + lp * M * w8:off[1] + (lp + 1) * M * w8].copy_(wss[2 + lp][off[0]:off[0] + M * w8])
    tlq_stage_reduce(wss[2][off[1]:], wss[2][off[2]:], D2, M, N, 8, 4, G, rank=2)
    w4 = (off[3] - off[2]) // M
    wss[0][off[3] + w4:off[3] + 2 * w4].copy_(wss[2][off[2]:off[2] + w4])   # from node 1 (slot m''=1)
    wss[0][off[3]:off[3] + w4].copy_(wss[0][off[2]:off[2] + w4])            # own unit (slot m''=0)
    out = ar.carve(S, torch.float32)
    tlq_stage_final(wss[0][off[3]:], out, D2, M, N, 4, G, 64, True)
    torch.cuda.synchronize()
    ok, where = ar.guards_intact()
    assert ok, f"a stage kernel wrote outside its buffers near bytes {where}"
    want = oracle.tlq_hs_reduce_scatter([g.float().numpy() for g in g0], oracle.Topology(M, N), G, 64, 8, 4,
                                        True).out[0]
    assert _same(out.cpu().numpy(), want)
