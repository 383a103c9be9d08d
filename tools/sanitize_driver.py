"""Small-size run of every kernel path through the C ABI, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run -- SURVEY sec. 4(5)):

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py

P = 1 calls of the product entry points (qWD step and two-call, qW with int2/4/8, TLq-HS on
bf16/fp32 gradients with b in {0, 64, 256} and bits {8/4, 4/4, 32/32}, nearest and stochastic
rounding, the ring), and the stage entry points on an emulated 2 x 2 topology (K3 / K4 / K5
with multi-source reductions), at sizes spanning several tiles and a ragged tail.  Checks
nothing itself: the sanitizer's report is the result."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2410_15526_b200 import (Comm, tlq_stage_final, tlq_stage_quantize, tlq_stage_reduce,  # noqa: E402
                                   tlq_workspace_bytes, tlq_workspace_offset)


def main():
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    comm = Comm()
    D = 16384 * 3 + 128 * 5   # several K3/K4/K5 tiles and a ragged tail
    G = 128
    w_model = synth.model_weights(D, seed=1).to(dev)
    w_main = synth.main_weights(w_model.cpu(), seed=2).to(dev)
    ws = torch.zeros(comm.qwd_workspace_bytes(D, 8, G), dtype=torch.uint8, device=dev)
    comm.qwd_step(w_main, w_model, ws, 4, G)
    comm.qwd_quantize(w_main, w_model, ws, 4, G, seed=7)
    comm.qwd_allgather_apply(ws, w_model, 4, G)
    for bits in (2, 4, 8):
        comm.qw_quantize(w_main, D, ws, bits, G)
        comm.qw_allgather_apply(ws, w_model, bits, G)
    out = torch.empty(D, dtype=torch.float32, device=dev)
    for dt in (torch.bfloat16, torch.float32):
        grad = synth.gradient(D, seed=3, dtype=dt).to(dev)
        for (bi, be, b, seed) in ((8, 4, 64, None), (8, 4, 0, None), (4, 4, 128, None), (8, 4, 64, 11),
                                  (32, 32, 64, None)):
            tws = torch.zeros(comm.tlq_workspace_bytes(D, bi, be, G), dtype=torch.uint8, device=dev)
            comm.tlq_hs_reduce_scatter(grad, out, tws, bi, be, G, b, True, seed=seed)
        rws = torch.zeros(comm.ring_workspace_bytes(D, 4, G), dtype=torch.uint8, device=dev)
        comm.ring_reduce_scatter(grad, out, rws, 4, G, True)
    # emulated 2 x 2: four ranks' K3 outputs routed by hand into rank 0's receive regions
    M, N = 2, 2
    P = M * N
    D2 = P * (16384 + 128 * 3)
    S = D2 // P
    off = [tlq_workspace_offset(M, N, D2, 8, 4, G, r) for r in range(4)]
    nbytes = tlq_workspace_bytes(M, N, D2, 8, 4, G)
    wss = [torch.zeros(nbytes, dtype=torch.uint8, device=dev) for _ in range(P)]
    grads = [synth.gradient(D2, seed=20 + r, dtype=torch.bfloat16).to(dev) for r in range(P)]
    for r in range(P):
        tlq_stage_quantize(grads[r], wss[r][off[0]:], M, N, 8, G, 64, rank=r)
    w8 = (off[1] - off[0]) // (N * M) if N > 1 else 0
    for lp in range(N):   # rank 0 = (m 0, l 0) receives block 0 of every local rank of group 0
        src = wss[lp][off[0]:off[0] + M * w8]
        wss[0][off[1] + lp * M * w8:off[1] + (lp + 1) * M * w8].copy_(src)
    tlq_stage_reduce(wss[0][off[1]:], wss[0][off[2]:], D2, M, N, 8, 4, G, rank=0)
    tlq_stage_reduce(wss[0][off[1]:], wss[0][off[2]:], D2, M, N, 8, 4, G, seed=5, rank=0)
    w4 = (off[3] - off[2]) // M
    wss[0][off[3] + w4:off[3] + 2 * w4].copy_(wss[0][off[2]:off[2] + w4])
    wss[0][off[3]:off[3] + w4].copy_(wss[0][off[2] + w4:off[2] + 2 * w4])
    o = torch.empty(S, dtype=torch.float32, device=dev)
    tlq_stage_final(wss[0][off[3]:], o, D2, M, N, 4, G, 64, True)
    torch.cuda.synchronize()
    comm.close()
    print("sanitize driver done", flush=True)


if __name__ == "__main__":
    main()
