"""Time the TLq-HS stage kernels alone (K3 / K4 / K5 through the stage entry points) on the
bench workload's shapes, with CUDA events: a quick loop for kernel tuning and ncu captures.

    python tools/kbench.py [--kernels K3,K4,K5] [--numel D] [--M 1 --N 1] [--iters 20]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2410_15526_b200 import (tlq_stage_final, tlq_stage_quantize, tlq_stage_reduce,  # noqa: E402
                                   tlq_workspace_bytes, tlq_workspace_offset, wire_unit_bytes)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernels", default="K3,K4,K5")
    ap.add_argument("--numel", type=int, default=synth.gpt_numel("1.3B"))
    ap.add_argument("--M", type=int, default=1)
    ap.add_argument("--N", type=int, default=1)
    ap.add_argument("--G", type=int, default=128)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--bits", default="8,4")
    ap.add_argument("--grad", default="bf16")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    bi, be = (int(x) for x in a.bits.split(","))
    M, N, G = a.M, a.N, a.G
    P = M * N
    D = a.numel - a.numel % (P * max(G, 64))
    S = D // P
    dev = torch.device("cuda", 0)
    grad = synth.gradient(D, seed=3, device=dev, dtype=torch.bfloat16 if a.grad == "bf16" else torch.float32)
    ws = torch.zeros(tlq_workspace_bytes(M, N, D, bi, be, G), dtype=torch.uint8, device=dev)
    r = [tlq_workspace_offset(M, N, D, bi, be, G, k) for k in range(4)]
    send8, recv8 = ws[r[0]:], ws[r[1]:]
    send4, recv4 = ws[r[2]:], ws[r[3]:]
    out = torch.empty(S, dtype=torch.float32, device=dev)
    tlq_stage_quantize(grad, send8, M, N, bi, G, a.b)
    if N > 1:   # every source block holds this rank's own quantized data (timing only)
        w8 = wire_unit_bytes(S, bi, G)
        for lp in range(N):
            recv8[lp * M * w8:(lp + 1) * M * w8].copy_(send8[:M * w8])
    tlq_stage_reduce(recv8, send4, D, M, N, bi, be, G)
    if M > 1:
        w4 = wire_unit_bytes(S, be, G)
        for mp in range(M):
            recv4[mp * w4:(mp + 1) * w4].copy_(send4[:w4])
    calls = {
        "K3": (lambda: tlq_stage_quantize(grad, send8, M, N, bi, G, a.b),
               D * grad.element_size() + D * (bi / 8 + 4 / G)),
        "K4": (lambda: tlq_stage_reduce(recv8, send4, D, M, N, bi, be, G),
               D * (bi / 8 + 4 / G) + D / N * (be / 8 + 4 / G)),
        "K5": (lambda: tlq_stage_final(recv4, out, D, M, N, be, G, a.b, True),
               S * M * (be / 8 + 4 / G) + 4 * S),
    }
    res = {}
    for k in a.kernels.split(","):
        fn, nbytes = calls[k]
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        res[k] = {"ms": round(ms, 4), "GBps": round(nbytes / ms / 1e6, 1)}
    print(json.dumps({"D": D, "M": M, "N": N, "G": G, "bits": [bi, be], "grad": a.grad, "kernels": res}))


if __name__ == "__main__":
    main()
