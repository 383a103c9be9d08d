"""Sharded-data-parallel SGD with SDP4Bit on a synthetic least-squares task (Alg. 2 / Alg. 4,
P:252-270 and P:426-440): the NEXT-4 training harness.

Every rank holds the full model replica w~ (bf16, as the paper's model weights), its
fp32 main-weight shard w[r] and its own data shard (X_r, y_r).  One step:

    g_r   = X_r^T (X_r w~ - y_r) / n                 (local gradient at the replica, torch)
    g~[r] = TLq-HS reduce-scatter of the g_r          (libsdp4, Alg. 3; mean over ranks)
    w[r] <- w[r] - lr * g~[r]                          (SGD on the shard, torch)
    w~   <- w~ + AllGather(Q(w[r] - w~[r]))            (libsdp4 qWD, Alg. 2 l.2-5)

`mode` selects the weight path: "qwd" (SDP4Bit), "qw" (direct 4-bit weight quantization,
QSDP / ZeRO++, Alg. 1) or "exact" (no weight quantization: w~ = bf16(w)); `grad` selects
"tlq_hs" (SDP4Bit) or "exact" (torch reduce-scatter).  The history records the loss of the
replica and the drift e_t = ||w~ - w|| / ||w|| between the replica and the main weights.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 examples/sgd_harness.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2410_15526_b200 import Comm  # noqa: E402


def make_task(d: int, n: int, rank: int, world: int, device, noise: float = 0.01):
    """Least squares with a planted solution; rank r draws its own n samples."""
    g = torch.Generator(device="cpu").manual_seed(1234)
    w_star = torch.randn(d, generator=g) / d ** 0.5
    gr = torch.Generator(device="cpu").manual_seed(5678 + rank)
    X = torch.randn(n, d, generator=gr) / d ** 0.5
    y = X @ w_star + noise * torch.randn(n, generator=gr)
    return X.to(device), y.to(device), w_star.to(device)


def run(comm: Comm, steps: int = 200, d: int = 1 << 16, n: int = 2048, lr: float = 2.0, mode: str = "qwd",
        grad: str = "tlq_hs", G: int = 128, b: int = 64, device=None):
    torch.backends.cuda.matmul.allow_tf32 = False
    device = device or torch.device("cuda", torch.cuda.current_device())
    P, r = comm.world, comm.rank
    S = d // P
    X, y, _ = make_task(d, n, r, P, device)
    w_main = torch.zeros(S, dtype=torch.float32, device=device)              # w[r]
    w_model = torch.zeros(d, dtype=torch.bfloat16, device=device)            # replica w~
    out = torch.empty(S, dtype=torch.float32, device=device)
    p2p = comm.transport == "p2p"
    ws_q = None if p2p else torch.empty(comm.qwd_workspace_bytes(d, 4, G), dtype=torch.uint8, device=device)
    ws_t = None if p2p else torch.empty(comm.tlq_workspace_bytes(d, 8, 4, G), dtype=torch.uint8, device=device)
    hist = []
    for t in range(steps):
        wm = w_model.float()
        res = X @ wm - y
        g_local = X.t() @ res / n
        loss = torch.tensor([float((res * res).mean()) / 2], device=device)
        if P > 1:
            dist.all_reduce(loss)
            loss /= P
        if grad == "tlq_hs":
            comm.tlq_hs_reduce_scatter(g_local, out, ws_t, 8, 4, G, b, True)
        elif P > 1:
            dist.reduce_scatter_tensor(out, g_local, op=dist.ReduceOp.AVG)
        else:
            out.copy_(g_local)
        w_main -= lr * out
        if mode == "qwd":
            comm.qwd_quantize(w_main, w_model, ws_q, 4, G)
            comm.qwd_allgather_apply(ws_q, w_model, 4, G)
        elif mode == "qw":
            comm.qw_quantize(w_main, d, ws_q, 4, G)
            comm.qw_allgather_apply(ws_q, w_model, 4, G)
        else:
            full = torch.empty(d, dtype=torch.float32, device=device)
            if P > 1:
                dist.all_gather_into_tensor(full, w_main)
            else:
                full.copy_(w_main)
            w_model.copy_(full.to(torch.bfloat16))
        shard = w_model[r * S:(r + 1) * S].float()
        drift = torch.tensor([float((shard - w_main).pow(2).sum()), float(w_main.pow(2).sum())], device=device)
        if P > 1:
            dist.all_reduce(drift)
        hist.append({"t": t, "loss": float(loss), "drift": float(drift[0].sqrt() / drift[1].sqrt().clamp_min(1e-30))})
    # replicas must be identical on every rank
    h = torch.tensor([float(w_model.float().double().mul(torch.arange(1, d + 1, device=device)).sum())],
                     dtype=torch.float64, device=device)
    same = True
    if P > 1:
        hs = [torch.zeros_like(h) for _ in range(P)]
        dist.all_gather(hs, h)
        same = len({float(x) for x in hs}) == 1
    return hist, same


def main():
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = Comm.from_process_group()
    else:
        comm = Comm()
    res = {}
    for mode, grad in (("exact", "exact"), ("qwd", "tlq_hs"), ("qw", "tlq_hs")):
        hist, same = run(comm, mode=mode, grad=grad)
        res[f"{mode}+{grad}"] = {"final_loss": hist[-1]["loss"], "max_drift": max(h["drift"] for h in hist[5:]),
                                 "replicas_identical": same}
    if rank == 0:
        print(json.dumps(res), flush=True)
    comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
