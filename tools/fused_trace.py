"""Phase timeline of the one-launch P2P kernels on real GPUs (run under torchrun with
SDP4_FUSED_TRACE=1: the library synchronizes after each one-launch call and prints its phase
stamps to stderr).  A few back-to-back calls at each size; a barrier between sizes."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2410_15526_b200 import Comm  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = Comm.from_process_group(None, dev)
    for mb in [int(x) for x in os.environ.get("TRACE_MB", "1,16").split(",")]:
        D = mb << 18
        S = D // world
        g = torch.randn(D, device=dev).to(torch.bfloat16)
        out = torch.empty(S, device=dev)
        wm = torch.randn(D, device=dev).to(torch.bfloat16)
        main_w = torch.randn(S, device=dev)
        for it in range(4):
            sys.stderr.write(f"# rank {rank} {mb} MB call {it}\n")
            comm.tlq_hs_reduce_scatter(g, out, None, 8, 4, 128, 64)
            comm.qwd_step(main_w, wm, None, 4, 128)
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
