"""Device time of the one-launch kernels on an emulated job (one GPU, all ranks in one launch,
no cross-GPU latency) next to the multi-launch path at P = 1, to separate kernel cost from
exchange latency.  Prints one JSON line per case."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_15526_b200 import (Comm, emu_qwd_step, emu_qwd_workspace_bytes,  # noqa: E402
                                   emu_tlq_hs_reduce_scatter, emu_tlq_workspace_bytes)


def timed(fn, iters=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3  # us


def main():
    comm = Comm()
    import os
    for mb in [int(x) for x in os.environ.get("FUSED_PROBE_MB", "1,4,16").split(",")]:
        D = mb << 18
        for M, N in ((1, 1), (2, 1), (1, 2), (2, 2)):
            P = M * N
            S = D // P
            g = [torch.randn(D, device="cuda").to(torch.bfloat16) for _ in range(P)]
            o = [torch.empty(S, device="cuda") for _ in range(P)]
            wm = [torch.randn(D, device="cuda").to(torch.bfloat16) for _ in range(P)]
            mains = [torch.randn(S, device="cuda") for _ in range(P)]
            row = {"mbytes": mb, "split": f"{M}x{N}"}
            if P == 1:
                ws = torch.empty(comm.tlq_workspace_bytes(D, 8, 4, 128), dtype=torch.uint8, device="cuda")
                row["tlq_multi_launch_us"] = timed(lambda: comm.tlq_hs_reduce_scatter(g[0], o[0], ws, 8, 4, 128, 64))
                wq = torch.empty(comm.qwd_workspace_bytes(D, 4, 128), dtype=torch.uint8, device="cuda")
                row["qwd_multi_launch_us"] = timed(lambda: comm.qwd_step(mains[0], wm[0], wq, 4, 128))
            else:
                ws = torch.empty(emu_tlq_workspace_bytes(M, N, D, 8, 4, 128), dtype=torch.uint8, device="cuda")
                emu_tlq_hs_reduce_scatter(M, N, g, o, ws, 8, 4, 128, 64, fresh=True)
                row["tlq_one_launch_us"] = timed(lambda: emu_tlq_hs_reduce_scatter(M, N, g, o, ws, 8, 4, 128, 64,
                                                                                  fresh=False))
                wq = torch.empty(emu_qwd_workspace_bytes(P, D, 4, 128), dtype=torch.uint8, device="cuda")
                emu_qwd_step(mains, wm, wq, 4, 128, fresh=True)
                row["qwd_one_launch_us"] = timed(lambda: emu_qwd_step(mains, wm, wq, 4, 128, fresh=False))
            print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in row.items()}), flush=True)
    comm.close()


if __name__ == "__main__":
    main()
