"""Message-size sweep (BASELINE.json configs[4]): qWD all-gather and TLq-HS reduce-scatter
through libsdp4 vs torch.distributed's unquantized NCCL all-gather / reduce-scatter on the
same buffers, from 1 MB to 4 GB of fp32 data (D*4 bytes).  One process per GPU:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/size_sweep.py [--groups M] [--out F]

Times are CUDA events on the launch stream, max over ranks, after warm-up (as bench.py).
The model replica is bf16, the gradient fp32 (so the reduce-scatter comparator moves the
same D*4 bytes the size names), G = 128, b = 64, bits 4/8/4."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2410_15526_b200 import Comm, default_split, pad_numel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, default=None)
    ap.add_argument("--sizes-mb", type=str, default="1,2,4,8,16,32,64,128,256,512,1024,2048,4096")
    ap.add_argument("--graphs", action="store_true", help="also time CUDA-graph replays of every call")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out", type=str, default=None)
    ap.add_argument("--fused-limit", type=int, default=None,
                    help="sdp4_comm_set_fused_limit (elements; 0 = always multi-launch)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    M, N = default_split(world, a.groups)
    comm = Comm.from_process_group(a.groups, dev)
    if a.fused_limit is not None:
        comm.set_fused_limit(a.fused_limit)
    P, G, b = world, 128, 64

    def timed(fn, iters=None):
        # median of three timed runs (each: max over ranks of the per-call device time), the
        # same method for libsdp4 and NCCL; small messages run more calls per run
        iters = iters or a.iters
        for _ in range(3):
            fn()
        runs = []
        for _ in range(3):
            dist.barrier(device_ids=[local])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / iters], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            runs.append(float(t.item()))
        return sorted(runs)[1]

    rows = []
    for mb in [int(x) for x in a.sizes_mb.split(",")]:
        D = pad_numel(mb * (1 << 20) // 4, P, G)
        S = D // P
        w_model = synth.model_weights(D, seed=1, device=dev)
        w_main = synth.main_weights(w_model[rank * S:(rank + 1) * S], seed=synth.seed_for(rank, 2))
        grad = synth.gradient(D, seed=synth.seed_for(rank, 3), device=dev, dtype=torch.float32)
        out = torch.empty(S, dtype=torch.float32, device=dev)
        ws_q = torch.empty(comm.qwd_workspace_bytes(D, 4, G), dtype=torch.uint8, device=dev)
        ws_t = torch.empty(comm.tlq_workspace_bytes(D, 8, 4, G), dtype=torch.uint8, device=dev)
        fq = lambda: comm.qwd_step(w_main, w_model, ws_q, 4, G)  # noqa: E731
        ft = lambda: comm.tlq_hs_reduce_scatter(grad, out, ws_t, 8, 4, G, b, True)  # noqa: E731
        it = max(a.iters, 50) if mb <= 64 else a.iters
        t_q = timed(fq, it)
        t_t = timed(ft, it)
        big = torch.empty(D, dtype=torch.float32, device=dev)
        shard = torch.empty(S, dtype=torch.float32, device=dev)
        fag = lambda: dist.all_gather_into_tensor(big, shard)  # noqa: E731
        frs = lambda: dist.reduce_scatter_tensor(out, grad, op=dist.ReduceOp.AVG)  # noqa: E731
        t_ag = timed(fag, it)
        t_rs = timed(frs, it)
        row = {"mbytes": mb, "D": D, "qwd_ms": round(t_q, 4), "nccl_all_gather_ms": round(t_ag, 4),
               "ag_speedup": round(t_ag / t_q, 3), "tlq_ms": round(t_t, 4), "nccl_reduce_scatter_ms": round(t_rs, 4),
               "rs_speedup": round(t_rs / t_t, 3)}
        if a.graphs:   # libsdp4's calls captured in CUDA graphs and replayed (the P2P flags carry no
            # epoch); NCCL stays eager (torch's process group hangs at teardown once its
            # collectives have been captured)
            gs = {}
            side = torch.cuda.Stream()
            for name, fn in (("qwd", fq), ("tlq", ft)):
                g = torch.cuda.CUDAGraph()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.graph(g, stream=side):
                    fn()
                torch.cuda.synchronize()
                gs[name] = timed(g.replay, it)
                del g
            row.update({"graph_qwd_ms": round(gs["qwd"], 4), "graph_ag_speedup": round(t_ag / gs["qwd"], 3),
                        "graph_tlq_ms": round(gs["tlq"], 4), "graph_rs_speedup": round(t_rs / gs["tlq"], 3)})
        rows.append(row)
        if rank == 0:
            print(json.dumps(rows[-1]), flush=True)
        del w_model, w_main, grad, out, ws_q, ws_t, big, shard
        torch.cuda.empty_cache()
    if os.environ.get("SDP4_SWEEP_TRACE"):
        print(f"rank {rank}: sweep done, closing", flush=True)
    if rank == 0 and a.out:
        with open(a.out, "w") as f:
            json.dump({"n_gpus": P, "split": f"{M}x{N}", "transport": comm.transport, "G": G, "b": b,
                       "bits": "4/8/4", "rows": rows}, f, indent=1)
    comm.close()
    if os.environ.get("SDP4_SWEEP_TRACE"):
        print(f"rank {rank}: comm closed", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
