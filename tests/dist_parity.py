"""Distributed parity of the full path (run with torchrun, one process per rank).

    torchrun --nproc-per-node P --master-addr 127.0.0.1 tests/dist_parity.py [--groups M]
    torchrun --nproc-per-node P ... tests/dist_parity.py --shared-gpu [--splits all]

Default: one process per GPU, NCCL bootstrap, both transports.  --shared-gpu: every rank on
cuda:0, bootstrapped over a gloo process group (sdp4_comm_init_p2p, no NCCL), so the product
P2P transport -- K1/K2 all-gather pull, K3/K4 all-to-all pushes and pulls, the flag protocol --
runs for any M x N on a single GPU; --splits all checks every M dividing P.  Ranks sharing a
GPU wait with stream memory operations only (no kernel ever waits for another rank).

Every rank draws all P ranks' synthetic inputs (seeded, CPU), runs
  qWD:    sdp4_qwd_quantize + sdp4_qwd_allgather_apply  (ncclAllGather), and sdp4_qwd_step
  TLq-HS: sdp4_tlq_hs_reduce_scatter                     (2 x ncclAlltoAll, intra/inter split)
through the C ABI, and checks against the oracle (bit-exact codes/outputs), plus the
replica identity of w_model across ranks, and the ablation baselines (qW all-gather,
ring reduce-scatter with per-hop quantization).  Prints one PASS/FAIL line per rank.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2410_15526_b200 import Comm, SDP4Error, default_split  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, default=None)
    ap.add_argument("--splits", type=str, default=None, help="'all' or comma-separated M values (virtual mode)")
    ap.add_argument("--G", type=int, default=128)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--chunks", type=str, default="1,3,0", help="NCCL pipeline chunk counts to check (0 = auto)")
    ap.add_argument("--transports", type=str, default="p2p,nccl")
    ap.add_argument("--full", action="store_true", help="GPT-1.3B-sized buffer, sampled windows (bench config)")
    ap.add_argument("--shared-gpu", dest="virtual", action="store_true", help="all ranks on cuda:0, host (gloo) bootstrap, P2P only")
    ap.add_argument("--timeout-test", action="store_true", help="rank 1 skips a call; rank 0 must time out")
    ap.add_argument("--graph", action="store_true", help="also replay CUDA-graph-captured P2P calls")
    ap.add_argument("--wait", type=str, default="kernel", help="P2P waits: kernel (timeout) or memop (unbounded)")
    ap.add_argument("--fused-limit", type=int, default=None, help="timeout test: sdp4_comm_set_fused_limit value")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = 0 if a.virtual else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if a.virtual:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if a.timeout_test:
        ok, msg = run_timeout_test(rank, world, fused_limit=a.fused_limit)
        print(f"rank {rank}/{world} {'PASS' if ok else 'FAIL'} timeout test: {msg}", flush=True)
        dist.barrier()
        dist.destroy_process_group()
        sys.exit(0 if ok else 1)
    if a.virtual and a.full:   # the bench workload at full size on ranks sharing one GPU
        M = int(a.splits or 2)
        comm = Comm.from_process_group(M, bootstrap="host")
        ok, msgs = run_full(comm, rank, world, M, world // M)
        comm.close()
        print(f"rank {rank}/{world} ({M}x{world // M}) {'PASS' if ok else 'FAIL'} full-size shared-GPU "
              f"{'; '.join(msgs)}", flush=True)
        dist.barrier()
        dist.destroy_process_group()
        sys.exit(0 if ok else 1)
    if a.virtual:
        splits = [m for m in range(1, world + 1) if world % m == 0] if a.splits in (None, "all") \
            else [int(x) for x in a.splits.split(",")]
        ok, out = True, []
        for M in splits:
            comm = Comm.from_process_group(M, bootstrap="host")
            try:   # ranks sharing a GPU never wait in a kernel: polling waits are refused
                comm.set_timeout(5.0)
                ok, out = False, out + [f"{M}: set_timeout accepted with ranks sharing a GPU"]
            except SDP4Error:
                pass
            N = world // M
            runs = [("p2p", 0, None), ("p2p", 0, 2 ** 34 + 2410), ("p2p", -1, None), ("p2p", -3, 2410),
                    ("p2p", 2, None), ("p2p", 3, 2411)]
            ok_m, msgs = run_matrix(comm, rank, world, M, N, a.G, a.b, runs, graph=a.graph)
            if world == 8 and M == 2:   # BASELINE.json config 1: 2^20 elements, G 128, b 64, 2 x 4
                comm.set_chunks(0)
                comm.set_intra_pull(1, 2)
                ok_c, m_c = run_checks(comm, rank, world, M, N, 128, 64, (1 << 20) // world, None)
                ok_m &= ok_c
                msgs += [f"config 1 (D = 2^20, 2x4): {m}" for m in m_c] + ["config 1 (D = 2^20, 2x4) checked"]
            comm.close()
            ok &= ok_m
            out.append(f"{M}x{N} {'PASS' if ok_m else 'FAIL'} {'; '.join(msgs)}")
        print(f"rank {rank}/{world} virtual {'PASS' if ok else 'FAIL'} " + " | ".join(out), flush=True)
        dist.barrier()
        dist.destroy_process_group()
        sys.exit(0 if ok else 1)
    M, N = default_split(world, a.groups)
    comm = Comm.from_process_group(a.groups)
    if a.wait == "memop":
        comm.set_timeout(0)
    P, G, b = world, a.G, a.b
    if a.full:
        ok, msgs = run_full(comm, rank, P, M, N)
        comm.close()
        print(f"rank {rank}/{world} ({M}x{N}) {'PASS' if ok else 'FAIL'} full-size {comm.transport} {'; '.join(msgs)}",
              flush=True)
        dist.barrier()
        dist.destroy_process_group()
        sys.exit(0 if ok else 1)
    runs = []
    for tr in a.transports.split(","):
        runs += [(tr, ch, None) for ch in ([int(x) for x in a.chunks.split(",")] if tr == "nccl" else [0])]
        runs.append((tr, 3 if tr == "nccl" else 0, 2 ** 34 + 2410))     # stochastic rounding (R14)
    if "p2p" in a.transports:   # intra all-to-all split between K3 pushes and K4 pulls; chunked P2P
        runs += [("p2p", -1, None), ("p2p", -3, 2410), ("p2p", 2, None), ("p2p", 3, 2411)]
    ok, msgs = run_matrix(comm, rank, P, M, N, G, b, runs, graph=a.graph)
    comm.close()
    print(f"rank {rank}/{world} ({M}x{N}) {'PASS' if ok else 'FAIL'} runs={runs} {'; '.join(msgs)}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


def run_matrix(comm, rank, P, M, N, G, b, runs, graph=False):
    """Every (transport, chunks / push-pull split, seed) run at two shard sizes (several K3
    tiles and a ragged tail), then optionally the CUDA-graph replays."""
    ok, msgs = True, []
    for tr, chunks, seed in runs:
        comm.set_transport(tr)
        comm.set_chunks(max(chunks, 0))
        if tr == "p2p":      # chunks -1: push only; -3: pull 2 of 3 tiles; else the default split
            if chunks in (-1, -3):
                comm.set_intra_pull(*{-1: (0, 1), -3: (2, 3)}[chunks])
            else:
                comm.set_intra_pull(1, 2) if N > 2 else comm.set_intra_pull(0, 1)
        # P2P single-chunk calls run as one kernel per rank below the fused limit (k_fused.cu) and
        # multi-launch above it: both, on the same comm, interleaved call by call
        limits = (0, 1 << 40) if tr == "p2p" and chunks in (0, -1, -3) else (0,)
        for lim in limits:
            comm.set_fused_limit(lim)
            for S in (16384 * 2 + 64 * 5 * max(1, G // 64), 16384 * 12 + 640):
                S -= S % max(G, 64)
                ok_c, m_c = run_checks(comm, rank, P, M, N, G, b, S, seed)
                ok &= ok_c
                msgs += [f"{tr} chunks={chunks} seed={seed} fused={lim > 0} S={S} ({comm.chunks(P * S, G)} used): {m}"
                         for m in m_c]
    if graph and comm.transport == "p2p":
        for lim in (0, 1 << 40):
            comm.set_fused_limit(lim)
            ok_g, m_g = run_graph(comm, rank, P, M, N, G, b)
            ok &= ok_g
            msgs += [f"fused={lim > 0}: {m}" for m in m_g]
    msgs.append(f"{len(runs)} runs x 2 sizes{' + graph replays' if graph else ''}")
    return ok, msgs


def run_graph(comm, rank, P, M, N, G, b, S=16384 * 2 + 640, replays=3):
    """P2P calls captured in CUDA graphs replay correctly (binary flags, no host epoch): the
    TLq-HS reduce-scatter and the qWD step, each replayed on new inputs copied into the
    captured buffers, every replay checked against the oracle."""
    S -= S % max(G, 64)
    D = P * S
    comm.set_chunks(0)
    ok, msgs = True, []
    g_in = torch.empty(D, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(S, dtype=torch.float32, device="cuda")
    w_model = torch.empty(D, dtype=torch.bfloat16, device="cuda")
    w_main = torch.empty(S, dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):   # eager warm-up of the same sizes: no buffer grows in capture
        comm.tlq_hs_reduce_scatter(g_in.zero_(), out, None, 8, 4, G, b, True)
        comm.qwd_step(w_main.zero_(), w_model.zero_(), None, 4, G)
    side.synchronize()
    g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1, stream=side):
        comm.tlq_hs_reduce_scatter(g_in, out, None, 8, 4, G, b, True)
    with torch.cuda.graph(g2, stream=side):
        comm.qwd_step(w_main, w_model, None, 4, G)
    for it in range(replays):
        grads = [synth.gradient(D, seed=synth.seed_for(r, 50 + it), dtype=torch.bfloat16) for r in range(P)]
        g_in.copy_(grads[rank])
        torch.cuda.synchronize()
        g1.replay()
        torch.cuda.synchronize()
        want = oracle.tlq_hs_reduce_scatter([g.float().numpy() for g in grads], oracle.Topology(M, N), G, b, 8, 4,
                                            True).out[rank]
        if not np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32)):
            ok = False
            msgs.append(f"graph replay {it}: TLq-HS differs")
        wm0 = synth.model_weights(D, seed=70 + it)
        mains = [synth.main_weights(wm0[r * S:(r + 1) * S], seed=synth.seed_for(r, 80 + it)) for r in range(P)]
        w_model.copy_(wm0)
        w_main.copy_(mains[rank])
        torch.cuda.synchronize()
        g2.replay()
        torch.cuda.synchronize()
        _, want = oracle.qwd_step([m.numpy() for m in mains], synth.bf16_bits(wm0), 4, G, model_bf16=True)
        if not np.array_equal(synth.bf16_bits(w_model.cpu()), want):
            ok = False
            msgs.append(f"graph replay {it}: qWD replica differs")
    del g1, g2
    comm.check()
    msgs.append(f"{replays} graph replays (TLq-HS, qWD step)")
    return ok, msgs


def run_timeout_test(rank, world, timeout_s=1.0, fused_limit=None):
    """Bounded waits: after one good call on both ranks, rank 1 skips the next collective call.
    Rank 0's flag waits must give up at the deadline (the stream drains, no hang) and the
    following call must return SDP4_ETIMEOUT; rank 1 is unaffected."""
    import time
    from paper_2410_15526_b200 import sdp4
    comm = Comm.from_process_group(1 if world == 2 else None)
    if fused_limit is not None:   # 0: the multi-launch path's wait kernels; else the one-launch kernel's waits
        comm.set_fused_limit(fused_limit)
    P = world
    S = 16384 * 2
    D = P * S
    g = synth.gradient(D, seed=synth.seed_for(rank, 3), dtype=torch.bfloat16).cuda()
    out = torch.empty(S, dtype=torch.float32, device="cuda")
    comm.tlq_hs_reduce_scatter(g, out, None, 8, 4, 128, 64, True)
    torch.cuda.synchronize()
    dist.barrier()
    ok, msg = True, ""
    if rank == 0:
        comm.set_timeout(timeout_s)
        t0 = time.time()
        comm.tlq_hs_reduce_scatter(g, out, None, 8, 4, 128, 64, True)   # rank 1 never joins
        torch.cuda.synchronize()
        el = time.time() - t0
        try:
            comm.tlq_hs_reduce_scatter(g, out, None, 8, 4, 128, 64, True)
            ok, msg = False, "the call after the timed-out one succeeded"
        except SDP4Error as ex:
            ok = ex.status == sdp4.ETIMEOUT
            msg = f"drained in {el:.1f} s (timeout {timeout_s} s per wait); next call: {ex}"
        try:
            comm.check()
            ok = False
        except SDP4Error:
            pass
    else:
        msg = "skipped the call"
    dist.barrier()
    comm.close()
    return ok, msg


def run_full(comm, rank, P, M, N, G=128, b=64, win=16384, nwin=6):
    """bench.py's workload and calls (GPT-1.3B-shaped, bf16 grads/model, G=128, b=64, 4/8/4
    bits); windows of every shard checked against the oracle (groups are position-local)."""
    from paper_2410_15526_b200 import pad_numel
    dev = torch.device("cuda", torch.cuda.current_device())
    D = pad_numel(synth.gpt_numel("1.3B"), P, G)
    S = D // P
    lr = synth.GPT_LR["1.3B"]

    def one_at_a_time(fn):
        """Generate full-size inputs rank by rank: ranks sharing one GPU must not hold their
        generators' fp32 temporaries (~16 GB each) at the same time."""
        res = None
        for turn in range(P):
            if turn == rank:
                res = fn()
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
            dist.barrier()
        return res

    def inputs():
        wm = synth.model_weights(D, seed=synth.seed_for(0, 1), device=dev)
        wmain = synth.main_weights(wm[rank * S:(rank + 1) * S], seed=synth.seed_for(rank, 2), lr=lr)
        g = synth.gradient(D, seed=synth.seed_for(rank, 3), device=dev, dtype=torch.bfloat16)
        return wm, wm.clone(), wmain, g
    w_model, w_model0, w_main, grad = one_at_a_time(inputs)
    p2p = comm.transport == "p2p"   # exchanges through libsdp4's own buffers: no workspace
    ws_q = None if p2p else torch.empty(comm.qwd_workspace_bytes(D, 4, G), dtype=torch.uint8, device=dev)
    ws_t = None if p2p else torch.empty(comm.tlq_workspace_bytes(D, 8, 4, G), dtype=torch.uint8, device=dev)
    out = torch.empty(S, dtype=torch.float32, device=dev)
    comm.qwd_step(w_main, w_model, ws_q, 4, G)   # the call bench.py times
    comm.tlq_hs_reduce_scatter(grad, out, ws_t, 8, 4, G, b, True)
    torch.cuda.synchronize()
    del grad, ws_q, ws_t
    rng = np.random.default_rng(7)
    offs = sorted(set(int(x) * win for x in rng.integers(0, S // win - 1, size=nwin)) | {0, S - win})
    ok, msgs = True, []
    # qWD: replica windows inside every shard j need rank j's main weights
    for j in range(P):
        mj = one_at_a_time(lambda: synth.main_weights(w_model0[j * S:(j + 1) * S], seed=synth.seed_for(j, 2), lr=lr))
        for o in offs[:3] + offs[-1:]:
            e = j * S + o
            _, want = oracle.qwd_step([mj[o:o + win].cpu().numpy()], synth.bf16_bits(w_model0[e:e + win]), 4, G,
                                      model_bf16=True)
            if not np.array_equal(synth.bf16_bits(w_model[e:e + win]), want):
                ok = False
                msgs.append(f"qWD replica window shard {j} +{o}")
        del mj
    # TLq-HS: windows of this rank's output shard need every rank's gradient at shard `rank`
    pieces = {o: [] for o in offs}
    for q in range(P):
        def windows():
            gq = synth.gradient(D, seed=synth.seed_for(q, 3), device=dev, dtype=torch.bfloat16)
            # a P-shard mini problem whose shard j holds the window of shard j (all shards are
            # needed only for the layout; the oracle's output shard `rank` uses column `rank`)
            return {o: torch.cat([gq[j * S + o:j * S + o + win] for j in range(P)]).float().cpu().numpy()
                    for o in offs}
        got_w = one_at_a_time(windows)
        for o in offs:
            pieces[o].append(got_w[o])
    for o in offs:
        tr = oracle.tlq_hs_reduce_scatter(pieces[o], oracle.Topology(M, N), G, b, 8, 4, True)
        got = out[o:o + win].cpu().numpy()
        if not np.array_equal(got.view(np.uint32), tr.out[rank].view(np.uint32)):
            ok = False
            msgs.append(f"TLq-HS output window +{o}: {int((got != tr.out[rank]).sum())} differ")
    msgs.append(f"{len(offs)} windows of {win}")
    return ok, msgs


def run_checks(comm, rank, P, M, N, G, b, S, seed=None):
    D = P * S
    ok = True
    msgs = []

    # ---- qWD (Alg. 2 l.2-5)
    w_model = synth.model_weights(D, seed=1)
    mains = [synth.main_weights(w_model[r * S:(r + 1) * S], seed=synth.seed_for(r, 2)) for r in range(P)]
    p2p = comm.transport == "p2p"      # P2P exchanges through libsdp4's buffers: no workspace
    ws = None if p2p else torch.zeros(comm.qwd_workspace_bytes(D, 4, G), dtype=torch.uint8, device="cuda")
    wm = w_model.cuda()
    comm.qwd_quantize(mains[rank].cuda(), wm, ws, 4, G, seed=seed)
    comm.qwd_allgather_apply(ws, wm, 4, G)
    torch.cuda.synchronize()
    _, want = oracle.qwd_step([m.numpy() for m in mains], synth.bf16_bits(w_model), 4, G, model_bf16=True, seed=seed)
    got = synth.bf16_bits(wm.cpu())
    if not np.array_equal(got, want):
        ok = False
        msgs.append(f"qWD replica differs from oracle in {int(np.sum(got != want))} elements")
    h = torch.tensor([int(np.uint64(np.sum(got.astype(np.uint64) * np.arange(1, D + 1, dtype=np.uint64))) & 0x7FFFFFFF)],
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    hs = [torch.zeros_like(h) for _ in range(P)]
    dist.all_gather(hs, h)
    if len({int(x.item()) for x in hs}) != 1:
        ok = False
        msgs.append("w_model replicas differ across ranks")
    # the same iteration in one call (owner's update fused into K1, K2 skips unit `rank`)
    wm = w_model.cuda()
    comm.qwd_step(mains[rank].cuda(), wm, ws, 4, G, seed=seed)
    torch.cuda.synchronize()
    got = synth.bf16_bits(wm.cpu())
    if not np.array_equal(got, want):
        ok = False
        msgs.append(f"qwd_step replica differs from oracle in {int(np.sum(got != want))} elements")

    # ---- TLq-HS (Alg. 3)
    for dtype in (torch.bfloat16, torch.float32):
        grads = [synth.gradient(D, seed=synth.seed_for(r, 3), dtype=dtype) for r in range(P)]
        tws = None if p2p else torch.zeros(comm.tlq_workspace_bytes(D, 8, 4, G), dtype=torch.uint8, device="cuda")
        out = torch.empty(S, dtype=torch.float32, device="cuda")
        comm.tlq_hs_reduce_scatter(grads[rank].cuda(), out, tws, 8, 4, G, b, True, seed=seed)
        torch.cuda.synchronize()
        tr = oracle.tlq_hs_reduce_scatter([g.float().numpy() for g in grads], oracle.Topology(M, N), G, b, 8, 4, True,
                                          seed=seed)
        o = out.cpu().numpy()
        w = tr.out[rank]
        same = (o.view(np.uint32) == w.view(np.uint32)) | (np.isnan(o) & np.isnan(w))
        if not same.all():
            ok = False
            msgs.append(f"TLq-HS {dtype} out shard: {int((~same).sum())} of {S} elements differ")
    # ---- ablation baselines (NEXT-3): qW all-gather (Alg. 1) and the per-hop-quantized
    # ring reduce-scatter, same transports
    if seed is None:
        ws = torch.zeros(comm.qwd_workspace_bytes(D, 4, G), dtype=torch.uint8, device="cuda")
        wq = torch.empty(D, dtype=torch.bfloat16, device="cuda")
        comm.qw_quantize(mains[rank].cuda(), D, ws, 4, G)
        comm.qw_allgather_apply(ws, wq, 4, G)
        torch.cuda.synchronize()
        _, want = oracle.qw_step([m.numpy() for m in mains], 4, G, model_bf16=True)
        if not np.array_equal(synth.bf16_bits(wq.cpu()), want):
            ok = False
            msgs.append("qW replica differs from oracle")
        grads = [synth.gradient(D, seed=synth.seed_for(r, 4), dtype=torch.bfloat16) for r in range(P)]
        for bits in (4, 32):
            rws = torch.zeros(comm.ring_workspace_bytes(D, bits, G), dtype=torch.uint8, device="cuda")
            out = torch.empty(S, dtype=torch.float32, device="cuda")
            comm.ring_reduce_scatter(grads[rank].cuda(), out, rws, bits, G, True)
            comm.ring_reduce_scatter(grads[rank].cuda(), out, rws, bits, G, True)   # slot reuse across calls
            torch.cuda.synchronize()
            w = oracle.ring_reduce_scatter([g.float().numpy() for g in grads], bits, G, True).out[rank]
            if not np.array_equal(out.cpu().numpy().view(np.uint32), w.view(np.uint32)):
                ok = False
                msgs.append(f"ring k={bits} out shard differs from oracle")
    return ok, msgs


if __name__ == "__main__":
    main()
