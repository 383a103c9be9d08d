"""Multi-process (world_size > 1) host-side tests on CPU with the gloo backend.

The data plan of the NCCL transport -- which bytes go where in the two all-to-alls of
Alg. 3 (routing reading R9) and in the qWD all-gather (Alg. 2 l.4) --
is replayed here with real torch.distributed collectives between processes: messages are
produced by the oracle, placed at the offsets the library's layout API returns
(sdp4_wire_unit_bytes / sdp4_tlq_workspace_offset / sdp4_qwd_workspace_bytes, host
functions of libsdp4.so), exchanged with gloo over the same process groups libsdp4 builds
with ncclCommSplit (intra: color r / N, inter: color r mod N), and checked against the
oracle's single-process simulation.  Also: the ring schedule of the ablation baseline (R18)
with point-to-point send/recv, and bench.py's reference arm under torchrun (rank 0 prints
one line, the other ranks exit 0).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _groups(world, M, N):
    """The two communicator splits of sdp4_comm_init: intra = {mN .. mN+N-1},
    inter = {l, N+l, ..}.  new_group is collective, so every rank creates all of them."""
    intra = [dist.new_group([m * N + q for q in range(N)]) for m in range(M)]
    inter = [dist.new_group([q * N + l for q in range(M)]) for l in range(N)]
    return intra, inter


def _spawn(fn, world, *args):
    mp.spawn(fn, args=(world, _free_port()) + args, nprocs=world, join=True)


# --------------------------------------------------------------------------- TLq-HS plan
def _tlq_worker(rank, world, port, M, N, G, b):
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    from paper_2410_15526_b200 import tlq_workspace_offset, wire_unit_bytes
    _init(rank, world, port)
    try:
        intra, inter = _groups(world, M, N)
        m, l = divmod(rank, N)
        P = world
        D = P * 16384 + P * G * 3
        S = D // P
        grads = [synth.gradient(D, seed=synth.seed_for(r, 3)).numpy() for r in range(P)]
        tr = oracle.tlq_hs_reduce_scatter(grads, oracle.Topology(M, N), G, b, 8, 4, True)
        w8, w4 = wire_unit_bytes(S, 8, G), wire_unit_bytes(S, 4, G)
        off = [tlq_workspace_offset(M, N, D, 8, 4, G, k) for k in range(4)]
        ws = np.zeros(off[0] + N * M * w8, dtype=np.uint8)
        # region 0 intra_send: block l' unit m' = shard m'N + l' of this rank (R9)
        for lp in range(N):
            for mp_ in range(M):
                c, s = tr.intra_send[rank][lp][mp_]
                o = off[0] + (lp * M + mp_) * w8
                ws[o:o + w8] = oracle.wire_unit(c, s, 8, G)
        send = torch.from_numpy(ws[off[0]:off[0] + N * M * w8].copy())
        recv = torch.empty_like(send)
        if N > 1:   # ncclAlltoAll(send8, recv8, M*w8, intra): equal splits in group-rank order
            dist.all_to_all_single(recv, send, group=intra[m])
        else:
            recv = send
        # K4 reads block l'' of intra_recv as the message from local rank l''
        for lpp in range(N):
            for mp_ in range(M):
                c, s = tr.intra_send[m * N + lpp][l][mp_]
                got = recv[(lpp * M + mp_) * w8:(lpp * M + mp_ + 1) * w8].numpy()
                assert np.array_equal(got, oracle.wire_unit(c, s, 8, G)), (rank, lpp, mp_)
        # region 2 inter_send: unit m' = shard m'N + l (after K4's reduce + requantize)
        send4 = torch.from_numpy(np.concatenate([oracle.wire_unit(*tr.inter_send[rank][q], 4, G) for q in range(M)]))
        recv4 = torch.empty_like(send4)
        if M > 1:   # ncclAlltoAll(send4, recv4, w4, inter)
            dist.all_to_all_single(recv4, send4, group=inter[l])
        else:
            recv4 = send4
        # K5 reads unit m'' of inter_recv as the message from group m''; decoding and reducing
        # them in order m'' = 0..M-1 is exactly the oracle's output shard `rank`
        for mpp in range(M):
            c, s = tr.inter_send[mpp * N + l][m]
            assert np.array_equal(recv4[mpp * w4:(mpp + 1) * w4].numpy(), oracle.wire_unit(c, s, 4, G)), (rank, mpp)
        assert off[1] == (0 if N == 1 else N * M * w8) and off[2] == off[1] + N * M * w8
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M,N", [(2, 1, 2), (2, 2, 1), (4, 2, 2), (4, 1, 4), (4, 4, 1)])
def test_tlq_exchange_plan_gloo(world, M, N):
    _spawn(_tlq_worker, world, M, N, 128, 64)


# ------------------------------------------------------------------------- qWD all-gather
def _qwd_worker(rank, world, port, G):
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    from paper_2410_15526_b200 import qwd_workspace_bytes, wire_unit_bytes
    _init(rank, world, port)
    try:
        P = world
        D = P * G * 40
        S = D // P
        w_model = synth.model_weights(D, seed=1)
        wbits = synth.bf16_bits(w_model)
        mains = [synth.main_weights(w_model[r * S:(r + 1) * S], seed=synth.seed_for(r, 2)).numpy() for r in range(P)]
        W = wire_unit_bytes(S, 4, G)
        assert qwd_workspace_bytes(P, D, 4, G) >= P * W
        c, s, _ = oracle.qwd_quantize(mains[rank], oracle.bf16_widen(wbits)[rank * S:(rank + 1) * S], 4, G)
        mine = torch.from_numpy(oracle.wire_unit(c, s, 4, G))
        # in-place all-gather: unit r at r * W (ncclAllGather on the world comm)
        gathered = torch.empty(P * W, dtype=torch.uint8)
        dist.all_gather_into_tensor(gathered, mine)
        units = [oracle.wire_unit_decode(gathered[r * W:(r + 1) * W].numpy(), S, 4, G) for r in range(P)]
        new = oracle.qwd_allgather_apply(units, oracle.bf16_widen(wbits), 4, G, model_bf16=True)
        _, want = oracle.qwd_step(mains, wbits, 4, G, model_bf16=True)
        assert np.array_equal(new, want)
        # replicas identical across ranks
        h = torch.tensor([int(np.sum(new.astype(np.int64) * np.arange(1, D + 1)) % (2 ** 61 - 1))])
        hs = [torch.zeros_like(h) for _ in range(P)]
        dist.all_gather(hs, h)
        assert len({int(x) for x in hs}) == 1
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_qwd_allgather_plan_gloo(world):
    _spawn(_qwd_worker, world, 128)


# --------------------------------------------------------------------------- ring (R18)
def _ring_worker(rank, world, port, k, G):
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    _init(rank, world, port)
    try:
        P = world
        D = P * G * 12
        S = D // P
        grads = [synth.gradient(D, seed=synth.seed_for(r, 4)).numpy() for r in range(P)]
        g = grads[rank]
        nxt, prv = (rank + 1) % P, (rank - 1) % P
        acc = None
        for t in range(P - 1):   # hop t: forward chunk (r - t - 1) mod P
            c = (rank - t - 1) % P
            part = g[c * S:(c + 1) * S] if t == 0 else (acc + g[c * S:(c + 1) * S]).astype(np.float32)
            codes, scales = oracle.quantize(part, k, G)
            msg = torch.from_numpy(oracle.wire_unit(codes, scales, k, G))
            buf = torch.empty_like(msg)
            reqs = [dist.isend(msg, nxt), dist.irecv(buf, prv)]
            for q in reqs:
                q.wait()
            acc = oracle.dequantize(*oracle.wire_unit_decode(buf.numpy(), S, k, G), k, G)
        out = (acc + g[rank * S:(rank + 1) * S]).astype(np.float32) if P > 1 else g[:S].copy()
        out = (out * np.float32(np.float32(1.0) / np.float32(P))).astype(np.float32)
        want = oracle.ring_reduce_scatter(grads, k, G, True).out[rank]
        assert np.array_equal(out.view(np.uint32), want.view(np.uint32))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 4), (3, 8), (4, 4)])
def test_ring_schedule_gloo(world, k):
    _spawn(_ring_worker, world, k, 128)


# ------------------------------------------------------------------ bench reference arm
def test_reference_arm_under_torchrun():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "1", "--cpu-seconds", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
