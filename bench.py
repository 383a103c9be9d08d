#!/usr/bin/env python
"""bench.py -- SDP4Bit hot path: qWD all-gather + TLq-HS reduce-scatter, GB/s of pre-quant bytes.

One step = one pass of the whole hot path over one synthetic GPT-shaped buffer:
  qWD   sdp4_qwd_step (= sdp4_qwd_quantize + sdp4_qwd_allgather_apply, owner's update in K1;
        Alg. 2 l.2-5; --qwd-two-call times the two calls instead)
  TLq-HS sdp4_tlq_hs_reduce_scatter                     (Alg. 3)
Pre-quant bytes per rank per step = D*4 (the fp32 weight-difference buffer gathered) +
D*g (the gradient reduce-scattered, g = 2 for bf16); `value` sums them over all ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sdp4|reference] [--model 1.3B]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "qWD all-gather + TLq-HS reduce-scatter GB/s (pre-quant bytes) at 1/2/4/8 B200"
SMI_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="sdp4", choices=["sdp4", "reference"])
    p.add_argument("--model", default="1.3B", help="GPT shape of the flat buffer (tab:model_size_params)")
    p.add_argument("--numel", type=int, default=0, help="override D (message-size sweeps)")
    p.add_argument("--groups", type=int, default=None, help="M (default: 2 groups when N is even)")
    p.add_argument("--group", type=int, default=128, help="G of TLq-HS (P:689)")
    p.add_argument("--qwd-group", type=int, default=128, help="G of qWD (BASELINE config G; paper uses 2048)")
    p.add_argument("--hadamard", type=int, default=64, help="Hadamard block b (BASELINE config 1)")
    p.add_argument("--bits-intra", type=int, default=8)
    p.add_argument("--bits-inter", type=int, default=4)
    p.add_argument("--bits-w", type=int, default=4)
    p.add_argument("--grad-dtype", default="bf16", choices=["bf16", "fp32"])
    p.add_argument("--model-dtype", default="bf16", choices=["bf16", "fp32"])
    p.add_argument("--chunks", type=int, default=0, help="pipeline chunks (0 = library default, 1 = off)")
    p.add_argument("--nccl-ctas", type=int, default=0, help="SMs left to NCCL while pipelining (0 = default)")
    p.add_argument("--transport", default="auto", choices=["auto", "p2p", "nccl"],
                   help="exchange transport (auto = fused P2P push when available)")
    p.add_argument("--qwd-two-call", action="store_true",
                   help="qWD as sdp4_qwd_quantize + sdp4_qwd_allgather_apply (K2 applies every unit)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-comparators", action="store_true")
    p.add_argument("--intra-pull", type=str, default=None,
                   help="P2P: num/den of the intra all-to-all pulled by K4 (default: the library's auto split)")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the oracle timing")
    p.add_argument("--steps-only", action="store_true",
                   help="only the warm-up and the K timed steps (for an ncu launch list of exactly those)")
    p.add_argument("--no-variants", action="store_true", help="skip the fp32-gradient step variant")
    p.add_argument("--overlap", action="store_true",
                   help="issue the qWD step on a second stream, concurrent with TLq-HS (experiment)")
    return p.parse_args()


# ----------------------------------------------------------------------------- helpers
def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={SMI_FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[3]) for r in self.rows if r[3].replace(".", "").isdigit()), default=None)}


def kernel_bytes(name, D, S, P, M, N, a):
    """Algorithmic HBM bytes per launch of each kernel."""
    g = 2 if a.grad_dtype == "bf16" else 4
    m = 2 if a.model_dtype == "bf16" else 4

    def wire(n, k, G):
        return n * k / 8 + (4 * n / G if k != 32 else 0)
    own = 0 if a.qwd_two_call else 1          # sdp4_qwd_step: K1 applies the owner's unit
    if name.startswith("K1"):
        return S * (4 + m) + wire(S, a.bits_w, a.qwd_group) + own * S * m
    if name.startswith("K2"):
        return wire(D - own * S, a.bits_w, a.qwd_group) + 2 * m * (D - own * S)
    if name.startswith("K345"):                 # world 1: K3 -> K4 -> K5 in one kernel (k_local.cu)
        return D * g + 4 * S
    if name.startswith("K34"):                  # N = 1: K3 + K4 in one kernel (k_local34.cu)
        return D * g + wire(D, a.bits_inter, a.group)
    if name.startswith("K3"):
        return D * g + wire(D, a.bits_intra, a.group)
    if name.startswith("K4"):
        return wire(D, a.bits_intra, a.group) + wire(D // N, a.bits_inter, a.group)
    if name.startswith("K5"):
        return wire(M * S, a.bits_inter, a.group) + 4 * S
    return None


NVLINK_PEAK_GBS = 770.0  # B200_PROFILING.md: measured peer copy, per direction per GPU (900 nominal)


def kernel_nvlink_bytes(name, D, S, P, M, N, a, transport):
    """Bytes a fused kernel moves over NVLink per launch (P2P transport; the larger of this
    rank's egress and ingress): K2 pulls the P-1 peer units of the qWD all-gather, K3 pushes
    the N-1 peer blocks of the intra all-to-all, K4 the M-1 peer units of the inter one."""
    if transport != "p2p" or P == 1:
        return 0

    def wire(n, k, G):
        return n * k / 8 + (4 * n / G if k != 32 else 0)
    if name.startswith("K2"):
        return (P - 1) * wire(S, a.bits_w, a.qwd_group)
    num, den = [int(x) for x in (a.intra_pull or ("0/1" if N <= 2 else "1/2")).split("/")]   # library default
    f = num / den if N > 1 else 0.0                      # share of intra tiles K4 pulls
    intra = (N - 1) * M * wire(S, a.bits_intra, a.group)
    if name.startswith("K34"):                           # N = 1: the inter units it pushes
        return (M - 1) * wire(S, a.bits_inter, a.group)
    if name.startswith("K3"):                            # pushed intra tiles (egress)
        return (1 - f) * intra
    if name.startswith("K4"):                            # max(pulled intra ingress, inter egress)
        return max(f * intra, (M - 1) * wire(S, a.bits_inter, a.group))
    return 0


def ncu_traffic(kernel, workload):
    """dram read+write bytes per launch from the committed ncu summary, if it matches."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        if d.get("workload") == workload and kernel in d.get("kernels", {}):
            return d["kernels"][kernel]
    except Exception:
        pass
    return None


# ------------------------------------------------------------------- oracle (CPU) legs
def _oracle_window(args):
    """Worker: one oracle step (qWD + TLq-HS at P=1) on a window of the workload, repeated for
    `seconds`; returns (elements processed, seconds).  Imports only numpy and the oracle."""
    w_main, wm, grad, cfg, seconds = args
    import oracle
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.qwd_step([w_main], wm, cfg["bits_w"], cfg["qwd_group"], model_bf16=cfg["model_bf16"])
        oracle.tlq_hs_reduce_scatter([grad], oracle.Topology(1, 1), cfg["group"], cfg["hadamard"], cfg["bits_intra"],
                                     cfg["bits_inter"], True)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            return reps * grad.size, el


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample_rate(a, seconds: float, D_full: int, cores: int = 1):
    """Time the oracle (as it stands) on a bounded sample of the workload: the full step
    (qWD at P=1 + TLq-HS at P=1) on `cores` independent 2M-element windows of the workload,
    one per worker process (numpy is single-threaded per process), each repeated for
    `seconds`.  Returns (GB/s of pre-quant bytes summed over the workers, description, cores)."""
    import torch

    import synth
    n = min(D_full, 1 << 21)
    n -= n % max(a.group, a.qwd_group, 64)
    g = 2 if a.grad_dtype == "bf16" else 4
    gdt = torch.bfloat16 if a.grad_dtype == "bf16" else torch.float32
    mdt = torch.bfloat16 if a.model_dtype == "bf16" else torch.float32
    w_model = synth.model_weights(n, seed=synth.seed_for(0, 1), dtype=mdt)
    w_main = synth.main_weights(w_model, seed=synth.seed_for(0, 2), lr=synth.GPT_LR.get(a.model, 2e-4)).numpy()
    grad = synth.gradient(n, seed=synth.seed_for(0, 3), dtype=gdt).float().numpy()
    wm = synth.bf16_bits(w_model) if mdt == torch.bfloat16 else w_model.numpy()
    cfg = {"bits_w": a.bits_w, "qwd_group": a.qwd_group, "model_bf16": mdt == torch.bfloat16, "group": a.group,
           "hadamard": a.hadamard, "bits_intra": a.bits_intra, "bits_inter": a.bits_inter}
    jobs = [(w_main, wm, grad, cfg, seconds)] * cores
    if cores == 1:
        res = [_oracle_window(jobs[0])]
    else:
        import multiprocessing as mp
        with mp.get_context("spawn").Pool(cores) as pool:
            res = pool.map(_oracle_window, jobs)
    elems = sum(r[0] for r in res)
    el = max(r[1] for r in res)
    rate = elems * (4 + g) / el / 1e9
    desc = (f"{elems // n} oracle steps (qWD + TLq-HS, P=1) on {cores} x {n}-element windows of the workload "
            f"({cores} worker process{'es' if cores > 1 else ''}, single-threaded numpy fp32 each), {el:.1f} s")
    return rate, desc, cores


def run_reference(a, rank, world):
    """--impl reference: the oracle on the host cores, rank 0 only."""
    if rank != 0:
        return
    import synth
    D = a.numel or synth.gpt_numel(a.model)
    per = max(1.0, a.cpu_seconds / max(1, a.steps))
    cores = min(os.cpu_count() or 1, 64)
    rates = []
    for _ in range(a.warmup):
        oracle_sample_rate(a, 0.1, D)
    desc = ""
    for _ in range(a.steps):
        r, desc, cores = oracle_sample_rate(a, per, D, cores)
        rates.append(r)
    v = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"GPT-{a.model}-shaped flat buffer (bounded CPU sample)", "D": D},
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": cores, "cpu_model": cpu_model(),
                             "kind": "oracle", "sample": desc},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    emit(line)


# --------------------------------------------------------------------------- GPU arm
def run_sdp4(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2410_15526_b200 import Comm, default_split, pad_numel

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    M, N = default_split(world, a.groups)
    P = world
    D0 = a.numel or synth.gpt_numel(a.model)
    D = pad_numel(D0, P, max(a.group, a.qwd_group))
    S = D // P
    gdt = torch.bfloat16 if a.grad_dtype == "bf16" else torch.float32
    mdt = torch.bfloat16 if a.model_dtype == "bf16" else torch.float32
    g_bytes = 2 if gdt == torch.bfloat16 else 4

    comm = Comm.from_process_group(a.groups, dev, a.nccl_ctas, a.chunks) if world > 1 else Comm()
    if world > 1 and a.transport != "auto":
        comm.set_transport(a.transport)
    if a.intra_pull:
        comm.set_intra_pull(*[int(x) for x in a.intra_pull.split("/")])
    lr = synth.GPT_LR.get(a.model, 2e-4)
    # synthetic inputs: w_model identical on all ranks, w_main shard r, grad per rank
    w_model = synth.model_weights(D, seed=synth.seed_for(0, 1), device=dev, dtype=mdt)
    w_main = synth.main_weights(w_model[rank * S:(rank + 1) * S], seed=synth.seed_for(rank, 2), lr=lr)
    grad = synth.gradient(D, seed=synth.seed_for(rank, 3), device=dev, dtype=gdt)
    out = torch.empty(S, dtype=torch.float32, device=dev)
    local_fused = P == 1 and a.bits_intra == 8 and a.bits_inter == 4   # world 1: K345, no TLq workspace
    if comm.transport == "p2p":   # exchanges through libsdp4's own symmetric buffers
        ws_q = ws_t = None
    else:
        ws_q = torch.empty(comm.qwd_workspace_bytes(D, a.bits_w, a.qwd_group), dtype=torch.uint8, device=dev)
        ws_t = None if local_fused else torch.empty(comm.tlq_workspace_bytes(D, a.bits_intra, a.bits_inter, a.group),
                                                    dtype=torch.uint8, device=dev)
    # the three-kernel variant's TLq-HS workspace (world 1), allocated with the inputs -- not
    # after the other measurements have fragmented the allocator -- when it fits
    ws3_bytes = comm.tlq_workspace_bytes(D, a.bits_intra, a.bits_inter, a.group)
    ws3 = None
    if local_fused and not a.no_variants and torch.cuda.mem_get_info(dev)[0] > ws3_bytes + (8 << 30):
        ws3 = torch.empty(ws3_bytes, dtype=torch.uint8, device=dev)

    def qwd(wmain):
        if a.qwd_two_call:
            comm.qwd_quantize(wmain, w_model, ws_q, a.bits_w, a.qwd_group)
            comm.qwd_allgather_apply(ws_q, w_model, a.bits_w, a.qwd_group)
        else:
            comm.qwd_step(wmain, w_model, ws_q, a.bits_w, a.qwd_group)

    s_q = torch.cuda.Stream() if a.overlap else None
    ev_fork, ev_join = torch.cuda.Event(), torch.cuda.Event()

    def step():
        if s_q is None:
            qwd(w_main)
            comm.tlq_hs_reduce_scatter(grad, out, ws_t, a.bits_intra, a.bits_inter, a.group, a.hadamard, True)
            return
        # the two collectives are independent: qWD on a second stream, joined at the end
        ev_fork.record()
        with torch.cuda.stream(s_q):
            s_q.wait_event(ev_fork)
            qwd(w_main)
            ev_join.record()
        comm.tlq_hs_reduce_scatter(grad, out, ws_t, a.bits_intra, a.bits_inter, a.group, a.hadamard, True)
        torch.cuda.current_stream().wait_event(ev_join)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps, warm=0):
        for _ in range(warm):   # comparators: first-call setup (NCCL channels, symmetric buffers) untimed
            fn()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / steps)

    for _ in range(max(3, a.warmup)):
        step()
    # headline: K steps, no instrumentation, clocks sampled during the region
    comm.launch_count(reset=True)
    with ClockSampler(local_rank) as clk:
        ms = timed(step, a.steps)
    launches = comm.launch_count(reset=True)
    pre_bytes_rank = D * (4 + g_bytes)
    value = P * pre_bytes_rank / (ms * 1e-3) / 1e9
    if a.steps_only:   # the launch list of exactly the warm-up + timed steps (ncu), nothing else
        if rank == 0:
            emit({"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": a.steps,
                  "warmup": max(3, a.warmup), "ms_per_step": round(ms, 4), "higher_is_better": True,
                  "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                  "config": {"workload": f"GPT-{a.model} D={D} P={P} ({M}x{N})", "steps_only": True},
                  "gpu_launches": int(launches), "clocks": clk.summary()})
        comm.close()
        return
    # per-kernel device times: the same K steps again with every launch bracketed by events
    comm.profile_enable(True)
    comm.profile_read()
    ms_prof = timed(step, a.steps)
    prof = comm.profile_read()
    comm.profile_enable(False)
    if os.environ.get("SDP4_BENCH_RANKS"):   # diagnostics: every rank's per-kernel / wait times
        print(f"rank {rank}: " + ", ".join(f"{n} {t / a.steps:.3f}" for n, (t, c) in sorted(prof.items())),
              file=sys.stderr, flush=True)

    # roofline for the dominant kernel (largest summed device time in the timed region)
    workload = f"GPT-{a.model} D={D} P={P} ({M}x{N}) G={a.group} Gw={a.qwd_group} b={a.hadamard} " \
               f"bits={a.bits_w}/{a.bits_intra}/{a.bits_inter} grad={a.grad_dtype} model={a.model_dtype}"
    peak, peak_src = peaks()
    kern = {}
    transport = comm.transport if world > 1 else "local"
    for name, (tms, cnt) in prof.items():
        if name.startswith("nccl_") or name.startswith("wait_"):
            continue
        per_step = max(1, round(cnt / a.steps))          # launches per step (pipeline chunks)
        kb = kernel_bytes(name, D, S, P, M, N, a) / per_step   # algorithmic bytes per launch
        nb = kernel_nvlink_bytes(name, D, S, P, M, N, a, transport) / per_step
        avg = tms / max(cnt, 1)
        kern[name] = {"avg_ms": round(avg, 4), "launches": cnt, "share": None,
                      "alg_bytes": kb, "gbs": round(kb / (avg * 1e-3) / 1e9, 1) if kb and avg > 0 else None}
        if nb:
            kern[name]["nvlink_bytes"] = nb
            kern[name]["nvlink_gbs"] = round(nb / (avg * 1e-3) / 1e9, 1)
    comm_ops = {n: {"ms_per_step": round(t / a.steps, 4), "calls": c} for n, (t, c) in prof.items()
                if n.startswith("nccl_") or n.startswith("wait_")}
    tot = sum(v["avg_ms"] * v["launches"] for v in kern.values()) or 1.0
    for v in kern.values():
        v["share_of_kernel_time"] = round(v["avg_ms"] * v["launches"] / tot, 4)
        v.pop("share")
    dom = max(kern, key=lambda k: kern[k]["avg_ms"] * kern[k]["launches"]) if kern else None
    roofline = None
    if dom:
        ach = kern[dom]["gbs"]
        tr = ncu_traffic(dom, workload)
        roofline = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4) if ach else None, "traffic": tr,
                    "alg_bytes_per_launch": kern[dom]["alg_bytes"], "peak_source": peak_src}
        nv = kern[dom].get("nvlink_gbs")
        if nv and nv / NVLINK_PEAK_GBS > (ach or 0) / peak:
            # the fused kernel is bound by its NVLink traffic, not by HBM
            roofline.update({"bound": "nvlink", "achieved": nv, "peak": NVLINK_PEAK_GBS,
                             "frac": round(nv / NVLINK_PEAK_GBS, 4), "traffic": None,
                             "alg_bytes_per_launch": kern[dom]["nvlink_bytes"],
                             "hbm_frac": round(ach / peak, 4) if ach else None,
                             "peak_source": "B200_PROFILING.md measured peer copy per direction (fallback)"})

    # each collective alone (K steps each): effective pre-quantization GB/s and, with the P2P
    # transport, the NVLink bytes this rank moves against the 900 GB/s per-direction NVLink 5
    # figure the north star names (the fused kernels are the collectives: no NCCL kernel runs)
    t_qwd = timed(lambda: qwd(w_main), a.steps)
    t_tlq = timed(lambda: comm.tlq_hs_reduce_scatter(grad, out, ws_t, a.bits_intra, a.bits_inter, a.group,
                                                     a.hadamard, True), a.steps)
    nv_q = kernel_nvlink_bytes("K2", D, S, P, M, N, a, transport)
    def wire_b(n, k, G):
        return n * k / 8 + (4 * n / G if k != 32 else 0)
    # per-direction NVLink bytes of one TLq-HS call: intra (N-1) blocks + inter (M-1) units
    nv_t = ((N - 1) * M * wire_b(S, a.bits_intra, a.group) + (M - 1) * wire_b(S, a.bits_inter, a.group)
            if transport == "p2p" else 0)
    collectives = {}
    for name, t, pre, nv in (("qwd_all_gather", t_qwd, D * 4, nv_q), ("tlq_hs_reduce_scatter", t_tlq, D * g_bytes, nv_t)):
        collectives[name] = {"ms": round(t, 4), "pre_quant_GBps": round(P * pre / (t * 1e-3) / 1e9, 1),
                             "nvlink_bytes_per_rank": int(nv),
                             "nvlink_GBps": round(nv / (t * 1e-3) / 1e9, 1) if nv else None,
                             "nvlink_frac_of_900": round(nv / (t * 1e-3) / 900e9, 4) if nv else None}

    variants = None
    if ws3 is not None and "K345_tlq_local" in prof:
        # the same step through the three kernels K3 -> K4 -> K5 (what every rank of a P > 1 job
        # runs), with each kernel's roofline; they need the TLq-HS workspace K345 does without
        comm.set_local_fusion(False)
        for _ in range(2):
            qwd(w_main)
            comm.tlq_hs_reduce_scatter(grad, out, ws3, a.bits_intra, a.bits_inter, a.group, a.hadamard, True)

        def step3():
            qwd(w_main)
            comm.tlq_hs_reduce_scatter(grad, out, ws3, a.bits_intra, a.bits_inter, a.group, a.hadamard, True)
        ms3 = timed(step3, a.steps)
        comm.profile_enable(True)
        comm.profile_read()
        timed(step3, a.steps)
        prof3 = comm.profile_read()
        comm.profile_enable(False)
        comm.set_local_fusion(True)
        k3k = {}
        for n, (tt, cc) in prof3.items():
            if n.startswith("K3") or n.startswith("K4") or n.startswith("K5"):
                avg = tt / max(1, cc)
                kb = kernel_bytes(n, D, S, P, M, N, a)
                k3k[n] = {"avg_ms": round(avg, 4), "gbs": round(kb / (avg * 1e-3) / 1e9, 1),
                          "frac_of_peak": round(kb / (avg * 1e-3) / 1e9 / peak, 4)}
        variants = dict(variants or {})
        variants["three_kernel_tlq"] = {"ms_per_step": round(ms3, 4),
                                        "value": round(P * pre_bytes_rank / (ms3 * 1e-3) / 1e9, 2),
                                        "unit": "GB/s", "kernels": k3k}
    ws3 = None
    torch.cuda.empty_cache()

    # the paper's FP32-gradient setting: the same step with fp32 gradients
    t_tlq32 = None
    if not a.no_variants and gdt == torch.bfloat16:
        g32 = grad.float()

        def step32():
            qwd(w_main)
            comm.tlq_hs_reduce_scatter(g32, out, ws_t, a.bits_intra, a.bits_inter, a.group, a.hadamard, True)
        for _ in range(2):
            step32()
        ms32 = timed(step32, a.steps)
        comm.profile_enable(True)
        comm.profile_read()
        timed(step32, a.steps)
        prof32 = comm.profile_read()
        comm.profile_enable(False)
        t_tlq32 = timed(lambda: comm.tlq_hs_reduce_scatter(g32, out, ws_t, a.bits_intra, a.bits_inter, a.group,
                                                           a.hadamard, True), a.steps)
        a32 = argparse.Namespace(**dict(vars(a), grad_dtype="fp32"))
        # the kernel that reads the gradient: K3, or at world 1 the fused K345
        tk = "K345_tlq_local" if "K345_tlq_local" in prof32 else "K3_tlq_had_quant"
        k_t, k_c = prof32.get(tk, (0.0, 0))
        k_ms = k_t / max(1, k_c)
        k_bytes = kernel_bytes(tk, D, S, P, M, N, a32)
        variants = dict(variants or {})
        variants["fp32_grad"] = {"ms_per_step": round(ms32, 4),
                                  "value": round(P * D * (4 + 4) / (ms32 * 1e-3) / 1e9, 2), "unit": "GB/s",
                                  "tlq_hs_reduce_scatter_ms": round(t_tlq32, 4),
                                  "grad_kernel": tk, "grad_kernel_avg_ms": round(k_ms, 4),
                                  "grad_kernel_gbs": round(k_bytes / (k_ms * 1e-3) / 1e9, 1) if k_ms else None,
                                  "grad_kernel_frac_of_peak":
                                      round(k_bytes / (k_ms * 1e-3) / 1e9 / peak, 4) if k_ms else None}
        del g32
    # ablation (NEXT-3): TLq-HS with the Hadamard transforms as separate passes ("SDP4Bit (HS
    # w/o fused)") -- K3 identity codec forward pass, the b = 0 reduce-scatter, K5
    # identity codec inverse pass -- against the fused path
    ablation = None
    if not a.no_comparators and a.hadamard > 0:
        from paper_2410_15526_b200 import tlq_stage_final, tlq_stage_quantize
        hbuf = torch.empty(D, dtype=torch.float32, device=dev)
        red = torch.empty(S, dtype=torch.float32, device=dev)
        out2 = torch.empty(S, dtype=torch.float32, device=dev)

        def unfused():
            tlq_stage_quantize(grad, hbuf.view(torch.uint8), 1, 1, 32, a.group, a.hadamard)
            comm.tlq_hs_reduce_scatter(hbuf, red, ws_t, a.bits_intra, a.bits_inter, a.group, 0, True)
            tlq_stage_final(red.view(torch.uint8), out2, S, 1, 1, 32, a.group, a.hadamard, False)
        t_unf = timed(unfused, max(3, a.steps // 2), 2)
        ablation = {"tlq_hs_fused_ms": round(t_tlq, 4), "tlq_hs_unfused_hadamard_ms": round(t_unf, 4),
                    "fusion_speedup": round(t_unf / t_tlq, 3)}
    if not a.no_comparators:   # qWD as two calls (K2 applies every unit, the owner's included)
        def qwd_two():
            comm.qwd_quantize(w_main, w_model, ws_q, a.bits_w, a.qwd_group)
            comm.qwd_allgather_apply(ws_q, w_model, a.bits_w, a.qwd_group)
        t_two = timed(qwd_two, a.steps, 1)
        ablation = dict(ablation or {}, qwd_step_ms=round(t_qwd, 4), qwd_two_call_ms=round(t_two, 4),
                        qwd_own_fusion_speedup=round(t_two / t_qwd, 3))
        del hbuf, red, out2

    # unquantized NCCL comparators (sec. 2.1), N > 1 only, torch.distributed's own NCCL
    # communicator (default configuration).  Like for like: qWD against the bf16 all-gather of
    # the model weights it replaces, TLq-HS against a reduce-scatter of the SAME gradient dtype
    # (bf16 and, for the paper's FP32-gradient setting P:502, fp32); plus the "same buffers"
    # pair SURVEY sec. 8(d) names (fp32 weight-difference all-gather + gradient reduce-scatter).
    comparators = None
    if world > 1 and not a.no_comparators:
        reps = max(3, a.steps // 2)
        big = torch.empty(D, dtype=torch.float32, device=dev)
        d_shard = torch.empty(S, dtype=torch.float32, device=dev)
        t_ag32 = timed(lambda: dist.all_gather_into_tensor(big, d_shard), reps, 2)
        w_shard16 = torch.empty(S, dtype=torch.bfloat16, device=dev)
        big16 = big.view(torch.bfloat16)[:D]
        t_ag16 = timed(lambda: dist.all_gather_into_tensor(big16, w_shard16), reps, 2)
        del big16, w_shard16, big, d_shard
        g16 = grad if gdt == torch.bfloat16 else grad.bfloat16()
        rs16 = torch.empty(S, dtype=torch.bfloat16, device=dev)
        t_rs16 = timed(lambda: dist.reduce_scatter_tensor(rs16, g16, op=dist.ReduceOp.AVG), reps, 2)
        del g16, rs16
        g32 = grad.float() if gdt != torch.float32 else grad
        rs32 = torch.empty(S, dtype=torch.float32, device=dev)
        t_rs32 = timed(lambda: dist.reduce_scatter_tensor(rs32, g32, op=dist.ReduceOp.AVG), reps, 2)
        del g32, rs32
        t_rs_grad = t_rs16 if gdt == torch.bfloat16 else t_rs32
        # ablation baselines through libsdp4 (NEXT-3): 4-bit ring reduce-scatter with per-hop
        # quantization
        ws_r = None if comm.transport == "p2p" else torch.empty(comm.ring_workspace_bytes(D, a.bits_inter, a.group),
                                                                 dtype=torch.uint8, device=dev)
        t_ring = timed(lambda: comm.ring_reduce_scatter(grad, out, ws_r, a.bits_inter, a.group, True), reps, 2)
        del ws_r
        ms32 = variants["fp32_grad"]["ms_per_step"] if variants else None
        comparators = {
            "nccl_ms": {"all_gather_bf16_weights": round(t_ag16, 3), "all_gather_fp32_weight_diff": round(t_ag32, 3),
                        "reduce_scatter_bf16": round(t_rs16, 3), "reduce_scatter_fp32": round(t_rs32, 3)},
            "like_for_like": {
                "qwd_vs_all_gather_bf16_weights": round(t_ag16 / t_qwd, 3),
                f"tlq_hs_vs_reduce_scatter_{a.grad_dtype}": round(t_rs_grad / t_tlq, 3),
                "tlq_hs_vs_reduce_scatter_fp32": round(t_rs32 / t_tlq32, 3) if t_tlq32 else None,
                f"step_vs_pair_bf16_weights_{a.grad_dtype}_grads": round((t_ag16 + t_rs_grad) / ms, 3),
                "step_vs_pair_bf16_weights_fp32_grads (Megatron, P:502)":
                    round((t_ag16 + t_rs32) / ms32, 3) if ms32 else None},
            "same_buffers (SURVEY 8(d): fp32 weight-difference all-gather + gradient reduce-scatter)": {
                "unquantized_ms_per_step": round(t_ag32 + t_rs_grad, 3),
                "unquantized_GBps": round(P * pre_bytes_rank / ((t_ag32 + t_rs_grad) * 1e-3) / 1e9, 2),
                "speedup": round((t_ag32 + t_rs_grad) / ms, 3)},
            f"ring_q{a.bits_inter}_reduce_scatter_ms": round(t_ring, 3)}

    # end to end through the public API with host buffers (pinned), copies inside the region.
    # Pipelined like a data loader: step i+1's inputs are copied host->device on one stream
    # while step i computes and its output shard is read back on another (double-buffered
    # device inputs/outputs), so PCIe runs both directions at once.  Every step's copies are
    # inside the timed region.
    e2e = None
    if not a.no_e2e:
        h_grad = grad.cpu().pin_memory()
        h_main = w_main.cpu().pin_memory()
        h_out = torch.empty(S, dtype=torch.float32).pin_memory()
        del grad
        torch.cuda.empty_cache()
        comp = torch.cuda.current_stream()
        # each direction's copies are split over 4 streams: with H2D and D2H in flight together,
        # one copy per direction gets ~28 GB/s each way on this PCIe link, four ~41 GB/s
        # (tools/pcie_probe.py)
        NS = 4
        s_ins = [torch.cuda.Stream() for _ in range(NS)]
        s_outs = [torch.cuda.Stream() for _ in range(NS)]
        gd = [torch.empty_like(h_grad, device=dev) for _ in range(2)]
        wmn = [torch.empty_like(h_main, device=dev) for _ in range(2)]
        outs = [torch.empty(S, dtype=torch.float32, device=dev) for _ in range(2)]
        ev = {k: [[torch.cuda.Event() for _ in range(NS)] for _ in range(2)] for k in ("in_ready", "out_free")}
        ev.update({k: [torch.cuda.Event() for _ in range(2)] for k in ("in_free", "out_ready")})
        for e in ev["in_free"]:
            e.record(comp)
        for es in ev["out_free"]:
            for e in es:
                e.record(comp)
        it = [0]

        def split_copy(dst, src, streams):
            n, k = dst.numel(), len(streams)
            for i, st_ in enumerate(streams):
                with torch.cuda.stream(st_):
                    dst[i * n // k:(i + 1) * n // k].copy_(src[i * n // k:(i + 1) * n // k], non_blocking=True)

        def e2e_step():
            sl = it[0] % 2
            it[0] += 1
            for st_ in s_ins:
                st_.wait_event(ev["in_free"][sl])
            split_copy(gd[sl], h_grad, s_ins)
            split_copy(wmn[sl], h_main, s_ins)
            for i, st_ in enumerate(s_ins):
                ev["in_ready"][sl][i].record(st_)
                comp.wait_event(ev["in_ready"][sl][i])
            for e in ev["out_free"][sl]:
                comp.wait_event(e)
            qwd(wmn[sl])
            comm.tlq_hs_reduce_scatter(gd[sl], outs[sl], ws_t, a.bits_intra, a.bits_inter, a.group, a.hadamard, True)
            ev["in_free"][sl].record(comp)
            ev["out_ready"][sl].record(comp)
            for st_ in s_outs:
                st_.wait_event(ev["out_ready"][sl])
            split_copy(h_out, outs[sl], s_outs)
            for i, st_ in enumerate(s_outs):
                ev["out_free"][sl][i].record(st_)

        def e2e_run(n):
            for _ in range(n):
                e2e_step()
            for st_ in s_outs + s_ins:   # the region ends when the last readback has landed
                comp.wait_stream(st_)

        e2e_run(2)
        steps_e2e = max(3, min(a.steps, 6))
        ms_e2e = timed(lambda: e2e_run(steps_e2e), 1) / steps_e2e
        e2e = {"value": round(P * pre_bytes_rank / (ms_e2e * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(h_grad.numel() * h_grad.element_size() + h_main.numel() * 4),
               "d2h_bytes_per_step": int(h_out.numel() * 4), "ms_per_step": round(ms_e2e, 3),
               "steps": steps_e2e,
               "schedule": "double-buffered: H2D of step i+1 and D2H of step i overlap step i's kernels; "
                           "each direction split over 4 copy streams"}
        del h_grad, h_main, h_out, gd, wmn, outs

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:   # host-only and single-rank: a failure here must not cost the GPU line
            # all host cores (one worker process per core, the oracle as it stands) and one core
            ncores = min(os.cpu_count() or 1, 64)
            v, desc, cores = oracle_sample_rate(a, a.cpu_seconds / 2, D, ncores)
            v1, desc1, _ = oracle_sample_rate(a, a.cpu_seconds / 2, D, 1)
            cpu = {"value": round(v, 4), "unit": "GB/s", "cores": cores, "cpu_model": cpu_model(),
                   "nproc": os.cpu_count(), "kind": "oracle", "sample": desc,
                   "single_thread": {"value": round(v1, 4), "cores": 1, "sample": desc1}}
        except Exception as ex:  # noqa: BLE001
            cpu = {"error": f"{type(ex).__name__}: {ex}"[:300], "kind": "oracle"}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": a.steps,
                "warmup": max(3, a.warmup), "ms_per_step": round(ms, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": workload, "D": D, "D_unpadded": D0, "M": M, "N": N, "G": a.group,
                           "pipeline_chunks": comm.chunks(D, a.group),
                           "transport": comm.transport if world > 1 else "local",
                           "intra_pull": a.intra_pull or ("auto: " + ("0/1" if N <= 2 else "1/2")),
                           "G_w": a.qwd_group, "hadamard_block": a.hadamard,
                           "qwd_call": "two calls" if a.qwd_two_call else "sdp4_qwd_step",
                           "bits": {"qwd": a.bits_w, "intra": a.bits_intra, "inter": a.bits_inter},
                           "grad_dtype": a.grad_dtype, "model_dtype": a.model_dtype,
                           "l2": "inputs larger than L2 (>= 2.6 GB per tensor), no flush",
                           "pre_quant_bytes_per_rank": pre_bytes_rank,
                           "storage": "bf16/fp32 storage, fp32 arithmetic, int8/int4 wire codes"},
                "clocks": clk.summary(), "gpu_launches": int(launches), "kernels": kern, "comm_ops": comm_ops,
                "ms_per_step_profiled": round(ms_prof, 4), "roofline": roofline,
                "collectives": collectives, "e2e": e2e, "comparators": comparators, "ablation": ablation,
                "variants": variants,
                "cpu_baseline": cpu}
        emit(line)
    comm.close()


_JSON_FD = None


def emit(line: dict):
    """The ONE JSON line of the contract, on the original stdout (library noise such as
    NCCL's version banner is redirected to stderr in main())."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _JSON_FD
    _JSON_FD = os.dup(1)
    sys.stdout.flush()
    os.dup2(2, 1)
    a = parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if a.gpus != world and world == 1 and a.gpus > 1:
        raise SystemExit(f"--gpus {a.gpus} needs torchrun --nproc-per-node {a.gpus}")
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_sdp4(a, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
