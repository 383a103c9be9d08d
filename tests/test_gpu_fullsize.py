"""Parity at the full BASELINE size (GPT-1.3B-shaped buffer, D = 1,315,819,520) in the launch
configuration bench.py times (same Comm defaults, same calls, same dtypes and group sizes).

The oracle cannot simulate 1.3e9 elements, but every output group depends only on the
same group positions of the inputs (R1: groups never straddle shards; Hadamard blocks lie
inside groups), so sampled windows are checked exactly: for each window the oracle
runs the whole path on the window's inputs and the GPU's codes, scales, updated replica and
output shard must match bit for bit.  Windows: random tile-aligned offsets + the first and
the last window of the buffer (ragged tail of the last tile).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2410_15526_b200 import Comm, pad_numel, tlq_workspace_offset, wire_unit_bytes

pytestmark = pytest.mark.gpu

G, GW, B, BITS_W, BI, BE = 128, 128, 64, 4, 8, 4   # bench.py defaults
WIN = 16384


def windows(D, k, seed):
    rng = np.random.default_rng(seed)
    starts = set(int(x) * WIN for x in rng.integers(0, D // WIN - 1, size=k))
    starts |= {0, D - WIN}
    return sorted(starts)


@pytest.fixture(scope="module")
def run():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    free = torch.cuda.mem_get_info()[0]
    if free < 40 * 2 ** 30:
        pytest.skip("needs ~40 GB of free device memory")
    dev = torch.device("cuda", 0)
    D = pad_numel(synth.gpt_numel("1.3B"), 1, G)
    comm = Comm()
    w_model = synth.model_weights(D, seed=synth.seed_for(0, 1), device=dev)
    w_main = synth.main_weights(w_model, seed=synth.seed_for(0, 2), lr=synth.GPT_LR["1.3B"])
    grad = synth.gradient(D, seed=synth.seed_for(0, 3), device=dev, dtype=torch.bfloat16)
    wm0 = w_model.clone()
    ws_q = torch.empty(comm.qwd_workspace_bytes(D, BITS_W, GW), dtype=torch.uint8, device=dev)
    ws_t = torch.empty(comm.tlq_workspace_bytes(D, BI, BE, G), dtype=torch.uint8, device=dev)
    out = torch.empty(D, dtype=torch.float32, device=dev)
    comm.qwd_step(w_main, w_model, ws_q, BITS_W, GW)   # the calls bench.py times: at world 1
    comm.tlq_hs_reduce_scatter(grad, out, ws_t, BI, BE, G, B, True)   # TLq-HS is one kernel (K345)
    # the three-kernel path (K3 -> K4 -> K5, what each rank of a P > 1 job runs): its wire
    # units land in the workspace and are checked too
    out3 = torch.empty(D, dtype=torch.float32, device=dev)
    comm.set_local_fusion(False)
    comm.tlq_hs_reduce_scatter(grad, out3, ws_t, BI, BE, G, B, True)
    comm.set_local_fusion(True)
    torch.cuda.synchronize()
    yield dict(D=D, w_model0=wm0, w_model=w_model, w_main=w_main, grad=grad, out=out, out3=out3, ws_q=ws_q,
               ws_t=ws_t)
    comm.close()


def unit_window(ws, base, D, k, Gx, start, n):
    """codes and scales of elements [start, start + n) of a one-unit wire layout at `base`."""
    cb = ws[base + start * k // 8: base + (start + n) * k // 8].cpu().numpy()
    so = base + D * k // 8
    sc = ws[so + start // Gx * 4: so + (start + n) // Gx * 4].cpu().numpy().view(np.float32)
    return cb, sc


def test_fullsize_qwd_windows(run):
    D = run["D"]
    for s in windows(D, 12, seed=1):
        wm = synth.bf16_bits(run["w_model0"][s:s + WIN])
        units, new = oracle.qwd_step([run["w_main"][s:s + WIN].cpu().numpy()], wm, BITS_W, GW, model_bf16=True)
        c, sc = units[0]
        cb, gsc = unit_window(run["ws_q"], 0, D, BITS_W, GW, s, WIN)
        assert np.array_equal(cb, oracle.pack_codes(c, BITS_W)), f"qWD codes differ in window {s}"
        assert np.array_equal(gsc.view(np.uint32), sc.view(np.uint32)), f"qWD scales differ in window {s}"
        assert np.array_equal(synth.bf16_bits(run["w_model"][s:s + WIN]), new), f"w_model differs in window {s}"


def test_fullsize_tlq_hs_windows(run):
    D = run["D"]
    o_inter = tlq_workspace_offset(1, 1, D, BI, BE, G, 2)
    for s in windows(D, 12, seed=2):
        g = run["grad"][s:s + WIN].float().cpu().numpy()
        tr = oracle.tlq_hs_reduce_scatter([g], oracle.Topology(1, 1), G, B, BI, BE, True)
        c8, s8 = tr.intra_send[0][0][0]
        cb, gsc = unit_window(run["ws_t"], 0, D, BI, G, s, WIN)
        assert np.array_equal(cb, oracle.pack_codes(c8, BI)), f"K3 codes differ in window {s}"
        assert np.array_equal(gsc.view(np.uint32), s8.view(np.uint32)), f"K3 scales differ in window {s}"
        c4, s4 = tr.inter_send[0][0]
        cb, gsc = unit_window(run["ws_t"], o_inter, D, BE, G, s, WIN)
        assert np.array_equal(cb, oracle.pack_codes(c4, BE)), f"K4 codes differ in window {s}"
        assert np.array_equal(gsc.view(np.uint32), s4.view(np.uint32)), f"K4 scales differ in window {s}"
        for key in ("out", "out3"):   # the fused kernel (bench) and the three kernels
            got = run[key][s:s + WIN].cpu().numpy()
            assert np.array_equal(got.view(np.uint32), tr.out[0].view(np.uint32)), f"{key} differs in window {s}"


def test_fullsize_output_sanity(run):
    # properties that hold at any size: finite everywhere, close to the gradient mean (P = 1:
    # the reduce-scatter returns the rank's own gradient up to the two quantizations)
    out = run["out"]
    assert torch.isfinite(out).all()
    g = run["grad"].float()
    rel = (torch.linalg.vector_norm(out - g) / torch.linalg.vector_norm(g)).item()
    assert rel < 0.2
    assert wire_unit_bytes(run["D"], 4, 128) > 0
