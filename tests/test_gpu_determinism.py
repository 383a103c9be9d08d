"""Run-to-run determinism: the kernels claim tiles from a dynamic
scheduler, so which CTA computes which tile changes from launch to launch -- the outputs must
not.  The bench workload (GPT-1.3B-shaped buffer, bf16, G = 128, b = 64, bits 4/8/4) is run
repeatedly through sdp4_qwd_step and sdp4_tlq_hs_reduce_scatter on identical inputs; every
repeat must be bit-identical to the first (and the first is the oracle's, by
tests/test_gpu_fullsize.py's sampled windows)."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def test_repeated_runs_bit_identical():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2410_15526_b200 import Comm
    dev = torch.device("cuda", 0)
    D = synth.gpt_numel("1.3B")
    G = 128
    comm = Comm()
    w0 = synth.model_weights(D, seed=synth.seed_for(0, 1), device=dev)
    main = synth.main_weights(w0, seed=synth.seed_for(0, 2), lr=synth.GPT_LR["1.3B"])
    grad = synth.gradient(D, seed=synth.seed_for(0, 3), device=dev, dtype=torch.bfloat16)
    ws_q = torch.empty(comm.qwd_workspace_bytes(D, 4, G), dtype=torch.uint8, device=dev)
    ws_t = torch.empty(comm.tlq_workspace_bytes(D, 8, 4, G), dtype=torch.uint8, device=dev)
    out_ref, wm_ref = None, None
    for rep in range(4):
        wm = w0.clone()
        out = torch.empty(D, dtype=torch.float32, device=dev)
        comm.qwd_step(main, wm, ws_q, 4, G)
        comm.tlq_hs_reduce_scatter(grad, out, ws_t, 8, 4, G, 64, True)
        comm.tlq_hs_reduce_scatter(grad, out, ws_t, 8, 4, G, 64, True, seed=2410 + 0)  # stochastic pass too
        torch.cuda.synchronize()
        if rep == 0:
            out_ref, wm_ref = out.view(torch.int32).clone(), wm.view(torch.int16).clone()
        else:
            assert torch.equal(out.view(torch.int32), out_ref), f"TLq-HS output changed on repeat {rep}"
            assert torch.equal(wm.view(torch.int16), wm_ref), f"qWD replica changed on repeat {rep}"
        del wm, out
    comm.close()
