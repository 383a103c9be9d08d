"""K34 alone in one process (sdp4_tlq_stage_quantize_reduce, every unit local): device time
at the GPT-1.3B size for M = 2 and 4, to profile it with ncu (the multi-rank path cannot be)."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2410_15526_b200 import tlq_stage_quantize_reduce, wire_unit_bytes  # noqa: E402


def main():
    D = synth.padded_numel(synth.gpt_numel("1.3B"), 8, 128)
    g = synth.gradient(D, seed=3, device="cuda", dtype=torch.bfloat16)
    for M in (2, 4):
        S = D // M
        buf = torch.empty(M * wire_unit_bytes(S, 4, 128), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            tlq_stage_quantize_reduce(g, buf, M, 128, 64)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            tlq_stage_quantize_reduce(g, buf, M, 128, 64)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        byt = D * 2 + M * wire_unit_bytes(S, 4, 128)
        print(f"K34 M={M}: {ms:.4f} ms, {byt / ms / 1e6:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
