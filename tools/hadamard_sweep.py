"""(De)quantization throughput with and without the fused Hadamard transform, mirroring the
paper's Table 5 (tab:quantization-throughput): K3
(blockwise Hadamard + 8-bit group quantization of an fp32 buffer) and K5 (4-bit dequantize +
inverse Hadamard into an fp32 buffer), b = 0 vs b = 64, G = 128, at 8 MB .. 2 GB of fp32
data, one GPU, through the stage entry points (no communication).  Throughput = fp32 bytes
(quantization input / dequantization output) per second, mean +- std over 20 timed launches
after warm-up; the HBM fraction uses each kernel's algorithmic bytes.

    python tools/hadamard_sweep.py [--out profiles/r01/hadamard_sweep.json]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2410_15526_b200 import tlq_stage_final, tlq_stage_quantize, wire_unit_bytes  # noqa: E402


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="8,16,64,512,1024,2048")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6551.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6551.0
    G = 128
    rows = []
    for mb in [int(x) for x in a.sizes_mb.split(",")]:
        D = (mb << 20) // 4
        D -= D % 16384
        x = synth.gradient(D, seed=3, device="cuda", dtype=torch.float32)
        q8 = torch.empty(wire_unit_bytes(D, 8, G), dtype=torch.uint8, device="cuda")
        q4 = torch.empty(wire_unit_bytes(D, 4, G), dtype=torch.uint8, device="cuda")
        y = torch.empty(D, dtype=torch.float32, device="cuda")
        tlq_stage_quantize(x, q4, 1, 1, 4, G, 0)          # a valid 4-bit unit to dequantize
        row = {"mbytes": mb, "D": D}
        for b in (0, 64):
            tq = timed(lambda: tlq_stage_quantize(x, q8, 1, 1, 8, G, b))
            td = timed(lambda: tlq_stage_final(q4, y, D, 1, 1, 4, G, b, True))
            for name, ts, alg in (("quant", tq, D * (4 + 1 + 4 / G)), ("dequant", td, D * (0.5 + 4 / G + 4))):
                m, sd = statistics.mean(ts), statistics.pstdev(ts)
                row[f"{name}_b{b}_GBps"] = round(D * 4 / (m * 1e-3) / 1e9, 1)
                row[f"{name}_b{b}_std"] = round(D * 4 / (m * 1e-3) / 1e9 * sd / m, 1)
                row[f"{name}_b{b}_hbm_frac"] = round(alg / (m * 1e-3) / 1e9 / peak, 3)
        rows.append(row)
        print(json.dumps(row), flush=True)
        del x, q8, q4, y
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"gpu": torch.cuda.get_device_name(), "G": G, "peak_hbm_gbs": peak, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
