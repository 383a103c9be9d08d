#!/usr/bin/env python
"""Summarize an ncu report (+ optional launch list) into profiles/<round>/ files.

    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep gpurun_out/launches.csv profiles/r01 "<workload>"

Writes <outdir>/ncu_summary.md (per-kernel duration, DRAM bytes, achieved DRAM GB/s vs the
measured peak, issue activity, registers, occupancy, top stall reasons), the launch share
table from the launch list, and profiles/ncu_traffic.json (dram read+write bytes per launch
per kernel, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

NAMES = {"k1_": "K1_qwd_quantize", "k2_": "K2_qwd_apply", "k3_": "K3_tlq_had_quant",
         "k4_": "K4_tlq_dq_reduce_q", "k5_": "K5_tlq_dq_reduce_had"}


def short(name):
    for k, v in NAMES.items():
        if k in name:
            return v
    return name[:40]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[0], rows[2:]
    return [{h: r[i] for i, h in enumerate(hdr)} for r in data]


def f(x):
    try:
        return float(x)
    except Exception:
        return 0.0


def main():
    rep, launches, outdir, workload = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = raw(rep)
    lines = [f"# ncu --set full summary ({os.path.basename(rep)})", "",
             f"Workload: `{workload}`.  Peak: {peak} GB/s (MEASURED_PEAKS.json hbm_gbs).  ncu serialises "
             "launches with cold caches (clock-control none); compare shares, not absolutes.", "",
             "| kernel | ms | DRAM read GB | DRAM write GB | DRAM GB/s | of peak | issue active % | warps active % | "
             "regs | top stalls (cycles/issue) |", "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for r in rows:
        name = short(r["Kernel Name"])
        ms = f(r["gpu__time_duration.sum"])
        rd, wr = f(r["dram__bytes_read.sum"]), f(r["dram__bytes_write.sum"])
        unit = 1.0
        traffic.setdefault(name, (rd + wr) * 1e9)
        gbs = (rd + wr) / (ms * 1e-3) if ms else 0
        stalls = sorted(((f(v), k.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", "")) for k, v in r.items()
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
            reverse=True)[:3]
        lines.append(f"| {name} | {ms:.3f} | {rd * unit:.3f} | {wr * unit:.3f} | {gbs:.0f} | {gbs / peak:.2f} | "
                     f"{f(r['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
                     f"{f(r['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
                     f"{r['launch__registers_per_thread']} | "
                     + ", ".join(f"{n} {v:.2f}" for v, n in stalls) + " |")
    if os.path.exists(launches):
        txt = open(launches).read()
        txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
        lr = list(csv.DictReader(io.StringIO(txt)))
        tot, per = 0.0, {}
        for r in lr:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            u = r.get("Metric Unit", "")
            v = f(r["Metric Value"]) * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3}.get(u, 1.0)
            n = short(r["Kernel Name"])
            per.setdefault(n, [0.0, 0])
            per[n][0] += v
            per[n][1] += 1
            tot += v
        ours = {n: v for n, v in per.items() if n in NAMES.values()}
        tot_ours = sum(v[0] for v in ours.values()) or 1.0
        lines += ["", "## Launch list (every launch, `--metrics gpu__time_duration.sum`)", "",
                  "Shares are of libsdp4 kernel time (torch kernels are the synthetic-input generators, "
                  "outside the timed region).", "",
                  "| kernel | launches | total ms | avg ms | share of libsdp4 time |", "|---|---|---|---|---|"]
        for n, (v, c) in sorted(ours.items(), key=lambda x: -x[1][0]):
            lines.append(f"| {n} | {c} | {v:.3f} | {v / c:.3f} | {v / tot_ours:.3f} |")
        other = sum(v[0] for n, v in per.items() if n not in ours)
        lines.append(f"| (torch input generation) | {sum(v[1] for n, v in per.items() if n not in ours)} | "
                     f"{other:.3f} | | |")
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, "ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(os.path.join(root, "profiles", "ncu_traffic.json"), "w") as fh:
        json.dump({"workload": workload, "source": os.path.join(outdir, "ncu_summary.md"),
                   "kernels": {k: int(v) for k, v in traffic.items()}}, fh, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
