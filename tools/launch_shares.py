"""Per-kernel launch counts, mean device times and shares of libsdp4 kernel time from an ncu
launch list (`--metrics gpu__time_duration.sum --csv`), skipping each kernel's first `warmup`
launches -- to check the bench's share_of_kernel_time against the serialised ncu pass.
    python tools/launch_shares.py launches.csv [warmup] [bench.json]"""
import collections
import csv
import io
import json
import sys

KERNELS = ("k1_qwd_quantize", "k2_qwd_apply", "k3_tlq_had_quant", "k4_tlq_dq_reduce_q", "k5_tlq_dq_reduce_had",
           "k6_ring_hop", "k_wait_flags", "k_tlq_local", "k_tlq_q84", "kf_qwd_step", "kf_tlq")


def main():
    path = sys.argv[1]
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    text = open(path).read()
    text = text[text.index('"ID"'):]
    times = collections.defaultdict(list)
    for r in csv.DictReader(io.StringIO(text)):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = next((k for k in KERNELS if k in r["Kernel Name"]), None)
        if name:
            times[name].append(float(r["Metric Value"]) * (1e-6 if r["Metric Unit"] == "ns" else 1e-3))
    tot = sum(sum(v[warm:]) for v in times.values())
    out = {n: {"launches": len(v), "timed_launches": len(v[warm:]), "avg_ms": round(sum(v[warm:]) / max(1, len(v[warm:])), 4),
               "share": round(sum(v[warm:]) / tot, 4)} for n, v in sorted(times.items())}
    if len(sys.argv) > 3:
        d = json.load(open(sys.argv[3]))
        bench_names = {"K345": "k_tlq_local", "K34": "k_tlq_q84", "KF": None}
        for n, v in d.get("kernels", {}).items():
            tag = n.split("_")[0]
            k = bench_names[tag] if tag in bench_names else next(
                (x for x in KERNELS if x.split("_")[0].upper() == tag), None)
            if k in out:
                out[k]["bench_share"] = v["share_of_kernel_time"]
                out[k]["bench_avg_ms"] = v["avg_ms"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
