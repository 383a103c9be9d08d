"""PCIe copy ceilings for the e2e leg: pinned host -> device and device -> host of 4 GB,
one stream vs the copy split into chunks over 2 / 4 streams, and H2D + D2H at once."""
import json

import torch


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    n = 4 << 30
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    res = {}
    for k in (1, 2, 4):
        ss = [torch.cuda.Stream() for _ in range(k)]

        def h2d():
            cur = torch.cuda.current_stream()
            for i, s in enumerate(ss):
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    d[i * n // k:(i + 1) * n // k].copy_(h[i * n // k:(i + 1) * n // k], non_blocking=True)
            for s in ss:
                cur.wait_stream(s)

        def d2h():
            cur = torch.cuda.current_stream()
            for i, s in enumerate(ss):
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    h2[i * n // k:(i + 1) * n // k].copy_(d2[i * n // k:(i + 1) * n // k], non_blocking=True)
            for s in ss:
                cur.wait_stream(s)
        res[f"h2d_{k}streams_GBps"] = round(n / t(h2d) / 1e6, 1)
        res[f"d2h_{k}streams_GBps"] = round(n / t(d2h) / 1e6, 1)

        def both():
            cur = torch.cuda.current_stream()
            s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            with torch.cuda.stream(s1):
                h2d()
            with torch.cuda.stream(s2):
                d2h()
            cur.wait_stream(s1)
            cur.wait_stream(s2)
        res[f"both_{k}streams_GBps_each_way"] = round(n / t(both) / 1e6, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
