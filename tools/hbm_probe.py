"""HBM ceilings by read/write mix on this GPU (CUDA events, 4 GiB buffers, best of 10):
write-only (fill), read-only (sum), copy (1:1), and 1-read:4-write / 4-read:1-write mixes
built from torch ops.  Used to judge the write-heavy kernels (K5 writes 88% of its bytes)."""
import json

import torch


def t(fn, reps=10):
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
    n = 1 << 30  # fp32 elements = 4 GiB
    x = torch.empty(n, device="cuda")
    y = torch.empty(n, device="cuda")
    small = torch.empty(n // 8, device="cuda")
    res = {}
    ms = t(lambda: x.fill_(1.0))
    res["write_only_fill_GBps"] = 4 * n / ms / 1e6
    ms = t(lambda: x.sum())
    res["read_only_sum_GBps"] = 4 * n / ms / 1e6
    ms = t(lambda: y.copy_(x))
    res["copy_1r1w_GBps"] = 8 * n / ms / 1e6
    # 1 read : 8 write -- broadcast a small tensor into a large one (expand + copy)
    big = x.view(8, n // 8)
    ms = t(lambda: big.copy_(small.expand(8, n // 8)))
    res["read1_write8_GBps"] = (4 * n // 8 + 4 * n) / ms / 1e6
    # in-place read-modify-write of a bf16 buffer (K2's replica pattern) vs a bf16 copy
    wb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    wb2 = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    ms = t(lambda: wb.add_(1.0))
    res["bf16_inplace_rmw_GBps"] = 4 * n / ms / 1e6
    ms = t(lambda: wb2.copy_(wb))
    res["bf16_copy_GBps"] = 4 * n / ms / 1e6
    print(json.dumps({k: round(v, 1) for k, v in res.items()}))


if __name__ == "__main__":
    main()
