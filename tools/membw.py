"""Achievable HBM read bandwidth on this GPU (context for the scan roofline).

Reads an 8 GiB buffer with torch reductions and a copy; CUDA events, best of 5.
"""
import json

import torch


def bw(fn, nbytes, reps=5):
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return nbytes / (best * 1e-3) / 1e9


x = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
x.fill_(1)
xi = x.view(torch.int64)
y = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
out = {
    "read_sum_int64_GBs": bw(lambda: xi.sum(), x.numel()),
    "read_amax_int64_GBs": bw(lambda: xi.amax(), x.numel()),
    "copy_4GiB_rw_GBs": bw(lambda: y.copy_(x[: 4 << 30]), 2 * (4 << 30)),
}
print(json.dumps(out))
