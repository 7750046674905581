#!/usr/bin/env python
"""Pure-write and copy HBM bandwidth on this GPU (torch fill_ / copy_ over
1 GiB, best of 20, CUDA events): the ceiling for the output-bound expand
kernels, whose DRAM traffic is almost all writes."""
import json

import torch


def best(fn, reps=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        out.append(s.elapsed_time(e) / 1e3)
    return min(out)


n = 1 << 28  # 1 GiB of int32
a = torch.empty(n, dtype=torch.int32, device="cuda")
b = torch.empty(n, dtype=torch.int32, device="cuda")
a.fill_(1)
t_w = best(lambda: a.fill_(7))
t_c = best(lambda: b.copy_(a))
print(json.dumps({"write_GBps": round(4 * n / t_w / 1e9, 1),
                  "copy_GBps_read_plus_write": round(8 * n / t_c / 1e9, 1)}))
