"""Write-only and copy HBM bandwidth on this box (the live QFT pass's floor):
a 16 GiB buffer written by cudaMemsetAsync (torch.zero_), by torch fill_ with
a complex128 value, and copied (read + write), CUDA events, best of 5."""
import json

import torch

n = 2**30
t = torch.empty(n, dtype=torch.complex128, device="cuda")
u = torch.empty(n // 2, dtype=torch.complex128, device="cuda")
res = {}


def best(f, nbytes, reps=5):
    f()
    torch.cuda.synchronize()
    b = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        b = ms if b is None else min(b, ms)
    return {"ms": b, "GBps": nbytes / b / 1e6}


res["memset_16GiB"] = best(lambda: t.zero_(), t.numel() * 16)
res["fill_c128_16GiB"] = best(lambda: t.fill_(0.5 + 0.25j), t.numel() * 16)
res["copy_8GiB_rw"] = best(lambda: u.copy_(t[: n // 2]), (n // 2) * 16 * 2)
print(json.dumps(res))
