"""Host-staged execution (row f4): QFT(n) with the state
in pinned host memory, slices streamed through one B200.  Prints one JSON
line: seconds per circuit, host<->device bytes per circuit (from the plan:
every sweep moves the state down and up once, every exchange too) and the
achieved host-link GB/s.  Usage: python tools/bench_host.py [n] [nslices] [dtype]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2203_08826_b200 as qj
from paper_2203_08826_b200 import qj as Q
from workloads import circuits as C

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dt = sys.argv[3] if len(sys.argv) > 3 else "c128"
tdt = torch.complex128 if dt == "c128" else torch.complex64
amp = 16 if dt == "c128" else 8
circ = C.qft(n)
steps, _ = Q.plan_circuit(n, ns, circ.gates, fuse=True, amp_bytes=amp)
sweeps, exch, prev_ex = 0, 0, True
for s in steps:
    if s["type"] == 1:
        exch += 1
        prev_ex = True
    else:
        if prev_ex:
            sweeps += 1
        prev_ex = False
state = amp << n
moved = 2 * state * sweeps  # exchanges relabel half-slices: no bytes move
t0 = time.perf_counter()
h = torch.empty(1 << n, dtype=tdt).pin_memory()
alloc = time.perf_counter() - t0
stream = torch.cuda.Stream()
st = qj.State.host(h, ns, basis=5, stream=stream)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
times = []
for rep in range(3):
    st.reset(5)
    st.sync()
    ev[0].record(stream)
    st.apply_circuit(circ.gates, fuse=True)
    ev[1].record(stream)
    st.sync()
    times.append(ev[0].elapsed_time(ev[1]) / 1e3)
t = min(times[1:]) if len(times) > 1 else times[0]
# spot parity: |amplitude| = 2^(-n/2) everywhere for QFT|x>
st.canonicalize()
st.sync()
idx = torch.randint(0, 1 << n, (4096,))
err = float((h[idx].abs() - 2 ** (-n / 2)).abs().max())
# host-link roofline on this box: pinned 2 GiB copies, one direction and both at once
def link_peaks():
    nb = 2 << 30
    hs = torch.empty(nb, dtype=torch.uint8).pin_memory()
    hd = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name in ("h2d", "d2h", "both"):
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if name in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d1.copy_(hs, non_blocking=True)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    hd.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = max(best, (2 if name == "both" else 1) * nb / dt / 1e9)
        out[name + "_gbs"] = best
    return out


peaks = link_peaks()
print(json.dumps({"workload": f"qft{n}_{dt}_host", "nslices": ns, "state_bytes": state, "s_per_circuit": t,
                  "sweeps": sweeps, "exchanges": exch, "host_link_bytes": moved,
                  "host_link_gbs": moved / t / 1e9, "per_direction_gbs": moved / 2 / t / 1e9, "times": times, "pin_alloc_s": alloc,
                  "max_abs_err_modulus": err, "link_peaks": peaks,
                  "link_frac": moved / t / 1e9 / peaks["both_gbs"]}))
