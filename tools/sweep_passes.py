"""Per-pass micro-benchmark sweep: where the per-pass HBM
fraction is won or lost.  30 qubits complex128 (16 GiB) and complex64 (8 GiB):

  * 1q dense pass at every target bit 0..29;
  * CU1 / CZ at bit pairs (0,1) (1,2) (0,29) (14,15) (28,29);
  * SWAP at (0,29) (14,15) (28,29); fSim at (0,1) (14,15) (28,29);
  * fused window tile passes (12-bit windows) of pure-diagonal, 1q-only and
    mixed programs;
  * references: torch copy_ of the state's bytes and an in-place
    read-modify-write (psi.mul_(1)), the practical roofline of an in-place pass.

Each entry: library per-launch device time (CUDA events on the state's
stream, profiling mode) over REPS launches, algorithmic bytes (C15), GB/s and
the fraction of the measured HBM peak.  One JSON line per entry on stdout.
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_08826_b200 as qj  # noqa: E402
from workloads import gates as G  # noqa: E402

PEAK, _ = bench.load_peaks()
REPS = int(os.environ.get("SWEEP_REPS", "5"))
n = 30


def emit(d):
    print(json.dumps(d), flush=True)


FILTER = os.environ.get("SWEEP_FILTER")  # only entries whose label contains it


def timed_gates(st, gates, fuse, label, dt):
    if FILTER and FILTER not in label:
        return
    packed = st.pack_circuit(gates)
    st.apply_circuit(None, fuse=fuse, packed=packed)  # plan + JIT
    st.sync()
    st.set_profiling(True)
    st.profile_launches(reset=True)
    for _ in range(REPS):
        st.apply_circuit(None, fuse=fuse, packed=packed)
    recs = st.profile_launches(reset=True)
    st.set_profiling(False)
    ms = sum(r[1] for r in recs)
    byts = sum(r[2] for r in recs)
    kinds = sorted({r[0] for r in recs})
    gbs = byts / (ms / 1e3) / 1e9 if ms > 0 else None
    emit({"entry": label, "dtype": dt, "kinds": kinds, "launches_per_rep": len(recs) / REPS,
          "us_per_launch": ms / len(recs) * 1e3 if recs else None, "alg_bytes_per_launch": byts / max(len(recs), 1),
          "GBps": gbs, "frac": gbs / PEAK if gbs else None})


def reference(t, dt):
    stream = torch.cuda.current_stream()
    u = torch.empty_like(t)
    for name, f, byts in (("torch copy_", lambda: u.copy_(t), 2 * t.numel() * t.element_size()),
                          ("in-place RMW psi.mul_(1)", lambda: t.mul_(1), 2 * t.numel() * t.element_size())):
        f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(REPS):
            f()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / REPS
        emit({"entry": "reference: " + name, "dtype": dt, "us_per_launch": ms * 1e3, "alg_bytes_per_launch": byts,
              "GBps": byts / (ms / 1e3) / 1e9, "frac": byts / (ms / 1e3) / 1e9 / PEAK})
    del u
    torch.cuda.empty_cache()


def main():
    rng = np.random.default_rng(8)
    for dt, tdt in (("c128", torch.complex128), ("c64", torch.complex64)):
        t = torch.empty(2**n, dtype=tdt, device="cuda")
        t.fill_(1.0 / math.sqrt(2**n))
        reference(t, dt)
        st = qj.State(t, basis=None, stream=torch.cuda.Stream())
        q = lambda b: n - 1 - b  # noqa: E731  qubit holding physical bit b
        u = G.random_unitary(1, rng)
        for b in range(n):
            timed_gates(st, [G.unitary("U", (q(b),), u)], False, f"1q dense bit {b}", dt)
        for (a, b) in ((0, 1), (1, 2), (0, 29), (14, 15), (28, 29)):
            timed_gates(st, [G.CU1(q(a), q(b), 0.7)], False, f"CU1 bits ({a},{b})", dt)
            timed_gates(st, [G.CZ(q(a), q(b))], False, f"CZ bits ({a},{b})", dt)
        for (a, b) in ((0, 29), (14, 15), (28, 29)):
            timed_gates(st, [G.SWAP(q(a), q(b))], False, f"SWAP bits ({a},{b})", dt)
        for (a, b) in ((0, 1), (14, 15), (28, 29)):
            timed_gates(st, [G.FSIM(q(a), q(b), 0.9, 0.4)], False, f"fSim bits ({a},{b})", dt)
        u5 = G.random_unitary(5, rng)
        for bits in ((25, 26, 27, 28, 29), (5, 6, 7, 8, 9), (0, 1, 2, 3, 4)):
            timed_gates(st, [G.unitary("U5", tuple(q(b) for b in bits), u5)], False,
                        f"5q dense bits {bits[0]}..{bits[-1]}" + (" (tensor cores)" if dt == "c64" else ""), dt)
        for w0 in (0, 9, 18):  # window = the 3 / 4 low bits + 9 / 8 more starting at bit w0 + C
            bits = list(range(12)) if w0 == 0 else list(range(3 if dt == "c128" else 4)) + \
                list(range(w0 + 3, w0 + 12 - (0 if dt == "c128" else 1)))
            qs = [q(b) for b in bits]
            diag = [G.CU1(qs[i], qs[(i + 5) % 12], 0.3 + i) for i in range(12)] + [G.RZ(x, 0.2) for x in qs]
            one = [G.H(x) for x in qs] + [G.RY(x, 0.4) for x in qs]
            mixed = [G.H(x) for x in qs] + [G.CU1(qs[i], qs[(i + 1) % 12], 0.5) for i in range(12)] + \
                [G.unitary("U", (x,), u) for x in qs[:6]]
            for name, gl in (("pure-diagonal", diag), ("1q-only", one), ("mixed", mixed)):
                timed_gates(st, gl, True, f"tile w=12 bits {bits[0]}..{bits[-1]} ({len(bits)} bits) {name}", dt)
        st.free()
        del st, t
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
