"""Tile-pass memory-path probe: time fused passes with little compute (H on
high qubits) against QFT30's first pass, on a 2^30 complex128 state."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_08826_b200 as qj  # noqa: E402
from workloads import gates as G  # noqa: E402
from workloads import circuits as C  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "c128"
n = 30 if dt == "c128" else 31
t = torch.empty(2**n, dtype=torch.complex128 if dt == "c128" else torch.complex64, device="cuda")
stream = torch.cuda.Stream()
st = qj.State(t, basis=0, stream=stream)
peak = 6464.9
cases = {
    "h9_high": [G.H(q) for q in range(9)],
    "h9_high_x2": [G.H(q) for q in range(9)] * 2,
    "h4_high": [G.H(q) for q in range(4)],
    "qft": C.qft(n).gates,
    "h9_low": [G.H(q) for q in range(n - 9, n)],
    "h6_mid": [G.H(q) for q in range(n - 18, n - 12)],
}
res = {}
for name, gates in cases.items():
    packed = st.pack_circuit(gates)
    for _ in range(3):
        st.apply_circuit(None, fuse=True, packed=packed)
    st.set_profiling(True)
    st.profile(reset=True)
    for _ in range(5):
        st.apply_circuit(None, fuse=True, packed=packed)
    prof = st.profile(reset=True)
    st.set_profiling(False)
    d = prof.get("tile")
    if d:
        us = d["total_ms"] / d["launches"] * 1e3
        res[name] = {"passes_per_circuit": d["launches"] / 5, "us_per_pass": us,
                     "frac": d["alg_bytes"] / (d["total_ms"] / 1e3) / 1e9 / peak}
    else:
        res[name] = {k: v for k, v in prof.items()}
print(json.dumps(res, indent=1))
