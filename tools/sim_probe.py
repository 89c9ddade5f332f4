"""QFT30 c128 step timing: reset + apply_circuit + marginal as three calls vs
one qj_simulate call (CUDA events, after warm-up)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_08826_b200 as qj  # noqa: E402
from workloads import circuits as C  # noqa: E402

import bench  # noqa: E402

wl = bench.make_workload(sys.argv[1] if len(sys.argv) > 1 else "qft30_c128")
n, x, circ = wl["n"], wl["basis"], wl["circ"]
t = torch.empty(2**n, dtype=torch.complex128 if wl["dtype"] == "c128" else torch.complex64, device="cuda")
stream = torch.cuda.Stream()
st = qj.State(t, basis=0, stream=stream)
packed = st.pack_circuit(circ.gates)
pb = torch.empty(1024, dtype=st.real_dtype, device="cuda")
q = list(range(10))


FG = int(os.environ.get("QJ_PROBE_FG", "0"))  # gate-fusion width before tiling (0 = none)


def sep():
    st.reset(x)
    st.apply_circuit(None, fuse=True, packed=packed, fuse_gates=FG)
    st.probabilities(q, out=pb)


def sim():
    st.simulate(x, qubits=q, packed=packed, out=pb, fuse_gates=FG)


res = {}
for name, f in (("separate", sep), ("simulate", sim)):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        f()
    e1.record(stream)
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 5
res["marginal_sum"] = float(pb.sum())
# per-pass device times (profiling: event pairs around every pass, no graph)
st.set_profiling(True)
for name, f in (("separate", sep), ("simulate", sim)):
    st.profile(reset=True)
    f()
    res[name + "_launches"] = [(k, round(ms, 4), round(b / ms / 1e6 / 6450.9, 3) if ms > 0 else None)
                               for k, ms, b in st.profile_launches(reset=True)]
st.set_profiling(False)
print(json.dumps(res))
