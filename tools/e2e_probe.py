"""Where the headline's end-to-end overhead goes (QFT30 c128 simulate):
host packing of the gate list, the call with a packed list, the call with
the Python gate list, each + D2H of the marginal + sync (wall clock)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_08826_b200 as qj  # noqa: E402
from paper_2203_08826_b200 import qj as qjm  # noqa: E402

wl = bench.make_workload(sys.argv[1] if len(sys.argv) > 1 else "qft30_c128")
t = torch.empty(2 ** wl["n"], dtype=torch.complex128 if wl["dtype"] == "c128" else torch.complex64, device="cuda")
stream = torch.cuda.Stream()
st = qj.State(t, basis=None, stream=stream)
gates = wl["circ"].gates
packed = st.pack_circuit(gates)
pb = torch.empty(1 << len(wl["readout"]), dtype=st.real_dtype, device="cuda")
host = torch.empty(pb.numel(), dtype=pb.dtype, pin_memory=True)


def run(f, reps=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    return (time.perf_counter() - t0) / reps * 1e3


def sim_packed():
    st.simulate(wl["basis"], qubits=wl["readout"], packed=packed, out=pb)
    with torch.cuda.stream(stream):
        host.copy_(pb, non_blocking=True)
    stream.synchronize()


def sim_gates():
    st.simulate(wl["basis"], gates, qubits=wl["readout"], fuse=True, out=pb)
    with torch.cuda.stream(stream):
        host.copy_(pb, non_blocking=True)
    stream.synchronize()


res = {"pack_ms": run(lambda: qjm.pack_gates(gates), 20), "sim_packed_ms": run(sim_packed), "sim_gates_ms": run(sim_gates)}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(10):
    st.simulate(wl["basis"], qubits=wl["readout"], packed=packed, out=pb)
e1.record(stream)
torch.cuda.synchronize()
res["device_ms"] = e0.elapsed_time(e1) / 10
print(json.dumps(res))
