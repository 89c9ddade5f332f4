"""Run exactly one bench section's step a few times (for ncu launch lists):
    python tools/step_probe.py WORKLOAD SECTION [STEPS]
SECTION: simulate (qj_simulate, the headline), separate (reset +
apply_circuit(QJ_FUSE) + marginal), unfused (per-gate passes), paper_fusion
(<= 2-qubit greedy fusion + per-gate passes).  The launches of every step are
the same, so per-kind averages over the whole run are per-launch figures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_08826_b200 as qj  # noqa: E402

wl_name, section = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
wl = bench.make_workload(wl_name)
dev = torch.device("cuda", 0)
tdt = torch.complex128 if wl["dtype"] == "c128" else torch.complex64
stream = torch.cuda.Stream(dev)
psi = torch.empty(1 << wl["n"], dtype=tdt, device=dev)
st = qj.State(psi, basis=None, stream=stream)
packed = st.pack_circuit(wl["circ"].gates)
pbuf = torch.empty(1 << len(wl["readout"]), dtype=st.real_dtype, device=dev)
for _ in range(steps):
    if section == "simulate":
        st.simulate(wl["basis"], qubits=wl["readout"], packed=packed, out=pbuf)
    else:
        st.reset(wl["basis"])
        st.apply_circuit(None, fuse=section == "separate", fuse_gates=section == "paper_fusion", packed=packed)
        st.probabilities(wl["readout"], out=pbuf)
st.sync()
print("ok", wl_name, section, steps)
