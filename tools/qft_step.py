"""QFT30 c128 steps for ncu captures: `simulate` (the headline, live tiles)
or `separate` (reset + every-tile fused passes + marginal), K times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_08826_b200 as qj  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "simulate"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = bench.make_workload(sys.argv[3] if len(sys.argv) > 3 else "qft30_c128")
t = torch.empty(2 ** wl["n"], dtype=torch.complex128 if wl["dtype"] == "c128" else torch.complex64, device="cuda")
st = qj.State(t, basis=None, stream=torch.cuda.Stream())
packed = st.pack_circuit(wl["circ"].gates)
pb = torch.empty(1024, dtype=st.real_dtype, device="cuda")
for _ in range(k):
    if mode == "simulate":
        st.simulate(wl["basis"], qubits=wl["readout"], packed=packed, out=pb)
    else:
        st.reset(wl["basis"])
        st.apply_circuit(None, fuse=True, packed=packed)
        st.probabilities(wl["readout"], out=pb)
st.sync()
print("ok", mode, k)
