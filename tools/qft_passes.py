"""Apply the fused QFT(n) circuit a few times (ncu target: -k regex:qj_tile_jit)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_08826_b200 as qj  # noqa: E402
from workloads import circuits as C  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
st = qj.State(t, basis=0)
which = os.environ.get("QJ_CIRC", "qft")
if which == "qft":
    gates = C.qft(n).gates
else:  # hK: H on the K highest qubits (window = low bits + K high bits)
    from workloads import gates as G
    gates = [G.H(q) for q in range(int(which[1:]))]
packed = st.pack_circuit(gates)
for _ in range(reps):
    st.reset(0)  # canonical qubit map: every repetition runs the same plan
    st.apply_circuit(None, fuse=True, packed=packed)
st.sync()
print("ok")
