"""Run the tfim10 circuit through the whole-state SMEM kernel a few times
(for ncu captures of small_kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2203_08826_b200 as qj
from workloads import evolution as E

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
circ = E.adiabatic_circuit(n, 1.0, 0.01)
t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
st = qj.State(t, basis=0)
packed = st.pack_circuit(circ.gates)
for _ in range(3):
    st.reset(0)
    st.apply_circuit(None, fuse=True, packed=packed)
st.sync()
print("ok", float(t.abs().pow(2).sum()))
