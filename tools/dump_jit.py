"""Apply one fused circuit with QJ_DUMP_JIT set (the caller exports it) so
the generated tile-pass sources land in that directory."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_08826_b200 as qj  # noqa: E402
from workloads import circuits as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qft30"
if name.startswith("qft"):
    n = int(name[3:])
    circ, dt = C.qft(n), torch.complex128
elif name == "sup32":
    n = 32
    circ, dt = C.supremacy(4, 8, 20), torch.complex64
t = torch.empty(2**n, dtype=dt, device="cuda")
st = qj.State(t, basis=0)
st.apply_circuit(circ.gates, fuse=True)
st.sync()
print("ok")
