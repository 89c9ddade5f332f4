"""Repro: tile passes of pure-diagonal / 1q-only / mixed programs on 12 window bits (ring form)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2203_08826_b200 as qj  # noqa: E402
from workloads import circuits as C  # noqa: E402
from workloads import gates as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
which = sys.argv[2] if len(sys.argv) > 2 else "all"
dt = np.complex128
q = lambda b: n - 1 - b  # noqa: E731
rng = np.random.default_rng(3)
u = G.random_unitary(1, rng)
for w0 in (0, 9):
    bits = list(range(12)) if w0 == 0 else list(range(3)) + list(range(w0 + 3, w0 + 12))
    qs = [q(b) for b in bits]
    progs = {"diag": [G.CU1(qs[i], qs[(i + 5) % 12], 0.3 + i) for i in range(12)] + [G.RZ(x, 0.2) for x in qs],
             "one": [G.H(x) for x in qs] + [G.RY(x, 0.4) for x in qs],
             "mixed": [G.H(x) for x in qs] + [G.CU1(qs[i], qs[(i + 1) % 12], 0.5) for i in range(12)] +
             [G.unitary("U", (x,), u) for x in qs[:6]]}
    for name, gl in progs.items():
        if which != "all" and which != name:
            continue
        circ = C.Circuit(n, list(gl))
        v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
        psi = v / np.linalg.norm(v)
        exp = oracle.run(circ, psi)
        x = torch.from_numpy(psi.copy()).cuda()
        st = qj.State(x, basis=None)
        st.apply_circuit(gl, fuse=True)
        st.canonicalize()
        st.sync()
        err = float(np.max(np.abs(x.cpu().numpy() - exp)))
        print(w0, name, err, flush=True)
        assert err < 1e-12
print("repro ok")
