"""Small invocations of every kernel family -- for compute-sanitizer runs
(closed on this pool) and for the bounds-checked JIT mode (QJ_JIT_CHECK=1,
tests/test_gpu_fullsize.py::test_checked_tile_kernels_subprocess): per-gate passes, the whole-state SMEM program, JIT
tile passes in the two-CTA, CTA-pair, live-tile and ring (TMA) forms, the
tensor-core dense pass, readout and measurement.  Each result is checked
against the oracle so a silent corruption fails the run too."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2203_08826_b200 as qj  # noqa: E402
from workloads import circuits as C  # noqa: E402
from workloads import gates as G  # noqa: E402


def check(t, exp, tol, what):
    err = float(np.max(np.abs(t.cpu().numpy().astype(np.complex128) - exp)))
    assert err <= tol, f"{what}: {err}"
    print("ok", what, f"{err:.1e}", flush=True)


dev = torch.device("cuda:0")
# per-gate passes + SMEM program (n = 10), c128 and c64
rc = C.random_circuit(10, 60, 3, max_targets=3, max_controls=2)
exp = oracle.run(rc, oracle.basis_state(10, 5))
for fuse in (False, True):
    t = torch.empty(2**10, dtype=torch.complex128, device=dev)
    st = qj.State(t, basis=5)
    st.apply_circuit(rc.gates, fuse=fuse)
    st.canonicalize()
    st.sync()
    check(t, exp, 1e-12, f"random10 fuse={fuse}")
# JIT tile passes (n = 16: two-CTA / pair forms) and the live-tile simulate path
n = 16
qf = C.qft(n)
t = torch.empty(2**n, dtype=torch.complex128, device=dev)
st = qj.State(t, basis=None, stream=torch.cuda.Stream())
st.simulate(77, qf.gates, qubits=[0, 1, 2])
st.sync()
e, _ = oracle.qft_basis_maxerr(t.cpu().numpy(), n, 77, phys=st.layout())
assert e < 1e-12
print("ok simulate qft16", e, flush=True)
st.reset(77)
st.apply_circuit(qf.gates, fuse=True)
st.canonicalize()
st.sync()
e, _ = oracle.qft_basis_maxerr(t.cpu().numpy(), n, 77)
assert e < 1e-12
print("ok fused qft16", e, flush=True)
# live-tile simulate with paired tiles (n = 25: several tiles per CTA, odd counts)
for n, dtp, tol in ((25, torch.complex128, 1e-12), (25, torch.complex64, 1e-5)):
    t = torch.empty(2**n, dtype=dtp, device=dev)
    st = qj.State(t, basis=None, stream=torch.cuda.Stream())
    st.simulate(4242, C.qft(n).gates, qubits=[0, 1, 2])
    st.sync()
    e, _ = oracle.qft_basis_maxerr(t.cpu().numpy().astype(np.complex128), n, 4242, phys=st.layout())
    assert e < tol, e
    print("ok simulate qft25", dtp, e, flush=True)
    del st, t
# ring form (TMA): needs >= 148 tiles -> n = 20 c128
n = 20
t = torch.empty(2**n, dtype=torch.complex128, device=dev)
st = qj.State(t, basis=12345)
st.apply_circuit(C.qft(n).gates, fuse=True)
st.canonicalize()
st.sync()
e, _ = oracle.qft_basis_maxerr(t.cpu().numpy(), n, 12345)
assert e < 1e-12
print("ok ring qft20", e, flush=True)
# complex64 fused random circuit over several tiles, and a sharded fused run
sc = C.supremacy(4, 5, 8)
exp = oracle.run(sc, oracle.basis_state(sc.n, 0), [g.matrix().astype(np.complex64).astype(np.complex128) for g in sc.gates])
t = torch.empty(2**sc.n, dtype=torch.complex64, device=dev)
st = qj.State(t, basis=0)
st.apply_circuit(sc.gates, fuse=True)
st.canonicalize()
st.sync()
check(t, exp, 1e-5, "supremacy20 c64 fused")
shards = [torch.empty(2**18, dtype=torch.complex128, device=dev) for _ in range(4)]
sh = qj.State.sharded(shards, 20, basis=12345)
sh.apply_circuit(C.qft(20).gates, fuse=True)
sh.canonicalize()
sh.sync()
e, _ = oracle.qft_basis_maxerr(torch.cat(shards).cpu().numpy(), 20, 12345)
assert e < 1e-12
print("ok sharded qft20", e, flush=True)
# tensor-core dense 5-qubit pass (complex64, n = 12)
rng = np.random.default_rng(1)
psi = rng.standard_normal(2**12) + 1j * rng.standard_normal(2**12)
psi = (psi / np.linalg.norm(psi)).astype(np.complex64)
g5 = G.unitary("U5", (0, 3, 7, 9, 11), G.random_unitary(5, rng))
circ = C.Circuit(12, [g5])
exp = oracle.run(circ, psi.astype(np.complex128), [g5.matrix().astype(np.complex64).astype(np.complex128)])
x = torch.from_numpy(psi.copy()).to(dev)
st = qj.State(x, basis=None)
st.apply_gate(g5.targets, g5.data[0])
st.sync()
check(x, exp, 1e-5, "dense5 tensor cores")
# readout + measurement
p = st.probabilities([0, 5, 11])
pr = st.collapse([2], 1)
s, _ = qj.sample_distribution(p.double(), 1000, 7)
st.sync()
print("ok readout/measure", float(p.sum()), pr, flush=True)
print("sanitize driver done")
