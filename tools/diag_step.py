"""Diagnose one bench step: host enqueue time of each call and device time of
each phase (reset / circuit / probabilities) for QFT30 c128."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_08826_b200 as qj
from workloads import circuits as C

WL = os.environ.get("WL", "qft")
n = int(os.environ.get("N", 30))
fuse = os.environ.get("FUSE", "1") == "1"
dev = torch.device("cuda", 0)
s = torch.cuda.Stream(dev)
psi = torch.empty(1 << n, dtype=torch.complex128, device=dev)
st = qj.State(psi, basis=None, stream=s)
circ = C.qft(n) if WL == "qft" else C.variational(n, layers=20)
packed = st.pack_circuit(circ.gates)
pb = torch.empty(1024, dtype=torch.float64, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for it in range(4):
    torch.cuda.synchronize()
    h = []
    t0 = time.perf_counter(); ev[0].record(s); st.reset(5); h.append(time.perf_counter() - t0)
    ev[1].record(s)
    t0 = time.perf_counter(); st.apply_circuit(None, fuse=fuse, packed=packed); h.append(time.perf_counter() - t0)
    ev[2].record(s)
    t0 = time.perf_counter(); st.probabilities(list(range(10)), out=pb); h.append(time.perf_counter() - t0)
    ev[3].record(s)
    torch.cuda.synchronize()
    d = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
    print(f"iter {it}: host ms reset/circuit/prob = " + "/".join(f"{x*1e3:.2f}" for x in h) +
          "   device ms = " + "/".join(f"{x:.2f}" for x in d), flush=True)
