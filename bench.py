#!/usr/bin/env python
"""bench.py -- seconds per circuit and effective HBM GB/s of the hot path
(BASELINE.json metric) on the 30-qubit complex128 QFT (BASELINE.json
configs[2], the configuration the north-star target is quoted on).

One step = one pass of the whole hot path over one synthetic input:
    qj_state_reset(|x>)            (a1: state layout / init)
    qj_apply_circuit(QFT30)        (a2-a6: every gate of the circuit)
    qj_probabilities(10 qubits)    (a7: Born-rule marginal readout)
Timed with CUDA events on the state's stream; the 16 GiB state is far larger
than the 126 MB L2, so no flush is needed between steps.

Arms:
  default          the sm_100a library through the C ABI (paper_2203_08826_b200)
  --impl reference the CPU oracle (oracle/, plain fp64 C/OpenMP Eq. 1) on the
                   host cores: each step applies a bounded sample of the QFT30
                   gates to a 2^30 state and extrapolates to s/circuit.

By default the fused planner runs (window tile passes, one HBM round trip per
run of gates); the per-gate-pass numbers (`--no-fuse` path) are measured in the
same run and reported under "unfused".

Multi-GPU (torchrun, N>1): the headline is ONE QFT circuit sharded over the
N ranks on its top log2 N qubits -- the north star's 35-qubit complex128 QFT
(512 GiB) at N = 4 / 8, 34 qubits at N = 2 -- fused tile passes
per rank, global-qubit swaps as pipelined NCCL exchanges; max over ranks of
the device time; with exchange bandwidth, E(N) per SURVEY C14 and a per-rank
closed-form check.  Independent per-rank QFT30 replicas are a side field.
`--sharded-n K` runs the sharded path at N = 1 too (one NCCL rank).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QFT/random-circuit sec per circuit and effective HBM GB/s vs peak, 1/2/4/8 B200"
SEED_X = 0b101101110001011100101101011011  # the seeded 30-bit basis input |x>


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    """DRAM read+write bytes per launch, measured by ncu on this workload and
    section (tools/ncu_traffic.py -> profiles/<round>/ncu_traffic.json, keyed
    workload -> section -> kernel kind); the newest round's file wins."""
    base = os.path.join(ROOT, "profiles")
    for name in sorted(os.listdir(base), reverse=True) if os.path.isdir(base) else []:
        p = os.path.join(base, name, "ncu_traffic.json")
        if name.startswith("r") and os.path.exists(p):
            try:
                with open(p) as f:
                    return json.load(f), os.path.relpath(p, ROOT)
            except Exception:
                pass
    return {}, None


def traffic_for(traffic, workload, section):
    return (traffic or {}).get(workload, {}).get(section, {})


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        self.reasons |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception:
                        pass
                    time.sleep(0.05)
            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=1)

    def summary(self):
        r = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": r, "samples": len(self.samples)}


# ----------------------------------------------------------------- workloads
def make_workload(name):
    from workloads import circuits as C
    if name == "qft30_c128":
        return dict(n=30, dtype="c128", circ=C.qft(30), basis=SEED_X, readout=list(range(10)))
    if name == "qft28_c128":
        return dict(n=28, dtype="c128", circ=C.qft(28), basis=SEED_X & ((1 << 28) - 1), readout=list(range(10)))
    if name == "var20_c128":
        return dict(n=20, dtype="c128", circ=C.variational(20, layers=20), basis=0, readout=list(range(10)))
    if name == "var20_c64":
        return dict(n=20, dtype="c64", circ=C.variational(20, layers=20), basis=0, readout=list(range(10)))
    if name == "sup32_c64":
        return dict(n=32, dtype="c64", circ=C.supremacy(4, 8, 20), basis=0, readout=list(range(10)))
    if name in ("tfim10_c128", "tfim20_c128"):
        # adiabatic TFIM evolution on 10 / 20 qubits by Trotter
        # decomposition; T = 1, dt = 0.01 (100 second-order steps, R24)
        from workloads import evolution as E
        nq = 10 if name.startswith("tfim10") else 20
        return dict(n=nq, dtype="c128", circ=E.adiabatic_circuit(nq, 1.0, 0.01), basis=0,
                    readout=list(range(10)))
    if name == "bv30_c128":  # SPEC S:520-528, Table 2 row bv (89 gates, secret all-ones)
        return dict(n=30, dtype="c128", circ=C.bv(30), basis=0, readout=list(range(10)))
    if name == "qaoa30_c128":  # north-star extra: QAOA-MaxCut p=2 on a seeded 3-regular graph
        return dict(n=30, dtype="c128", circ=C.qaoa(30, 2), basis=0, readout=list(range(10)))
    if name == "qft10_c128":
        return dict(n=10, dtype="c128", circ=C.qft(10), basis=SEED_X & 1023, readout=list(range(10)))
    raise SystemExit(f"unknown workload {name}")


# ----------------------------------------------------------------- oracle timing
WHOLE_CIRCUIT_MAX_N = 22  # the oracle runs whole circuits up to here; above, a per-class sample


def oracle_time(wl, threads=0, budget_s=30.0):
    """Seconds per circuit of the CPU oracle (plain fp64 Eq. 1, OpenMP) on
    this workload, measured on `threads` host threads (0 = all).

    n <= 22: the circuit's gates in order from |basis> until the whole circuit
    ran or `budget_s` passed; a partial run is extrapolated by gate count.
    n > 22: one gate of each (targets, controls) class applied to a full 2^n
    state, weighted by the class counts (the oracle's cost per gate depends
    only on the class).  Returns (s/circuit, sample text, cores used,
    extrapolated?, wall seconds spent)."""
    import numpy as np
    import oracle

    if threads:
        oracle.set_num_threads(threads)
    cores = oracle.num_threads()
    n = wl["n"]
    gates = wl["circ"].gates
    t_all = time.perf_counter()
    psi = oracle.basis_state(n, wl["basis"])
    out = np.empty_like(psi)
    try:
        if n <= WHOLE_CIRCUIT_MAX_N:
            t0 = time.perf_counter()
            done = 0
            for g in gates:
                oracle.apply_matrix(psi, out, n, g.targets, g.controls, g.matrix())
                psi, out = out, psi
                done += 1
                if time.perf_counter() - t0 > budget_s:
                    break
            el = time.perf_counter() - t0
            value = el * len(gates) / done
            extra = done < len(gates)
            sample = (f"whole circuit ({len(gates)} gates) from |basis>" if not extra else
                      f"first {done} of {len(gates)} gates from |basis>, extrapolated by gate count")
        else:
            per = oracle_class_times(psi, out, n, gates)
            counts = class_counts(gates)
            value = sum(per[k] * c for k, c in counts.items())
            extra = True
            sample = f"one gate per class on a 2^{n} state, extrapolated by class counts: " + "; ".join(
                f"{counts[k]}x[{k[0]}t,{k[1]}c] {per[k]:.3f}s" for k in sorted(per))
    finally:
        if threads:
            oracle.set_num_threads(os.cpu_count() or 1)
    return value, sample, cores, extra, time.perf_counter() - t_all


def class_counts(gates):
    counts = {}
    for g in gates:
        key = (len(g.targets), len(g.controls))
        counts[key] = counts.get(key, 0) + 1
    return counts


def oracle_class_times(psi, out, n, gates):
    """Seconds the oracle takes for one gate of each (targets, controls)
    class present in `gates` on the 2^n state psi (out = second buffer)."""
    import oracle
    first = {}
    for g in gates:
        first.setdefault((len(g.targets), len(g.controls)), g)
    per = {}
    for key, g in sorted(first.items()):
        t0 = time.perf_counter()
        oracle.apply_matrix(psi, out, n, g.targets, g.controls, g.matrix())
        per[key] = time.perf_counter() - t0
    return per


def cpu_baseline_of(wl):
    v, sample, cores, extra, _ = oracle_time(wl)
    cpu = {"value": v, "unit": "s/circuit", "cores": cores, "kind": "oracle", "sample": sample,
           "extrapolated": extra}
    if wl["n"] <= 20:  # the small configs also on one host thread
        v1, s1, c1, x1, _ = oracle_time(wl, threads=1, budget_s=20.0)
        cpu["single_thread"] = {"value": v1, "unit": "s/circuit", "cores": c1, "sample": s1, "extrapolated": x1}
    return cpu


def config_of(args, wl, world):
    """The config dict both arms print (same workload, same keys)."""
    amp = 16 if wl["dtype"] == "c128" else 8
    state_bytes = amp << wl["n"]
    return {"workload": args.workload, "n": wl["n"], "state": wl["dtype"], "gates": len(wl["circ"]),
            "basis": wl["basis"], "fuse": bool(args.fuse),
            "step": ("qj_simulate: state reset + apply_circuit + 10-qubit marginal probabilities in one call"
                     if args.fuse else "state_reset + apply_circuit + 10-qubit marginal probabilities"),
            "l2": (f"state {state_bytes >> 20} MiB >> 126 MB L2: inputs larger than L2, no flush"
                   if not needs_flush(wl) else
                   f"state {state_bytes >> 20} MiB fits L2: 256 MiB L2 flush before every timed step "
                   "(outside its CUDA-event pair; per-step event pairs summed)"),
            "parallelism": "1 GPU" if world == 1 else f"{world} ranks"}


def run_reference(args, rank, world):
    """The reference arm: the CPU oracle as it stands, on the host cores.  Each
    step is one bounded oracle run of this workload (whole circuit for n <= 22,
    else one gate per class on the full state); `value` is seconds per circuit
    (extrapolated where the step is a sample), `ms_per_step` the wall time one
    step actually took, so ms_per_step x steps is this run's oracle time."""
    if rank != 0:
        return 0
    if world > 1 or args.sharded_n:
        return run_reference_sharded(args, world)
    wl = make_workload(args.workload)
    vals, walls = [], []
    for i in range(args.warmup + args.steps):
        v, sample, cores, extra, wall = oracle_time(wl)
        if i >= args.warmup:
            vals.append(v)
            walls.append(wall)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s/circuit",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(walls) * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args, wl, 1),
        "extrapolated": extra,
        "cpu_baseline": {"value": value, "unit": "s/circuit", "cores": cores, "kind": "oracle", "sample": sample,
                         "extrapolated": extra},
        "e2e": {"value": value, "unit": "s/circuit", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference_sharded(args, world):
    """Reference arm for the N > 1 headline (one QFT(34 / 35) circuit): the
    oracle cannot hold 2^35 complex128 amplitudes (512 GiB, two buffers) in
    host memory, so each step times one gate per (targets, controls) class of
    that circuit on a 2^30 state and scales by 2^(n - 30) -- the oracle's cost
    per gate is linear in the state size (labelled extrapolated)."""
    import numpy as np
    import oracle
    from workloads import circuits as C
    n = args.sharded_n or sharded_n(world)
    big = C.qft(n)
    counts = class_counts(big.gates)
    small = [g for g in C.qft(30).gates]  # same gate classes, on qubits a 2^30 state has
    cores = oracle.num_threads()
    vals, walls = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        psi = oracle.basis_state(30, SEED_X)
        out = np.empty_like(psi)
        per = oracle_class_times(psi, out, 30, small)
        del psi, out
        v = sum(per[k] * c for k, c in counts.items()) * 2.0 ** (n - 30)
        walls.append(time.perf_counter() - t0)
        if i >= args.warmup:
            vals.append(v)
    walls = walls[args.warmup:]
    sample = "; ".join(f"{counts[k]}x[{k[0]}t,{k[1]}c] {per[k]:.3f}s" for k in sorted(per))
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s/circuit", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(walls) * 1e3,
            "higher_is_better": False, "scaling": "strong" if world >= 4 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "extrapolated": True,
            "config": sharded_config(n, world),
            "cpu_baseline": {"value": value, "unit": "s/circuit", "cores": cores, "kind": "oracle", "extrapolated": True,
                             "sample": f"one gate per class on a 2^30 state, scaled by class counts of QFT{n} and "
                                       f"2^{n - 30} (oracle cost linear in the state size): {sample}"},
            "e2e": {"value": value, "unit": "s/circuit", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- qj arm
L2_FLUSH_BELOW = 256 << 20  # states smaller than 2x the 126 MB L2 are timed with a flush between steps


def needs_flush(wl):
    return ((16 if wl["dtype"] == "c128" else 8) << wl["n"]) < L2_FLUSH_BELOW


def timed_steps(torch, stream, steps, step, flush_buf):
    """Device time (ms) of `steps` calls of step() on `stream`.  Without a
    flush buffer: one event pair around all steps (the state is larger than
    L2).  With one: every step is preceded by a 256 MiB write of the flush
    buffer (outside the events) and timed by its own event pair; the sum is
    returned."""
    if flush_buf is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        stream.synchronize()
        return e0.elapsed_time(e1)
    pairs = []
    for i in range(steps):
        with torch.cuda.stream(stream):
            flush_buf.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        pairs.append((a, b))
    stream.synchronize()
    return sum(a.elapsed_time(b) for a, b in pairs)


def measure(qj, torch, wl, fuse, steps, warmup, dev, world, profile=True, fuse_gates=False, simulate=False):
    """Time `steps` steps (state reset + circuit + 10-qubit marginal) on the
    device with CUDA events; returns timings, per-kind profile and counters.
    simulate=True runs the step as ONE qj_simulate call (the first tile pass
    synthesises |basis>, the last one accumulates the marginal); otherwise as
    qj_state_reset + qj_apply_circuit + qj_probabilities."""
    n = wl["n"]
    tdt = torch.complex128 if wl["dtype"] == "c128" else torch.complex64
    stream = torch.cuda.Stream(dev)
    flush_buf = torch.empty(L2_FLUSH_BELOW, dtype=torch.uint8, device=dev) if needs_flush(wl) else None
    torch.cuda.synchronize(dev)
    free0 = torch.cuda.mem_get_info(dev)[0]
    psi = torch.empty(1 << n, dtype=tdt, device=dev)
    torch.cuda.synchronize(dev)
    free1 = torch.cuda.mem_get_info(dev)[0]
    st = qj.State(psi, basis=None, stream=stream)
    packed = st.pack_circuit(wl["circ"].gates)
    readout = wl["readout"]
    pbuf = torch.empty(1 << len(readout), dtype=st.real_dtype, device=dev)

    def step():
        if simulate:
            st.simulate(wl["basis"], qubits=readout, fuse=fuse, fuse_gates=fuse_gates, packed=packed, out=pbuf)
            return
        st.reset(wl["basis"])
        st.apply_circuit(None, fuse=fuse, packed=packed, fuse_gates=fuse_gates)
        st.probabilities(readout, out=pbuf)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    step()  # dry run: first circuit of this configuration
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    dry = ev0.elapsed_time(ev1) / 1e3
    for _ in range(max(0, warmup - 1)):
        step()
    barrier()
    st.counters(reset=True)
    barrier()
    with ClockSampler(dev.index) as clk:
        ms = timed_steps(torch, stream, steps, step, flush_buf)
        torch.cuda.synchronize(dev)
    barrier()
    ctr = st.counters(reset=True)
    free2 = torch.cuda.mem_get_info(dev)[0]
    # Table 3: m = device memory of the run, dm = what the
    # library holds beyond the caller's state buffer (plans, program buffers,
    # staging, bins, JIT modules); the free-memory deltas include allocator
    # rounding
    mem = {"state_bytes": psi.numel() * psi.element_size(), "state_alloc_bytes": free0 - free1,
           "library_bytes": free1 - free2, "m_bytes": free0 - free2,
           "how": "cudaMemGetInfo deltas: before the state alloc, after it, after the timed steps"}
    # per-pass device times: a profiled repeat of the same timed steps (CUDA
    # events around every pass on the state's stream; no graph replay)
    prof, ms_prof = {}, ms
    if profile:
        st.set_profiling(True)
        st.profile(reset=True)
        ms_prof = timed_steps(torch, stream, steps, step, flush_buf)
        prof = st.profile(reset=True)
        st.set_profiling(False)
        st.counters(reset=True)
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_max = float(t.item())
    return dict(st=st, psi=psi, stream=stream, pbuf=pbuf, ms=ms, ms_max=ms_max, prof=prof, ctr=ctr,
                clk=clk, dry=dry, ms_prof=ms_prof, flush_buf=flush_buf, mem=mem)


def roofline_of(prof, ms_step_total, peak, peak_src, traffic, traffic_src):
    if not prof:
        return None
    k, d = max(prof.items(), key=lambda kv: kv[1]["total_ms"])
    ach = d["alg_bytes"] / (d["total_ms"] / 1e3) / 1e9
    tr = traffic.get(k) if traffic else None
    return {"bound": "hbm", "kernel": k, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "peak_source": peak_src, "alg_bytes_per_launch": d["alg_bytes"] / d["launches"],
            "avg_launch_us": d["total_ms"] / d["launches"] * 1e3,
            "share_of_step": d["total_ms"] / max(ms_step_total, 1e-9),
            "traffic": (tr["dram_bytes_per_launch"] if tr else None),
            "traffic_source": (traffic_src if tr else None)}


def kinds_of(prof, steps, peak):
    return {k: {"launches_per_step": v["launches"] / steps, "ms_per_step": v["total_ms"] / steps,
                "GBps": v["alg_bytes"] / max(v["total_ms"], 1e-12) / 1e6,
                "frac": v["alg_bytes"] / max(v["total_ms"], 1e-12) / 1e6 / peak} for k, v in prof.items()}


def sharded_n(world):
    """Qubits of the N>1 headline: the north star's 35-qubit QFT (512 GiB
    complex128) at P = 4 / 8 (128 / 64 GiB per GPU); 34 qubits at P = 2
    (35 q would need 256 GiB per GPU); 30 + log2 P below that."""
    g = world.bit_length() - 1
    return 35 if world >= 4 else 34 if world == 2 else 30 + g


def sharded_basis(n):
    x = SEED_X | (0b10110 << 30) if n > 30 else SEED_X
    return x & ((1 << n) - 1)


def sharded_config(n, world):
    """The config dict of the N > 1 headline (both arms)."""
    from workloads import circuits as C
    g = world.bit_length() - 1
    nl = n - g
    return {"workload": f"qft{n}_c128_sharded", "n": n, "state": "c128", "gates": len(C.qft(n)),
            "basis": sharded_basis(n), "fuse": True, "global_qubits": g, "shard_gib": (16 << nl) / 2**30,
            "step": "qj_state_reset + qj_apply_circuit(QJ_FUSE) + 10-qubit marginal (NCCL all-reduce)",
            "l2": f"shard {(16 << nl) >> 30} GiB >> 126 MB L2: no flush",
            "parallelism": f"state sharded over {world} ranks on the top {g} qubits (NCCL exchanges)"}


def run_sharded(args, rank, world):
    """N>1 headline: one QFT(n) complex128
    circuit sharded over the N ranks on its top log2 N qubits; fused window
    tile passes on every rank, global-qubit work through local<->global swaps
    exchanged with NCCL (grouped send/recv, pipelined through the staging
    ring).  Step = reset(|x>) + circuit + 10-qubit marginal (all-reduced).
    Timed with CUDA events on each rank's stream, max over ranks.  A
    profiled repeat splits each rank's time into local passes and exchanges:
    E(N) = T1_hat / (N T_N) with T1_hat = the local-pass time of all N shards
    back to back on one GPU at the same per-pass bandwidth;
    exchange bandwidth = bytes each rank sends / exchange time.  Replicas
    (each rank its own QFT30) are reported as a side field."""
    import threading

    import numpy as np
    import torch

    import paper_2203_08826_b200 as qj
    from workloads import circuits as C

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    g = world.bit_length() - 1
    n = args.sharded_n or sharded_n(world)
    nl = n - g
    x = sharded_basis(n)
    peak, peak_src = load_peaks()
    steps = args.steps
    line = {"metric": METRIC, "unit": "s/circuit", "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "higher_is_better": False, "scaling": "strong" if world >= 4 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": sharded_config(n, world)}

    def emit_error(msg):
        if rank == 0:
            line["value"] = None
            line["error"] = msg
            print(json.dumps(line), flush=True)
        os._exit(0)

    wd = threading.Timer(args.sharded_timeout, lambda: emit_error(f"timeout after {args.sharded_timeout}s"))
    wd.daemon = True
    wd.start()
    t = torch.empty(1 << nl, dtype=torch.complex128, device=dev)
    stream = torch.cuda.Stream(dev)
    st = qj.State.distributed(t, n, basis=x, stream=stream)
    circ = C.qft(n)
    packed = st.pack_circuit(circ.gates)
    readout = list(range(10))
    pb = torch.empty(1 << len(readout), dtype=torch.float64, device=dev)

    def step():
        st.reset(x)
        st.apply_circuit(None, fuse=True, packed=packed)
        st.probabilities(readout, out=pb)

    def barrier():
        torch.cuda.synchronize(dev)
        torch.distributed.barrier()

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step()  # dry run (plan, JIT, NCCL setup)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    dry = e0.elapsed_time(e1) / 1e3
    for _ in range(max(0, args.warmup - 1)):
        step()
    barrier()
    st.counters(reset=True)
    barrier()
    with ClockSampler(dev.index) as clk:
        ms = timed_steps(torch, stream, steps, step, None)
        torch.cuda.synchronize(dev)
    barrier()
    ctr = st.counters(reset=True)
    # e2e: the public API with the host gate list packed every step and the
    # marginal read back to pinned host memory
    host_out = torch.empty(1 << len(readout), dtype=torch.float64, pin_memory=True)

    def e2e_step():
        st.reset(x)
        st.apply_circuit(circ.gates, fuse=True)
        st.probabilities(readout, out=pb)
        with torch.cuda.stream(stream):
            host_out.copy_(pb, non_blocking=True)
        stream.synchronize()

    barrier()
    e2e_ms = timed_steps(torch, stream, steps, e2e_step, None)
    gsz = ctypes.sizeof(qj.qj.qj_gate)
    h2d = sum(gsz + (4 ** len(gg.targets) * 16 if gg.kind == "dense" else 2 ** len(gg.targets) * 16
                     if gg.kind == "diag" else 0) for gg in circ.gates)
    # profiled repeat: per-kind device times on this rank (events around every
    # pass / exchange on the state's stream)
    st.set_profiling(True)
    st.profile(reset=True)
    ms_prof = timed_steps(torch, stream, steps, step, None)
    prof = st.profile(reset=True)
    st.set_profiling(False)
    torch.cuda.synchronize(dev)
    ex = prof.get("exchange", {"total_ms": 0.0, "alg_bytes": 0.0, "launches": 0})
    local_ms = sum(v["total_ms"] for k, v in prof.items() if k != "exchange")
    # per-rank closed-form check of the final state (canonical slice of this
    # rank): a contiguous 2^22-amplitude chunk at a seeded offset + 4096 samples
    st.canonicalize()
    rng = np.random.default_rng(35 + rank)
    off = int(rng.integers(0, (1 << nl) - (1 << 22))) if nl > 22 else 0
    idx = np.unique(np.concatenate([np.arange(off, off + min(1 << 22, 1 << nl)), rng.integers(0, 1 << nl, 4096)]))
    got = t[torch.from_numpy(idx.astype(np.int64)).to(dev)].cpu().numpy()
    y = (np.uint64(rank) << np.uint64(nl)) | idx.astype(np.uint64)
    mm = (np.uint64(x) * y) & np.uint64((1 << n) - 1)
    exp = 2 ** (-n / 2) * np.exp(2j * np.pi * mm.astype(np.float64) / (1 << n))
    err = float(np.max(np.abs(got - exp)))
    marg = float(np.max(np.abs(pb.cpu().numpy() - 2.0 ** -len(readout))))
    vals = torch.tensor([ms, ms_prof, local_ms, ex["total_ms"], err, marg, e2e_ms], device=dev, dtype=torch.float64)
    mx = vals.clone()
    torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
    ms_max, msp_max, local_max, ex_max, err_max, marg_max, e2e_max = (float(v) for v in mx.tolist())
    st.free()
    del t
    torch.cuda.empty_cache()
    wd.cancel()
    # replicas (side field): every rank its own 2^30 QFT, no data-path collective
    replicas = None
    if not args.no_replicas:
        wl = make_workload("qft30_c128")
        r = measure(qj, torch, wl, True, max(1, min(steps, 3)), 2, dev, world, profile=False, simulate=True)
        rs = max(1, min(steps, 3))
        replicas = {"workload": "qft30_c128 x N (independent circuits)", "value": r["ms_max"] / 1e3 / (rs * world),
                    "unit": "s/circuit (aggregate over ranks)", "steps": rs, "scaling": "weak"}
        r["st"].free()
        del r
        torch.cuda.empty_cache()
    T_N = msp_max / steps / 1e3
    # every rank's non-exchange device time (passes, reset, readout) is work one
    # GPU would do for that shard at the same per-pass bandwidth
    T1_hat = world * (msp_max - ex_max) / steps / 1e3
    xbytes = ex["alg_bytes"] / steps  # bytes this rank sends per step (= receives)
    line.update({
        "value": ms_max / 1e3 / steps, "ms_per_step": ms_max / steps,
        "efficiency": {"E": T1_hat / (world * T_N), "T1_hat_s": T1_hat, "T_N_s": T_N,
                       "definition": "SURVEY C14: T1_hat = N x (profiled step time - exchange time), max over "
                                     "ranks = one GPU doing every shard's local work (passes, reset, readout) at "
                                     "the same per-pass bandwidth; T_N = profiled step time (max over ranks); "
                                     "E = 1 - the exchange share of the slowest rank's step"},
        "exchange": {"exchanges_per_step": ctr["exchanges"] / steps, "bytes_per_rank_per_step": xbytes,
                     "ms_per_step": ex_max / steps,
                     "GBps_per_direction": xbytes / max(ex_max / steps / 1e3, 1e-12) / 1e9,
                     "link_ref_GBps": 770.0, "link_ref": "measured NVLink peer copy per direction (B200_PROFILING.md)"},
        "local_passes": {"ms_per_step": local_max / steps,
                         "alg_bytes_per_rank_per_step": ctr["alg_bytes"] / steps,
                         "GBps": ctr["alg_bytes"] / steps / max(local_max / steps / 1e3, 1e-12) / 1e9,
                         "frac": ctr["alg_bytes"] / steps / max(local_max / steps / 1e3, 1e-12) / 1e9 / peak},
        "kinds": kinds_of(prof, steps, peak),
        "roofline": roofline_of({k: v for k, v in prof.items() if k != "exchange"}, ms_prof, peak, peak_src,
                                None, None),
        "gpu_launches": ctr["launches"],
        "clocks": clk.summary(), "dry_run_s": dry,
        "parity_max_abs_err_sampled": max(err_max, marg_max),
        "parity_check": "per rank: canonical slice, contiguous 2^22 chunk + 4096 samples vs the QFT|x> closed form; "
                        "marginal vs uniform 2^-10",
        "replicas": replicas,
        "cpu_baseline": None,
        "e2e": {"value": e2e_max / 1e3 / steps, "unit": "s/circuit", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": host_out.numel() * 8},
    })
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def run_qj(args, rank, world):
    import numpy as np
    import torch

    import paper_2203_08826_b200 as qj

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    wl = make_workload(args.workload)
    n = wl["n"]
    amp_bytes = 16 if wl["dtype"] == "c128" else 8
    t_load0 = time.perf_counter()
    qj.lib()
    load_s = time.perf_counter() - t_load0
    steps = args.steps
    peak, peak_src = load_peaks()
    traffic, traffic_src = load_traffic()

    # ---- headline: the default planner (fused window passes unless --no-fuse),
    # the step as one qj_simulate call
    m = measure(qj, torch, wl, args.fuse, steps, args.warmup, dev, world, simulate=args.fuse)
    st, psi, stream = m["st"], m["psi"], m["stream"]

    # ---- e2e: the public API with host buffers each step ----
    readout = wl["readout"]
    host_out = torch.empty(1 << len(readout), dtype=st.real_dtype, pin_memory=True)
    h2d = 0
    gates = wl["circ"].gates
    for g in gates:
        h2d += ctypes.sizeof(qj.qj.qj_gate)
        if g.kind in ("dense", "diag", "fsim"):
            cnt = {"dense": 4 ** len(g.targets), "diag": 2 ** len(g.targets), "fsim": 5}[g.kind]
            h2d += cnt * amp_bytes
    d2h = host_out.numel() * host_out.element_size()
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()

    def e2e_step():
        if args.fuse:  # packs the host gate list each step
            p = st.simulate(wl["basis"], gates, qubits=readout, fuse=True, out=m["pbuf"])
        else:
            st.reset(wl["basis"])
            st.apply_circuit(gates, fuse=False)
            p = st.probabilities(readout, out=m["pbuf"])
        with torch.cuda.stream(stream):
            host_out.copy_(p, non_blocking=True)
        stream.synchronize()

    e2e_ms = timed_steps(torch, stream, steps, e2e_step, m["flush_buf"])
    torch.cuda.synchronize(dev)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- parity spot check of the benched state (not timed) ----
    check = None
    if args.workload.startswith("qft"):
        st.canonicalize()
        rng = np.random.default_rng(30)
        idx = np.unique(np.concatenate([rng.integers(0, 1 << n, 4096), [0, (1 << n) - 1]])).astype(np.int64)
        got = psi[torch.from_numpy(idx).to(dev)].cpu().numpy()
        mm = (np.uint64(wl["basis"]) * idx.astype(np.uint64)) % np.uint64(1 << n)
        exp = 2 ** (-n / 2) * np.exp(2j * np.pi * mm.astype(np.float64) / (1 << n))
        check = float(np.max(np.abs(got - exp)))
        # |QFT|x>|^2 is uniform: every bin of the 10-qubit marginal is 2^-10
        marg_err = float(np.max(np.abs(m["pbuf"].cpu().numpy() - 2.0 ** -len(wl["readout"]))))
        check = max(check, marg_err)
    st.free()
    del psi, m["psi"]
    torch.cuda.empty_cache()

    # ---- the same fused passes as three calls (reset + apply_circuit + probabilities) ----
    separate = None
    if args.fuse and not args.no_unfused:
        sc = measure(qj, torch, wl, True, max(1, min(steps, 3)), 1, dev, world)
        ss = max(1, min(steps, 3))
        separate = {"value": sc["ms_max"] / 1e3 / (ss * world), "unit": "s/circuit", "steps": ss,
                    "step": "qj_state_reset + qj_apply_circuit(QJ_FUSE) + qj_probabilities",
                    "roofline": roofline_of(sc["prof"], sc["ms_prof"], peak, peak_src,
                                            traffic_for(traffic, args.workload, "separate"), traffic_src)}
        sc["st"].free()
        del sc
        torch.cuda.empty_cache()

    # ---- per-gate passes (the north star's "per gate pass" bandwidth) ----
    unfused = None
    if args.fuse and not args.no_unfused:
        u = measure(qj, torch, wl, False, max(1, min(steps, 3)), 1, dev, world)
        us = max(1, min(steps, 3))
        ub = u["ctr"]["alg_bytes"] / us
        unfused = {"value": u["ms_max"] / 1e3 / (us * world), "unit": "s/circuit", "steps": us,
                   "effective_gbs": ub / (u["ms_max"] / us / 1e3) / 1e9,
                   "effective_frac": ub / (u["ms_max"] / us / 1e3) / 1e9 / peak,
                   "roofline": roofline_of(u["prof"], u["ms_prof"], peak, peak_src,
                                           traffic_for(traffic, args.workload, "unfused"), traffic_src),
                   "kinds": kinds_of(u["prof"], us, peak), "gpu_launches": u["ctr"]["launches"]}
        u["st"].free()
        del u
        torch.cuda.empty_cache()

    # ---- the paper's own fusion: greedy <= 2-qubit dense
    # gates, then one pass per fused gate (row f1 of SURVEY 8(f))
    paper = None
    if args.fuse and not args.no_unfused:
        pf = measure(qj, torch, wl, False, max(1, min(steps, 3)), 1, dev, world, fuse_gates=True)
        ps = max(1, min(steps, 3))
        pb = pf["ctr"]["alg_bytes"] / ps
        paper = {"value": pf["ms_max"] / 1e3 / (ps * world), "unit": "s/circuit", "steps": ps,
                 "passes_per_circuit": pf["ctr"]["passes"] / ps,
                 "effective_gbs": pb / (pf["ms_max"] / ps / 1e3) / 1e9,
                 "effective_frac": pb / (pf["ms_max"] / ps / 1e3) / 1e9 / peak,
                 "roofline": roofline_of(pf["prof"], pf["ms_prof"], peak, peak_src,
                                         traffic_for(traffic, args.workload, "paper_fusion"), traffic_src)}
        pf["st"].free()
        del pf
        torch.cuda.empty_cache()

    ms_max = m["ms_max"]
    value = ms_max / 1e3 / (steps * world)
    per_step_bytes = m["ctr"]["alg_bytes"] / steps
    cpu = None
    if world == 1 and not args.no_cpu_baseline and rank == 0:
        cpu = cpu_baseline_of(wl)
    line = {
        "metric": METRIC, "value": value, "unit": "s/circuit", "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms_max / steps, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if wl["dtype"] == "c128" else "f32",
        "data": "synthetic",
        "config": config_of(args, wl, world),
        "effective_gbs": per_step_bytes / (ms_max / steps / 1e3) / 1e9,
        "effective_frac": per_step_bytes / (ms_max / steps / 1e3) / 1e9 / peak,
        "alg_bytes_per_step": per_step_bytes,
        "roofline": roofline_of(m["prof"], m["ms_prof"], peak, peak_src,
                                traffic_for(traffic, args.workload, "simulate" if args.fuse else "unfused"),
                                traffic_src),
        "kinds": kinds_of(m["prof"], steps, peak),
        "memory": m["mem"],
        "profiled_ms_per_step": m["ms_prof"] / steps,
        "separate_calls": separate,
        "unfused": unfused,
        "paper_fusion": paper,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_ms / 1e3 / (steps * world), "unit": "s/circuit",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "inputs": "every step: the Python gate list packed into qj_gate records + coefficients "
                          "(h2d_bytes_per_step) and passed with the basis index through the C ABI; the library "
                          "compares every record and coefficient with its cached plan's key and, when equal, "
                          "replays the plan whose device tables hold those same values (a changed gate list "
                          "re-plans and uploads); the marginal is copied to pinned host memory and synchronised"},
        "gpu_launches": m["ctr"]["launches"],
        "clocks": m["clk"].summary(),
        "dry_run_s": m["dry"], "lib_load_s": load_s,
        "parity_max_abs_err_sampled": check,
    }

    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="qj", choices=["qj", "reference"])
    ap.add_argument("--workload", default="qft30_c128")
    ap.add_argument("--fuse", dest="fuse", action="store_true", default=True)
    ap.add_argument("--no-fuse", dest="fuse", action="store_false")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-unfused", action="store_true", help="skip the per-gate-pass measurement")
    ap.add_argument("--no-replicas", action="store_true", help="N>1: skip the independent-replica side field")
    ap.add_argument("--sharded-n", type=int, default=0,
                    help="qubits of the sharded headline (default: 35 at N>=4, 34 at N=2); at N=1 runs the "
                         "sharded path on one NCCL rank")
    ap.add_argument("--sharded-timeout", type=float, default=600.0)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1 or args.sharded_n:  # (--sharded-n at N=1: the sharded path on one NCCL rank)
        import torch
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        torch.distributed.init_process_group(
            "nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
    try:
        if world > 1 or args.sharded_n:
            return run_sharded(args, rank, world)
        return run_qj(args, rank, world)
    finally:
        if world > 1 or args.sharded_n:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
