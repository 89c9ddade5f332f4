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

Multi-GPU (torchrun, N>1): every rank runs its own QFT30 circuit (independent
problems, weak scaling, no data-path collective); the max over ranks of the
device time is used and value = that time / (steps * N).  The same run then
times QFT(30 + log2 N) sharded over the N ranks through NCCL global-qubit
swaps and reports it under "sharded" (a watchdog keeps a hang from losing the
line).
"""

from __future__ import annotations

import argparse
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
    """dram read+write bytes per launch from the committed ncu --set full capture."""
    for name in sorted(os.listdir(os.path.join(ROOT, "profiles")), reverse=True) if os.path.isdir(
            os.path.join(ROOT, "profiles")) else []:
        if name.startswith("ncu_traffic") and name.endswith(".json"):
            try:
                with open(os.path.join(ROOT, "profiles", name)) as f:
                    return json.load(f), name
            except Exception:
                pass
    return {}, None


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
    if name == "qft10_c128":
        return dict(n=10, dtype="c128", circ=C.qft(10), basis=SEED_X & 1023, readout=list(range(10)))
    raise SystemExit(f"unknown workload {name}")


# ----------------------------------------------------------------- oracle timing
def oracle_sample(wl, reps=1):
    """Time the CPU oracle on a bounded sample of the workload's gates applied
    to a full 2^n state and extrapolate to seconds per circuit: one gate of each
    (kind, #targets, #controls) class present in the circuit, weighted by the
    class counts (the oracle's cost per gate depends only on that class)."""
    import numpy as np
    import oracle

    n = wl["n"]
    classes = {}
    for g in wl["circ"].gates:
        key = (len(g.targets), len(g.controls))
        classes.setdefault(key, [g, 0])
        classes[key][1] += 1
    psi = oracle.basis_state(n, wl["basis"])
    out = np.empty_like(psi)
    total = 0.0
    parts = []
    for key, (g, cnt) in sorted(classes.items()):
        t0 = time.perf_counter()
        for _ in range(reps):
            oracle.apply_matrix(psi, out, n, g.targets, g.controls, g.matrix())
        dt = (time.perf_counter() - t0) / reps
        total += dt * cnt
        parts.append(f"{cnt}x[{key[0]}t,{key[1]}c] {dt:.3f}s")
    return total, "; ".join(parts), oracle.num_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    wl = make_workload(args.workload)
    vals = []
    for i in range(args.warmup + args.steps):
        v, sample, cores = oracle_sample(wl)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s/circuit",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "n": wl["n"], "gates": len(wl["circ"])},
        "cpu_baseline": {"value": value, "unit": "s/circuit", "cores": cores, "kind": "oracle",
                         "sample": f"one gate per class on a 2^{wl['n']} state, extrapolated by class "
                                   f"counts: {sample}"},
        "e2e": {"value": value, "unit": "s/circuit", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
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
    psi = torch.empty(1 << n, dtype=tdt, device=dev)
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
                clk=clk, dry=dry, ms_prof=ms_prof, flush_buf=flush_buf)


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
            "traffic": (tr["dram_bytes_per_launch"] if tr else None), "traffic_source": traffic_src}


def kinds_of(prof, steps, peak):
    return {k: {"launches_per_step": v["launches"] / steps, "ms_per_step": v["total_ms"] / steps,
                "GBps": v["alg_bytes"] / max(v["total_ms"], 1e-12) / 1e6,
                "frac": v["alg_bytes"] / max(v["total_ms"], 1e-12) / 1e6 / peak} for k, v in prof.items()}


def sharded_section(qj, torch, dev, world, rank, timeout_s, emit):
    """QFT(30 + log2 N) complex128 sharded over the N ranks (16 GiB per GPU):
    fused tile passes per rank, global-qubit swaps as NCCL exchanges.  One warm-up and one timed
    circuit; a watchdog keeps a hang from losing the main line."""
    import threading
    from workloads import circuits as C

    g = world.bit_length() - 1
    n = 30 + g

    def on_timeout():
        emit({"error": f"timeout after {timeout_s}s"})
        os._exit(0)

    wd = threading.Timer(timeout_s, on_timeout)
    wd.daemon = True
    wd.start()
    try:
        t = torch.empty(1 << (n - g), dtype=torch.complex128, device=dev)
        stream = torch.cuda.Stream(dev)
        with torch.cuda.stream(stream):
            st = qj.State.distributed(t, n, basis=SEED_X, stream=stream)
        circ = C.qft(n)
        packed = st.pack_circuit(circ.gates)
        pb = torch.empty(1 << 10, dtype=torch.float64, device=dev)
        st.apply_circuit(None, fuse=True, packed=packed)
        st.sync()
        st.reset(SEED_X)
        torch.cuda.synchronize(dev)
        torch.distributed.barrier()
        st.counters(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st.apply_circuit(None, fuse=True, packed=packed)
        st.probabilities(list(range(10)), out=pb)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        ctr = st.counters(reset=True)
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        psum = float(pb.sum().item())
        res = {"workload": f"qft{n}_c128_sharded", "n": n, "ranks": world, "s_per_circuit": float(tt.item()) / 1e3,
               "exchanges": ctr["exchanges"], "exchange_bytes_per_rank": ctr["exchange_bytes"],
               "alg_bytes_per_rank": ctr["alg_bytes"], "marginal_sum": psum,
               "note": "fused window tile passes per rank + NCCL local<->global swaps between them"}
        st.free()
        return res
    except Exception as e:  # report, never lose the main line
        return {"error": f"{type(e).__name__}: {e}"[:300]}
    finally:
        wd.cancel()


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
        h2d += 112  # sizeof(qj_gate)
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
                    "roofline": roofline_of(sc["prof"], sc["ms_prof"], peak, peak_src, traffic, traffic_src)}
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
                   "roofline": roofline_of(u["prof"], u["ms_prof"], peak, peak_src, traffic, traffic_src),
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
                 "roofline": roofline_of(pf["prof"], pf["ms_prof"], peak, peak_src, traffic, traffic_src)}
        pf["st"].free()
        del pf
        torch.cuda.empty_cache()

    ms_max = m["ms_max"]
    value = ms_max / 1e3 / (steps * world)
    per_step_bytes = m["ctr"]["alg_bytes"] / steps
    cpu = None
    if world == 1 and not args.no_cpu_baseline and rank == 0:
        v, sample, cores = oracle_sample(wl)
        cpu = {"value": v, "unit": "s/circuit", "cores": cores, "kind": "oracle",
               "sample": f"one gate per class on a 2^{n} state, extrapolated by class counts: {sample}"}
    state_bytes = amp_bytes << n
    line = {
        "metric": METRIC, "value": value, "unit": "s/circuit", "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms_max / steps, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if wl["dtype"] == "c128" else "f32",
        "data": "synthetic",
        "config": {"workload": args.workload, "n": n, "state": wl["dtype"], "gates": len(gates),
                   "basis": wl["basis"], "fuse": bool(args.fuse),
                   "step": ("qj_simulate: state reset + apply_circuit + 10-qubit marginal probabilities in one call"
                            if args.fuse else "state_reset + apply_circuit + 10-qubit marginal probabilities"),
                   "l2": (f"state {state_bytes >> 20} MiB >> 126 MB L2: inputs larger than L2, no flush"
                          if not needs_flush(wl) else
                          f"state {state_bytes >> 20} MiB fits L2: 256 MiB L2 flush before every timed step "
                          "(outside its CUDA-event pair; per-step event pairs summed)"),
                   "parallelism": f"{world} independent replicas (weak scaling)" if world > 1 else "1 GPU"},
        "effective_gbs": per_step_bytes / (ms_max / steps / 1e3) / 1e9,
        "effective_frac": per_step_bytes / (ms_max / steps / 1e3) / 1e9 / peak,
        "alg_bytes_per_step": per_step_bytes,
        "roofline": roofline_of(m["prof"], m["ms_prof"], peak, peak_src, traffic, traffic_src),
        "kinds": kinds_of(m["prof"], steps, peak),
        "profiled_ms_per_step": m["ms_prof"] / steps,
        "separate_calls": separate,
        "unfused": unfused,
        "paper_fusion": paper,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_ms / 1e3 / (steps * world), "unit": "s/circuit",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": m["ctr"]["launches"],
        "clocks": m["clk"].summary(),
        "dry_run_s": m["dry"], "lib_load_s": load_s,
        "parity_max_abs_err_sampled": check,
    }

    def emit(sharded):
        if rank == 0:
            line["sharded"] = sharded
            print(json.dumps(line), flush=True)

    if world > 1 and not args.no_sharded:
        emit(sharded_section(qj, torch, dev, world, rank, args.sharded_timeout, emit))
    else:
        emit(None)
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
    ap.add_argument("--no-sharded", action="store_true", help="N>1: skip the NCCL-sharded QFT section")
    ap.add_argument("--sharded-timeout", type=float, default=240.0)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        torch.distributed.init_process_group(
            "nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
    try:
        return run_qj(args, rank, world)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
