"""Full-size GPU parity: every amplitude of the BASELINE-sized states, in the
launch configuration bench.py times, against the oracle side.

* QFT30 (complex128, 16 GiB; complex64, 8 GiB) from the seeded basis input
  |x>: the whole device state is streamed to host memory in 1 GiB chunks and
  every one of the 2^30 amplitudes is checked against the closed form
  QFT|x> = 2^{-n/2} sum_y e^{2 pi i x y / 2^n} |y> by the oracle's
  or_qft_basis_maxerr (integer phase numerator; pinned in
  tests/test_oracle_pins.py).  qj_simulate is checked in the physical layout
  it leaves (its final SWAP layer is a relabelling, R21), so the
  exact bench output is what is compared.
* supremacy-style random circuits (complex64, SURVEY 8(d) config 4 on a 4x6
  grid, 24 qubits) element-wise against the gate-by-gate oracle; the 4x7 grid
  (28 qubits) runs when QJ_SLOW_TESTS=1 (minutes of oracle time).
* controlled fSim at every bit position, sharded amplitudes (not only |psi|^2),
  the in-place invariant (device memory the library takes across a 16 GiB
  circuit), and a live-tile pass whose window repeats the first one.

Tolerances: north star / reading R8 (1e-12 complex128, 1e-5 complex64).
"""

import math
import os

import numpy as np
import pytest

import oracle
from workloads import circuits as C
from workloads import gates as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
qjp = pytest.importorskip("paper_2203_08826_b200")

TOL = {np.complex128: 1e-12, np.complex64: 1e-5}
TDT = {np.complex128: torch.complex128, np.complex64: torch.complex64}
SEED_X = 0b101101110001011100101101011011  # bench.py's basis input
CHUNK = 1 << 26                            # amplitudes per host chunk (1 GiB complex128)


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2203_08826_b200 import build
    build.build()


def qft_check_full(t, n, x, phys=None):
    """(max abs error, l2 error) of the whole device state `t` against
    QFT|x>, streamed through a pinned host buffer."""
    chunk = min(CHUNK, t.numel())
    host = torch.empty(chunk, dtype=t.dtype, pin_memory=True)
    worst, ss = 0.0, 0.0
    for off in range(0, t.numel(), chunk):
        host.copy_(t[off:off + chunk])
        m, s = oracle.qft_basis_maxerr(host.numpy(), n, x, offset=off, phys=phys)
        worst = max(worst, m)
        ss += s
    return worst, math.sqrt(ss)


def free_bytes():
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info()[0]


# ------------------------------------------------ QFT30, all 2^30 amplitudes
@pytest.mark.slow
@pytest.mark.parametrize("dt", [np.complex128, np.complex64], ids=["c128", "c64"])
def test_qft30_simulate_every_amplitude(dt):
    """The bench step exactly: qj_simulate(QFT30, |x>, 10-qubit marginal) on a
    non-default stream, third call (the first plans, the second captures the
    CUDA graph, the third replays it).  All 2^30 amplitudes in the layout the
    step leaves, plus the marginal (uniform for QFT|x>)."""
    n = 30
    stream = torch.cuda.Stream()
    t = torch.empty(2**n, dtype=TDT[dt], device="cuda")
    st = qjp.State(t, basis=None, stream=stream)
    packed = st.pack_circuit(C.qft(n).gates)
    q = list(range(10))
    for _ in range(3):
        with torch.cuda.stream(stream):
            t.fill_(float("nan"))  # nothing stale can pass (ordered on the state's stream)
        p = st.simulate(SEED_X, qubits=q, packed=packed)
        st.sync()
    phys = st.layout()
    assert sorted(phys) == list(range(n))
    worst, l2 = qft_check_full(t, n, SEED_X, phys)
    assert worst <= TOL[dt], f"max abs err {worst:.3e}"
    assert l2 <= (1e-10 if dt == np.complex128 else 1e-3), f"l2 err {l2:.3e}"
    assert np.max(np.abs(p.cpu().numpy() - 2.0**-10)) <= TOL[dt]
    del st, t
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dt", [np.complex128, np.complex64], ids=["c128", "c64"])
@pytest.mark.parametrize("n", [13, 17, 23, 25, 27])
def test_qft_simulate_every_amplitude_sizes(dt, n):
    """qj_simulate(QFT n, |x>) at sizes whose live-tile passes give CTAs odd
    tile counts (paired live tiles: the last pair's second tile is absent) and
    one or two tiles in all (n = 13); every amplitude against the closed form."""
    x = (0x2D5A3C9 * n + 777) & ((1 << n) - 1)
    t = torch.empty(2**n, dtype=TDT[dt], device="cuda")
    st = qjp.State(t, basis=None)
    t.fill_(float("nan"))
    p = st.simulate(x, C.qft(n).gates, qubits=[0, n // 2, n - 1], fuse=True)
    st.sync()
    phys = st.layout()
    worst, _ = qft_check_full(t, n, x, phys)
    assert worst <= TOL[dt], f"max abs err {worst:.3e}"
    assert np.max(np.abs(p.cpu().numpy() - 1 / 8)) <= TOL[dt]


@pytest.mark.slow
@pytest.mark.parametrize("dt,fuse", [(np.complex128, True), (np.complex64, True), (np.complex128, False)],
                         ids=["c128-fused", "c64-fused", "c128-unfused"])
def test_qft30_apply_circuit_every_amplitude(dt, fuse):
    """reset + qj_apply_circuit: the every-tile fused passes (each reads and
    writes the whole state) and the per-gate passes, then canonicalize; all
    2^30 amplitudes against the closed form."""
    n = 30
    t = torch.empty(2**n, dtype=TDT[dt], device="cuda")
    st = qjp.State(t, basis=SEED_X)
    st.apply_circuit(C.qft(n).gates, fuse=fuse)
    st.canonicalize()
    st.sync()
    assert st.layout() == [n - 1 - q for q in range(n)]
    worst, l2 = qft_check_full(t, n, SEED_X)
    assert worst <= TOL[dt], f"max abs err {worst:.3e}"
    assert l2 <= (1e-10 if dt == np.complex128 else 1e-3)
    del st, t
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_qft30_in_place_memory():
    """In place (reading R6): across a fused and
    an unfused QFT30 c128 circuit (16 GiB state) and a qj_simulate step the
    library takes at most 256 MiB of device memory beyond the caller's state
    buffer (program buffers, staging ring, reduction bins, JIT modules) -- no
    second state-sized buffer."""
    n = 30
    free0 = free_bytes()
    t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
    free1 = free_bytes()
    st = qjp.State(t, basis=SEED_X)
    st.apply_circuit(C.qft(n).gates, fuse=True)
    st.sync()
    low = free_bytes()
    st.reset(SEED_X)
    st.apply_circuit(C.qft(n).gates, fuse=False)
    st.sync()
    low = min(low, free_bytes())
    st.simulate(SEED_X, C.qft(n).gates, qubits=list(range(10)))
    st.sync()
    low = min(low, free_bytes())
    taken = free1 - low
    print(f"state {free0 - free1} B, library scratch {taken} B")
    assert free0 - free1 >= 2**n * 16
    assert taken <= 256 << 20, f"library took {taken / 2**20:.1f} MiB"
    del st, t
    torch.cuda.empty_cache()


# ------------------------------------------------ supremacy-style c64 vs the oracle
def _oracle_c64(circ, basis=0):
    mats = [g.matrix().astype(np.complex64).astype(np.complex128) for g in circ.gates]
    return oracle.run(circ, oracle.basis_state(circ.n, basis), mats)


def _supremacy_check(rows, cols, cycles):
    circ = C.supremacy(rows, cols, cycles)
    n = circ.n
    exp = _oracle_c64(circ)
    t = torch.empty(2**n, dtype=torch.complex64, device="cuda")
    st = qjp.State(t, basis=0)
    st.apply_circuit(circ.gates, fuse=True)  # every-tile passes
    st.canonicalize()
    st.sync()
    err = np.max(np.abs(t.cpu().numpy().astype(np.complex128) - exp))
    assert err <= 1e-5, f"fused apply_circuit max abs err {err:.3e}"
    t.fill_(float("nan"))
    p = st.simulate(0, circ.gates, qubits=[0, 1, 2], fuse=True)  # live tiles from |0>
    st.canonicalize()
    st.sync()
    err = np.max(np.abs(t.cpu().numpy().astype(np.complex128) - exp))
    assert err <= 1e-5, f"simulate max abs err {err:.3e}"
    pe = oracle.probabilities(exp, n, [0, 1, 2])
    assert np.max(np.abs(p.cpu().numpy() - pe)) <= 1e-5
    del st, t


@pytest.mark.slow
def test_supremacy24_c64_vs_oracle():
    """SURVEY 8(d) config 4's generator (sqrt-X/Y/W + fSim(pi/2, pi/6) on the
    ABCDCDAB couplers, 20 cycles) on a 4x6 grid: every amplitude of the fused
    GPU result against the gate-by-gate oracle (same complex64 matrices)."""
    _supremacy_check(4, 6, 20)


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("QJ_SLOW_TESTS") != "1", reason="QJ_SLOW_TESTS=1: minutes of oracle time")
def test_supremacy28_c64_vs_oracle():
    _supremacy_check(4, 7, 20)


# ------------------------------------------------ controlled fSim
@pytest.mark.parametrize("dt", [np.complex128, np.complex64], ids=["c128", "c64"])
@pytest.mark.parametrize("n", [3, 6, 12])
def test_controlled_fsim_every_position(dt, n):
    """fSim(theta, phi) with 1-2 controls on every ordered target pair: the
    per-gate entry point (qj_apply_fsim) and the fused circuit path, against
    the oracle's dense 4x4 matrix with the control projector."""
    rng = np.random.default_rng(100 + n)
    v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    psi = (v / np.linalg.norm(v)).astype(dt)
    gates = []
    for a in range(n):
        for b in range(n):
            if a == b:
                continue
            rest = [q for q in range(n) if q not in (a, b)]
            nc = int(rng.integers(1, min(2, len(rest)) + 1)) if rest else 0
            ctrls = tuple(int(q) for q in rng.permutation(rest)[:nc])
            th, ph = rng.uniform(0, 2 * math.pi, 2)
            gates.append(G.FSIM(a, b, float(th), float(ph), ctrls))
    if n == 12:
        gates = [gates[i] for i in rng.permutation(len(gates))[:60]]
    circ = C.Circuit(n, name="cfsim")
    for g in gates:
        circ.append(g)
    mats = [g.matrix().astype(dt).astype(np.complex128) for g in circ.gates]
    exp = oracle.run(circ, psi.astype(np.complex128), mats)
    for mode in ("per_gate", "fused"):
        x = torch.from_numpy(psi.copy()).cuda()
        st = qjp.State(x, basis=None)
        if mode == "per_gate":
            for g in gates:
                st.fsim(g.targets[0], g.targets[1], g.data[0], g.data[1], g.controls)
        else:
            st.apply_circuit(gates, fuse=True)
            st.canonicalize()
        st.sync()
        err = np.max(np.abs(x.cpu().numpy().astype(np.complex128) - exp))
        assert err <= TOL[dt], f"{mode}: max abs err {err:.3e}"


@pytest.mark.parametrize("dt", [np.complex128, np.complex64], ids=["c128", "c64"])
def test_controlled_fsim_tile_pass(dt):
    """Controlled fSims inside fused window tile passes (n = 18: several
    tiles, controls on bits inside and outside the window)."""
    n = 18
    rng = np.random.default_rng(7)
    circ = C.Circuit(n, name="cfsim18")
    for i in range(80):
        qs = [int(q) for q in rng.permutation(n)]
        th, ph = rng.uniform(0, 2 * math.pi, 2)
        circ.append(G.FSIM(qs[0], qs[1], float(th), float(ph), tuple(qs[2:2 + (i % 3)])))
        circ.append(G.unitary("U", (qs[3],), G.random_unitary(1, rng), ()))
    v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    psi = (v / np.linalg.norm(v)).astype(dt)
    mats = [g.matrix().astype(dt).astype(np.complex128) for g in circ.gates]
    exp = oracle.run(circ, psi.astype(np.complex128), mats)
    x = torch.from_numpy(psi.copy()).cuda()
    st = qjp.State(x, basis=None)
    st.apply_circuit(circ.gates, fuse=True)
    st.canonicalize()
    st.sync()
    err = np.max(np.abs(x.cpu().numpy().astype(np.complex128) - exp))
    assert err <= TOL[dt], f"max abs err {err:.3e}"


# ------------------------------------------------ sharded: amplitudes, not |psi|^2
@pytest.mark.parametrize("dt", [np.complex128, np.complex64], ids=["c128", "c64"])
@pytest.mark.parametrize("nshards", [2, 4, 8])
@pytest.mark.parametrize("fuse", [False, True], ids=["unfused", "fused"])
def test_sharded_amplitudes_vs_oracle(dt, nshards, fuse):
    """Virtual-rank sharded states (global-qubit swaps): after canonicalize
    every shard holds its canonical slice; amplitudes (phases included) match
    the oracle and the single-shard run."""
    n = 16 if fuse else 11
    circ = C.random_circuit(n, 150, 70 + nshards, max_targets=2, max_controls=2)
    circ.gates += C.qft(n).gates
    rng = np.random.default_rng(31 + nshards)
    v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    psi = (v / np.linalg.norm(v)).astype(dt)
    exp = oracle.run(circ, psi.astype(np.complex128), [g.matrix().astype(dt).astype(np.complex128) for g in circ.gates])
    g = nshards.bit_length() - 1
    nl = n - g
    shards = [torch.from_numpy(psi[r << nl:(r + 1) << nl].copy()).cuda() for r in range(nshards)]
    sh = qjp.State.sharded(shards, n, basis=None)
    sh.apply_circuit(circ.gates, fuse=fuse)
    sh.canonicalize()
    sh.sync()
    assert sh.layout() == [n - 1 - q for q in range(n)]
    got = np.concatenate([s.cpu().numpy() for s in shards]).astype(np.complex128)
    err = np.max(np.abs(got - exp))
    assert err <= TOL[dt], f"sharded max abs err {err:.3e}"
    x1 = torch.from_numpy(psi.copy()).cuda()
    s1 = qjp.State(x1, basis=None)
    s1.apply_circuit(circ.gates, fuse=fuse)
    s1.canonicalize()
    s1.sync()
    assert np.max(np.abs(x1.cpu().numpy().astype(np.complex128) - got)) <= TOL[dt]
    assert sh.counters()["exchanges"] > 0


@pytest.mark.parametrize("nshards", [2, 8])
def test_sharded_amplitudes_bit_identical_exact_gates(nshards):
    """Permutation / sign / single-phase gates: canonicalised sharded
    amplitudes equal the single-shard amplitudes bit for bit (R20)."""
    n, dt = 10, np.complex128
    circ = C.random_circuit(n, 200, 40 + nshards, kinds=("x", "z", "swap", "diag"), max_targets=2)
    rng = np.random.default_rng(24)
    v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    psi = (v / np.linalg.norm(v)).astype(dt)
    g = nshards.bit_length() - 1
    nl = n - g
    shards = [torch.from_numpy(psi[r << nl:(r + 1) << nl].copy()).cuda() for r in range(nshards)]
    sh = qjp.State.sharded(shards, n, basis=None)
    sh.apply_circuit(circ.gates)
    sh.canonicalize()
    x1 = torch.from_numpy(psi.copy()).cuda()
    s1 = qjp.State(x1, basis=None)
    s1.apply_circuit(circ.gates)
    s1.canonicalize()
    sh.sync()
    s1.sync()
    got = np.concatenate([s.cpu().numpy() for s in shards])
    assert np.array_equal(got, x1.cpu().numpy())


# ------------------------------------------------ live-tile pass that repeats the first window
@pytest.mark.parametrize("dt", [np.complex128, np.complex64], ids=["c128", "c64"])
def test_simulate_repeated_window_single_tile(dt):
    """A deep circuit on 12 qubits of a 16-qubit state: the planner's budget
    splits it into several tile passes on the same window, so every pass after
    the synthesised one runs exactly one live tile (ntiles == 1, grid 1).
    qj_simulate against the oracle, element-wise."""
    n = 16
    rng = np.random.default_rng(12)
    circ = C.Circuit(n, name="deep12")
    qs = list(range(4, 16))  # bits 0..11
    for _ in range(400):
        a, b = (int(q) for q in rng.choice(qs, 2, replace=False))
        circ.append(G.unitary("U", (a,), G.random_unitary(1, rng), ()))
        circ.append(G.unitary("U", (a, b), G.random_unitary(2, rng), ()))
    basis = 0b1011000000000000 | 0b101
    x = torch.full((2**n,), float("nan"), dtype=TDT[dt], device="cuda")
    st = qjp.State(x, basis=None)
    p = st.simulate(basis, circ.gates, qubits=[4, 15], fuse=True)
    st.canonicalize()
    st.sync()
    exp = oracle.run(circ, oracle.basis_state(n, basis), [g.matrix().astype(dt).astype(np.complex128) for g in circ.gates])
    err = np.max(np.abs(x.cpu().numpy().astype(np.complex128) - exp))
    assert err <= TOL[dt], f"max abs err {err:.3e}"
    assert np.max(np.abs(p.cpu().numpy() - oracle.probabilities(exp, n, [4, 15]))) <= TOL[dt]
    assert st.counters()["launches"] > 0


# ------------------------------------------------ wider gate fusion (QJ_FUSE_GATES_K)
@pytest.mark.parametrize("dt", [np.complex128, np.complex64], ids=["c128", "c64"])
@pytest.mark.parametrize("k", [2, 3, 4, 5])
@pytest.mark.parametrize("fuse", [False, True], ids=["passes", "tiles"])
def test_fuse_gates_width_vs_oracle(dt, k, fuse):
    """Greedy fusion into <= k-qubit dense gates
    followed by per-gate passes or window tile passes: every amplitude
    against the oracle on the unfused circuit (n = 16: several tiles)."""
    n = 16
    circ = C.supremacy(4, 4, 8)
    circ.gates += C.random_circuit(n, 60, 77 + k, max_targets=2, max_controls=1).gates
    rng = np.random.default_rng(k)
    v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    psi = (v / np.linalg.norm(v)).astype(dt)
    exp = oracle.run(circ, psi.astype(np.complex128), [g.matrix().astype(dt).astype(np.complex128) for g in circ.gates])
    x = torch.from_numpy(psi.copy()).cuda()
    st = qjp.State(x, basis=None)
    st.apply_circuit(circ.gates, fuse=fuse, fuse_gates=k)
    st.canonicalize()
    st.sync()
    err = np.max(np.abs(x.cpu().numpy().astype(np.complex128) - exp))
    assert err <= TOL[dt], f"max abs err {err:.3e}"


# ------------------------------------------------ complex64 5-qubit dense passes on the tensor cores
@pytest.mark.parametrize("n", [12, 14, 20])
def test_dense5_c64_tensor_core_pass(n):
    """Dense 5-qubit gates on complex64 states run as 3xTF32 tcgen05.mma
    contractions (dense_tc.cu): targets on high, low and mixed bits, unsorted
    listed order, with and without controls, against the oracle (R8 1e-5)."""
    rng = np.random.default_rng(500 + n)
    v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    psi = (v / np.linalg.norm(v)).astype(np.complex64)
    circ = C.Circuit(n, name="dense5")
    sets = [tuple(range(n - 5, n)), tuple(range(5)), (0, n - 1, 3, n // 2, 5)]
    for _ in range(5):
        sets.append(tuple(int(q) for q in rng.permutation(n)[:5]))
    for i, ts in enumerate(sets):
        rest = [q for q in range(n) if q not in ts]
        ctrls = tuple(int(q) for q in rng.permutation(rest)[: i % 3]) if n >= 14 else ()
        circ.append(G.unitary("U5", ts, G.random_unitary(5, rng), ctrls))
    mats = [g.matrix().astype(np.complex64).astype(np.complex128) for g in circ.gates]
    exp = oracle.run(circ, psi.astype(np.complex128), mats)
    x = torch.from_numpy(psi.copy()).cuda()
    st = qjp.State(x, basis=None)
    for g in circ.gates:
        st.apply_gate(g.targets, g.data[0], g.controls)
    st.sync()
    err = np.max(np.abs(x.cpu().numpy().astype(np.complex128) - exp))
    assert err <= 1e-5, f"max abs err {err:.3e}"
    # and the same gates as a fused circuit at width 5 (QJ_FUSE_GATES_K(5))
    x2 = torch.from_numpy(psi.copy()).cuda()
    s2 = qjp.State(x2, basis=None)
    s2.apply_circuit(circ.gates, fuse_gates=5)
    s2.sync()
    assert np.max(np.abs(x2.cpu().numpy().astype(np.complex128) - exp)) <= 1e-5


# ------------------------------------------------ bounds-checked JIT kernels (QJ_JIT_CHECK=1)
def test_checked_tile_kernels_subprocess():
    """compute-sanitizer is closed on this pool, so the JIT tile kernels carry
    their own bounds checks when QJ_JIT_CHECK=1 (every global load / store /
    bulk copy checked against the state size; a violation sets a device flag
    that qj_sync reports instead of touching memory).  Run every tile-kernel
    form -- two-CTA, CTA pair, ring (TMA), live tile, synthesised pass, fused
    marginal, complex64 -- in a fresh process with the checks compiled in."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QJ_JIT_CHECK="1")
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "sanitize_driver.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "sanitize driver done" in r.stdout


# ------------------------------------------------ BV30: every amplitude against its closed form
@pytest.mark.slow
def test_bv30_simulate_every_amplitude():
    """Bernstein-Vazirani (Table 2 row bv, secret all ones,
    ancilla = qubit 29): the output is |1...1>_data (x) |->_anc, i.e. +1/sqrt2 at
    canonical index 2^30 - 2, -1/sqrt2 at 2^30 - 1 and exactly 0 elsewhere.  The
    bench step (qj_simulate, fused marginal over qubits 0..9 = all ones with
    probability 1); all 2^30 amplitudes checked after canonicalisation."""
    n = 30
    t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
    st = qjp.State(t, basis=None)
    t.fill_(float("nan"))
    p = st.simulate(0, C.bv(n).gates, qubits=list(range(10)))
    st.canonicalize()
    st.sync()
    pc = p.cpu().numpy()
    assert abs(pc[1023] - 1.0) <= 1e-12 and np.max(np.abs(pc[:1023])) <= 1e-12
    chunk = CHUNK
    host = torch.empty(chunk, dtype=t.dtype, pin_memory=True)
    worst = 0.0
    for off in range(0, 2**n, chunk):
        host.copy_(t[off:off + chunk])
        a = host.numpy().copy()
        if off + chunk == 2**n:
            assert abs(a[-2] - 2**-0.5) <= 1e-12 and abs(a[-1] + 2**-0.5) <= 1e-12
            a[-2:] = 0
        worst = max(worst, float(np.max(np.abs(a))))
    assert worst <= 1e-12, f"max |amp| off the two basis states {worst:.3e}"
    del st, t
    torch.cuda.empty_cache()
