"""GPU parity: the sm_100a CUDA path (through the C ABI) vs the CPU oracle,
element by element, on seeded inputs.

Tolerances (north star, reading R8): max |psi_gpu - psi_oracle| <= 1e-12 for
complex128 and 1e-5 for complex64; X / Z / SWAP (and controlled versions) are
exact (IEEE ==, reading R9); probabilities' index ordering is exact (a basis
state gives exactly one 1).  For complex64 runs the oracle is fed the same
complex64-rounded matrices and input state, widened to double (reading R7).
"""

import math

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


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2203_08826_b200 import build
    build.build()


def rand_state(n, rng, dt):
    v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    v = (v / np.linalg.norm(v)).astype(dt)
    return v


def to_gpu(psi, dt):
    return torch.from_numpy(np.ascontiguousarray(psi.astype(dt))).to("cuda")


def gate_matrix_for(g, dt):
    """Dense matrix as the GPU sees it: rounded to the state dtype, widened."""
    return g.matrix().astype(dt).astype(np.complex128)


def oracle_circuit(circ, psi, dt):
    mats = [gate_matrix_for(g, dt) for g in circ.gates]
    return oracle.run(circ, psi.astype(np.complex128), mats)


def run_gpu_gate(st, g):
    if g.kind == "dense":
        st.apply_gate(g.targets, g.data[0], g.controls)
    elif g.kind == "x":
        st.x(g.targets[0], g.controls)
    elif g.kind == "z":
        st.z(g.targets[0], g.controls)
    elif g.kind == "swap":
        st.swap(g.targets[0], g.targets[1], g.controls)
    elif g.kind == "fsim":
        st.fsim(g.targets[0], g.targets[1], g.data[0], g.data[1], g.controls)
    elif g.kind == "diag":
        st.diagonal(g.targets, g.data[0], g.controls)
    else:
        raise ValueError(g.kind)


def check_close(got, exp, dt, exact=False):
    if exact:
        assert np.array_equal(got.astype(np.complex128), exp), "not value-exact"
        return
    err = np.max(np.abs(got.astype(np.complex128) - exp))
    assert err <= TOL[dt], f"max abs err {err:.3e} > {TOL[dt]}"


DTYPES = [np.complex128, np.complex64]


# ------------------------------------------------ every bit position, 1 target
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 6, 7, 9, 12])
def test_one_qubit_every_position(dt, n):
    rng = np.random.default_rng(n)
    psi = rand_state(n, rng, dt)
    for t in range(n):
        for nc in range(0, min(2, n - 1) + 1):
            ctrls = tuple(int(q) for q in rng.permutation([q for q in range(n) if q != t])[:nc])
            g = G.unitary("U", (t,), G.random_unitary(1, rng), ctrls)
            x = to_gpu(psi, dt)
            st = qjp.State(x, basis=None)
            st.apply_gate(g.targets, g.data[0], g.controls)
            st.sync()
            exp = np.empty(2**n, dtype=np.complex128)
            oracle.apply_matrix(psi.astype(np.complex128), exp, n, g.targets, g.controls,
                                gate_matrix_for(g, dt))
            check_close(x.cpu().numpy(), exp, dt)


# ------------------------------------------------ random gates of every kind
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("seed", range(12))
def test_random_gates(dt, seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 13))
    psi = rand_state(n, rng, dt)
    for i in range(30):
        g = C.random_gate(n, rng, max_targets=5, max_controls=3)
        x = to_gpu(psi, dt)
        st = qjp.State(x, basis=None)
        run_gpu_gate(st, g)
        st.sync()
        exp = np.empty(2**n, dtype=np.complex128)
        oracle.apply_matrix(psi.astype(np.complex128), exp, n, g.targets, g.controls,
                            gate_matrix_for(g, dt))
        check_close(x.cpu().numpy(), exp, dt, exact=g.kind in ("x", "z", "swap"))


@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("k", [2, 3, 4, 5, 6, 7, 8])
def test_multi_target_dense(dt, k):
    """k-target dense gates on every kind of bit mix (vector, lane, outer)."""
    rng = np.random.default_rng(77 + k)
    n = 12
    psi = rand_state(n, rng, dt)
    for trial in range(6):
        qs = [int(q) for q in rng.permutation(n)]
        if trial == 0:
            qs = list(range(n - 1, -1, -1))  # lowest bits (lane / vector)
        elif trial == 1:
            qs = list(range(n))              # highest bits (outer)
        t = tuple(qs[:k])
        c = tuple(qs[k:k + int(rng.integers(0, 3))])
        g = G.unitary("U", t, G.random_unitary(k, rng), c)
        x = to_gpu(psi, dt)
        st = qjp.State(x, basis=None)
        st.apply_gate(g.targets, g.data[0], g.controls)
        st.sync()
        exp = np.empty(2**n, dtype=np.complex128)
        oracle.apply_matrix(psi.astype(np.complex128), exp, n, t, c, gate_matrix_for(g, dt))
        check_close(x.cpu().numpy(), exp, dt)


@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
def test_specialised_exact_every_position(dt):
    """X, CX, SWAP, CSWAP, Z, CZ are value-exact vs Eq. 1 with their matrices (R9)."""
    rng = np.random.default_rng(5)
    n = 11
    psi = rand_state(n, rng, dt)
    cases = []
    for t in range(n):
        cases.append(G.X(t))
        cases.append(G.Z(t))
        cases.append(G.X(t, controls=((t + 3) % n,)))
        cases.append(G.Z(t, controls=((t + 5) % n, (t + 1) % n)))
        cases.append(G.SWAP(t, (t + 1) % n))
        cases.append(G.SWAP(t, (t + 6) % n, controls=((t + 2) % n,)))
    for g in cases:
        x = to_gpu(psi, dt)
        st = qjp.State(x, basis=None)
        run_gpu_gate(st, g)
        st.sync()
        exp = np.empty(2**n, dtype=np.complex128)
        oracle.apply_matrix(psi.astype(np.complex128), exp, n, g.targets, g.controls, g.matrix())
        check_close(x.cpu().numpy(), exp, dt, exact=True)


# ------------------------------------------------ circuits
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("name", ["qft10", "variational12", "supremacy3x4", "qaoa10", "bv10", "random10",
                                  "qft15", "variational16", "supremacy4x4", "qaoa16", "bv15", "random16"])
def test_circuits_vs_oracle(dt, name):
    """n <= 13 (c128) / 14 (c64) runs fused circuits as whole-state SMEM
    programs; the larger cases exercise the window tile passes."""
    circ = {"qft10": lambda: C.qft(10), "variational12": lambda: C.variational(12, layers=3),
            "supremacy3x4": lambda: C.supremacy(3, 4, 12), "qaoa10": lambda: C.qaoa(10, 2),
            "bv10": lambda: C.bv(10), "random10": lambda: C.random_circuit(10, 300, 3),
            "qft15": lambda: C.qft(15), "variational16": lambda: C.variational(16, layers=3),
            "supremacy4x4": lambda: C.supremacy(4, 4, 12), "qaoa16": lambda: C.qaoa(16, 2),
            "bv15": lambda: C.bv(15), "random16": lambda: C.random_circuit(16, 300, 4)}[name]()
    n = circ.n
    rng = np.random.default_rng(11)
    psi = rand_state(n, rng, dt)
    for fuse, fg in ((False, False), (True, False), (False, True), (True, True)):
        x = to_gpu(psi, dt)
        st = qjp.State(x, basis=None)
        st.apply_circuit(circ.gates, fuse=fuse, fuse_gates=fg)
        pf = st.probabilities([0, n - 1]).cpu().numpy()  # canonical through the map
        st.canonicalize()
        st.sync()
        exp = oracle_circuit(circ, psi, dt)
        pe = oracle.probabilities(exp, n, [0, n - 1])
        assert np.max(np.abs(pf - pe)) < TOL[dt]
        check_close(x.cpu().numpy(), exp, dt)


@pytest.mark.parametrize("n,x", [(10, 0b1011001110), (16, 40503), (20, 0xB1E05)])
def test_qft_basis_closed_form(n, x):
    y = np.arange(2**n, dtype=np.uint64)
    m = (np.uint64(x) * y) % np.uint64(2**n)
    exp = 2 ** (-n / 2) * np.exp(2j * np.pi * m.astype(np.float64) / 2**n)
    for fuse in (False, True):
        t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
        st = qjp.State(t, basis=x)
        st.apply_circuit(C.qft(n).gates, fuse=fuse)
        st.canonicalize()
        st.sync()
        assert np.max(np.abs(t.cpu().numpy() - exp)) < 1e-12


# ------------------------------------------------ probabilities
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
def test_probabilities(dt):
    rng = np.random.default_rng(3)
    for n in [1, 3, 7, 12]:
        psi = rand_state(n, rng, dt)
        st = qjp.State(to_gpu(psi, dt), basis=None)
        full = st.probabilities().cpu().numpy()
        exp = oracle.probabilities(psi.astype(np.complex128), n)
        assert np.max(np.abs(full - exp)) < (1e-15 if dt == np.complex128 else 1e-7)
        for m in range(1, n + 1):
            qs = [int(q) for q in rng.permutation(n)[:m]]
            p = st.probabilities(qs).cpu().numpy()
            e = oracle.probabilities(psi.astype(np.complex128), n, qs)
            assert np.max(np.abs(p - e)) < (1e-14 if dt == np.complex128 else 1e-6)


def test_probabilities_basis_ordering_exact():
    n, x = 14, 0b10110011100101
    t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
    st = qjp.State(t, basis=x)
    p = st.probabilities().cpu().numpy()
    assert p[x] == 1.0 and np.count_nonzero(p) == 1
    q = [3, 0, 7]
    pm = st.probabilities(q).cpu().numpy()
    o = int("".join(str((x >> (n - 1 - qq)) & 1) for qq in q), 2)
    assert pm[o] == 1.0 and np.count_nonzero(pm) == 1


# ------------------------------------------------ sharded (virtual ranks)
def _shard_run(circ, psi, dt, nshards):
    n = circ.n
    g = nshards.bit_length() - 1
    x1 = to_gpu(psi, dt)
    s1 = qjp.State(x1, basis=None)
    s1.apply_circuit(circ.gates)
    s1.sync()
    shards = [to_gpu(psi[r << (n - g):(r + 1) << (n - g)], dt) for r in range(nshards)]
    sh = qjp.State.sharded(shards, n, basis=None)
    sh.apply_circuit(circ.gates)
    sh.sync()
    return s1, sh


@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("nshards", [2, 4, 8])
def test_sharded_vs_single_and_oracle(dt, nshards):
    """The sharded path (global-qubit swaps between shards) matches the
    single-shard path and the oracle within tolerance (dense gates may land on
    different physical bits after a remap, which changes the summation order)."""
    n = 11
    circ = C.random_circuit(n, 120, 17 + nshards, max_targets=3)
    circ.gates += C.qft(n).gates
    rng = np.random.default_rng(23)
    psi = rand_state(n, rng, dt)
    s1, sh = _shard_run(circ, psi, dt, nshards)
    full = sh.probabilities().cpu().numpy()
    single = s1.probabilities().cpu().numpy()
    assert np.max(np.abs(full - single)) < TOL[dt]
    qs = [0, n - 1, 3]
    assert np.max(np.abs(sh.probabilities(qs).cpu().numpy() - s1.probabilities(qs).cpu().numpy())) < TOL[dt]
    exp = oracle_circuit(circ, psi, dt)
    assert np.max(np.abs(full - np.abs(exp) ** 2)) < TOL[dt]
    assert sh.counters()["exchanges"] > 0


@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("nshards", [2, 8])
def test_sharded_bit_identical_exact_gates(dt, nshards):
    """With only permutation / sign / single-phase gates every amplitude sees
    the same arithmetic wherever it lives: sharded == single, bit for bit."""
    n = 10
    circ = C.random_circuit(n, 200, 40 + nshards, kinds=("x", "z", "swap", "diag"), max_targets=2)
    rng = np.random.default_rng(24)
    psi = rand_state(n, rng, dt)
    s1, sh = _shard_run(circ, psi, dt, nshards)
    assert np.array_equal(sh.probabilities().cpu().numpy(), s1.probabilities().cpu().numpy())


# ------------------------------------------------ full-size sampled checks
@pytest.mark.slow
@pytest.mark.parametrize("fuse", [False, True])
def test_qft30_c128_sampled_closed_form(fuse):
    """The bench workload (30-qubit QFT, complex128, bench launch config): every
    amplitude is checked on a seeded sample of 2^16 indices plus the ends
    against the exact closed form (integer phase numerator)."""
    n, x = 30, 0b101101110001011100101101011011
    t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
    st = qjp.State(t, basis=x)
    st.apply_circuit(C.qft(n).gates, fuse=fuse)
    p = st.probabilities([0, 1, 2, 3])
    assert abs(float(p.sum()) - 1) < 1e-10
    st.canonicalize()
    st.sync()
    rng = np.random.default_rng(30)
    idx = np.unique(np.concatenate([rng.integers(0, 2**n, 1 << 16), [0, 1, 2**n - 1]])).astype(np.int64)
    got = t[torch.from_numpy(idx).cuda()].cpu().numpy()
    m = (np.uint64(x) * idx.astype(np.uint64)) % np.uint64(2**n)
    exp = 2 ** (-n / 2) * np.exp(2j * np.pi * m.astype(np.float64) / 2**n)
    assert np.max(np.abs(got - exp)) < 1e-12
    p = st.probabilities([0, 1, 2, 3])
    assert abs(float(p.sum()) - 1) < 1e-10
    del st, t
    torch.cuda.empty_cache()


# ------------------------------------------------ NCCL path (1 rank on 1 GPU)
def _nccl_worker(port, q):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    try:
        n = 12
        circ = C.qft(n)
        t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
        st = qjp.State.distributed(t, n, basis=5)
        st.apply_circuit(circ.gates)
        p = st.probabilities([0, 3, 7]).cpu().numpy()    # NCCL all-reduce of the bins
        full = st.probabilities().cpu().numpy()
        st.sync()
        exp = oracle.run(circ, oracle.basis_state(n, 5))
        # the exchange data path (pipelined grouped send / recv through the
        # staging ring, both streams, pack / unpack) with this rank as its own
        # partner: a 1 GiB shard (two 256 MiB chunks per half), the top local
        # bit (in-place halves) and a low bit (pack / unpack); unchanged after
        n2 = 26
        t2 = torch.randn(2**n2, dtype=torch.complex128, device="cuda")
        ref = t2.clone()
        s2 = qjp.State.distributed(t2, n2, basis=None)
        for bit in (n2 - 1, 3, 0):
            s2.debug_self_exchange(bit)
        s2.sync()
        self_ok = bool(torch.equal(t2, ref))
        q.put((float(np.max(np.abs(t.cpu().numpy() - exp))),
               float(np.max(np.abs(p - oracle.probabilities(exp, n, [0, 3, 7])))),
               float(np.max(np.abs(full - np.abs(exp) ** 2))), st.info()["nshards"], self_ok))
    finally:
        dist.destroy_process_group()


def test_nccl_single_rank_state():
    import multiprocessing as mpm
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mpm.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(port, q))
    p.start()
    p.join(timeout=300)
    assert p.exitcode == 0
    e_amp, e_marg, e_full, nsh, self_ok = q.get(timeout=10)
    assert nsh == 1 and e_amp < 1e-12 and e_marg < 1e-12 and e_full < 1e-12
    assert self_ok, "self exchange changed the state"


# ------------------------------------------------ edge cases
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
def test_empty_circuit_and_tiny_states(dt):
    rng = np.random.default_rng(9)
    psi = rand_state(12, rng, dt)
    x = to_gpu(psi, dt)
    st = qjp.State(x, basis=None)
    st.apply_circuit([], fuse=True)
    st.apply_circuit([], fuse=False)
    st.sync()
    assert np.array_equal(x.cpu().numpy(), psi)
    for n in (1, 2, 3):
        circ = C.random_circuit(n, 40, n, max_targets=min(3, n), max_controls=1)
        p0 = rand_state(n, rng, dt)
        for fuse in (False, True):
            x = to_gpu(p0, dt)
            s = qjp.State(x, basis=None)
            s.apply_circuit(circ.gates, fuse=fuse)
            s.canonicalize()
            s.sync()
            check_close(x.cpu().numpy(), oracle_circuit(circ, p0, dt), dt)


@pytest.mark.slow
def test_qft32_c128_max_size_closed_form():
    """64 GiB complex128 state (the largest power of two with room to spare on
    one B200 besides 33 q): fused QFT |x>, sampled against the closed form."""
    n, x = 32, 0xB5E3C1A7
    t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
    st = qjp.State(t, basis=x)
    st.apply_circuit(C.qft(n).gates, fuse=True)
    p = st.probabilities([0, 1, 2])
    assert abs(float(p.sum()) - 1) < 1e-10
    st.canonicalize()
    st.sync()
    rng = np.random.default_rng(32)
    idx = np.unique(np.concatenate([rng.integers(0, 2**n, 1 << 14), [0, 2**n - 1]])).astype(np.int64)
    got = t[torch.from_numpy(idx).cuda()].cpu().numpy()
    m = (np.uint64(x) * idx.astype(np.uint64)) % np.uint64(2**n)
    exp = 2 ** (-n / 2) * np.exp(2j * np.pi * m.astype(np.float64) / 2**n)
    assert np.max(np.abs(got - exp)) < 1e-12
    del st, t
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_supremacy32_c64_fused_vs_unfused():
    """BASELINE config 4 at full size (32 qubits, complex64, 32 GiB): fused and
    unfused paths agree amplitude by amplitude on a sample (no oracle fits), and
    the norm is preserved."""
    circ = C.supremacy(4, 8, 20)
    n = circ.n
    rng = np.random.default_rng(4)
    idx = torch.from_numpy(np.unique(rng.integers(0, 2**n, 1 << 14)).astype(np.int64)).cuda()
    t = torch.empty(2**n, dtype=torch.complex64, device="cuda")
    st = qjp.State(t, basis=0)
    st.apply_circuit(circ.gates, fuse=True)
    st.canonicalize()
    norm = float(st.probabilities([0, 1]).double().sum())
    a = t[idx].cpu().numpy()
    st.reset(0)
    st.apply_circuit(circ.gates, fuse=False)
    st.sync()
    b = t[idx].cpu().numpy()
    assert abs(norm - 1) < 1e-4
    assert np.max(np.abs(a.astype(np.complex128) - b)) < 1e-5
    del st, t
    torch.cuda.empty_cache()


# ------------------------------------------------ plan cache + CUDA graph replay
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("fuse", [False, True])
def test_plan_cache_graph_replay(dt, fuse):
    """The same circuit applied repeatedly on one handle: 1st call plans, 2nd
    captures a CUDA graph, later calls replay it (non-default stream)."""
    n = 16
    circ = C.random_circuit(n, 150, 77, max_targets=2, max_controls=1)
    circ.gates += C.qft(n).gates
    rng = np.random.default_rng(12)
    psi = rand_state(n, rng, dt)
    stream = torch.cuda.Stream()
    x = to_gpu(psi, dt)
    torch.cuda.synchronize()
    st = qjp.State(x, basis=None, stream=stream)
    packed = st.pack_circuit(circ.gates)
    exp = psi.astype(np.complex128)
    mats = [gate_matrix_for(g, dt) for g in circ.gates]
    for rep in range(4):
        st.apply_circuit(None, fuse=fuse, packed=packed)
        exp = oracle.run(circ, exp, mats)
    pf = st.probabilities([0, 5, n - 1]).cpu().numpy()
    st.canonicalize()
    st.sync()
    check_close(x.cpu().numpy(), exp, dt)
    assert np.max(np.abs(pf - oracle.probabilities(exp, n, [0, 5, n - 1]))) < TOL[dt]


# ------------------------------------------------ f3: Trotterized adiabatic TFIM
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("n,periodic", [(10, True), (13, False), (2, True)])
def test_tfim_trotter_vs_oracle(dt, n, periodic):
    """The Trotter circuit of the adiabatic TFIM run through
    the library (unfused, fused tile pass, paper fusion) vs the gate oracle."""
    from workloads import evolution as W
    circ = W.adiabatic_circuit(n, 1.0, 0.05, periodic=periodic)
    psi = np.zeros(2**n, dtype=dt)
    psi[0] = 1
    exp = oracle_circuit(circ, psi, dt)
    for fuse, fg in ((False, False), (True, False), (True, True)):
        x = torch.empty(2**n, dtype=TDT[dt], device="cuda")
        st = qjp.State(x, basis=0)
        st.apply_circuit(circ.gates, fuse=fuse, fuse_gates=fg)
        st.canonicalize()
        st.sync()
        check_close(x.cpu().numpy(), exp, dt)


def test_tfim_adiabatic_ground_energy_gpu():
    """n = 8, T = 20, dt = 0.05 on the GPU: <H1> within 2% of the exact ground
    energy of the dense oracle's H1 (SPEC S:576 at a larger n)."""
    from oracle import evolution as E
    from workloads import evolution as W
    n = 8
    circ = W.adiabatic_circuit(n, 20.0, 0.05)
    x = torch.empty(2**n, dtype=torch.complex128, device="cuda")
    st = qjp.State(x, basis=0)
    st.apply_circuit(circ.gates, fuse=True)
    st.canonicalize()
    st.sync()
    H1 = E.tfim_hamiltonian(n, 1.0)
    e0 = np.linalg.eigvalsh(H1)[0]
    assert abs(E.energy(x.cpu().numpy(), H1) - e0) <= 0.02 * abs(e0)


# ------------------------------------------------ whole-state SMEM programs (small states)
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
def test_small_state_programs_every_size(dt):
    """QJ_FUSE on n <= 13 (c128) / 14 (c64): runs of gates execute as one
    whole-state shared-memory program; dense gates on 5+ targets run as
    ordinary passes in between.  Every size up to the SMEM limit, vs the oracle."""
    nmax = 13 if dt == np.complex128 else 14
    for n in range(1, nmax + 1):
        rng = np.random.default_rng(500 + n)
        circ = C.random_circuit(n, 80, 900 + n, max_targets=min(5, n), max_controls=min(2, max(0, n - 1)))
        psi = rand_state(n, rng, dt)
        x = to_gpu(psi, dt)
        st = qjp.State(x, basis=None)
        st.apply_circuit(circ.gates, fuse=True)
        st.sync()
        check_close(x.cpu().numpy(), oracle_circuit(circ, psi, dt), dt)


def test_small_state_is_one_launch():
    n = 10
    circ = C.qft(n)
    t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
    st = qjp.State(t, basis=5)
    st.counters(reset=True)
    st.apply_circuit(circ.gates, fuse=True)
    st.sync()
    c = st.counters(reset=True)
    assert c["launches"] == 1 and c["passes"] == 1
    y = np.arange(2**n, dtype=np.uint64)
    exp = 2 ** (-n / 2) * np.exp(2j * np.pi * ((5 * y) % 2**n).astype(np.float64) / 2**n)
    assert np.max(np.abs(t.cpu().numpy() - exp)) < 1e-12


# ------------------------------------------------ f4: host-staged states
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("nslices", [1, 2, 8])
def test_host_staged_vs_oracle_and_sharded(dt, nslices):
    """State in (pinned) host memory, slices streamed through the GPU
    (PAPER.md:469-479): matches the oracle, and is bit-identical to the in-HBM
    virtual-sharded path with the same slice count (same plan, same kernels)."""
    n = 14
    circ = C.random_circuit(n, 200, 31, max_targets=3, max_controls=2)
    circ.gates += C.qft(n).gates
    rng = np.random.default_rng(77)
    psi = rand_state(n, rng, dt)
    h = torch.from_numpy(psi.copy()).pin_memory()
    st = qjp.State.host(h, nslices, basis=None)
    st.apply_circuit(circ.gates, fuse=True)
    pf = st.probabilities([0, 5, n - 1]).cpu().numpy()
    st.canonicalize()
    st.sync()
    got = h.numpy().copy()
    exp = oracle_circuit(circ, psi, dt)
    check_close(got, exp, dt)
    assert np.max(np.abs(pf - oracle.probabilities(exp, n, [0, 5, n - 1]))) < TOL[dt]
    if nslices > 1:
        parts = [torch.from_numpy(c.copy()).cuda() for c in np.split(psi, nslices)]
        sh = qjp.State.sharded(parts, n, basis=None)
        sh.apply_circuit(circ.gates, fuse=True)
        sh.canonicalize()
        sh.sync()
        ref = np.concatenate([t.cpu().numpy() for t in parts])
        assert np.array_equal(got, ref), "host-staged != in-HBM sharded"


def test_host_staged_measurement_and_reset():
    from oracle import measure as M
    n = 12
    psi = rand_state(n, np.random.default_rng(3), np.complex128)
    h = torch.from_numpy(psi.copy()).pin_memory()
    st = qjp.State.host(h, 4, basis=None)
    p = st.collapse([0, 7], 2)
    st.sync()
    exp, pe = M.collapse(psi, n, [0, 7], 2)
    assert abs(p - pe) < 1e-13
    check_close(h.numpy().copy(), exp, np.complex128)
    _, c = st.sample([7, 3], 20000, 5)
    assert c.cpu().numpy().sum() == 20000
    st.reset(0b101)
    st.sync()
    e = np.zeros(2**n)
    e[0b101] = 1
    assert np.array_equal(h.numpy().copy(), e.astype(np.complex128))


@pytest.mark.parametrize("mode", ["sharded", "host"])
@pytest.mark.parametrize("nshards", [4, 8])
def test_canonicalize_global_bit_permutation(mode, nshards):
    """QFT leaves global qubits permuted among themselves (its final SWAPs
    pair top and bottom qubits); canonicalize restores them through three
    exchanges per transposition."""
    n = 14
    x = 0b10110011101001
    circ = C.qft(n)
    if mode == "sharded":
        parts = [torch.empty(2**n // nshards, dtype=torch.complex128, device="cuda") for _ in range(nshards)]
        st = qjp.State.sharded(parts, n, basis=x)
    else:
        h = torch.empty(2**n, dtype=torch.complex128).pin_memory()
        st = qjp.State.host(h, nshards, basis=x)
    st.apply_circuit(circ.gates, fuse=True)
    st.canonicalize()
    st.sync()
    got = np.concatenate([t.cpu().numpy() for t in parts]) if mode == "sharded" else h.numpy().copy()
    y = np.arange(2**n, dtype=np.uint64)
    exp = 2 ** (-n / 2) * np.exp(2j * np.pi * ((np.uint64(x) * y) % np.uint64(2**n)).astype(np.float64) / 2**n)
    assert np.max(np.abs(got - exp)) < 1e-12


# ------------------------------------------------ fused tile passes on sharded states
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("mode,nshards", [("sharded", 2), ("sharded", 8), ("host", 4)])
@pytest.mark.parametrize("name", ["qft18", "random18", "variational18"])
def test_fused_sharded_vs_oracle(dt, mode, nshards, name):
    """QJ_FUSE on sharded / host-staged states: window tile passes per shard
    (global bits enter the tile predicates through gbase; global targets are
    exchanged in between).  Random circuits put controls and diagonal phases
    on global qubits."""
    n = 18
    circ = {"qft18": lambda: C.qft(n), "variational18": lambda: C.variational(n, layers=3),
            "random18": lambda: C.random_circuit(n, 250, 17, max_targets=2, max_controls=2)}[name]()
    rng = np.random.default_rng(170)
    psi = rand_state(n, rng, dt)
    if mode == "sharded":
        parts = [torch.from_numpy(c.copy()).cuda() for c in np.split(psi, nshards)]
        st = qjp.State.sharded(parts, n, basis=None)
    else:
        h = torch.from_numpy(psi.copy()).pin_memory()
        st = qjp.State.host(h, nshards, basis=None)
    st.counters(reset=True)
    st.apply_circuit(circ.gates, fuse=True)
    ctr = st.counters(reset=True)
    pf = st.probabilities([0, 1, n - 1]).cpu().numpy()
    st.canonicalize()
    st.sync()
    got = np.concatenate([t.cpu().numpy() for t in parts]) if mode == "sharded" else h.numpy().copy()
    exp = oracle_circuit(circ, psi, dt)
    check_close(got, exp, dt)
    assert np.max(np.abs(pf - oracle.probabilities(exp, n, [0, 1, n - 1]))) < TOL[dt]
    assert ctr["passes"] < len(circ.gates) * nshards / 2, ctr  # actually fused


# ------------------------------------------------ many tiles per CTA (prefetch ring)
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
def test_fused_many_tiles_per_block(dt):
    """n = 22: 1024 tiles per pass > the grid (SMs x blocks), so every CTA
    loops over several tiles and the cp.async prefetch ring carries data
    between iterations (at n <= 20 each CTA sees at most one tile)."""
    n = 22
    circ = C.random_circuit(n, 160, 22, max_targets=2, max_controls=1)
    circ.gates += C.qft(n).gates
    rng = np.random.default_rng(2222)
    psi = rand_state(n, rng, dt)
    x = to_gpu(psi, dt)
    st = qjp.State(x, basis=None)
    st.apply_circuit(circ.gates, fuse=True)
    st.canonicalize()
    st.sync()
    check_close(x.cpu().numpy(), oracle_circuit(circ, psi, dt), dt)


@pytest.mark.parametrize("n", [24, 26])
def test_qft_large_closed_form_fused(n):
    """QFT|x> closed form at 4096 / 16384 tiles per pass (c128)."""
    x = (0x2D5A3C9 * n) & ((1 << n) - 1)
    t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
    st = qjp.State(t, basis=x)
    st.apply_circuit(C.qft(n).gates, fuse=True)
    st.canonicalize()
    st.sync()
    rng = np.random.default_rng(n)
    idx = np.unique(np.concatenate([rng.integers(0, 2**n, 20000), [0, 2**n - 1]])).astype(np.int64)
    got = t[torch.from_numpy(idx).cuda()].cpu().numpy()
    m = (np.uint64(x) * idx.astype(np.uint64)) % np.uint64(2**n)
    exp = 2 ** (-n / 2) * np.exp(2j * np.pi * m.astype(np.float64) / 2**n)
    assert np.max(np.abs(got - exp)) < 1e-12


# ------------------------------------------------ qj_simulate (fused step ends)
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("name", ["qft22", "random22", "qft12", "variational16"])
def test_simulate_matches_separate_calls(dt, name):
    """qj_simulate == reset + apply_circuit + probabilities: the first tile
    pass synthesises |basis>, the last one accumulates the marginal (n >= 14);
    small states take the SMEM program path.  Repeated calls replay a graph."""
    n = int("".join(c for c in name if c.isdigit()))
    circ = {"qft": lambda: C.qft(n), "random": lambda: C.random_circuit(n, 200, 5, max_targets=2, max_controls=1),
            "variational": lambda: C.variational(n, layers=2)}[name.rstrip("0123456789")]()
    basis = (0x9E3779B97F4A7C15 >> (64 - n)) if n < 64 else 5
    qubits = [0, 3, n - 1, n // 2]
    tdt = TDT[dt]
    stream = torch.cuda.Stream()
    ref = torch.empty(2**n, dtype=tdt, device="cuda")
    sr = qjp.State(ref, basis=basis, stream=stream)
    sr.apply_circuit(circ.gates, fuse=True)
    pr = sr.probabilities(qubits)
    sr.canonicalize()
    sr.sync()
    x = torch.empty(2**n, dtype=tdt, device="cuda")
    st = qjp.State(x, basis=None, stream=stream)
    packed = st.pack_circuit(circ.gates)
    for rep in range(3):
        x.fill_(float("nan"))  # the synthesised first pass must not read the buffer
        p = st.simulate(basis, qubits=qubits, packed=packed)
        st.canonicalize()
        st.sync()
        tol = TOL[dt]
        assert np.max(np.abs(x.cpu().numpy().astype(np.complex128) - ref.cpu().numpy())) <= tol, rep
        assert np.max(np.abs(p.cpu().numpy() - pr.cpu().numpy())) <= tol, rep
    psi0 = np.zeros(2**n, dtype=dt)
    psi0[basis] = 1
    exp = oracle_circuit(circ, psi0, dt)
    check_close(x.cpu().numpy(), exp, dt)


@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("n", [26, 28])
def test_simulate_live_tiles_qft(dt, n):
    """Three or more tile passes: after the synthesised first pass, the later
    passes run only the tiles whose not-yet-windowed bits equal the basis bits
    (the rest are zero in and zero out).  Closed form QFT|x> on sampled
    amplitudes, marginals against the same closed form (uniform), and the
    same run with every tile (QJ_LIVE_TILES-free separate calls) agrees."""
    x = (0x2D5A3C9 * n + 12345) & ((1 << n) - 1)
    tdt = TDT[dt]
    t = torch.empty(2**n, dtype=tdt, device="cuda")
    st = qjp.State(t, basis=None)
    t.fill_(float("nan"))
    qubits = [0, 5, n - 1]
    p = st.simulate(x, C.qft(n).gates, qubits=qubits, fuse=True)
    st.canonicalize()
    st.sync()
    rng = np.random.default_rng(n)
    idx = np.unique(np.concatenate([rng.integers(0, 2**n, 20000), [0, 2**n - 1]])).astype(np.int64)
    got = t[torch.from_numpy(idx).cuda()].cpu().numpy().astype(np.complex128)
    m = (np.uint64(x) * idx.astype(np.uint64)) % np.uint64(2**n)
    exp = 2 ** (-n / 2) * np.exp(2j * np.pi * m.astype(np.float64) / 2**n)
    assert np.max(np.abs(got - exp)) < (1e-12 if dt == np.complex128 else 1e-5)
    assert np.max(np.abs(p.cpu().numpy() - 1 / 8)) < (1e-12 if dt == np.complex128 else 1e-5)
    assert not torch.isnan(t).any()


@pytest.mark.parametrize("n", [26])
def test_simulate_live_tiles_random(n):
    """A random circuit over several tile passes: qj_simulate (live tiles)
    equals reset + apply_circuit(fused, every tile) + probabilities."""
    circ = C.random_circuit(n, 300, 11, max_targets=2, max_controls=1)
    basis = 0x2F0F0F3 & ((1 << n) - 1)
    qubits = [1, n - 2, n // 2]
    ref = torch.empty(2**n, dtype=torch.complex128, device="cuda")
    sr = qjp.State(ref, basis=basis)
    sr.apply_circuit(circ.gates, fuse=True)
    pr = sr.probabilities(qubits)
    sr.canonicalize()
    sr.sync()
    x = torch.full((2**n,), float("nan"), dtype=torch.complex128, device="cuda")
    st = qjp.State(x, basis=None)
    p = st.simulate(basis, circ.gates, qubits=qubits, fuse=True)
    st.canonicalize()
    st.sync()
    assert torch.max(torch.abs(x - ref)).item() <= 1e-12
    assert np.max(np.abs(p.cpu().numpy() - pr.cpu().numpy())) <= 1e-12
    del ref, x


def test_simulate_fallbacks_and_no_readout():
    n = 15
    circ = C.qft(n)
    t = torch.empty(2**n, dtype=torch.complex128, device="cuda")
    st = qjp.State(t, basis=None)
    assert st.simulate(7, circ.gates, qubits=()) is None  # nq = 0
    st.canonicalize()
    st.sync()
    y = np.arange(2**n, dtype=np.uint64)
    exp = 2 ** (-n / 2) * np.exp(2j * np.pi * ((7 * y) % 2**n).astype(np.float64) / 2**n)
    assert np.max(np.abs(t.cpu().numpy() - exp)) < 1e-12
    p = st.simulate(7, circ.gates, qubits=list(range(11)), fuse=True)  # nq > 10: three-call path
    assert abs(float(p.sum()) - 1) < 1e-12
    p = st.simulate(7, circ.gates, qubits=[0, 1], fuse=False)  # unfused: three-call path
    assert abs(float(p.sum()) - 1) < 1e-12
