"""GPU parity for measurement through
the C ABI, against oracle/measure.py on the same seeded inputs:

* collapse: element-wise within 1e-12 (c128) / 1e-5 (c64), zeroed amplitudes
  exactly 0, on plain, remapped (fused SWAP relabels) and virtual-sharded
  states; zero-probability outcomes fail and leave the state bit-identical.
* samplers: given the ORACLE's probability array, the CUDA direct sampler
  (exact fixed-point CDF, R27) and both Metropolis variants (R28) reproduce
  the oracle's samples bit for bit (same Philox4x32-10 counters); counts are
  the exact histogram of the samples.
* state sampling / measurement: statistical agreement with the exact marginal
  (TV, zero-probability outcomes never drawn), determinism under a seed.
"""

import math

import numpy as np
import pytest

import oracle
from oracle import measure as M
from workloads import circuits as C
from workloads import gates as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
qjp = pytest.importorskip("paper_2203_08826_b200")
from paper_2203_08826_b200 import qj as Q  # noqa: E402

TOL = {np.complex128: 1e-12, np.complex64: 1e-5}
TDT = {np.complex128: torch.complex128, np.complex64: torch.complex64}
DTYPES = [np.complex128, np.complex64]


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2203_08826_b200 import build
    build.build()


def rand_state(n, seed, dt=np.complex128):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    return (v / np.linalg.norm(v)).astype(dt)


def check_collapsed(got, exp, dt):
    got = got.astype(np.complex128)
    assert np.all(got[exp == 0] == 0), "inconsistent amplitudes must be exactly 0"
    err = np.max(np.abs(got - exp))
    assert err <= TOL[dt], f"max abs err {err:.3e}"


# ------------------------------------------------------------------ collapse
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("qubits", [[0], [10], [9], [10, 0], [3, 10, 6], [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 0]])
def test_collapse_vs_oracle(dt, qubits):
    n = 11
    psi = rand_state(n, 7, dt)
    outs = range(2 ** len(qubits)) if len(qubits) <= 3 else [0, 1234, 2047]
    for outcome in outs:
        x = torch.from_numpy(psi.copy()).cuda()
        st = qjp.State(x, basis=None)
        try:
            exp, pe = M.collapse(psi.astype(np.complex128), n, qubits, outcome)
        except M.ZeroProbabilityOutcome:
            continue
        p = st.collapse(qubits, outcome)
        st.sync()
        assert abs(p - pe) <= (1e-14 if dt == np.complex128 else 1e-6)
        check_collapsed(x.cpu().numpy(), exp, dt)


@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
def test_collapse_after_fused_relabels(dt):
    """Fused circuits leave the state in a permuted bit order (SWAP relabels);
    collapse names logical qubits regardless."""
    n = 12
    circ = C.random_circuit(n, 120, 5, max_targets=2, max_controls=1)
    circ.gates += [G.SWAP(0, 11), G.SWAP(3, 7), G.H(2), G.SWAP(1, 10)]
    psi = rand_state(n, 3, dt)
    mats = [g.matrix().astype(dt).astype(np.complex128) for g in circ.gates]
    ref = oracle.run(circ, psi.astype(np.complex128), mats)
    for qubits, outcome in (([0], 1), ([11, 3], 2), ([10, 1, 0], 5)):
        x = torch.from_numpy(psi.copy()).cuda()
        st = qjp.State(x, basis=None)
        st.apply_circuit(circ.gates, fuse=True)
        p = st.collapse(qubits, outcome)
        st.canonicalize()
        st.sync()
        exp, pe = M.collapse(ref, n, qubits, outcome)
        assert abs(p - pe) < 1e-6
        check_collapsed(x.cpu().numpy(), exp, dt)


@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("nshards", [2, 8])
def test_collapse_sharded(dt, nshards):
    """Virtual ranks: global qubits select whole shards (zeroed or scaled)."""
    n = 11
    psi = rand_state(n, 11, dt)
    for qubits, outcome in (([0], 1), ([1, 9], 2), ([2, 0, 10], 6)):
        parts = [torch.from_numpy(c.copy()).cuda() for c in np.split(psi, nshards)]
        st = qjp.State.sharded(parts, n, basis=None)
        p = st.collapse(qubits, outcome)
        st.sync()
        exp, pe = M.collapse(psi.astype(np.complex128), n, qubits, outcome)
        assert abs(p - pe) < 1e-6
        got = np.concatenate([t.cpu().numpy() for t in parts])
        check_collapsed(got, exp, dt)


def test_collapse_spec_examples_and_zero_probability():
    bell = (np.array([1, 0, 0, 1]) / math.sqrt(2)).astype(np.complex128)
    x = torch.from_numpy(bell.copy()).cuda()
    st = qjp.State(x, basis=None)
    assert abs(st.collapse([0], 0) - 0.5) < 1e-15
    assert np.max(np.abs(x.cpu().numpy() - np.array([1, 0, 0, 0]))) < 1e-15
    # idempotent
    assert abs(st.collapse([0], 0) - 1.0) < 1e-15
    # zero probability: error, state bit-identical
    psi = rand_state(6, 1)
    psi[psi.size // 2:] = 0  # qubit 0 is 0 with certainty
    psi /= np.linalg.norm(psi)
    x = torch.from_numpy(psi.copy()).cuda()
    st = qjp.State(x, basis=None)
    with pytest.raises(Q.QJError) as e:
        st.collapse([0], 1)
    assert e.value.code == 10
    assert np.array_equal(x.cpu().numpy(), psi)


# ------------------------------------------------------------------ samplers: bit-exact parity
def gpu_probs(p):
    return torch.from_numpy(np.ascontiguousarray(p, dtype=np.float64)).cuda()


@pytest.mark.parametrize("m,nshots,seed", [(1, 1000, 1), (6, 100000, 2), (10, 4099, 3), (0, 10, 4)])
def test_direct_sampler_bit_exact(m, nshots, seed):
    p = M.marginal(rand_state(max(m, 1), 50 + m), max(m, 1), range(m)) if m else np.array([1.0])
    if m >= 6:
        p[3] = 0.0  # a zero bin inside the support
    s, c = qjp.sample_distribution(gpu_probs(p), nshots, seed)
    s = s.cpu().numpy()
    exp = M.sample_direct(p, nshots, seed)
    assert np.array_equal(s, exp)
    assert np.array_equal(c.cpu().numpy(), M.frequencies(exp, m))


def test_direct_sampler_large_marginal_bit_exact():
    """2^24 bins (several thousand scan tiles and a ragged shot count)."""
    rng = np.random.default_rng(24)
    p = rng.exponential(size=2**24)
    p[rng.integers(0, 2**24, 1000)] = 0
    p /= p.sum()
    s, _ = qjp.sample_distribution(gpu_probs(p), 100003, 99, counts=False)
    assert np.array_equal(s.cpu().numpy(), M.sample_direct(p, 100003, 99))


@pytest.mark.parametrize("method,proposal", [("metropolis", "uniform"), ("metropolis_flip", "flip")])
@pytest.mark.parametrize("m,nshots,nchains,burnin", [(4, 10000, 0, None), (8, 30001, 7, 13), (6, 5000, 5000, None),
                                                     (1, 100, 3, 0)])
def test_metropolis_bit_exact(method, proposal, m, nshots, nchains, burnin):
    p = M.marginal(rand_state(m, 60 + m), m, range(m))
    if m >= 4:
        p[1] = 0.0
    s, c = qjp.sample_distribution(gpu_probs(p), nshots, 77, method=method, nchains=nchains, burnin=burnin)
    exp = M.sample_metropolis(p, nshots, 77, nchains=nchains, burnin=burnin, proposal=proposal)
    assert np.array_equal(s.cpu().numpy(), exp)
    assert np.array_equal(c.cpu().numpy(), M.frequencies(exp, m))


def test_counts_only_and_zero_total():
    p = np.zeros(8)
    with pytest.raises(Q.QJError) as e:
        qjp.sample_distribution(gpu_probs(p), 10, 1)
    assert e.value.code == 10
    p[5] = 1.0
    s, c = qjp.sample_distribution(gpu_probs(p), 1000, 1, samples=False)
    assert s is None and c.cpu().numpy()[5] == 1000


# ------------------------------------------------------------------ sampling a state
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
@pytest.mark.parametrize("method", ["direct", "metropolis", "metropolis_flip"])
def test_state_sampling_statistics(dt, method):
    n = 8
    psi = rand_state(n, 21, dt)
    x = torch.from_numpy(psi.copy()).cuda()
    st = qjp.State(x, basis=None)
    qubits = [7, 0, 3, 4, 1, 6]
    s, c = st.sample(qubits, 10**6, 5, method=method)
    st.sync()
    pe = M.marginal(psi.astype(np.complex128), n, qubits)
    f = c.cpu().numpy() / 10**6
    assert 0.5 * np.abs(f - pe).sum() <= 0.02
    assert c.cpu().numpy().sum() == 10**6
    assert np.array_equal(np.bincount(s.cpu().numpy(), minlength=64), c.cpu().numpy())
    s2, c2 = st.sample(qubits, 10**6, 5, method=method)
    assert torch.equal(s, s2) and torch.equal(c, c2)
    # the state is untouched
    assert np.array_equal(x.cpu().numpy(), psi)


def test_state_sampling_bell_and_basis():
    bell = (np.array([1, 0, 0, 1]) / math.sqrt(2)).astype(np.complex128)
    for method in ("direct", "metropolis", "metropolis_flip"):
        st = qjp.State(torch.from_numpy(bell.copy()).cuda(), basis=None)
        _, c = st.sample([0, 1], 10**5, 3, method=method, samples=False)
        c = c.cpu().numpy()
        assert c[1] == 0 and c[2] == 0 and c.sum() == 10**5
        assert abs(c[0] - 50000) < 5 * math.sqrt(10**5 * 0.25) or method != "direct"
    t = torch.empty(2**12, dtype=torch.complex128, device="cuda")
    st = qjp.State(t, basis=0b101101001110)
    s, _ = st.sample(list(range(12)), 1000, 1)
    assert np.all(s.cpu().numpy() == 0b101101001110)


def test_state_sample_matches_oracle_on_oracle_marginal():
    """qj_sample draws from the state's marginal: with the direct method its
    samples equal the oracle's draws from the oracle's marginal except where
    a last-ulp difference of a bin moves a fixed-point boundary (none here)."""
    n = 14
    psi = rand_state(n, 8)
    st = qjp.State(torch.from_numpy(psi.copy()).cuda(), basis=None)
    qubits = [13, 2, 7, 0, 9]
    s, _ = st.sample(qubits, 50000, 123)
    exp = M.sample_direct(M.marginal(psi, n, qubits), 50000, 123)
    assert np.mean(s.cpu().numpy() == exp) > 0.9999


# ------------------------------------------------------------------ measurement
@pytest.mark.parametrize("dt", DTYPES, ids=["c128", "c64"])
def test_measure_draws_and_collapses(dt):
    n = 10
    psi = rand_state(n, 4, dt)
    qubits = [2, 9]
    pe = M.marginal(psi.astype(np.complex128), n, qubits)
    seen = set()
    for seed in range(40):
        x = torch.from_numpy(psi.copy()).cuda()
        st = qjp.State(x, basis=None)
        o, p = st.measure(qubits, seed)
        st.sync()
        if dt == np.complex128:  # same draw as the oracle (shot 0 of the seed)
            assert o == int(M.sample_direct(pe, 1, seed)[0])
        assert abs(p - pe[o]) < (1e-12 if dt == np.complex128 else 1e-6)
        exp, _ = M.collapse(psi.astype(np.complex128), n, qubits, o)
        check_collapsed(x.cpu().numpy(), exp, dt)
        seen.add(o)
    assert len(seen) == 4
