"""Pins for the CPU oracle (oracle/qj_oracle.c) against things other than itself.

Each pin is chosen so that a plausible mistake in the oracle (a dropped term,
a wrong sign, a bit-order flip, a transposed matrix, a mis-read control) fails
at least one of them:

  * closed forms: H^n|0> uniform, GHZ, QFT|x> = 2^{-n/2} sum_y e^{2 pi i x y / 2^n}|y>
    (the last one discriminates big- vs little-endian, reading R1, and a
    transposed G, since the QFT matrix is not symmetric under the circuit's
    gate order);
  * a textbook library routine: numpy.tensordot contraction of G over the
    target axes of psi.reshape((2,)*n) (reading R3: first target = MSB);
  * brute force: the full 2^n x 2^n operator built from Kronecker products
    sum_{tau,tau'} G(tau,tau') (x)_i |tau_i><tau'_i| plus the control projector;
  * invariants: norm after 1000 random unitaries, exact permutations;
  * SPEC worked examples (tests/golden/spec_examples.json);
  * probabilities vs numpy reshape-and-sum.
"""

import json
import math
import os

import numpy as np
import pytest

import oracle
from workloads import circuits as C
from workloads import gates as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-12


def rand_state(n, rng):
    v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    return v / np.linalg.norm(v)


def run(circ, x=0):
    return oracle.run(circ, oracle.basis_state(circ.n, x))


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("n", [1, 2, 5, 10])
def test_hadamard_all_uniform(n):
    c = C.Circuit(n)
    for q in range(n):
        c.append(G.H(q))
    psi = run(c)
    assert np.max(np.abs(psi - 2 ** (-n / 2))) < TOL


@pytest.mark.parametrize("n", [2, 5, 9])
def test_ghz(n):
    c = C.Circuit(n)
    c.append(G.H(0))
    for q in range(n - 1):
        c.append(G.CNOT(q, q + 1))
    psi = run(c)
    exp = np.zeros(2**n, dtype=complex)
    exp[0] = exp[-1] = 1 / math.sqrt(2)
    assert np.max(np.abs(psi - exp)) < TOL
    assert np.all(psi[1:-1] == 0)  # the other amplitudes are exactly zero


def qft_closed_form(n, x):
    y = np.arange(2**n, dtype=np.uint64)
    m = (np.uint64(x) * y) % np.uint64(2**n)   # exact integer phase numerator
    return 2 ** (-n / 2) * np.exp(2j * np.pi * m.astype(np.float64) / 2**n)


@pytest.mark.parametrize("n,x", [(3, 1), (4, 3), (6, 37), (8, 0), (8, 201), (10, 0b1011001110)])
def test_qft_basis_closed_form(n, x):
    psi = run(C.qft(n), x)
    assert np.max(np.abs(psi - qft_closed_form(n, x))) < TOL


def test_qft_without_swaps_is_bit_reversed():
    n, x = 6, 45
    psi = run(C.qft(n, swaps=False), x)
    rev = [int(format(i, f"0{n}b")[::-1], 2) for i in range(2**n)]
    assert np.max(np.abs(psi[rev] - qft_closed_form(n, x))) < TOL


# ------------------------------------------------ textbook tensordot formulation
def tensordot_apply(psi, n, targets, controls, M):
    """Contract G over the target axes of psi viewed as a rank-n tensor
    (axis q = qubit q, axis 0 = most significant), on the control=1 slice."""
    T = psi.reshape((2,) * n).copy()
    k = len(targets)
    Gt = np.asarray(M).reshape((2,) * (2 * k))
    idx = tuple(1 if q in controls else slice(None) for q in range(n))
    sub = T[idx]
    rest = [q for q in range(n) if q not in controls]
    tpos = [rest.index(t) for t in targets]
    new = np.tensordot(Gt, sub, axes=(list(range(k, 2 * k)), tpos))
    new = np.moveaxis(new, list(range(k)), tpos)
    T[idx] = new
    return T.reshape(-1)


# ------------------------------------------------ brute-force Kronecker operator
def kron_operator(n, targets, controls, M):
    """U = P (x) sum_{tau,tau'} G(tau,tau') (x)_i |tau_i><tau'_i| + (I - P)."""
    k = len(targets)
    E = [[np.array([[1, 0], [0, 0]]), np.array([[0, 1], [0, 0]])],
         [np.array([[0, 0], [1, 0]]), np.array([[0, 0], [0, 1]])]]
    I2 = np.eye(2)
    P1 = np.array([[0, 0], [0, 1]])
    U = np.zeros((2**n, 2**n), dtype=complex)
    for r in range(2**k):
        for c in range(2**k):
            if M[r, c] == 0:
                continue
            f = []
            for q in range(n):
                if q in targets:
                    i = targets.index(q)
                    f.append(E[(r >> (k - 1 - i)) & 1][(c >> (k - 1 - i)) & 1])
                elif q in controls:
                    f.append(P1)
                else:
                    f.append(I2)
            t = np.array([[1.0]])
            for x in f:
                t = np.kron(t, x)
            U += M[r, c] * t
    Pc = np.array([[1.0]])
    for q in range(n):
        Pc = np.kron(Pc, P1 if q in controls else I2)
    return U + (np.eye(2**n) - Pc)


@pytest.mark.parametrize("seed", range(40))
def test_three_formulations_agree(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 7))
    k = int(rng.integers(1, min(3, n) + 1))
    qs = [int(q) for q in rng.permutation(n)]
    targets = qs[:k]                                   # unsorted on purpose
    controls = qs[k:k + int(rng.integers(0, min(2, n - k) + 1))]
    M = G.random_unitary(k, rng)
    psi = rand_state(n, rng)
    out = np.empty_like(psi)
    oracle.apply_matrix(psi, out, n, targets, controls, M)
    td = tensordot_apply(psi, n, targets, controls, M)
    bf = kron_operator(n, targets, controls, M) @ psi
    assert np.max(np.abs(out - td)) < TOL
    assert np.max(np.abs(out - bf)) < TOL


@pytest.mark.parametrize("seed", range(6))
def test_random_circuit_vs_kron(seed):
    n = 6
    circ = C.random_circuit(n, 25, seed)
    rng = np.random.default_rng(100 + seed)
    psi = rand_state(n, rng)
    out = oracle.run(circ, psi)
    ref = psi.copy()
    for g in circ.gates:
        ref = kron_operator(n, list(g.targets), list(g.controls), g.matrix()) @ ref
    assert np.max(np.abs(out - ref)) < TOL


# --------------------------------------------------------------- invariants
def test_norm_after_1000_random_gates():
    n = 8
    circ = C.random_circuit(n, 1000, 7)
    psi = run(circ)
    assert abs(np.linalg.norm(psi) - 1) < 1e-10


@pytest.mark.parametrize("seed", range(5))
def test_permutations_exact(seed):
    """X, CX, SWAP, CSWAP are exact permutations; Z, CZ exact sign flips (R9)."""
    rng = np.random.default_rng(seed)
    n = 7
    psi = rand_state(n, rng)
    out = np.empty_like(psi)
    idx = np.arange(2**n)
    bit = lambda i, q: (i >> (n - 1 - q)) & 1  # noqa: E731
    # CX control 2 target 5
    oracle.apply_matrix(psi, out, n, [5], [2], G.X(5).matrix())
    src = np.where(bit(idx, 2) == 1, idx ^ (1 << (n - 1 - 5)), idx)
    assert np.array_equal(out, psi[src])
    # SWAP 1 <-> 6
    oracle.apply_matrix(psi, out, n, [1, 6], [], G.SWAP(1, 6).matrix())
    b1, b6 = bit(idx, 1), bit(idx, 6)
    src = np.where(b1 != b6, idx ^ (1 << (n - 2)) ^ 1, idx)
    assert np.array_equal(out, psi[src])
    # CZ(0, 3): negate where both bits are 1
    oracle.apply_matrix(psi, out, n, [3], [0], G.Z(3).matrix())
    sign = np.where((bit(idx, 0) & bit(idx, 3)) == 1, -1, 1)
    assert np.array_equal(out, psi * sign)


def test_spec_examples():
    s2 = 1 / math.sqrt(2)
    # H on zero_state(1) -> [1/sqrt2, 1/sqrt2]
    c = C.Circuit(1)
    c.append(G.H(0))
    assert np.allclose(run(c), [s2, s2], atol=1e-15)
    # CNOT(control 0, target 1) on |10> -> |11>; on |00> -> |00>
    c = C.Circuit(2)
    c.append(G.CNOT(0, 1))
    assert np.array_equal(run(c, 0b10), [0, 0, 0, 1])
    assert np.array_equal(run(c, 0b00), [1, 0, 0, 0])
    # CCZ on uniform 3-qubit superposition -> sign flip on amps[7] only
    psi = np.full(8, 1 / math.sqrt(8), dtype=complex)
    out = np.empty_like(psi)
    oracle.apply_matrix(psi, out, 3, [2], [0, 1], G.Z(2).matrix())
    exp = psi.copy()
    exp[7] *= -1
    assert np.array_equal(out, exp)
    # X on zero_state(1) -> [0,1]; SWAP(0,1)|01> -> |10>
    c = C.Circuit(1)
    c.append(G.X(0))
    assert np.array_equal(run(c), [0, 1])
    c = C.Circuit(2)
    c.append(G.SWAP(0, 1))
    assert np.array_equal(run(c, 0b01), [0, 0, 1, 0])


# ------------------------------------------------------------- probabilities
def numpy_marginal(psi, n, qubits):
    p = (np.abs(psi) ** 2).reshape((2,) * n)
    drop = tuple(q for q in range(n) if q not in qubits)
    m = p.sum(axis=drop) if drop else p
    kept = [q for q in range(n) if q in qubits]
    m = np.transpose(m, [kept.index(q) for q in qubits])
    return m.reshape(-1)


def test_probabilities_golden():
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        gold = json.load(f)["probabilities"]
    for case in gold:
        n = case["n"]
        if case["state"] == "zero":
            psi = oracle.basis_state(n, 0)
        elif case["state"] == "uniform":
            psi = np.full(2**n, 2 ** (-n / 2), dtype=complex)
        else:
            psi = np.zeros(2**n, dtype=complex)
            psi[0] = psi[-1] = 1 / math.sqrt(2)
        p = oracle.probabilities(psi, n, case["qubits"])
        assert np.allclose(p, case["out"], atol=1e-15)


@pytest.mark.parametrize("seed", range(8))
def test_probabilities_vs_numpy(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 9))
    psi = rand_state(n, rng)
    m = int(rng.integers(1, n + 1))
    qubits = [int(q) for q in rng.permutation(n)[:m]]
    p = oracle.probabilities(psi, n, qubits)
    assert np.max(np.abs(p - numpy_marginal(psi, n, qubits))) < 1e-14
    assert abs(p.sum() - 1) < 1e-12
    full = oracle.probabilities(psi, n)
    assert np.max(np.abs(full - np.abs(psi) ** 2)) < 1e-15


def test_probabilities_basis_exact():
    n, x = 9, 0b101100111
    p = oracle.probabilities(oracle.basis_state(n, x), n)
    assert p[x] == 1.0 and np.count_nonzero(p) == 1


@pytest.mark.parametrize("n", [3, 6, 10])
def test_bv_marginal(n):
    psi = run(C.bv(n))
    p = oracle.probabilities(psi, n, list(range(n - 1)))
    assert abs(p[-1] - 1) < 1e-10


# ---------------------------------------------------------------- QFT|x> closed-form checker
# oracle.qft_basis_maxerr (or_qft_basis_maxerr) streams the full-size GPU
# states through the closed form; pinned here to a textbook library routine
# (numpy's inverse FFT: QFT|x> = sqrt(N) ifft(e_x)), to the gate-by-gate
# oracle, and to mutations it must reject.
@pytest.mark.parametrize("n,x", [(1, 1), (4, 11), (7, 0b1011001), (10, 0b1011001110), (12, 2**12 - 1)])
def test_qft_checker_vs_numpy_ifft(n, x):
    e = np.zeros(2**n, dtype=np.complex128)
    e[x] = 1.0
    ref = np.sqrt(2**n) * np.fft.ifft(e)
    m, ss = oracle.qft_basis_maxerr(ref, n, x)
    assert m < 1e-15 and ss < 1e-28
    got = run(C.qft(n), x) if n <= 10 else None
    if got is not None:
        assert oracle.qft_basis_maxerr(got, n, x)[0] < 1e-14


def test_qft_checker_rejects_mutations():
    n, x = 9, 0b100110101
    e = np.zeros(2**n, dtype=np.complex128)
    e[x] = 1.0
    ref = np.sqrt(2**n) * np.fft.ifft(e)
    bad = ref.copy()
    bad[300] += 1e-9
    assert oracle.qft_basis_maxerr(bad, n, x)[0] >= 0.99e-9
    assert oracle.qft_basis_maxerr(np.conj(ref), n, x)[0] > 1e-3        # wrong sign of the phase
    rev = np.array([ref[int(format(i, f"0{n}b")[::-1], 2)] for i in range(2**n)])
    assert oracle.qft_basis_maxerr(rev, n, x)[0] > 1e-3                 # missing final SWAP layer
    assert oracle.qft_basis_maxerr(ref, n, x ^ 1)[0] > 1e-3             # other basis input
    nan = ref.copy()
    nan[5] = np.nan
    assert not oracle.qft_basis_maxerr(nan, n, x)[0] < 1.0              # NaN is a failure
    # chunks: offsets address the same amplitudes
    assert oracle.qft_basis_maxerr(ref[100:200], n, x, offset=100)[0] < 1e-15
    assert oracle.qft_basis_maxerr(ref[100:200], n, x, offset=101)[0] > 1e-3
    # complex64 buffers are widened, not reinterpreted
    m64 = oracle.qft_basis_maxerr(ref.astype(np.complex64), n, x)[0]
    assert 1e-10 < m64 < 1e-7


def test_qft_checker_physical_layout():
    n, x = 8, 0b11010011
    rng = np.random.default_rng(5)
    e = np.zeros(2**n, dtype=np.complex128)
    e[x] = 1.0
    ref = np.sqrt(2**n) * np.fft.ifft(e)
    phys = [int(b) for b in rng.permutation(n)]  # qubit q at bit phys[q]
    buf = np.empty_like(ref)
    for y in range(2**n):
        i = sum(((y >> (n - 1 - q)) & 1) << phys[q] for q in range(n))
        buf[i] = ref[y]
    assert oracle.qft_basis_maxerr(buf, n, x, phys=phys)[0] < 1e-15
    assert oracle.qft_basis_maxerr(buf, n, x)[0] > 1e-3
    wrong = list(phys)
    wrong[0], wrong[1] = wrong[1], wrong[0]
    assert oracle.qft_basis_maxerr(buf, n, x, phys=wrong)[0] > 1e-3
