"""Row f3: Trotterized adiabatic TFIM evolution
as a circuit of gates.  The dense-exponential oracle (oracle/evolution.py, the
paper's "trivial algorithm") is pinned to SPEC's worked examples and
closed forms; the Trotter circuits, run through the gate oracle, are pinned to
it (second-order convergence slope, single-term exactness, adiabatic ground
energy)."""

import math

import numpy as np
import pytest

import oracle
from oracle import evolution as E
from workloads import evolution as W


def kron(*ms):
    out = np.array([[1.0 + 0j]])
    for m in ms:
        out = np.kron(out, m)
    return out


def test_dense_step_examples():
    plus = np.array([1, 1]) / math.sqrt(2)
    minus = np.array([1, -1]) / math.sqrt(2)
    # e^{-i (pi/2) Z} |+> = -i |->  (SPEC S:440-443 states dt = pi, which gives -|+>; reading R25)
    out = E.dense_step(plus, E.Z, math.pi / 2)
    assert abs(abs(np.vdot(minus, out)) - 1) < 1e-12
    assert np.allclose(E.dense_step(plus, E.Z, math.pi), -plus, atol=1e-12)
    assert np.allclose(E.dense_step(plus, np.zeros((2, 2)), 0.3), plus)
    assert np.allclose(E.dense_step(plus, E.Z, 0.0), plus)


def test_tfim_hamiltonian_examples():
    assert np.allclose(E.tfim_hamiltonian(2, 0.0), -(kron(E.X, E.I2) + kron(E.I2, E.X)))
    assert np.allclose(E.tfim_hamiltonian(2, 1.0, h=0.0), -2 * kron(E.Z, E.Z))
    for s in np.linspace(0, 1, 11):
        H = E.tfim_hamiltonian(5, s, h=0.7)
        assert np.allclose(H, H.conj().T, atol=1e-12)


def run_circuit(c, psi):
    return oracle.run(c, psi)


def test_single_term_step_is_exact():
    """n=2, s=1, h=0: one Trotter step is a pure ZZ rotation == dense step."""
    dt = 0.37
    c = W.evolution_circuit(2, 1.0, dt, dt, h=0.0)
    rng = np.random.default_rng(0)
    psi = rng.standard_normal(4) + 1j * rng.standard_normal(4)
    psi /= np.linalg.norm(psi)
    exp = E.dense_step(psi, E.tfim_hamiltonian(2, 1.0, h=0.0), dt)
    assert np.max(np.abs(run_circuit(c, psi) - exp)) < 1e-12


def test_second_order_convergence():
    """Global error of the adiabatic Trotter path vs the dense path at n = 6,
    T = 1: log-log slope 2.0 +- 0.2 over dt in {0.08, 0.04, 0.02, 0.01}."""
    n, T = 6, 1.0
    dts = [0.08, 0.04, 0.02, 0.01]
    errs = []
    for dt in dts:
        c = W.adiabatic_circuit(n, T, dt)
        psi_t = run_circuit(c, oracle.basis_state(n, 0))
        psi_d = E.adiabatic_dense(n, T, dt)
        errs.append(np.linalg.norm(psi_t - psi_d))
    slope = np.polyfit(np.log(dts), np.log(errs), 1)[0]
    assert 1.8 <= slope <= 2.2, (slope, errs)


def test_adiabatic_ground_energy():
    """n = 4, T = 50, dt = 0.05: <H1> within 2% of the exact ground energy."""
    n = 4
    c = W.adiabatic_circuit(n, 50.0, 0.05)
    psi = run_circuit(c, oracle.basis_state(n, 0))
    H1 = E.tfim_hamiltonian(n, 1.0)
    e0 = np.linalg.eigvalsh(H1)[0]
    assert abs(E.energy(psi, H1) - e0) <= 0.02 * abs(e0)
    # a diabatic schedule stays well above the ground energy
    fast = run_circuit(W.adiabatic_circuit(n, 0.1, 0.05), oracle.basis_state(n, 0))
    assert E.energy(fast, H1) > e0 + 0.05 * abs(e0)
