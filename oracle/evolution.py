"""Dense time-evolution oracle -- TEST INFRASTRUCTURE ONLY.

The paper's "trivial algorithm for unitary time evolution calculates the
exponential of the Hamiltonian matrix e^{-iH(t) dt} at each time t"
(PAPER.md:597-599).  Written out plainly: H(s) built from Kronecker products
of Pauli matrices, each step applied as V e^{-i Lambda dt} V^dagger
from the Hermitian eigendecomposition, numpy in complex128.
It checks the Trotter circuits (workloads/evolution.py) run through the gate
oracle and the GPU path.  Pins: tests/test_evolution.py (SPEC examples,
closed-form single-term steps, Hermiticity).
"""

from __future__ import annotations

import numpy as np

X = np.array([[0, 1], [1, 0]], dtype=complex)
Z = np.array([[1, 0], [0, -1]], dtype=complex)
I2 = np.eye(2, dtype=complex)


def op_on(n: int, ops: dict) -> np.ndarray:
    """Kronecker product with ops[q] at qubit q (qubit 0 = leftmost = MSB)."""
    m = np.array([[1.0 + 0j]])
    for q in range(n):
        m = np.kron(m, ops.get(q, I2))
    return m


def tfim_hamiltonian(n: int, s: float, h: float = 1.0, periodic: bool = True) -> np.ndarray:
    """H(s) = (1-s)(-sum X_i) + s(-sum (Z_i Z_{i+1} + h X_i))."""
    H = np.zeros((2**n, 2**n), dtype=complex)
    for q in range(n):
        H -= (1.0 - s) * op_on(n, {q: X})
        H -= s * h * op_on(n, {q: X})
    bonds = [(i, i + 1) for i in range(n - 1)]
    if periodic and n >= 2:
        bonds.append((n - 1, 0))  # on n = 2 the two ring bonds coincide
    for (a, b) in bonds:
        H -= s * op_on(n, {a: Z, b: Z})
    return H


def dense_step(psi: np.ndarray, H: np.ndarray, dt: float) -> np.ndarray:
    """psi <- V e^{-i Lambda dt} V^dagger psi."""
    lam, V = np.linalg.eigh(H)
    return V @ (np.exp(-1j * lam * dt) * (V.conj().T @ psi))


def adiabatic_dense(n: int, T: float, dt: float, h: float = 1.0, periodic: bool = True) -> np.ndarray:
    """|+>^n evolved with dense steps of H(s) at the step midpoints s = (k + 1/2) dt / T."""
    psi = np.full(2**n, 2 ** (-n / 2), dtype=complex)
    for k in range(int(round(T / dt))):
        psi = dense_step(psi, tfim_hamiltonian(n, (k + 0.5) * dt / T, h, periodic), dt)
    return psi


def energy(psi: np.ndarray, H: np.ndarray) -> float:
    return float(np.real(np.vdot(psi, H @ psi)))
