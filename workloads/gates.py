"""Gate definitions: the matrices G(tau, tau') of Eq. 1.

The paper names gates (X, Y, Z, SWAP at PAPER.md:238-240; H, CU1, CZ, RY through
the Table 2 circuits) but prints no matrices.  The conventions
below are DESIGN.md reading R5 (Qibo/Cirq/OpenQASM conventions); they are inputs
to both the oracle and the CUDA path and are pinned only by self-consistency
(unitarity, sqrt(P)^2 = P, U3(pi/2,0,pi) = H).

A `Gate` carries
  * ``targets``  qubit labels, first listed = most significant bit of the matrix
                 row/column index (reading R3),
  * ``controls`` qubit labels; the gate acts only where every control is 1
                 (reading R4),
  * ``kind``     which C-ABI entry point the CUDA side uses
                 ('dense' | 'x' | 'z' | 'swap' | 'fsim' | 'diag'),
  * ``data``     the kind-specific payload handed to that entry point.
``Gate.matrix()`` returns the dense 2^k x 2^k target matrix; the oracle only ever
sees this dense form (specialisation is the CUDA side's business).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

KINDS = ("dense", "x", "z", "swap", "fsim", "diag")


@dataclass(frozen=True)
class Gate:
    name: str
    kind: str
    targets: tuple
    controls: tuple = ()
    data: tuple = field(default=(), compare=False)

    @property
    def nt(self) -> int:
        return len(self.targets)

    @property
    def qubits(self) -> tuple:
        return tuple(self.targets) + tuple(self.controls)

    def matrix(self) -> np.ndarray:
        """Dense 2^k x 2^k complex128 matrix of the target action."""
        k = self.nt
        if self.kind == "dense":
            return np.array(self.data[0], dtype=np.complex128).reshape(2**k, 2**k)
        if self.kind == "x":
            return np.array([[0, 1], [1, 0]], dtype=np.complex128)
        if self.kind == "z":
            return np.array([[1, 0], [0, -1]], dtype=np.complex128)
        if self.kind == "swap":
            m = np.zeros((4, 4), dtype=np.complex128)
            m[0, 0] = m[1, 2] = m[2, 1] = m[3, 3] = 1
            return m
        if self.kind == "fsim":
            u, p = self.data
            u = np.asarray(u, dtype=np.complex128).reshape(2, 2)
            m = np.zeros((4, 4), dtype=np.complex128)
            m[0, 0] = 1
            m[1:3, 1:3] = u
            m[3, 3] = p
            return m
        if self.kind == "diag":
            return np.diag(np.asarray(self.data[0], dtype=np.complex128).reshape(2**k))
        raise ValueError(f"unknown kind {self.kind}")


def _dense(name, targets, m, controls=()):
    m = np.asarray(m, dtype=np.complex128)
    return Gate(name, "dense", tuple(targets), tuple(controls), (m,))


# ---- one-qubit gates ---------------------------------------------------------
SQ2 = 1.0 / math.sqrt(2.0)
H_M = np.array([[SQ2, SQ2], [SQ2, -SQ2]], dtype=np.complex128)
Y_M = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
X_M = np.array([[0, 1], [1, 0]], dtype=np.complex128)
I_M = np.eye(2, dtype=np.complex128)
W_M = (X_M + Y_M) / math.sqrt(2.0)


def H(q):
    return _dense("H", (q,), H_M)


def X(q, controls=()):
    return Gate("X" if not controls else "C" * len(controls) + "X", "x", (q,), tuple(controls))


def Y(q):
    return _dense("Y", (q,), Y_M)


def Z(q, controls=()):
    return Gate("Z" if not controls else "C" * len(controls) + "Z", "z", (q,), tuple(controls))


def CZ(a, b):
    """CZ = diag(1,1,1,-1) on (a, b): Z on b controlled by a."""
    return Z(b, controls=(a,))


def CNOT(c, t):
    return X(t, controls=(c,))


def S(q):
    return Gate("S", "diag", (q,), (), (np.array([1, 1j], dtype=np.complex128),))


def T(q):
    return Gate("T", "diag", (q,), (), (np.array([1, np.exp(1j * math.pi / 4)]),))


def RX(q, theta):
    c, s = math.cos(theta / 2), math.sin(theta / 2)
    return _dense("RX", (q,), [[c, -1j * s], [-1j * s, c]])


def RY(q, theta):
    c, s = math.cos(theta / 2), math.sin(theta / 2)
    return _dense("RY", (q,), [[c, -s], [s, c]])


def RZ(q, theta):
    return Gate("RZ", "diag", (q,), (),
                (np.array([np.exp(-0.5j * theta), np.exp(0.5j * theta)]),))


def U1(q, lam, controls=()):
    name = "U1" if not controls else "CU1"
    return Gate(name, "diag", (q,), tuple(controls), (np.array([1, np.exp(1j * lam)]),))


def CU1(c, t, lam):
    """Controlled U1(lam): control c, target t (SPEC S:505 QFT construction)."""
    return U1(t, lam, controls=(c,))


def U3(q, theta, phi, lam):
    c, s = math.cos(theta / 2), math.sin(theta / 2)
    return _dense("U3", (q,), [[c, -np.exp(1j * lam) * s],
                               [np.exp(1j * phi) * s, np.exp(1j * (phi + lam)) * c]])


def sqrt_pauli(P):
    """sqrt(P) = ((1+i)/2) I + ((1-i)/2) P for a Pauli-like involution P."""
    return 0.5 * (1 + 1j) * I_M + 0.5 * (1 - 1j) * P


SQRT_X_M = sqrt_pauli(X_M)
SQRT_Y_M = sqrt_pauli(Y_M)
SQRT_W_M = sqrt_pauli(W_M)


def SQRT_X(q):
    return _dense("SX", (q,), SQRT_X_M)


def SQRT_Y(q):
    return _dense("SY", (q,), SQRT_Y_M)


def SQRT_W(q):
    return _dense("SW", (q,), SQRT_W_M)


# ---- two-qubit gates ---------------------------------------------------------
def SWAP(a, b, controls=()):
    return Gate("SWAP" if not controls else "CSWAP", "swap", (a, b), tuple(controls))


def FSIM(a, b, theta, phi, controls=()):
    """fSim(theta, phi) = [[1,0,0,0],[0,c,-is,0],[0,-is,c,0],[0,0,0,e^{-i phi}]]
    (optionally controlled: acts where every control qubit is 1)."""
    c, s = math.cos(theta), math.sin(theta)
    u = np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)
    return Gate("FSIM", "fsim", (a, b), tuple(controls), (u, complex(np.exp(-1j * phi))))


def RZZ(a, b, gamma):
    e = np.exp(-0.5j * gamma)
    f = np.exp(0.5j * gamma)
    return Gate("RZZ", "diag", (a, b), (), (np.array([e, f, f, e]),))


def unitary(name, targets, m, controls=()):
    """An arbitrary dense gate (e.g. a random unitary or a fused matrix)."""
    return _dense(name, targets, m, controls)


def random_unitary(k: int, rng: np.random.Generator) -> np.ndarray:
    """Haar-ish random 2^k x 2^k unitary (QR of a complex Gaussian matrix)."""
    d = 2**k
    z = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return q * ph[None, :]
