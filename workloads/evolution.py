"""Trotterized adiabatic evolution of the transverse-field Ising model as a
circuit of gates ("the time evolution is decomposed into a
circuit of unitary gates"; SPEC S:417-489 for the conventions).

H(s) = (1 - s) H0 + s H1,  H0 = -sum_i X_i,  H1 = -sum_i (Z_i Z_{i+1} + h X_i)
(ring indexing when periodic; h = 1 by default -- the paper states no
coefficients, reading R24).  One second-order symmetric Trotter step
of length dt: half-step even ZZ bonds, half-step odd ZZ bonds, full X layer,
half-step odd, half-step even.  ZZ factors are RZZ diagonal
gates, X factors RX gates, so the GPU runs them through the ordinary gate path.
These are inputs (gate definitions); the dense-exponential oracle lives in
oracle/evolution.py.
"""

from __future__ import annotations

import math

from . import gates as G
from .circuits import Circuit


def bonds(n: int, periodic: bool = True):
    b = [(i, i + 1) for i in range(n - 1)]
    if periodic and n >= 2:
        b.append((n - 1, 0))  # on n = 2 the two ring bonds coincide
    return b


def trotter_step(c: Circuit, s: float, dt: float, h: float = 1.0, periodic: bool = True):
    n = c.n
    bb = bonds(n, periodic)
    even = [e for k, e in enumerate(bb) if k % 2 == 0]
    odd = [e for k, e in enumerate(bb) if k % 2 == 1]
    # e^{-i (-s) Z Z tau} = RZZ(gamma) with RZZ(gamma) = e^{-i gamma/2 ZZ}: gamma = -2 s tau
    zz_half = -2.0 * s * (dt / 2)
    cx = -(1.0 - s) - s * h  # X coefficient of H(s)
    for layer in (even, odd):
        for (a, b) in layer:
            c.append(G.RZZ(a, b, zz_half))
    for q in range(n):
        c.append(G.RX(q, 2.0 * cx * dt))  # RX(theta) = e^{-i theta/2 X}
    for layer in (odd, even):
        for (a, b) in layer:
            c.append(G.RZZ(a, b, zz_half))
    return c


def adiabatic_circuit(n: int, T: float, dt: float, h: float = 1.0, periodic: bool = True,
                      prepare: bool = True) -> Circuit:
    """|+>^n (ground state of H0), then T/dt Trotter steps with the linear
    schedule s = t/T evaluated at the step midpoint."""
    c = Circuit(n, name=f"tfim{n}_T{T}_dt{dt}")
    if prepare:
        for q in range(n):
            c.append(G.H(q))
    steps = int(round(T / dt))
    for k in range(steps):
        s = (k + 0.5) * dt / T
        trotter_step(c, s, dt, h, periodic)
    return c


def evolution_circuit(n: int, s: float, t: float, dt: float, h: float = 1.0, periodic: bool = True) -> Circuit:
    """Fixed-s evolution e^{-i H(s) t} by t/dt Trotter steps (no preparation)."""
    c = Circuit(n, name=f"tfim{n}_s{s}_t{t}_dt{dt}")
    for _ in range(int(round(t / dt))):
        trotter_step(c, s, dt, h, periodic)
    return c
