"""Pins for the shared input generators: Table 2 structure
and self-consistency of the gate definitions (reading R5: the paper prints no
matrices, so named-gate conventions are pinned only by these identities)."""

import json
import math
import os

import numpy as np
import pytest

from workloads import circuits as C
from workloads import gates as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_table2_counts_and_depths():
    with open(os.path.join(GOLD, "table2.json")) as f:
        t2 = json.load(f)
    n = t2["n"]
    for name, circ in (("qft", C.qft(n)), ("variational", C.variational(n, theta=0.1)),
                       ("bv", C.bv(n))):
        assert len(circ) == t2[name]["gates"], name
        assert C.depth(circ) == t2[name]["depth"], name


@pytest.mark.parametrize("n", range(2, 31))
def test_generator_count_formulas(n):
    assert len(C.qft(n)) == n + n * (n - 1) // 2 + n // 2
    assert len(C.bv(n)) == 3 * n - 1
    if n % 2 == 0:
        assert len(C.variational(n, theta=0.1)) == 3 * n


def test_supremacy_config4_shape():
    c = C.supremacy(4, 8, 20)
    one = [g for g in c if g.nt == 1]
    two = [g for g in c if g.kind == "fsim"]
    assert (c.n, len(one), len(two)) == (32, 640, 260)
    # consecutive 1q choices on a qubit always differ (after cycle 0)
    last = {}
    for g in one:
        q = g.targets[0]
        assert last.get(q) != g.name
        last[q] = g.name


def test_qaoa_graph_3_regular():
    c = C.qaoa(12, p=2)
    deg = np.zeros(12, int)
    zz = [g for g in c if g.name == "RZZ"]
    for g in zz[: len(zz) // 2]:
        for q in g.targets:
            deg[q] += 1
    assert np.all(deg == 3)


def _all_gates():
    th = 0.731
    return [G.H(0), G.X(0), G.Y(0), G.Z(0), G.S(0), G.T(0), G.RX(0, th), G.RY(0, th),
            G.RZ(0, th), G.U1(0, th), G.U3(0, th, 0.2, 1.1), G.SQRT_X(0), G.SQRT_Y(0),
            G.SQRT_W(0), G.SWAP(0, 1), G.FSIM(0, 1, th, 0.4), G.RZZ(0, 1, th)]


@pytest.mark.parametrize("g", _all_gates(), ids=lambda g: g.name)
def test_gate_unitary(g):
    m = g.matrix()
    assert np.max(np.abs(m.conj().T @ m - np.eye(len(m)))) < 1e-12


def test_gate_identities():
    assert np.max(np.abs(G.SQRT_X_M @ G.SQRT_X_M - G.X_M)) < 1e-15
    assert np.max(np.abs(G.SQRT_Y_M @ G.SQRT_Y_M - G.Y_M)) < 1e-15
    assert np.max(np.abs(G.SQRT_W_M @ G.SQRT_W_M - G.W_M)) < 1e-15
    assert np.max(np.abs(G.U3(0, math.pi / 2, 0, math.pi).matrix() - G.H_M)) < 1e-15
    assert np.allclose(G.RZ(0, 0.0).matrix(), np.eye(2))
    # sqrt(W) closed form
    sw = np.array([[(1 + 1j) / 2, -1j / math.sqrt(2)], [1 / math.sqrt(2), (1 + 1j) / 2]])
    assert np.max(np.abs(G.SQRT_W_M - sw)) < 1e-15
