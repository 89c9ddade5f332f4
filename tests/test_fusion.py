"""The paper's gate fusion as implemented by the library's
host planner (qj_fuse_circuit): pinned to Table 2's fused columns
(Gates* / Depth*), to the oracle (a fused circuit computes
the same state) and to SPEC's fusion examples."""

import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2203_08826_b200 import qj as Q
from workloads import circuits as C
from workloads import gates as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2203_08826_b200 import build
    build.build()


def fused_depth(gates, n):
    return C.depth(C.Circuit(n, list(gates)))


def test_table2_fused_columns():
    t2 = json.load(open(os.path.join(GOLD, "table2.json")))
    n = t2["n"]
    for name, circ in (("qft", C.qft(n)), ("variational", C.variational(n, theta=0.1)), ("bv", C.bv(n))):
        f = Q.fuse_circuit(n, circ.gates)
        assert len(f) == t2[name]["gates_fused"], name
        assert fused_depth(f, n) == t2[name]["depth_fused"], name
        assert all(len(g.qubits) <= 2 for g in f)


@pytest.mark.parametrize("seed", range(12))
def test_fused_circuit_equals_original(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 9))
    circ = C.random_circuit(n, 60, 500 + seed, max_targets=3, max_controls=2)
    f = Q.fuse_circuit(n, circ.gates)
    assert len(f) <= len(circ)
    psi = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    psi /= np.linalg.norm(psi)
    a = oracle.run(circ, psi)
    b = oracle.run(C.Circuit(n, f), psi, [g.m if hasattr(g, "m") else g.matrix() for g in f])
    assert np.max(np.abs(a - b)) < 1e-12  # global phase included


def test_fusion_idempotent_and_generators():
    for circ in (C.qft(12), C.variational(12, layers=2), C.bv(12), C.supremacy(3, 4, 8), C.qaoa(12, 2)):
        n = circ.n
        f = Q.fuse_circuit(n, circ.gates)
        f2 = Q.fuse_circuit(n, f)
        assert len(f2) == len(f)
        psi = oracle.basis_state(n, 5)
        a = oracle.run(circ, psi)
        b = oracle.run(C.Circuit(n, f), psi, [g.m if hasattr(g, "m") else g.matrix() for g in f])
        assert np.max(np.abs(a - b)) < 1e-12


def test_spec_fusion_examples():
    # [H on q0] alone -> 2x2 H
    f = Q.fuse_circuit(1, [G.H(0)])
    assert len(f) == 1 and np.allclose(f[0].matrix() if hasattr(f[0], "matrix") else f[0].m, G.H_M)
    # [X, X] -> identity
    f = Q.fuse_circuit(1, [G.Gate("X", "dense", (0,), (), (G.X_M,)), G.Gate("X", "dense", (0,), (), (G.X_M,))])
    assert len(f) == 1 and np.allclose(f[0].m, np.eye(2))
    # [RY(a), RY(b)] -> RY(a+b)
    a, b = 0.37, 1.21
    f = Q.fuse_circuit(1, [G.RY(0, a), G.RY(0, b)])
    assert np.max(np.abs(f[0].m - G.RY(0, a + b).matrix())) < 1e-12


# ---- wider fusion ("fusing gates up to about five [qubits]
# may provide additional advantage"): the same greedy rule with max_qubits 1..5
@pytest.mark.parametrize("k", [1, 3, 4, 5])
@pytest.mark.parametrize("seed", range(6))
def test_wide_fusion_equals_original(k, seed):
    rng = np.random.default_rng(100 * k + seed)
    n = int(rng.integers(k + 1, 10))
    circ = C.random_circuit(n, 80, 900 + 10 * k + seed, max_targets=3, max_controls=2)
    f = Q.fuse_circuit(n, circ.gates, k)
    assert len(f) <= len(circ)
    for g in f:  # fused groups never exceed k qubits; wider gates pass through unchanged
        assert len(g.qubits) <= k or any(g is h for h in circ.gates)
    psi = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    psi /= np.linalg.norm(psi)
    a = oracle.run(circ, psi)
    b = oracle.run(C.Circuit(n, f), psi, [g.m if hasattr(g, "m") else g.matrix() for g in f])
    assert np.max(np.abs(a - b)) < 1e-12


def test_wide_fusion_counts_monotone_and_generators():
    """Wider fusion never yields more gates than narrower on the BASELINE
    generators, k=2 reproduces Table 2, and every width computes the same state."""
    for circ in (C.qft(10), C.bv(10), C.supremacy(3, 4, 8), C.qaoa(10, 2), C.variational(10, layers=2)):
        n = circ.n
        counts = [len(Q.fuse_circuit(n, circ.gates, k)) for k in (1, 2, 3, 4, 5)]
        assert counts[1:] == sorted(counts[1:], reverse=True), (circ.name, counts)
        psi = oracle.basis_state(n, 3)
        a = oracle.run(circ, psi)
        for k in (3, 5):
            f = Q.fuse_circuit(n, circ.gates, k)
            b = oracle.run(C.Circuit(n, f), psi, [g.m if hasattr(g, "m") else g.matrix() for g in f])
            assert np.max(np.abs(a - b)) < 1e-12, (circ.name, k)


def test_fusion_width_rejected_above_5():
    with pytest.raises(Q.QJError):
        Q.fuse_circuit(3, [G.H(0)], 6)
