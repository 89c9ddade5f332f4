"""Pins for the measurement oracle (oracle/measure.py, SURVEY 8(f) row f2,
PAPER.md:239-242): Philox known-answer vectors, collapse against projectors
built from Kronecker products, SPEC's worked examples, and the
statistical properties of both samplers (chi-square against the exact
multinomial, total variation, zero-probability outcomes never drawn)."""

import json
import math
import os

import numpy as np
import pytest
from scipy import stats

import oracle
from oracle import measure as M

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.json")


def test_philox_known_answers():
    for v in json.load(open(GOLD))["philox4x32_10"]:
        c = [int(x, 16) for x in v["ctr"]]
        k = [int(x, 16) for x in v["key"]]
        out = [int(w) for w in M.philox4x32_10(*c, *k)]
        assert out == [int(x, 16) for x in v["out"]]


def test_uniform53_range_and_mean():
    i = np.arange(200000, dtype=np.uint64)
    w = M.philox4x32_10(i, 0, 0, 0, 7, 0)
    u = M.uniform53(w[0], w[1])
    assert u.min() >= 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 5 * math.sqrt(1 / 12 / len(u))
    assert M.uniform53(0xFFFFFFFF, 0xFFFFFFFF) == 1 - 2.0**-53


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    return v / np.linalg.norm(v)


def projector(n, qubits, outcome):
    P0 = np.diag([1.0, 0.0])
    P1 = np.diag([0.0, 1.0])
    ops = {}
    for j, q in enumerate(qubits):
        ops[q] = P1 if (outcome >> (len(qubits) - 1 - j)) & 1 else P0
    m = np.array([[1.0]])
    for q in range(n):
        m = np.kron(m, ops.get(q, np.eye(2)))
    return m


@pytest.mark.parametrize("qubits", [[0], [3], [4, 1], [2, 0, 3]])
def test_collapse_matches_projector(qubits):
    n = 5
    psi = rand_state(n, 3)
    for outcome in range(2 ** len(qubits)):
        P = projector(n, qubits, outcome)
        v = P @ psi
        p = float(np.vdot(v, v).real)
        got, pg = M.collapse(psi, n, qubits, outcome)
        assert abs(pg - p) < 1e-14
        assert np.max(np.abs(got - v / math.sqrt(p))) < 1e-14
        assert abs(np.linalg.norm(got) - 1) < 1e-12
        # idempotent
        again, p2 = M.collapse(got, n, qubits, outcome)
        assert abs(p2 - 1) < 1e-12 and np.max(np.abs(again - got)) < 1e-14
        # P(outcome) agrees with the marginal
        assert abs(M.marginal(psi, n, qubits)[outcome] - p) < 1e-14


def test_collapse_spec_examples():
    bell = np.array([1, 0, 0, 1]) / math.sqrt(2)
    got, p = M.collapse(bell, 2, [0], 0)
    assert np.array_equal(got, np.array([1, 0, 0, 0], dtype=complex)) and abs(p - 0.5) < 1e-15
    with pytest.raises(M.ZeroProbabilityOutcome):
        M.collapse(oracle.basis_state(1, 0), 1, [0], 1)
    uni = np.full(8, 8 ** -0.5)
    got, p = M.collapse(uni, 3, [1], 0)
    assert np.allclose(got, np.array([1, 1, 0, 0, 1, 1, 0, 0]) / 2) and abs(p - 0.5) < 1e-15


def test_marginal_spec_examples():
    assert np.allclose(M.marginal(oracle.basis_state(2, 0), 2, [0]), [1, 0])
    assert np.allclose(M.marginal(np.full(4, 0.5), 2, [0, 1]), [0.25] * 4)
    bell = np.array([1, 0, 0, 1]) / math.sqrt(2)
    assert np.allclose(M.marginal(bell, 2, [1]), [0.5, 0.5])
    psi = rand_state(6, 1)
    assert np.allclose(M.marginal(psi, 6, [2, 5]), oracle.probabilities(psi, 6, [2, 5]), atol=1e-15)


def chi2_ok(counts, p, nshots):
    keep = p > 0
    assert counts[~keep].sum() == 0
    e = p[keep] / p[keep].sum() * nshots
    return stats.chisquare(counts[keep], e).pvalue > 1e-3


def test_direct_sampler_statistics_and_determinism():
    p = M.marginal(rand_state(6, 9), 6, range(6))
    s = M.sample_direct(p, 100000, 42)
    assert chi2_ok(M.frequencies(s, 6), p, 100000)
    assert np.array_equal(s, M.sample_direct(p, 100000, 42))
    assert not np.array_equal(s, M.sample_direct(p, 100000, 43))
    # inverse CDF in plain floating point agrees except within 1e-15 of a bin edge
    cdf = np.cumsum(p)
    i = np.arange(1000, dtype=np.uint64)
    w = M.philox4x32_10(i, 0, 0, 0, 42, 0)
    u = M.uniform53(w[0], w[1])
    for k, uu in zip(s[:1000], u):
        kf = int(np.searchsorted(cdf / cdf[-1], uu, side="right"))
        assert k == kf or np.min(np.abs(cdf / cdf[-1] - uu)) < 1e-15


def test_fixed_point_cdf_exact():
    p = np.array([0.25, 0.0, 0.5, 0.25, 2.0**-70, -1.0, np.nan])
    C = M.fixed_point_cdf(p)
    assert [int(c) for c in C] == [2**58, 2**58, 3 * 2**58, 2**60, 2**60, 2**60, 2**60]


def test_direct_sampler_zero_bins_and_basis():
    assert np.all(M.sample_direct(np.array([1.0, 0, 0, 0]), 1000, 1) == 0)
    p = np.array([0, 0.5, 0, 0.5, 0, 0, 0, 0])
    s = M.sample_direct(p, 20000, 5)
    assert set(np.unique(s)) == {1, 3}


@pytest.mark.parametrize("proposal", ["uniform", "flip"])
def test_metropolis_converges(proposal):
    """TV <= 0.02 at 10^6 shots on random n <= 8 states."""
    for n, seed in ((4, 1), (8, 2)):
        p = M.marginal(rand_state(n, seed), n, range(n))
        s = M.sample_metropolis(p, 10**6, 1234, proposal=proposal)
        f = M.frequencies(s, n) / 10**6
        assert 0.5 * np.abs(f - p).sum() <= 0.02


@pytest.mark.parametrize("proposal", ["uniform", "flip"])
def test_metropolis_spec_examples(proposal):
    # |0...0>: all shots 0 once every chain has left the zero-probability
    # start; a single support point among 16 needs a burn-in of a few hundred
    # steps ((15/16)^1000 ~ 1e-28 per chain; the default 100 leaves ~0.2% of
    # chains outside, R28)
    s = M.sample_metropolis(np.eye(1, 16, 0)[0], 5000, 3, burnin=1000, proposal=proposal)
    assert np.all(s == 0)
    # uniform 1-qubit: each outcome within 5 sigma of n/2
    s = M.sample_metropolis(np.array([0.5, 0.5]), 10**5, 4, proposal=proposal)
    c = M.frequencies(s, 1)
    assert abs(c[0] - 50000) < 5 * math.sqrt(10**5 * 0.25)
    # Bell state: 01 / 10 never recorded after burn-in
    s = M.sample_metropolis(np.array([0.5, 0, 0, 0.5]), 10**5, 5, proposal=proposal)
    c = M.frequencies(s, 2)
    assert c[1] == 0 and c[2] == 0 and c.sum() == 10**5


@pytest.mark.parametrize("proposal", ["uniform", "flip"])
def test_metropolis_agrees_with_exact_chi2(proposal):
    """Metropolis vs the exact multinomial on 20 random 6-qubit states, 10^5
    shots.  Chi-square needs independent draws, so each of the
    10^5 chains records one shot after its burn-in (successive states of one
    chain are autocorrelated -- the default layout is checked by TV above)."""
    for seed in range(20):
        p = M.marginal(rand_state(6, 100 + seed), 6, range(6))
        s = M.sample_metropolis(p, 10**5, seed, nchains=10**5, proposal=proposal)
        assert chi2_ok(M.frequencies(s, 6), p, 10**5), seed


def test_metropolis_layout_and_determinism():
    shots, offs = M.chain_layout(10, 4)
    assert list(shots) == [3, 3, 2, 2] and list(offs) == [0, 3, 6, 8]
    p = M.marginal(rand_state(5, 3), 5, range(5))
    a = M.sample_metropolis(p, 3001, 9, nchains=7, burnin=11)
    assert np.array_equal(a, M.sample_metropolis(p, 3001, 9, nchains=7, burnin=11))
    assert len(a) == 3001 and a.min() >= 0 and a.max() < 32
