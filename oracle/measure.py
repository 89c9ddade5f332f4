"""Measurement oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module; the product path never does.

PAPER.md:239-242: "a custom operator for collapsing and re-normalizing states
and a method for sampling shot frequencies based on Metropolis algorithm".
Written plainly in numpy / fp64, following DESIGN.md readings R26-R28:

* collapse (R26): amplitudes inconsistent with the outcome are set to 0, the
  rest divided by sqrt(P(outcome)); P <= 1e-14 raises ZeroProbabilityOutcome
  (SPEC S:373-380).  Outcome bit i (MSB first) belongs to qubits[i].
* sample_direct (R27): exact multinomial draws by inverse CDF over the
  marginal, the CDF held in 2^-60 fixed point so that every
  prefix sum is exact: C = cumsum(rint(p * 2^60)), shot i takes the first k
  with C[k] > floor(r_i * C[-1] / 2^53), r_i 53 random bits.
* sample_metropolis (R28): independent Metropolis chains over the outcome
  space of the marginal; proposal uniform over all outcomes ("uniform") or a
  flip of one measured bit ("flip"); a move x -> y is accepted iff
  p(x) == 0 or u * p(x) < p(y) (i.e. with probability min(1, p(y)/p(x)),
  Metropolis 1953); after `burnin` steps every step records x.

Random numbers: Philox4x32-10 (Salmon et al., SC'11, the Random123 generator),
implemented here independently of the CUDA path with the same counter layout
(R27/R28).  Pinned to the Random123 known-answer vectors in
tests/test_measure_oracle.py.
"""

from __future__ import annotations

import numpy as np

M32 = np.uint64(0xFFFFFFFF)
_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)

STREAM_DIRECT = 0
STREAM_METROPOLIS = 1


class ZeroProbabilityOutcome(ValueError):
    pass


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds on arrays of 32-bit counters (uint64 holders).
    Round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2;
    c = (hi1^c1^k0, lo1, hi0^c3^k1, lo0); then the key is bumped by (W0, W1)."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & M32 for v in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & M32
    k1 = np.asarray(k1, dtype=np.uint64) & M32
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & M32
        hi1, lo1 = p1 >> np.uint64(32), p1 & M32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + _W0) & M32
        k1 = (k1 + _W1) & M32
    return c0, c1, c2, c3


def uniform53(w_hi, w_lo):
    """u = ((w_hi << 32 | w_lo) >> 11) * 2^-53, in [0, 1)."""
    x = (np.asarray(w_hi, dtype=np.uint64) << np.uint64(32)) | np.asarray(w_lo, dtype=np.uint64)
    return (x >> np.uint64(11)).astype(np.float64) * 2.0**-53


def _key(seed):
    seed = np.uint64(seed)
    return seed & M32, seed >> np.uint64(32)


def marginal(psi: np.ndarray, n: int, qubits) -> np.ndarray:
    """p(outcome) = sum |psi_i|^2 over i consistent with outcome; qubit q is bit n-1-q."""
    i = np.arange(2**n, dtype=np.uint64)
    o = np.zeros(2**n, dtype=np.int64)
    for q in qubits:
        o = (o << 1) | ((i >> np.uint64(n - 1 - q)) & np.uint64(1)).astype(np.int64)
    return np.bincount(o, weights=np.abs(psi.astype(np.complex128)) ** 2, minlength=2 ** len(qubits))


def collapse(psi: np.ndarray, n: int, qubits, outcome: int, eps: float = 1e-14):
    """Returns (collapsed state, P(outcome)); raises ZeroProbabilityOutcome."""
    psi = psi.astype(np.complex128)
    i = np.arange(2**n, dtype=np.uint64)
    keep = np.ones(2**n, dtype=bool)
    m = len(qubits)
    for j, q in enumerate(qubits):
        want = (outcome >> (m - 1 - j)) & 1
        keep &= ((i >> np.uint64(n - 1 - q)) & np.uint64(1)) == np.uint64(want)
    p = float(np.sum(np.abs(psi[keep]) ** 2))
    if p <= eps:
        raise ZeroProbabilityOutcome(f"P(outcome={outcome}) = {p:.3e}")
    out = np.where(keep, psi / np.sqrt(p), 0)
    return out, p


FIXED_SHIFT = 60  # CDF fixed point: q_k = rint(p_k * 2^60) (R27)


def fixed_point_cdf(p: np.ndarray) -> np.ndarray:
    """Inclusive prefix sums of q_k = rint(p_k 2^60) in exact integer arithmetic
    (negative / NaN entries count as 0; sum(p) must stay below 16)."""
    p = np.nan_to_num(np.asarray(p, dtype=np.float64), nan=0.0)
    q = np.rint(np.maximum(p, 0.0) * 2.0**FIXED_SHIFT).astype(np.uint64)
    return np.cumsum(q, dtype=np.uint64)


def sample_direct(p: np.ndarray, nshots: int, seed: int) -> np.ndarray:
    """Inverse CDF in exact integers.  Shot i:
    (w0,w1,.,.) = philox((i lo, i hi, 0, 0), seed); r = (w0<<32|w1) >> 11 (53 bits);
    v = floor(r * Q / 2^53) with Q = C[-1]; k = first index with C[k] > v."""
    C = fixed_point_cdf(p)
    Q = int(C[-1])
    if Q == 0:
        raise ZeroProbabilityOutcome("all probabilities are zero")
    i = np.arange(nshots, dtype=np.uint64)
    k0, k1 = _key(seed)
    w0, w1, _, _ = philox4x32_10(i & M32, i >> np.uint64(32), STREAM_DIRECT, 0, k0, k1)
    r = ((w0 << np.uint64(32)) | w1) >> np.uint64(11)
    v = np.array([(int(x) * Q) >> 53 for x in r], dtype=np.uint64)
    return np.searchsorted(C, v, side="right").astype(np.int64)


def chain_layout(nshots: int, nchains: int):
    """Chain c records nshots//C (+1 for c < nshots % C) shots at offset
    c*(nshots//C) + min(c, nshots % C) of the sample array."""
    base, extra = divmod(nshots, nchains)
    c = np.arange(nchains)
    return base + (c < extra), c * base + np.minimum(c, extra)


def default_chains(nshots: int) -> int:
    return int(min(nshots, 4096))


def default_burnin(nshots: int, nchains: int) -> int:
    per = -(-nshots // nchains)
    return int(max(100, -(-per // 10)))


def sample_metropolis(p: np.ndarray, nshots: int, seed: int, nchains: int = 0,
                      burnin: int | None = None, proposal: str = "uniform") -> np.ndarray:
    """Chain c, step t (t = 0 .. burnin + shots_c - 1):
    (w0,w1,w2,w3) = philox((t, c, 1, 0), seed); proposal y = (w0<<32|w1) mod 2^m
    ("uniform") or x ^ (1 << (w0 mod m)) ("flip"); u = uniform53(w2, w3); accept iff
    p[x] == 0 or u * p[x] < p[y]; for t >= burnin record x.  Start:
    (w0,w1,..) = philox((2^32-1, c, 1, 0), seed), x0 = (w0<<32|w1) mod 2^m."""
    p = np.asarray(p, dtype=np.float64)
    nb = len(p)
    m = nb.bit_length() - 1
    assert nb == 1 << m
    C = nchains or default_chains(nshots)
    B = default_burnin(nshots, C) if burnin is None else burnin
    shots, offs = chain_layout(nshots, C)
    k0, k1 = _key(seed)
    c = np.arange(C, dtype=np.uint64)
    mask = np.uint64(nb - 1)
    w0, w1, _, _ = philox4x32_10(M32, c, STREAM_METROPOLIS, 0, k0, k1)
    x = ((w0 << np.uint64(32)) | w1) & mask
    out = np.empty(nshots, dtype=np.int64)
    for t in range(B + int(shots.max(initial=0))):
        w0, w1, w2, w3 = philox4x32_10(np.uint64(t), c, STREAM_METROPOLIS, 0, k0, k1)
        if proposal == "uniform":
            y = ((w0 << np.uint64(32)) | w1) & mask
        elif proposal == "flip":
            y = x ^ (np.uint64(1) << (w0 % np.uint64(max(m, 1))))
            y &= mask
        else:
            raise ValueError(proposal)
        u = uniform53(w2, w3)
        px, py = p[x.astype(np.int64)], p[y.astype(np.int64)]
        acc = (px == 0) | (u * px < py)
        x = np.where(acc, y, x)
        r = t - B
        live = (r >= 0) & (r < shots)
        out[offs[live] + r] = x[live].astype(np.int64)
    return out


def frequencies(samples: np.ndarray, nbits: int) -> np.ndarray:
    return np.bincount(samples, minlength=2**nbits).astype(np.int64)
