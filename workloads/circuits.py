"""Circuit generators shaped like the paper's benchmark circuits.

Table 2 lists qft, variational, supremacy, qv and bv at 30
qubits.  qft / variational / bv follow SPEC S:502-528 and reproduce Table 2's
gate counts and depths (pinned in tests/test_workloads.py).  The supremacy-style
circuit is the Sycamore-style recipe of SURVEY.md section 8(d) config 4 (the
paper's own Cirq export is unavailable: reading R16, parity vs that exact circuit
is unpinned).  QAOA follows the BASELINE.json north star's workload list.

Every random choice is drawn from numpy PCG64 seeded from `SEED` plus a per-call
sub-seed, so the oracle and the CUDA path see the identical gate list.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import gates as G

SEED = 220308826


def rng_for(sub: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([SEED, int(sub)]))


@dataclass
class Circuit:
    n: int
    gates: list = field(default_factory=list)
    name: str = ""

    def __len__(self):
        return len(self.gates)

    def __iter__(self):
        return iter(self.gates)

    def append(self, g):
        for q in g.qubits:
            if not 0 <= q < self.n:
                raise ValueError(f"qubit {q} out of range for n={self.n}")
        self.gates.append(g)


def depth(c: Circuit) -> int:
    """ASAP layering depth: a gate sits one layer above the
    latest gate sharing any of its qubits (targets or controls)."""
    level = [0] * c.n
    d = 0
    for g in c.gates:
        lv = 1 + max(level[q] for q in g.qubits)
        for q in g.qubits:
            level[q] = lv
        d = max(d, lv)
    return d


# ---- Table 2 generators ------------------------------------------------------
def qft(n: int, swaps: bool = True) -> Circuit:
    """for j: H(j); CU1(pi/2^(k-j)) control k target j for k>j;
    then SWAP(i, n-1-i) for i < n//2.  Gate count n + n(n-1)/2 + n//2."""
    c = Circuit(n, name=f"qft{n}")
    for j in range(n):
        c.append(G.H(j))
        for k in range(j + 1, n):
            c.append(G.CU1(k, j, math.pi / 2 ** (k - j)))
    if swaps:
        for i in range(n // 2):
            c.append(G.SWAP(i, n - 1 - i))
    return c


def variational(n: int, layers: int = 1, theta=None, seed: int = 2) -> Circuit:
    """RY layer, CZ(0,1)(2,3)..., RY layer, CZ(1,2)...(n-1,0).
    theta=None draws each angle U[0, 2 pi) (reading R17); a float fixes all."""
    if n % 2:
        raise ValueError("variational circuit needs an even number of qubits")
    rng = rng_for(seed)
    c = Circuit(n, name=f"variational{n}x{layers}")

    def ang():
        return float(rng.uniform(0, 2 * math.pi)) if theta is None else float(theta)

    for _ in range(layers):
        for q in range(n):
            c.append(G.RY(q, ang()))
        for q in range(0, n, 2):
            c.append(G.CZ(q, q + 1))
        for q in range(n):
            c.append(G.RY(q, ang()))
        for q in range(1, n, 2):
            c.append(G.CZ(q, (q + 1) % n))
    return c


def bv(n: int) -> Circuit:
    """secret all-ones, ancilla n-1.  3n-1 gates, depth n+2."""
    c = Circuit(n, name=f"bv{n}")
    for q in range(n - 1):
        c.append(G.H(q))
    c.append(G.X(n - 1))
    c.append(G.H(n - 1))
    for q in range(n - 1):
        c.append(G.CNOT(q, n - 1))
    for q in range(n - 1):
        c.append(G.H(q))
    return c


def supremacy(rows: int, cols: int, cycles: int = 20, seed: int = 4) -> Circuit:
    """Sycamore-style random circuit: per cycle one of
    {sqrt X, sqrt Y, sqrt W} on every qubit (cycle 0 uniform, later uniform over
    the two differing from that qubit's previous choice), then fSim(pi/2, pi/6)
    on coupler pattern 'ABCDCDAB'[cycle % 8]; qubit q = cols*r + c."""
    rng = rng_for(seed)
    n = rows * cols
    c = Circuit(n, name=f"supremacy{rows}x{cols}m{cycles}")
    one = [G.SQRT_X, G.SQRT_Y, G.SQRT_W]
    prev = [-1] * n

    def couplers(kind):
        out = []
        for r in range(rows):
            for cc in range(cols):
                q = cols * r + cc
                if kind == "A" and cc % 2 == 0 and cc + 1 < cols:
                    out.append((q, q + 1))
                if kind == "B" and cc % 2 == 1 and cc + 1 < cols:
                    out.append((q, q + 1))
                if kind == "C" and r % 2 == 0 and r + 1 < rows:
                    out.append((q, q + cols))
                if kind == "D" and r % 2 == 1 and r + 1 < rows:
                    out.append((q, q + cols))
        return out

    for cyc in range(cycles):
        for q in range(n):
            if prev[q] < 0:
                ch = int(rng.integers(0, 3))
            else:
                opts = [i for i in range(3) if i != prev[q]]
                ch = opts[int(rng.integers(0, 2))]
            prev[q] = ch
            c.append(one[ch](q))
        for (a, b) in couplers("ABCDCDAB"[cyc % 8]):
            c.append(G.FSIM(a, b, math.pi / 2, math.pi / 6))
    return c


def random_3_regular(n: int, rng: np.random.Generator):
    """Seeded random 3-regular simple graph by the pairing model with retries."""
    if (3 * n) % 2 or n < 4:
        raise ValueError("3-regular graph needs n >= 4 and 3n even")
    for _ in range(10000):
        pts = np.repeat(np.arange(n), 3)
        rng.shuffle(pts)
        edges = set()
        ok = True
        for i in range(0, len(pts), 2):
            a, b = int(pts[i]), int(pts[i + 1])
            if a == b or (min(a, b), max(a, b)) in edges:
                ok = False
                break
            edges.add((min(a, b), max(a, b)))
        if ok:
            return sorted(edges)
    raise RuntimeError("could not draw a 3-regular graph")


def qaoa(n: int, p: int = 2, seed: int = 5) -> Circuit:
    """QAOA-MaxCut on a seeded random 3-regular graph: H on all qubits, then p
    rounds of RZZ(gamma) per edge (a diagonal gate) and RX(beta) mixers."""
    rng = rng_for(seed)
    edges = random_3_regular(n, rng)
    c = Circuit(n, name=f"qaoa{n}p{p}")
    for q in range(n):
        c.append(G.H(q))
    for _ in range(p):
        gamma = float(rng.uniform(0, 2 * math.pi))
        beta = float(rng.uniform(0, math.pi))
        for (a, b) in edges:
            c.append(G.RZZ(a, b, gamma))
        for q in range(n):
            c.append(G.RX(q, 2 * beta))
    return c


# ---- random circuits for parity tests ---------------------------------------
def random_gate(n: int, rng: np.random.Generator, max_targets: int = 3,
                max_controls: int = 2, kinds=None):
    kinds = kinds or ("dense", "x", "z", "swap", "fsim", "diag")
    kind = kinds[int(rng.integers(0, len(kinds)))]
    if kind in ("x", "z"):
        k = 1
    elif kind in ("swap", "fsim"):
        k = 2
    else:
        k = int(rng.integers(1, max_targets + 1))
    if k > n:
        kind, k = "dense", n
    qs = [int(x) for x in rng.permutation(n)]
    targets = tuple(qs[:k])
    nc = int(rng.integers(0, min(max_controls, n - k) + 1))
    controls = tuple(qs[k:k + nc])
    if kind == "dense":
        return G.unitary("U", targets, G.random_unitary(k, rng), controls)
    if kind == "x":
        return G.X(targets[0], controls)
    if kind == "z":
        return G.Z(targets[0], controls)
    if kind == "swap":
        return G.SWAP(targets[0], targets[1], controls)
    if kind == "fsim":
        th, ph = rng.uniform(0, 2 * math.pi, 2)
        return G.FSIM(targets[0], targets[1], float(th), float(ph), controls)
    d = np.exp(1j * rng.uniform(0, 2 * math.pi, 2**k))
    if rng.random() < 0.3:
        d[:-1] = 1.0  # single non-unit entry: the CU1/CZ-like phase shape
    return G.Gate("D", "diag", targets, controls, (d,))


def random_circuit(n: int, count: int, seed: int, **kw) -> Circuit:
    rng = rng_for(1000 + seed)
    c = Circuit(n, name=f"random{n}x{count}s{seed}")
    for _ in range(count):
        c.append(random_gate(n, rng, **kw))
    return c
