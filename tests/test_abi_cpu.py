"""CPU-only checks of the C-ABI library: it loads, exports every entry point
include/qj.h declares, its host index math (bit insertion)
partitions the index space exactly, and argument validation returns the
documented status codes before anything reaches a GPU."""

import ctypes
import itertools
import json
import os
import re

import numpy as np
import pytest

import paper_2203_08826_b200 as qjp
from paper_2203_08826_b200 import qj as Q

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2203_08826_b200 import build
    build.build()


def header_functions():
    txt = open(os.path.join(ROOT, "include", "qj.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(qj_\w+)\s*\(", txt)))


def test_exports_every_header_symbol():
    L = Q.lib()
    names = header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(Q.EXPORTS)
    assert Q.lib().qj_version().startswith(b"qj")


def insert_members(g, positions, n):
    """Group members for sorted `positions` via the library's bit insertion."""
    base = qjp.insert_zero_bits(g, sorted(positions))
    out = []
    for j in range(2 ** len(positions)):
        x = base
        for i, p in enumerate(sorted(positions)):
            if (j >> i) & 1:
                x |= 1 << p
        out.append(x)
    return sorted(out)


def test_spec_index_examples():
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))
    for c in gold["index_pair"]:
        assert insert_members(c["g"], [c["t"]], 8) == c["out"]
    for c in gold["multi_index_tuple"]:
        assert insert_members(c["g"], c["bits"], c["n"]) == c["out"]
    # the paper's listing literally: i1 = ((g >> m) << (m + 1)) + (g & (k - 1)), k = 1 << m
    for m in range(6):
        for g in range(64):
            assert qjp.insert_zero_bits(g, [m]) == ((g >> m) << (m + 1)) + (g & ((1 << m) - 1))


@pytest.mark.parametrize("n", [1, 2, 5, 8, 12])
def test_partition_exhaustive(n):
    """For every set of <= 3 positions the groups are disjoint and cover [0, 2^n)
    (SPEC S:156), checked exhaustively."""
    sets = [s for k in range(1, min(3, n) + 1) for s in itertools.combinations(range(n), k)]
    if n == 12:
        sets = sets[::7]  # keep the CPU suite fast; every position still appears
    for pos in sets:
        k = len(pos)
        seen = np.zeros(2**n, dtype=np.int8)
        for g in range(2 ** (n - k)):
            for x in insert_members(g, pos, n):
                seen[x] += 1
        assert np.all(seen == 1), pos


def fake_state(n=6, dtype=Q.QJ_C128):
    """A handle over a fake (aligned, never dereferenced) pointer: QJ_KEEP makes
    qj_state_init issue no CUDA call, so validation is testable without a GPU."""
    h = ctypes.c_void_p()
    rc = Q.lib().qj_state_init(ctypes.byref(h), ctypes.c_void_p(0x10000), n, dtype,
                               ctypes.c_uint64(Q.QJ_KEEP), None, None)
    assert rc == 0, Q.lib().qj_last_error()
    return h


def ints(xs):
    return (ctypes.c_int * max(1, len(xs)))(*xs)


def test_init_validation():
    L = Q.lib()
    h = ctypes.c_void_p()
    P = ctypes.c_void_p(0x10000)
    K = ctypes.c_uint64(Q.QJ_KEEP)
    assert L.qj_state_init(None, P, 4, 1, K, None, None) == 1
    assert L.qj_state_init(ctypes.byref(h), None, 4, 1, K, None, None) == 1
    assert L.qj_state_init(ctypes.byref(h), P, 0, 1, K, None, None) == 5
    assert L.qj_state_init(ctypes.byref(h), P, 41, 1, K, None, None) == 5
    assert L.qj_state_init(ctypes.byref(h), P, 4, 7, K, None, None) == 6
    assert L.qj_state_init(ctypes.byref(h), ctypes.c_void_p(0x10008), 4, 1, K, None, None) == 1
    assert L.qj_state_init(ctypes.byref(h), P, 4, 1, ctypes.c_uint64(16), None, None) == 2
    assert b"2^4" in L.qj_last_error()


def test_gate_validation_codes():
    L = Q.lib()
    h = fake_state(6)
    m = (ctypes.c_double * 8)()
    t, c = ints([1]), ints([2])
    assert L.qj_apply_gate(h, 5, t, 1, None, 0, m) == 1          # n mismatch
    assert L.qj_apply_gate(h, 6, t, 0, None, 0, m) == 1          # nt < 1
    assert L.qj_apply_gate(h, 6, ints(list(range(6)) + [0, 0, 0]), 9, None, 0, m) == 4
    assert L.qj_apply_gate(h, 6, ints([6]), 1, None, 0, m) == 2  # out of range
    assert L.qj_apply_gate(h, 6, ints([-1]), 1, None, 0, m) == 2
    assert L.qj_apply_gate(h, 6, t, 1, ints([1]), 1, m) == 3     # target == control
    assert L.qj_apply_gate(h, 6, ints([2, 2]), 2, None, 0, m) == 3
    assert L.qj_apply_gate(h, 6, t, 1, None, 0, None) == 1       # NULL matrix
    assert L.qj_apply_gate(h, 6, t, 1, None, 1, m) == 1          # NULL controls, nc=1
    assert L.qj_apply_x(h, 7, None, 0) == 2
    assert L.qj_apply_swap(h, 3, 3, None, 0) == 3
    assert L.qj_apply_diagonal(h, t, 1, None, None, 0) == 1
    assert L.qj_apply_fsim(h, 0, 1, None, m, None, 0) == 1
    # circuits: every gate is validated before anything is enqueued
    g = (Q.qj_gate * 2)()
    g[0].kind, g[0].nt, g[0].targets[0] = 1, 1, 0
    g[1].kind, g[1].nt, g[1].targets[0] = 1, 1, 9
    assert L.qj_apply_circuit(h, g, 2, 0) == 2
    assert L.qj_last_error().startswith(b"gate 1:")
    assert L.qj_apply_circuit(h, g, 1, 0x8) == 1                 # unknown flag
    g[1].kind = 42
    g[1].targets[0] = 1
    assert L.qj_apply_circuit(h, g, 2, 0) == 1
    # probabilities
    o = ctypes.c_void_p(0x20000)
    assert L.qj_probabilities(h, None, 3, o) == 1
    assert L.qj_probabilities(h, ints([0, 0]), 2, o) == 3
    assert L.qj_probabilities(h, ints([9]), 1, o) == 2
    assert L.qj_probabilities(h, ints([0]), 1, None) == 1
    info = [ctypes.c_int() for _ in range(4)]
    assert L.qj_state_info(h, *[ctypes.byref(x) for x in info]) == 0
    assert [x.value for x in info] == [6, 6, 1, 1]
    assert L.qj_state_free(h) == 0


def test_sharded_init_validation():
    L = Q.lib()
    h = ctypes.c_void_p()
    K = ctypes.c_uint64(Q.QJ_KEEP)
    P3 = (ctypes.c_void_p * 3)(0x10000, 0x20000, 0x30000)
    assert L.qj_state_init_sharded(ctypes.byref(h), P3, 3, 8, 1, K, None) == 1  # not a power of 2
    P4 = (ctypes.c_void_p * 4)(0x10000, 0x20000, 0x30000, 0x40000)
    assert L.qj_state_init_sharded(ctypes.byref(h), P4, 4, 2, 1, K, None) == 5  # g >= n
    assert L.qj_state_init_sharded(ctypes.byref(h), P4, 4, 8, 1, K, None) == 0
    info = [ctypes.c_int() for _ in range(4)]
    L.qj_state_info(h, *[ctypes.byref(x) for x in info])
    assert [x.value for x in info] == [8, 6, 1, 4]
    assert L.qj_state_free(h) == 0


def test_no_cpu_fallback_without_gpu():
    """A valid request on a machine without a GPU must fail loudly (QJ_ERR_CUDA),
    never silently compute on the host."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    L = Q.lib()
    h = fake_state(6)
    assert L.qj_apply_x(h, 0, None, 0) == 7
    assert b"cuda" in L.qj_last_error().lower() or b"CUDA" in L.qj_last_error()


def test_measurement_validation_codes():
    """qj_collapse / qj_sample / qj_measure / qj_sample_distribution reject bad
    arguments before any CUDA call (include/qj.h measurement section)."""
    L = Q.lib()
    h = fake_state(6)
    p = ctypes.c_double()
    U = ctypes.c_uint64
    assert L.qj_collapse(None, ints([0]), 1, U(0), ctypes.byref(p)) == 1
    assert L.qj_collapse(h, None, 1, U(0), None) == 1
    assert L.qj_collapse(h, ints([0]), 0, U(0), None) == 1
    assert L.qj_collapse(h, ints([0, 1]), 2, U(4), None) == 1
    assert L.qj_collapse(h, ints([6]), 1, U(0), None) == 2
    assert L.qj_collapse(h, ints([2, 2]), 2, U(0), None) == 3
    opts = Q.sample_opts("metropolis")
    dev = ctypes.c_void_p(0x20000)
    assert L.qj_sample(h, ints([0]), 1, U(0), U(1), ctypes.byref(opts), dev, None) == 1
    assert L.qj_sample(h, ints([0]), 1, U(5), U(1), ctypes.byref(opts), None, None) == 1
    assert L.qj_sample(h, ints([9]), 1, U(5), U(1), ctypes.byref(opts), dev, None) == 2
    o = ctypes.c_uint64()
    assert L.qj_measure(h, ints([0]), 1, U(1), None, None) == 1
    assert L.qj_measure(h, ints([1, 1]), 2, U(1), ctypes.byref(o), None) == 3
    assert L.qj_sample_distribution(None, 3, U(5), U(1), None, dev, None, None) == 1
    assert L.qj_sample_distribution(dev, 35, U(5), U(1), None, dev, None, None) == 5
    assert L.qj_sample_distribution(dev, 3, U(0), U(1), None, dev, None, None) == 1
    assert L.qj_sample_distribution(dev, 3, U(5), U(1), None, None, None, None) == 1
    bad = Q.qj_sample_opts(7, 0, Q.AUTO)
    assert L.qj_sample_distribution(dev, 3, U(5), U(1), ctypes.byref(bad), dev, None, None) == 1
    long_chain = Q.sample_opts("metropolis", nchains=1, burnin=2**32)
    assert L.qj_sample_distribution(dev, 3, U(5), U(1), ctypes.byref(long_chain), dev, None, None) == 5
    with pytest.raises(ValueError):
        Q.sample_opts("gibbs")
    assert L.qj_state_free(h) == 0


def test_host_state_init_validation():
    L = Q.lib()
    h = ctypes.c_void_p()
    buf = (ctypes.c_double * 64)()
    P = ctypes.cast(buf, ctypes.c_void_p)
    K = ctypes.c_uint64(Q.QJ_KEEP)
    assert L.qj_state_init_host(None, P, 4, 1, 2, K, None) == 1
    assert L.qj_state_init_host(ctypes.byref(h), None, 4, 1, 2, K, None) == 1
    assert L.qj_state_init_host(ctypes.byref(h), P, 4, 7, 2, K, None) == 6
    assert L.qj_state_init_host(ctypes.byref(h), P, 4, 1, 3, K, None) == 1
    assert L.qj_state_init_host(ctypes.byref(h), P, 4, 1, 16, K, None) == 5
    assert L.qj_state_init_host(ctypes.byref(h), P, 41, 1, 2, K, None) == 5
    assert L.qj_state_init_host(ctypes.byref(h), P, 4, 1, 2, K, None) == 0
    assert L.qj_state_free(h) == 0


def _pack_reference(gates, np_dtype):
    """Gate records built one field at a time from the qj_gate layout in
    include/qj.h (kind, nt, nc, targets[8], controls[16], data pointer)."""
    recs, coeffs = [], []
    for g in gates:
        r = Q.qj_gate()
        r.kind = Q.KIND[g.kind]
        r.nt, r.nc = len(g.targets), len(g.controls)
        for i, t in enumerate(g.targets):
            r.targets[i] = t
        for i, c in enumerate(g.controls):
            r.controls[i] = c
        if g.kind in ("dense", "diag"):
            coeffs.append(np.asarray(g.data[0], dtype=np_dtype).reshape(-1))
        elif g.kind == "fsim":
            coeffs.append(np.append(np.asarray(g.data[0]).reshape(-1), g.data[1]).astype(np_dtype))
        else:
            coeffs.append(None)
        recs.append(r)
    return recs, coeffs


@pytest.mark.parametrize("np_dtype", [np.complex128, np.complex64])
def test_pack_gates_matches_field_by_field(np_dtype):
    """The vectorised gate-list packing (qj.pack_gates) writes exactly the
    records and coefficients a field-by-field packing does, for every gate
    kind, with and without controls, coefficients given as arrays or lists."""
    from workloads import circuits as C
    from workloads.gates import Gate
    rng = np.random.default_rng(5)
    gates = list(C.random_circuit(12, 300, 3, max_targets=3, max_controls=3).gates)
    gates += [Gate("i", "dense", (4,), (), (np.eye(2).tolist(),)), Gate("cx", "x", (0,), (1, 2)),
              Gate("cswap", "swap", (3, 5), (7,)), Gate("d", "diag", (2, 6), (), ([1, 1j, -1, -1j],)),
              Gate("z", "z", (9,), ())]
    rng.shuffle(gates)
    arr, ng, keep = Q.pack_gates(gates, np_dtype)
    rec, coeff = keep
    ref, ref_coeffs = _pack_reference(gates, np_dtype)
    assert ng == len(gates)
    base = coeff.ctypes.data if coeff is not None else 0
    item = np.dtype(np_dtype).itemsize
    for i, (g, r, c) in enumerate(zip(gates, ref, ref_coeffs)):
        assert arr[i].kind == r.kind and arr[i].nt == r.nt and arr[i].nc == r.nc, i
        assert list(arr[i].targets) == list(r.targets) and list(arr[i].controls) == list(r.controls), i
        if c is None:
            assert rec["data"][i] == 0, i
        else:
            off = (int(rec["data"][i]) - base) // item
            assert np.array_equal(coeff[off:off + c.size], c), i
    with pytest.raises(Q.QJError):
        Q.pack_gates([Gate("x", "x", (0,), tuple(range(1, 18)))])
