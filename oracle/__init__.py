"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct complex128 implementation of Eq. 1
 and of Born-rule probabilities, in
``oracle/qj_oracle.c`` (C99 + OpenMP), wrapped here with ctypes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_2203_08826_b200`` never imports it, and the two share no
code; the only common inputs come from ``workloads/`` (seeded generators).

Every function is pinned in tests/test_oracle_pins.py against closed forms,
a textbook tensordot formulation, brute-force dense operators and Table 2.
Parity unpinned: the named-gate matrices themselves (the paper prints none;
reading R5) -- see DESIGN.md.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qj_oracle.c")
_LIB = os.path.join(_HERE, "libqj_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP).  Plain flags: no fast-math."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
               "-fcx-limited-range", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int
        L.or_apply_gate.argtypes = [P, P, I, P, I, P, I, P]
        L.or_apply_gate.restype = I
        L.or_basis_state.argtypes = [P, I, ctypes.c_uint64]
        L.or_basis_state.restype = None
        L.or_probabilities.argtypes = [P, I, P, I, P]
        L.or_probabilities.restype = None
        L.or_qft_basis_maxerr.argtypes = [P, I, I, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, P,
                                          ctypes.POINTER(ctypes.c_double)]
        L.or_qft_basis_maxerr.restype = ctypes.c_double
        L.or_set_num_threads.argtypes = [I]
        L.or_set_num_threads.restype = None
        L.or_num_threads.argtypes = []
        L.or_num_threads.restype = I
        _lib = L
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else None


def _ints(xs):
    return np.ascontiguousarray(np.asarray(list(xs), dtype=np.int32))


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_num_threads(t: int) -> None:
    lib().or_set_num_threads(int(t))


def basis_state(n: int, x: int = 0) -> np.ndarray:
    psi = np.empty(2**n, dtype=np.complex128)
    lib().or_basis_state(_ptr(psi), n, int(x))
    return psi


def apply_matrix(psi: np.ndarray, out: np.ndarray, n: int, targets, controls, matrix) -> None:
    """out <- Eq. 1 applied to psi (out-of-place; psi, out complex128, length 2^n)."""
    m = np.ascontiguousarray(np.asarray(matrix, dtype=np.complex128))
    t = _ints(targets)
    c = _ints(controls)
    assert psi.dtype == np.complex128 and out.dtype == np.complex128
    assert m.shape == (2 ** len(t), 2 ** len(t))
    lib().or_apply_gate(_ptr(psi), _ptr(out), n, _ptr(t), len(t), _ptr(c), len(c), _ptr(m))


def run(circuit, psi: np.ndarray, matrices=None) -> np.ndarray:
    """Apply every gate of `circuit` in order; returns the final state (a new array
    or one of the two ping-pong buffers).  `matrices` optionally overrides each
    gate's dense matrix (used to feed complex64-rounded matrices, reading R7)."""
    n = circuit.n
    a = np.array(psi, dtype=np.complex128, copy=True)
    b = np.empty_like(a)
    for idx, g in enumerate(circuit.gates):
        m = g.matrix() if matrices is None else matrices[idx]
        apply_matrix(a, b, n, g.targets, g.controls, m)
        a, b = b, a
    return a


def probabilities(psi: np.ndarray, n: int, qubits=None) -> np.ndarray:
    """Marginal probabilities over `qubits` (first listed = MSB); None = all qubits
    in canonical order."""
    q = _ints(range(n) if qubits is None else qubits)
    out = np.empty(2 ** len(q), dtype=np.float64)
    p = np.ascontiguousarray(psi, dtype=np.complex128)
    lib().or_probabilities(_ptr(p), n, _ptr(q), len(q), _ptr(out))
    return out


def qft_basis_maxerr(psi: np.ndarray, n: int, x: int, offset: int = 0, phys=None):
    """Closed-form QFT|x> check of a chunk of a state computed elsewhere
    (or_qft_basis_maxerr): element j of `psi` (complex128 or complex64) is
    buffer index offset + j; `phys` (qubit -> bit) gives a physical layout,
    None = canonical order.  Returns (max abs error, sum of squared errors)."""
    a = np.ascontiguousarray(psi)
    assert a.dtype in (np.complex128, np.complex64)
    ph = None if phys is None else _ints(phys)
    ss = ctypes.c_double(0.0)
    m = lib().or_qft_basis_maxerr(_ptr(a), int(a.dtype == np.complex64), n, int(x), int(offset), a.size,
                                  _ptr(ph), ctypes.byref(ss))
    return float(m), float(ss.value)
