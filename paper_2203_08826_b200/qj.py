"""Thin ctypes binding of libqj (include/qj.h).  Argument marshalling only:
every amplitude is touched by the library's sm_100a kernels.  torch supplies
device memory and streams; nothing here computes on the state.

The library is built in-tree (``python -m paper_2203_08826_b200.build``); if it
is missing, importing this module raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from itertools import chain
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libqj.so")

QJ_C64, QJ_C128 = 0, 1
QJ_KEEP = (1 << 64) - 1
QJ_FUSE = 1
QJ_FUSE_GATES = 2
MAX_TARGETS, MAX_CONTROLS = 8, 16
KIND = {"dense": 0, "x": 1, "z": 2, "swap": 3, "fsim": 4, "diag": 5}
STATUS = {0: "QJ_OK", 1: "QJ_ERR_INVALID_ARG", 2: "QJ_ERR_INDEX_OUT_OF_RANGE",
          3: "QJ_ERR_OVERLAPPING_QUBITS", 4: "QJ_ERR_TOO_MANY_TARGETS", 5: "QJ_ERR_CAPACITY",
          6: "QJ_ERR_DTYPE", 7: "QJ_ERR_CUDA", 8: "QJ_ERR_NCCL", 9: "QJ_ERR_UNSUPPORTED",
          10: "QJ_ERR_ZERO_PROBABILITY"}

SAMPLE_METHODS = {"direct": 0, "metropolis": 1, "metropolis_flip": 2}
AUTO = (1 << 64) - 1

EXPORTS = ["qj_state_init", "qj_state_init_sharded", "qj_state_reset", "qj_state_free",
           "qj_apply_gate", "qj_apply_x", "qj_apply_z", "qj_apply_swap", "qj_apply_fsim",
           "qj_apply_diagonal", "qj_apply_circuit", "qj_probabilities", "qj_sync",
           "qj_get_counters", "qj_state_info", "qj_last_error", "qj_version",
           "qj_insert_zero_bits", "qj_set_profiling", "qj_get_profile", "qj_state_canonicalize",
           "qj_plan_circuit", "qj_exchange_peer", "qj_fuse_circuit", "qj_collapse",
           "qj_sample_distribution", "qj_sample", "qj_measure", "qj_state_init_host",
           "qj_simulate", "qj_state_layout", "qj_plan_canonicalize", "qj_debug_tile_sources",
           "qj_debug_nccl_self_exchange"]


class QJError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class qj_gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("nt", ctypes.c_int), ("nc", ctypes.c_int),
                ("targets", ctypes.c_int * MAX_TARGETS), ("controls", ctypes.c_int * MAX_CONTROLS),
                ("data", ctypes.c_void_p)]


class qj_counters(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_uint64), ("passes", ctypes.c_uint64),
                ("exchanges", ctypes.c_uint64), ("alg_bytes", ctypes.c_double),
                ("exchange_bytes", ctypes.c_double)]


class qj_profile_entry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_uint64),
                ("total_ms", ctypes.c_double), ("alg_bytes", ctypes.c_double)]


class qj_sample_opts(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int), ("nchains", ctypes.c_uint32), ("burnin", ctypes.c_uint64)]


def sample_opts(method="direct", nchains=0, burnin=None):
    if method not in SAMPLE_METHODS:
        raise ValueError(f"unknown sampling method {method!r} (one of {sorted(SAMPLE_METHODS)})")
    return qj_sample_opts(SAMPLE_METHODS[method], int(nchains), AUTO if burnin is None else int(burnin))


class qj_plan_step(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("shard", ctypes.c_int), ("kind", ctypes.c_int), ("k", ctypes.c_int),
                ("tpos", ctypes.c_int * MAX_TARGETS), ("nfix", ctypes.c_int), ("fpos", ctypes.c_int * 64),
                ("fval", ctypes.c_int * 64), ("touch", ctypes.c_uint32), ("nm", ctypes.c_int),
                ("m", ctypes.c_double * 512), ("gbit", ctypes.c_int), ("lbit", ctypes.c_int),
                ("alg_bytes", ctypes.c_double)]


_lib = None


def lib():
    """Load libqj.so (raises if the CUDA library has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libqj.so not built: run `python -m paper_2203_08826_b200.build` ({LIB_PATH})")
    L = ctypes.CDLL(LIB_PATH)
    P, I, U64, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int
    IP = ctypes.POINTER(ctypes.c_int)
    sig = {
        "qj_state_init": ([ctypes.POINTER(P), P, I, I, U64, P, P], S),
        "qj_state_init_sharded": ([ctypes.POINTER(P), ctypes.POINTER(P), I, I, I, U64, P], S),
        "qj_state_reset": ([P, U64], S),
        "qj_state_free": ([P], S),
        "qj_apply_gate": ([P, I, IP, I, IP, I, P], S),
        "qj_apply_x": ([P, I, IP, I], S),
        "qj_apply_z": ([P, I, IP, I], S),
        "qj_apply_swap": ([P, I, I, IP, I], S),
        "qj_apply_fsim": ([P, I, I, P, P, IP, I], S),
        "qj_apply_diagonal": ([P, IP, I, P, IP, I], S),
        "qj_apply_circuit": ([P, ctypes.POINTER(qj_gate), I, ctypes.c_uint32], S),
        "qj_probabilities": ([P, IP, I, P], S),
        "qj_sync": ([P], S),
        "qj_get_counters": ([P, ctypes.POINTER(qj_counters), I], S),
        "qj_state_info": ([P, IP, IP, IP, IP], S),
        "qj_state_layout": ([P, IP], S),
        "qj_last_error": ([], ctypes.c_char_p),
        "qj_version": ([], ctypes.c_char_p),
        "qj_insert_zero_bits": ([U64, IP, I], U64),
        "qj_set_profiling": ([P, I], S),
        "qj_get_profile": ([P, ctypes.POINTER(qj_profile_entry), I, IP, I], S),
        "qj_state_canonicalize": ([P], S),
        "qj_plan_circuit": ([I, I, I, ctypes.POINTER(qj_gate), I, ctypes.c_uint32, ctypes.POINTER(qj_plan_step), I,
                             IP, IP], S),
        "qj_exchange_peer": ([I, I, IP, IP], None),
        "qj_plan_canonicalize": ([I, I, IP, ctypes.POINTER(qj_plan_step), I, IP], S),
        "qj_debug_tile_sources": ([I, I, ctypes.POINTER(qj_gate), I, ctypes.c_uint32, ctypes.c_char_p, I, IP], S),
        "qj_debug_nccl_self_exchange": ([P, I], S),
        "qj_fuse_circuit": ([I, ctypes.POINTER(qj_gate), I, I, ctypes.POINTER(qj_gate), ctypes.POINTER(ctypes.c_double),
                             I, IP, IP], S),
        "qj_collapse": ([P, IP, I, U64, ctypes.POINTER(ctypes.c_double)], S),
        "qj_state_init_host": ([ctypes.POINTER(P), P, I, I, I, U64, P], S),
        "qj_simulate": ([P, U64, ctypes.POINTER(qj_gate), I, ctypes.c_uint32, IP, I, P], S),
        "qj_sample_distribution": ([P, I, U64, U64, ctypes.POINTER(qj_sample_opts), P, P, P], S),
        "qj_sample": ([P, IP, I, U64, U64, ctypes.POINTER(qj_sample_opts), P, P], S),
        "qj_measure": ([P, IP, I, U64, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_double)], S),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(code: int):
    if code != 0:
        raise QJError(code, lib().qj_last_error().decode())


def _ints(xs):
    xs = [int(x) for x in (xs or ())]
    return (ctypes.c_int * max(1, len(xs)))(*xs), len(xs)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def sample_distribution(probs, nshots, seed, method="direct", nchains=0, burnin=None,
                        samples=True, counts=True, stream=None):
    """Shots from a fp64 device tensor of 2^m weights (qj_sample_distribution)
    on `stream` (default: torch's current stream).  Returns (samples, counts)."""
    import torch

    if probs.dtype != torch.float64 or not probs.is_cuda or not probs.is_contiguous():
        raise ValueError("probs must be a contiguous float64 CUDA tensor")
    nb = probs.numel()
    m = nb.bit_length() - 1
    if nb != 1 << m:
        raise ValueError("len(probs) must be a power of two")
    stream = stream or torch.cuda.current_stream(probs.device)
    opts = sample_opts(method, nchains, burnin)
    smp = torch.empty(int(nshots), dtype=torch.int64, device=probs.device) if samples else None
    cnt = None
    if counts:
        with torch.cuda.stream(stream):
            cnt = torch.zeros(nb, dtype=torch.int64, device=probs.device)
    _check(lib().qj_sample_distribution(ctypes.c_void_p(probs.data_ptr()), m, ctypes.c_uint64(int(nshots)),
                                        ctypes.c_uint64(int(seed)), ctypes.byref(opts), _ptr(smp), _ptr(cnt),
                                        ctypes.c_void_p(stream.cuda_stream)))
    return smp, cnt


def insert_zero_bits(g: int, sorted_positions) -> int:
    arr, n = _ints(sorted_positions)
    return int(lib().qj_insert_zero_bits(ctypes.c_uint64(g), arr, n))


def exchange_peer(rank: int, gbit: int):
    """(peer rank, value of the swapped local bit of the half this rank trades)."""
    p, h = ctypes.c_int(), ctypes.c_int()
    lib().qj_exchange_peer(int(rank), int(gbit), ctypes.byref(p), ctypes.byref(h))
    return p.value, h.value


_GATE_NP = np.dtype({"names": ["kind", "nt", "nc", "targets", "controls", "data"],
                     "formats": ["<i4", "<i4", "<i4", ("<i4", (MAX_TARGETS,)), ("<i4", (MAX_CONTROLS,)), "<u8"],
                     "offsets": [0, 4, 8, 12, 44, 112], "itemsize": 120})


def _scatter_rows(field, seqs, lens, ng):
    """field[i, :lens[i]] = seqs[i] for every row, in one vectorised store."""
    flat = np.fromiter(chain.from_iterable(seqs), dtype=np.int32)
    if flat.size:
        rows = np.repeat(np.arange(ng), lens)
        starts = np.cumsum(lens) - lens
        field[rows, np.arange(flat.size) - np.repeat(starts, lens)] = flat


def pack_gates(gates, np_dtype=np.complex128):
    """Marshal gate records (kind/targets/controls/data) into a qj_gate array:
    one numpy record array with the C struct's layout and one contiguous
    coefficient buffer in the state's dtype.  Returns (qj_gate*, n, keepalive).
    Vectorised over the gate list (it is on the end-to-end path of every
    simulate / apply_circuit call that passes Python gates)."""
    assert ctypes.sizeof(qj_gate) == _GATE_NP.itemsize
    gates = gates if isinstance(gates, list) else list(gates)
    ng = len(gates)
    rec = np.zeros(max(1, ng), dtype=_GATE_NP)
    coeff = None
    if ng:
        kl = [g.kind for g in gates]
        tl = [g.targets for g in gates]
        cl = [g.controls for g in gates]
        nts = np.fromiter(map(len, tl), dtype=np.int64, count=ng)
        ncs = np.fromiter(map(len, cl), dtype=np.int64, count=ng)
        bad = np.nonzero((nts > MAX_TARGETS) | (ncs > MAX_CONTROLS))[0]
        if bad.size:
            raise QJError(4, f"gate {int(bad[0])}: too many qubits")
        rec["kind"][:ng] = [KIND[k] for k in kl]
        rec["nt"][:ng] = nts
        rec["nc"][:ng] = ncs
        _scatter_rows(rec["targets"], tl, nts, ng)
        if ncs.any():
            _scatter_rows(rec["controls"], cl, ncs, ng)
        owner = [i for i, k in enumerate(kl) if k == "dense" or k == "diag" or k == "fsim"]
        if owner:
            # coefficients in C order, each gate's block converted to the state's
            # dtype, joined as bytes (numpy's concatenate costs ~0.3-0.6 us per
            # small array; thousands of 2x2 blocks are common)
            dt = np.dtype(np_dtype)
            parts = [gates[i].data[0] for i in owner]
            for j, i in enumerate(owner):
                if kl[i] == "fsim":
                    parts[j] = np.append(np.asarray(parts[j]).reshape(-1), gates[i].data[1])
            if {p.dtype if type(p) is np.ndarray else None for p in parts} != {dt}:
                parts = [np.asarray(p).astype(dt, copy=False) for p in parts]
            blobs = [p.tobytes() for p in parts]
            coeff = np.frombuffer(b"".join(blobs), dtype=dt).copy()
            lens = np.fromiter(map(len, blobs), dtype=np.uint64, count=len(blobs))
            offs = np.cumsum(lens) - lens
            rec["data"][owner] = np.uint64(coeff.ctypes.data) + offs
    arr = rec.ctypes.data_as(ctypes.POINTER(qj_gate))
    return arr, ng, (rec, coeff)


def plan_circuit(n, nshards, gates, fuse=False, amp_bytes=16, max_steps=1 << 16):
    """Run the library's host planner (no GPU): returns (steps, phys map)."""
    arr, ng, keep = pack_gates(gates)
    out = (qj_plan_step * max_steps)()
    cnt = ctypes.c_int()
    phys = (ctypes.c_int * n)()
    _check(lib().qj_plan_circuit(n, nshards, amp_bytes, arr, ng, QJ_FUSE if fuse else 0, out, max_steps,
                                 ctypes.byref(cnt), phys))
    del keep
    steps = []
    for i in range(cnt.value):
        o = out[i]
        m = np.array(o.m[:2 * o.nm]).view(np.complex128) if o.nm else np.zeros(0, np.complex128)
        steps.append({"type": o.type, "shard": o.shard, "kind": o.kind, "tpos": list(o.tpos[:o.k]),
                      "fix": [(o.fpos[j], o.fval[j]) for j in range(o.nfix)], "touch": o.touch, "m": m,
                      "gbit": o.gbit, "lbit": o.lbit, "alg_bytes": o.alg_bytes})
    return steps, list(phys)


def debug_tile_sources(n, gates, amp_bytes=16, out_dir=None, compile=True, fuse_gates=False):
    """Generate (and NVRTC-compile, no GPU needed) every JIT tile kernel of the
    fused plan; returns the number of tile passes."""
    arr, ng, keep = pack_gates(gates)
    cnt = ctypes.c_int()
    _check(lib().qj_debug_tile_sources(n, amp_bytes, arr, ng, _fuse_gates_flags(fuse_gates),
                                       out_dir.encode() if out_dir else None, 1 if compile else 0, ctypes.byref(cnt)))
    del keep
    return cnt.value


def plan_canonicalize(n, nshards, phys, max_steps=4096):
    """The steps qj_state_canonicalize runs for map `phys` (host only)."""
    out = (qj_plan_step * max_steps)()
    cnt = ctypes.c_int()
    ph = (ctypes.c_int * n)(*phys)
    _check(lib().qj_plan_canonicalize(n, nshards, ph, out, max_steps, ctypes.byref(cnt)))
    return [{"type": out[i].type, "shard": out[i].shard, "kind": out[i].kind, "tpos": list(out[i].tpos[:out[i].k]),
             "fix": [], "touch": out[i].touch, "m": np.zeros(0, np.complex128), "gbit": out[i].gbit,
             "lbit": out[i].lbit, "alg_bytes": out[i].alg_bytes} for i in range(cnt.value)]


class FusedGate:
    """A gate returned by fuse_circuit (dense matrix on `targets`, or an input
    gate passed through unchanged)."""

    def __init__(self, kind, targets, controls, matrix):
        self.kind, self.targets, self.controls = kind, tuple(targets), tuple(controls)
        self.m = matrix
        self.data = (matrix,) if kind in ("dense", "diag") else ()

    @property
    def qubits(self):
        return self.targets + self.controls


def fuse_circuit(n, gates, max_qubits=2):
    """The paper's greedy gate fusion run by the library:
    returns the fused gate list (FusedGate for fused groups; the original gate
    objects for gates passed through)."""
    gates = list(gates)
    arr, ng, keep = pack_gates(gates)
    out = (qj_gate * max(1, ng))()
    stride = 2 * 4 ** max_qubits
    mats = (ctypes.c_double * (stride * max(1, ng)))()
    cnt = ctypes.c_int()
    src = (ctypes.c_int * max(1, ng))()
    _check(lib().qj_fuse_circuit(n, arr, ng, max_qubits, out, mats, ng, ctypes.byref(cnt), src))
    res = []
    for i in range(cnt.value):
        o = out[i]
        if src[i] >= 0:
            res.append(gates[src[i]])      # passed through unchanged
        else:
            k = o.nt
            m = np.array(mats[stride * i:stride * i + 2 * 4 ** k]).view(np.complex128).reshape(2 ** k, 2 ** k)
            res.append(FusedGate("dense", o.targets[:o.nt], o.controls[:o.nc], m))
    del keep
    return res


def _fuse_gates_flags(fuse_gates):
    """fuse_gates: False, True (the paper's <= 2-qubit fusion) or a width 1..5."""
    if not fuse_gates:
        return 0
    k = 2 if fuse_gates is True else int(fuse_gates)
    return QJ_FUSE_GATES | ((k & 15) << 4)


class State:
    """A state vector living in caller-owned torch device memory.

    ``State(tensor, basis=0)`` wraps a contiguous complex64/complex128 CUDA
    tensor of 2^n elements and writes |basis> into it (``basis=None`` keeps the
    contents).  ``State.sharded([t0, t1, ...], n)`` wraps 2^g shards of
    2^(n-g) amplitudes (global qubits = the top g bits)."""

    def __init__(self, tensor=None, basis=0, stream=None, _shards=None, _n=None):
        import torch

        L = lib()
        self._h = ctypes.c_void_p()
        shards = _shards if _shards is not None else [tensor]
        t0 = shards[0]
        for t in shards:
            if not (t.is_cuda and t.is_contiguous()):
                raise ValueError("state tensors must be contiguous CUDA tensors")
            if t.dtype not in (torch.complex64, torch.complex128) or t.dtype != t0.dtype:
                raise ValueError("state tensors must all be complex64 or all complex128")
        self.dtype = QJ_C64 if t0.dtype == torch.complex64 else QJ_C128
        self.np_dtype = np.complex64 if self.dtype == QJ_C64 else np.complex128
        self.real_dtype = torch.float32 if self.dtype == QJ_C64 else torch.float64
        ntot = _n if _n is not None else int(t0.numel()).bit_length() - 1
        if _n is None and (1 << ntot) != t0.numel():
            raise ValueError("state length must be a power of two")
        self.n = ntot
        self.shards = shards
        self.device = t0.device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        basis = QJ_KEEP if basis is None else int(basis)
        if _shards is None:
            _check(L.qj_state_init(ctypes.byref(self._h), ctypes.c_void_p(t0.data_ptr()), ntot, self.dtype,
                                   ctypes.c_uint64(basis), ctypes.c_void_p(self.stream.cuda_stream), None))
        else:
            ptrs = (ctypes.c_void_p * len(shards))(*[t.data_ptr() for t in shards])
            _check(L.qj_state_init_sharded(ctypes.byref(self._h), ptrs, len(shards), ntot, self.dtype,
                                           ctypes.c_uint64(basis), ctypes.c_void_p(self.stream.cuda_stream)))

    @classmethod
    def sharded(cls, shards, n, basis=0, stream=None):
        return cls(None, basis=basis, stream=stream, _shards=list(shards), _n=n)

    @classmethod
    def distributed(cls, tensor, n, group=None, basis=0, stream=None):
        """One shard per process: `tensor` holds this rank's 2^(n - log2 P)
        amplitudes (global qubits = the top log2 P bits, shard index = rank).
        The NCCL communicator is torch's (ProcessGroupNCCL); it is initialised
        eagerly with a barrier before its pointer is taken."""
        import torch
        import torch.distributed as dist

        pg = group if group is not None else dist.group.WORLD
        dist.barrier(group=pg, device_ids=[tensor.device.index])
        comm = pg._get_backend(torch.device("cuda"))._comm_ptr()
        self = cls.__new__(cls)
        L = lib()
        self._h = ctypes.c_void_p()
        self.dtype = QJ_C64 if tensor.dtype == torch.complex64 else QJ_C128
        self.np_dtype = np.complex64 if self.dtype == QJ_C64 else np.complex128
        self.real_dtype = torch.float32 if self.dtype == QJ_C64 else torch.float64
        self.n = n
        self.shards = [tensor]
        self.device = tensor.device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(L.qj_state_init(ctypes.byref(self._h), ctypes.c_void_p(tensor.data_ptr()), n, self.dtype,
                               ctypes.c_uint64(QJ_KEEP if basis is None else int(basis)),
                               ctypes.c_void_p(self.stream.cuda_stream), ctypes.c_void_p(comm)))
        return self

    @classmethod
    def host(cls, tensor, nslices, basis=0, stream=None, device=None):
        """Host-staged state: `tensor` is a contiguous
        complex64/complex128 CPU tensor of 2^n amplitudes (pin it for
        overlapped copies); the library streams its `nslices` slices through
        the GPU.  Read the tensor only after sync()."""
        import torch

        if tensor.is_cuda or not tensor.is_contiguous():
            raise ValueError("a host-staged state needs a contiguous CPU tensor")
        if tensor.dtype not in (torch.complex64, torch.complex128):
            raise ValueError("state tensors must be complex64 or complex128")
        n = int(tensor.numel()).bit_length() - 1
        if (1 << n) != tensor.numel():
            raise ValueError("state length must be a power of two")
        self = cls.__new__(cls)
        self._h = ctypes.c_void_p()
        self.dtype = QJ_C64 if tensor.dtype == torch.complex64 else QJ_C128
        self.np_dtype = np.complex64 if self.dtype == QJ_C64 else np.complex128
        self.real_dtype = torch.float32 if self.dtype == QJ_C64 else torch.float64
        self.n = n
        self.shards = [tensor]
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(lib().qj_state_init_host(ctypes.byref(self._h), ctypes.c_void_p(tensor.data_ptr()), n, self.dtype,
                                        int(nslices), ctypes.c_uint64(QJ_KEEP if basis is None else int(basis)),
                                        ctypes.c_void_p(self.stream.cuda_stream)))
        return self

    # -- lifetime ----------------------------------------------------------
    def free(self):
        if self._h:
            _check(lib().qj_state_free(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def reset(self, basis=0):
        _check(lib().qj_state_reset(self._h, ctypes.c_uint64(QJ_KEEP if basis is None else basis)))

    def canonicalize(self):
        """Move the amplitudes back to canonical bit order (after fused circuits
        relabelled SWAPs or sharded remaps); probabilities never need this."""
        _check(lib().qj_state_canonicalize(self._h))

    def sync(self):
        _check(lib().qj_sync(self._h))

    # -- gates -------------------------------------------------------------
    def _mat(self, m, count):
        a = np.ascontiguousarray(np.asarray(m, dtype=self.np_dtype).reshape(-1))
        if a.size != count:
            raise ValueError(f"expected {count} complex values, got {a.size}")
        return a

    def apply_gate(self, targets, matrix, controls=()):
        t, nt = _ints(targets)
        c, nc = _ints(controls)
        m = self._mat(matrix, 4 ** nt)
        _check(lib().qj_apply_gate(self._h, self.n, t, nt, c, nc, ctypes.c_void_p(m.ctypes.data)))

    def x(self, target, controls=()):
        c, nc = _ints(controls)
        _check(lib().qj_apply_x(self._h, int(target), c, nc))

    def z(self, target, controls=()):
        c, nc = _ints(controls)
        _check(lib().qj_apply_z(self._h, int(target), c, nc))

    def swap(self, t0, t1, controls=()):
        c, nc = _ints(controls)
        _check(lib().qj_apply_swap(self._h, int(t0), int(t1), c, nc))

    def fsim(self, t0, t1, u2x2, phase11, controls=()):
        c, nc = _ints(controls)
        u = self._mat(u2x2, 4)
        p = self._mat([phase11], 1)
        _check(lib().qj_apply_fsim(self._h, int(t0), int(t1), ctypes.c_void_p(u.ctypes.data),
                                   ctypes.c_void_p(p.ctypes.data), c, nc))

    def diagonal(self, targets, diag, controls=()):
        t, nt = _ints(targets)
        c, nc = _ints(controls)
        d = self._mat(diag, 2 ** nt)
        _check(lib().qj_apply_diagonal(self._h, t, nt, ctypes.c_void_p(d.ctypes.data), c, nc))

    def pack_circuit(self, gates):
        """Marshal gate records (objects with kind/targets/controls/data, e.g.
        workloads.gates.Gate) into a qj_gate array; returns (array, n, keepalive)."""
        return pack_gates(gates, self.np_dtype)

    def apply_circuit(self, gates, fuse=False, packed=None, fuse_gates=False):
        """fuse: window tile passes (QJ_FUSE); fuse_gates: first the paper's
        greedy <= 2-qubit fusion (QJ_FUSE_GATES)."""
        arr, ng, keep = packed if packed is not None else self.pack_circuit(gates)
        flags = (QJ_FUSE if fuse else 0) | _fuse_gates_flags(fuse_gates)
        _check(lib().qj_apply_circuit(self._h, arr, ng, flags))
        del keep

    def simulate(self, basis, gates=None, qubits=(), fuse=True, fuse_gates=False, packed=None, out=None):
        """reset(basis) + apply_circuit + probabilities(qubits) in one call
        (qj_simulate: the step's ends fuse into the first / last tile pass).
        Returns the marginal tensor (or None when qubits is empty)."""
        import torch

        arr, ng, keep = packed if packed is not None else self.pack_circuit(gates)
        q, nq = _ints(qubits)
        if nq and out is None:
            out = torch.empty(1 << nq, dtype=self.real_dtype, device=self.device)
        flags = (QJ_FUSE if fuse else 0) | _fuse_gates_flags(fuse_gates)
        _check(lib().qj_simulate(self._h, ctypes.c_uint64(int(basis)), arr, ng, flags, q, nq,
                                 ctypes.c_void_p(out.data_ptr()) if nq else None))
        del keep
        return out if nq else None

    # -- readout -----------------------------------------------------------
    def probabilities(self, qubits=None, out=None):
        import torch

        if qubits is None:
            size = 1 << self.n
            q, nq = None, -1
        else:
            qa, nq = _ints(qubits)
            q = qa
            size = 1 << nq
        if out is None:
            out = torch.empty(size, dtype=self.real_dtype, device=self.device)
        _check(lib().qj_probabilities(self._h, q, nq, ctypes.c_void_p(out.data_ptr())))
        return out

    # ---- measurement (R26-R28)
    def collapse(self, qubits, outcome):
        """Project onto `outcome` of the listed qubits (first = MSB) and
        renormalise in place; returns P(outcome).  Raises QJError
        (QJ_ERR_ZERO_PROBABILITY) if P <= 1e-14, leaving the state untouched."""
        q, nq = _ints(qubits)
        p = ctypes.c_double()
        _check(lib().qj_collapse(self._h, q, nq, ctypes.c_uint64(int(outcome)), ctypes.byref(p)))
        return p.value

    def sample(self, qubits, nshots, seed, method="direct", nchains=0, burnin=None,
               samples=True, counts=True):
        """Shots over the marginal of `qubits`: returns (samples int64[nshots] or
        None, counts int64[2^nq] or None), device tensors on the handle's stream."""
        import torch

        q, nq = _ints(qubits)
        opts = sample_opts(method, nchains, burnin)
        smp = torch.empty(int(nshots), dtype=torch.int64, device=self.device) if samples else None
        cnt = None
        if counts:
            with torch.cuda.stream(self.stream):
                cnt = torch.zeros(1 << nq, dtype=torch.int64, device=self.device)
        _check(lib().qj_sample(self._h, q, nq, ctypes.c_uint64(int(nshots)), ctypes.c_uint64(int(seed)),
                               ctypes.byref(opts), _ptr(smp), _ptr(cnt)))
        return smp, cnt

    def measure(self, qubits, seed):
        """Draw one outcome of `qubits` (direct method) and collapse onto it:
        returns (outcome, probability)."""
        q, nq = _ints(qubits)
        o, p = ctypes.c_uint64(), ctypes.c_double()
        _check(lib().qj_measure(self._h, q, nq, ctypes.c_uint64(int(seed)), ctypes.byref(o), ctypes.byref(p)))
        return int(o.value), p.value

    def counters(self, reset=False):
        c = qj_counters()
        _check(lib().qj_get_counters(self._h, ctypes.byref(c), 1 if reset else 0))
        return {"launches": c.launches, "passes": c.passes, "exchanges": c.exchanges,
                "alg_bytes": c.alg_bytes, "exchange_bytes": c.exchange_bytes}

    def set_profiling(self, on=True):
        _check(lib().qj_set_profiling(self._h, 1 if on else 0))

    def profile(self, reset=True):
        """{kind: {"launches", "total_ms", "alg_bytes"}} of the passes enqueued
        while profiling was on (synchronises the stream)."""
        arr = (qj_profile_entry * 16)()
        cnt = ctypes.c_int()
        _check(lib().qj_get_profile(self._h, arr, 16, ctypes.byref(cnt), 1 if reset else 0))
        return {arr[i].name.decode(): {"launches": arr[i].launches, "total_ms": arr[i].total_ms,
                                       "alg_bytes": arr[i].alg_bytes} for i in range(cnt.value)}

    def debug_self_exchange(self, local_bit):
        """NCCL states only: the exchange path with this rank as its own partner
        (the state must come back unchanged)."""
        _check(lib().qj_debug_nccl_self_exchange(self._h, int(local_bit)))

    def layout(self):
        """Logical->physical bit map: qubit q is held at bit layout()[q]."""
        phys = (ctypes.c_int * self.n)()
        _check(lib().qj_state_layout(self._h, phys))
        return list(phys)

    def profile_launches(self, reset=True):
        """Per-launch records in enqueue order: [(kind, ms, alg_bytes)]."""
        arr = (qj_profile_entry * 4096)()
        cnt = ctypes.c_int()
        _check(lib().qj_get_profile(self._h, arr, 4096, ctypes.byref(cnt), (1 if reset else 0) | 2))
        return [(arr[i].name.decode(), arr[i].total_ms, arr[i].alg_bytes) for i in range(cnt.value)]

    def info(self):
        v = [ctypes.c_int() for _ in range(4)]
        _check(lib().qj_state_info(self._h, *[ctypes.byref(x) for x in v]))
        return {"n": v[0].value, "n_local": v[1].value, "dtype": v[2].value, "nshards": v[3].value}
