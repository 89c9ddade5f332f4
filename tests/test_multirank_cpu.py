"""World-size-2 (and 4) CPU tests of the multi-GPU layer's host logic over
torch.distributed 'gloo' (the paper's multi-device scheme is
PAPER.md:469-489).

Each rank owns one shard (global qubits = the top log2 P bits).  The steps come
from the library's own planner (qj_plan_circuit, no GPU): per-shard passes on
physical local bits, and EXCHANGE steps that swap a global bit with a local
bit; the exchange partner and the half traded come from the library's
exchange rule (qj_exchange_peer) -- the same code the NCCL path runs.  A
test-side numpy interpreter applies each pass (an independent restatement of
the pass semantics: dense / X / SWAP / diagonal / phase / sign flip on fixed-bit
subspaces) and gloo moves the halves.  The gathered state, read through the
final logical->physical map, must equal the CPU oracle.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from workloads import circuits as C  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def apply_pass(psi, nl, st):
    """Test-side interpreter of one planned pass on a shard (physical bits)."""
    idx = np.arange(psi.size, dtype=np.int64)
    act = np.ones(psi.size, dtype=bool)
    for (p, v) in st["fix"]:
        act &= ((idx >> p) & 1) == v
    kind, t, m = st["kind"], st["tpos"], st["m"]
    out = psi.copy()
    if kind in (3, 4, 5):  # diag / phase / neg
        if kind == 5:
            out[act] = -psi[act]
        elif kind == 4:
            out[act] = m[0] * psi[act]
        else:
            row = np.zeros(psi.size, dtype=np.int64)
            for b in t:
                row = (row << 1) | ((idx >> b) & 1)
            out[act] = m[row[act]] * psi[act]
        return out
    k = len(t)
    if kind == 1:      # X
        M = np.array([[0, 1], [1, 0]], dtype=complex)
        touch = 0x3
    elif kind == 2:    # SWAP
        M = np.eye(4, dtype=complex)[[0, 2, 1, 3]]
        touch = 0x6
    else:
        M = m.reshape(2**k, 2**k)
        touch = st["touch"]
    row = np.zeros(psi.size, dtype=np.int64)
    clear = idx.copy()
    for b in t:
        row = (row << 1) | ((idx >> b) & 1)
        clear &= ~(1 << b)
    for r in range(2**k):
        if not (touch >> r) & 1:
            continue
        sel = act & (row == r)
        acc = np.zeros(int(sel.sum()), dtype=complex)
        for c in range(2**k):
            src = clear[sel].copy()
            for i, b in enumerate(t):
                if (c >> (k - 1 - i)) & 1:
                    src |= 1 << b
            acc += M[r, c] * psi[src]
        out[sel] = acc
    return out


def _run_steps(steps, shard, rank, nl, Q):
    nex = 0
    for st in steps:
        if st["type"] == 0:
            if st["shard"] == rank:
                shard = apply_pass(shard, nl, st)
        elif st["type"] == 1:
            nex += 1
            peer, hb = Q.exchange_peer(rank, st["gbit"])
            L = st["lbit"]
            idx = np.arange(shard.size)
            sel = np.nonzero(((idx >> L) & 1) == hb)[0]
            send = torch.from_numpy(np.ascontiguousarray(shard[sel]).view(np.float64))
            recv = torch.empty_like(send)
            req = dist.isend(send, peer)
            dist.recv(recv, peer)
            req.wait()
            shard[sel] = recv.numpy().view(np.complex128)
        else:
            raise AssertionError("unexpected fused step")
    return shard, nex


def _worker(rank, world, port, n, seed, which, result_q, canon=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_08826_b200 import qj as Q

        circ = {"random": lambda: C.random_circuit(n, 80, seed, max_targets=3),
                "qft": lambda: C.qft(n),
                "supremacy": lambda: C.supremacy(2, n // 2, 6)}[which]()
        g = world.bit_length() - 1
        nl = n - g
        rng = np.random.default_rng(seed)
        full = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
        full /= np.linalg.norm(full)
        shard = full[rank << nl:(rank + 1) << nl].copy()
        steps, phys = Q.plan_circuit(n, world, circ.gates)
        shard, nex = _run_steps(steps, shard, rank, nl, Q)
        if canon:  # qj_state_canonicalize's plan: every rank ends in canonical order
            shard, _ = _run_steps(Q.plan_canonicalize(n, world, phys), shard, rank, nl, Q)
            phys = [n - 1 - q for q in range(n)]
        parts = [torch.empty(2 * shard.size, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(shard.view(np.float64)))
        if rank == 0:
            phys_full = np.concatenate([p.numpy().view(np.complex128) for p in parts])
            # canonical index c: bit (n-1-q) of c = bit phys[q] of the physical index
            c = np.arange(2**n, dtype=np.int64)
            p = np.zeros_like(c)
            for q in range(n):
                p |= ((c >> (n - 1 - q)) & 1) << phys[q]
            canon = phys_full[p]
            import oracle
            exp = oracle.run(circ, full)
            result_q.put((float(np.max(np.abs(canon - exp))), nex))
    finally:
        dist.destroy_process_group()


def _run(world, n, seed, which, canon=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, seed, which, q, canon)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return q.get(timeout=10)


@pytest.mark.parametrize("which,seed", [("random", 1), ("random", 2), ("qft", 0), ("supremacy", 3)])
def test_world2_matches_oracle(which, seed):
    err, nex = _run(2, 8, seed, which)
    assert err < 1e-12, err
    assert nex > 0


def test_world4_matches_oracle():
    err, nex = _run(4, 8, 7, "random")
    assert err < 1e-12, err
    assert nex > 0


def test_exchange_rule_pairs_up():
    from paper_2203_08826_b200 import qj as Q
    for world in (2, 4, 8):
        for j in range(world.bit_length() - 1):
            for r in range(world):
                peer, hb = Q.exchange_peer(r, j)
                back, hb2 = Q.exchange_peer(peer, j)
                assert back == r and peer != r
                assert hb + hb2 == 1  # the two halves traded are complementary
                assert hb == 1 - ((r >> j) & 1)


@pytest.mark.parametrize("world,seed", [(2, 11), (4, 12)])
def test_canonicalize_plan_per_rank(world, seed):
    """After a circuit that remaps global qubits, every rank runs
    qj_state_canonicalize's plan for its own shard index (SWAP passes on
    local pairs are emitted for every shard, not only shard 0); the gathered
    shards are then the oracle's state in canonical order."""
    err, nex = _run(world, 8, seed, "random", canon=True)
    assert err < 1e-12, err
    assert nex > 0


def test_canonicalize_plan_covers_every_shard():
    from paper_2203_08826_b200 import qj as Q
    n, world = 9, 4
    rng = np.random.default_rng(3)
    for _ in range(20):
        phys = [int(b) for b in rng.permutation(n)]
        steps = Q.plan_canonicalize(n, world, phys)
        passes = [s for s in steps if s["type"] == 0]
        for i in range(0, len(passes), world):
            assert sorted(s["shard"] for s in passes[i:i + world]) == list(range(world))
        # replaying the plan on the map gives the canonical map
        cur = list(phys)
        for s in steps:
            if s["type"] == 0:
                if s["shard"] == 0:
                    a, b = s["tpos"]
                    cur = [b if p == a else a if p == b else p for p in cur]
            else:  # exchange: global bit nl + gbit <-> local bit lbit (nl = n - 2 at 4 shards)
                gb, b = (n - 2) + s["gbit"], s["lbit"]
                cur = [b if p == gb else gb if p == b else p for p in cur]
        assert cur == [n - 1 - q for q in range(n)], (phys, cur)
