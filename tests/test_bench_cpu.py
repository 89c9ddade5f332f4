"""CPU checks of bench.py's contract plumbing (no GPU): every configured
workload builds with the BASELINE shapes, both arms print the same config
dict, and the oracle timing reports what it actually ran."""
import argparse
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

WORKLOADS = ["qft10_c128", "var20_c128", "var20_c64", "tfim10_c128", "tfim20_c128", "qft30_c128", "bv30_c128",
             "qaoa30_c128", "sup32_c64"]


@pytest.mark.parametrize("name", WORKLOADS)
def test_workloads_build(name):
    wl = bench.make_workload(name)
    assert wl["n"] >= 10 and len(wl["circ"]) > 0 and wl["circ"].n == wl["n"]
    assert wl["dtype"] in ("c128", "c64") and 0 <= wl["basis"] < 2 ** wl["n"]
    args = argparse.Namespace(workload=name, fuse=True)
    cfg = bench.config_of(args, wl, 1)
    assert cfg["workload"] == name and cfg["gates"] == len(wl["circ"])
    assert ("flush before every timed step" in cfg["l2"]) == bench.needs_flush(wl)


def test_baseline_shapes():
    assert len(bench.make_workload("qft30_c128")["circ"]) == 480    # Table 2: qft(30) 480 gates
    assert len(bench.make_workload("bv30_c128")["circ"]) == 89      # Table 2: bv(30) 89 gates
    assert len(bench.make_workload("sup32_c64")["circ"]) == 900
    assert bench.sharded_n(2) == 34 and bench.sharded_n(4) == 35 and bench.sharded_n(8) == 35


def test_sharded_config_shared_by_both_arms():
    for world in (2, 4, 8):
        n = bench.sharded_n(world)
        cfg = bench.sharded_config(n, world)
        assert cfg == bench.sharded_config(n, world)
        assert cfg["basis"] < 2 ** n and cfg["global_qubits"] == world.bit_length() - 1
        assert cfg["shard_gib"] == 16 * 2 ** (n - cfg["global_qubits"]) / 2**30


def test_oracle_time_whole_and_sampled():
    from workloads import circuits as C
    wl = dict(n=10, dtype="c128", circ=C.qft(10), basis=5, readout=list(range(10)))
    v, sample, cores, extra, wall = bench.oracle_time(wl)
    assert not extra and "whole circuit (60 gates)" in sample and v > 0 and cores >= 1
    wl = dict(n=23, dtype="c128", circ=C.qft(23), basis=5, readout=list(range(10)))
    v, sample, cores, extra, wall = bench.oracle_time(wl)
    assert extra and "one gate per class" in sample and v > wall / 10
    counts = bench.class_counts(C.qft(35).gates)
    assert counts == {(1, 0): 35, (1, 1): 595, (2, 0): 17}
