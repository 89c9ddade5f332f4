"""CPU-only checks of the JIT tile-kernel generator's launch-shape decisions
(sources generated without compiling, no GPU): the forms the round-2
measurements chose must be the ones the headline and the every-tile passes
get (paired live tiles, the 1/sqrt2 factors up front, two ring
buffers for short-row windows whose factor tables would not fit beside
three)."""
import os
import re

import pytest

from paper_2203_08826_b200 import qj as Q
from workloads import circuits as C


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2203_08826_b200 import build
    build.build()


def sources(n, gates, amp_bytes, tmp, live=None):
    old = os.environ.get("QJ_DEBUG_LIVE")
    if live is not None:
        os.environ["QJ_DEBUG_LIVE"] = hex(live)
    try:
        k = Q.debug_tile_sources(n, gates, amp_bytes, out_dir=str(tmp), compile=False)
    finally:
        if live is not None:
            if old is None:
                del os.environ["QJ_DEBUG_LIVE"]
            else:
                os.environ["QJ_DEBUG_LIVE"] = old
    return [open(os.path.join(str(tmp), f"qj_tile_{i}.cu")).read() for i in range(k)]


def test_qft30_live_pass_is_paired(tmp_path):
    src = sources(30, C.qft(30).gates, 16, tmp_path, live=0x2DC5CB5B)
    assert len(src) == 3
    last = src[2]
    assert "const int tid = tid_e0;" in last and "tid_e1" in last  # paired through the sparse segments
    assert "if (has1) {  // tile t + 1" in last  # the last segment twice
    assert "scale_all" not in last  # (1/sqrt2)^12 applied to the one input register
    assert re.search(r"v\[\d+\] = Cx<RT>\{v\[\d+\]\.re \* \(RT\)0\.0156", last)
    loop = last[last.index("for (uint64_t tile = t_lo"):]
    assert loop.count("TILE_SYNC();") == 2 and loop.count("__syncthreads();") == 1  # barriers per pair


def test_qft30_every_tile_ring_buffers(tmp_path):
    src = sources(30, C.qft(30).gates, 16, tmp_path)
    nbuf = [int(re.search(r"#define TILE_NBUF (\d+)", s).group(1)) for s in src]
    pairs = ["#define RING_TILE(i) (2 *" in s for s in src]
    assert nbuf == [2, 2, 3] and pairs == [False, False, False]


def test_bv30_every_tile_keeps_three_buffers_and_pairs(tmp_path):
    src = sources(30, C.bv(30).gates, 16, tmp_path)
    short = [s for s in src if "#define TILE_NBUF" in s]
    assert short and all("#define TILE_NBUF 3" in s for s in short)
    assert any("#define RING_TILE(i) (2 *" in s for s in short)
