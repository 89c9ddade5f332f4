"""Summarise ncu outputs from gpurun_out/ into profiles/<tag>/.

  python tools/ncu_summary.py --tag r01 --launches gpurun_out/launches.csv \
      --full gpurun_out/prof_diag.ncu-rep gpurun_out/prof_gate_hi.ncu-rep ...

Writes
  profiles/<tag>/launches_summary.txt  per-kernel count, time share, DRAM bytes / launch
                                        (from the --metrics launch list: cold-cache,
                                        serialised -- compare SHARES, not absolutes)
  profiles/<tag>/launches.csv.gz        the raw launch list
  profiles/<tag>/ncu_full_summary.txt   key counters of each --set full capture
  profiles/ncu_traffic_<tag>.json       dram read+write bytes per launch per pass kind
                                        (read by bench.py for roofline.traffic)
"""

import argparse
import collections
import csv
import gzip
import json
import os
import re
import shutil
import subprocess

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
        "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}

# kernel template -> bench pass-kind name (qj_get_profile names)
KIND = [(r"diag_kernel<\w+, 0>", "diag_table"), (r"diag_kernel<\w+, 1>", "diag_phase"),
        (r"diag_kernel<\w+, 2>", "diag_neg"), (r"gate_warp_kernel<\w+, \d, \d, \d, 0>", "gate_dense"),
        (r"gate_warp_kernel<\w+, \d, \d, \d, 1>", "gate_x"), (r"gate_warp_kernel<\w+, \d, \d, \d, 2>", "gate_swap"),
        (r"tile_kernel|qj_tile_jit", "tile"), (r"exchange_kernel", "exchange")]


def kind_of(name):
    for pat, k in KIND:
        if re.search(pat, name):
            return k
    return None


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = per.setdefault(r[idi], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--root", default="profiles", help="output root (use /tmp for scratch)")
    a = ap.parse_args()
    out = os.path.join(a.root, a.tag)
    os.makedirs(out, exist_ok=True)
    traffic = {}
    if a.launches:
        per = read_launches(a.launches)
        agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
        kagg = collections.defaultdict(lambda: [0, 0.0])
        for d in per.values():
            name = d["name"].split("(")[0]
            g = agg[name]
            g[0] += 1
            g[1] += d.get("gpu__time_duration.sum", 0.0)
            g[2] += d.get("dram__bytes_read.sum", 0.0)
            g[3] += d.get("dram__bytes_write.sum", 0.0)
            k = kind_of(name)
            if k:
                kagg[k][0] += 1
                kagg[k][1] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        tot = sum(g[1] for g in agg.values()) or 1.0
        with open(os.path.join(out, "launches_summary.txt"), "w") as f:
            f.write(f"# ncu launch list ({a.launches}); {len(per)} launches; gpu__time_duration "
                    f"cold-cache + serialised: compare shares\n")
            f.write(f"{'kernel':64s} {'launches':>8s} {'time_ms':>10s} {'share':>6s} {'rd_GB/l':>8s} {'wr_GB/l':>8s}\n")
            for name, g in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                f.write(f"{name[:64]:64s} {g[0]:8d} {g[1] * 1e3:10.2f} {g[1] / tot:6.3f} "
                        f"{g[2] / g[0] / 1e9:8.3f} {g[3] / g[0] / 1e9:8.3f}\n")
        with open(a.launches, "rb") as fi, gzip.open(os.path.join(out, "launches.csv.gz"), "wb") as fo:
            shutil.copyfileobj(fi, fo)
        for k, (cnt, by) in kagg.items():
            traffic[k] = {"dram_bytes_per_launch": by / cnt, "launches": cnt, "source": f"profiles/{a.tag}/launches.csv.gz"}
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__average_warp_latency_issue_stalled_long_scoreboard", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
            "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum"]
    if a.full:
        with open(os.path.join(out, "ncu_full_summary.txt"), "w") as f:
            for rep in a.full:
                r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
                rows = list(csv.reader(r.stdout.splitlines()))
                if len(rows) < 3:
                    continue
                h, units = rows[0], rows[1]
                f.write(f"== {os.path.basename(rep)} (ncu --set full --clock-control none)\n")
                for row in rows[2:]:
                    f.write(f"  kernel: {row[h.index('Kernel Name')]}\n")
                    for w in want:
                        if w in h:
                            f.write(f"    {w:60s} {row[h.index(w)]} {units[h.index(w)]}\n")
    with open(os.path.join(a.root, f"ncu_traffic_{a.tag}.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()
