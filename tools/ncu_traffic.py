"""Fold ncu launch lists (csv, --metrics dram__bytes_read.sum,
dram__bytes_write.sum,gpu__time_duration.sum) into per-kind DRAM bytes per
launch, keyed workload -> section -> kind, merged into a JSON file that
bench.py reads for roofline.traffic:

    python tools/ncu_traffic.py OUT.json WORKLOAD SECTION launches.csv
"""
import collections
import csv
import json
import os
import re
import sys


def kind_of(name):
    if "qj_tile_jit" in name or "tile_kernel" in name:
        return "tile"
    m = re.search(r"gate_warp_kernel<[^>]*,\s*(\d+)>", name)
    if m:
        return {"0": "gate_dense", "1": "gate_x", "2": "gate_swap"}[m.group(1)]
    if "gate_bigk_kernel" in name or "gate_simple_kernel" in name:
        return "gate_dense"
    m = re.search(r"diag_kernel<[^,]*,\s*(\d+)>", name)
    if m:
        return {"0": "diag_table", "1": "diag_phase", "2": "diag_neg"}[m.group(1)]
    if "small" in name:
        return "small"
    if "init_kernel" in name:
        return "init"
    if "exchange" in name or "half_pack" in name or "half_unpack" in name:
        return "exchange"
    return "other:" + name.split("(")[0].split("<")[0].replace("void ", "").strip()


def main():
    out, workload, section, path = sys.argv[1:5]
    rows = [l for l in open(path) if l.startswith('"')]
    r = csv.DictReader(rows)
    per = collections.defaultdict(dict)
    for row in r:
        per[(row["ID"], row["Kernel Name"])][row["Metric Name"]] = (float(row["Metric Value"].replace(",", "")),
                                                                    row["Metric Unit"])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
    agg = collections.defaultdict(lambda: {"dram": 0.0, "ms": 0.0, "launches": 0})
    for (_, name), met in per.items():
        k = kind_of(name)
        d = agg[k]
        d["launches"] += 1
        for mname in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if mname in met:
                v, u = met[mname]
                d["dram"] += v * scale.get(u, 1)
        if "gpu__time_duration.sum" in met:
            v, u = met["gpu__time_duration.sum"]
            d["ms"] += v * scale.get(u, 1) * 1e3
    res = json.load(open(out)) if os.path.exists(out) else {}
    sec = res.setdefault(workload, {}).setdefault(section, {})
    for k, d in agg.items():
        sec[k] = {"dram_bytes_per_launch": d["dram"] / d["launches"], "launches": d["launches"],
                  "ncu_ms_per_launch": d["ms"] / d["launches"],
                  "source": f"{os.path.basename(path)}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                            f"gpu__time_duration.sum --clock-control none, tools/step_probe.py {workload} {section}"}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
