"""Per-kernel key counters + stall breakdown + top SASS opcodes of an ncu report.
  python tools/ncu_stalls.py gpurun_out/x.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
for r in rows[2:]:
    print("---", r[hdr.index("Kernel Name")])
    for w in want:
        if w in hdr:
            print(f"  {w:70s} {r[hdr.index(w)]} {units[hdr.index(w)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
        continue
    if cur is not None:
        cur.append(r)
for b in blocks:
    h, data = b[0], b[1:]
    iS, iI = h.index("Source"), h.index("Instructions Executed")
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = {c: sum(int(x[h.index(c)] or 0) for x in data) for c in cols}
    T = sum(tot.values()) or 1
    print("stalls:", {c[6:]: round(100 * v / T, 1) for c, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v > 0.01 * T})
    inst = sum(int(x[iI] or 0) for x in data) or 1
    op = collections.Counter()
    for x in data:
        t = x[iS].strip().split()
        if not t:
            continue
        m = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        op[m.split(".")[0]] += int(x[iI] or 0)
    print("inst:", inst, {m: round(100 * c / inst, 1) for m, c in op.most_common(14)})
