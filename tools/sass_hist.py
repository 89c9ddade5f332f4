"""Opcode histogram (+ hottest stall sites) from `ncu --page source --csv` of one kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
his = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[his[0]]
end = his[1] if len(his) > 1 else len(rows)
data = [r for r in rows[his[0] + 1:end] if len(r) == len(h)]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


ie, st, src = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
namp = float(sys.argv[2]) if len(sys.argv) > 2 else 2 ** 30
tot = sum(f(r[ie]) for r in data)
stot = sum(f(r[st]) for r in data) or 1
op, ops = collections.Counter(), collections.Counter()
for r in data:
    t = r[src].split()
    if not t:
        continue
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    op[o] += f(r[ie])
    ops[o] += f(r[st])
print(f"warp inst {tot:.3e}  thread-inst/amp {tot * 32 / namp:.1f}")
for k, v in op.most_common(16):
    print(f"  {k:10s} {v / tot:6.3f} ({v * 32 / namp:6.1f}/amp)  stall {ops[k] / stot:6.3f}")
print("hottest stall sites:")
for r in sorted(data, key=lambda r: -f(r[st]))[:12]:
    print(f"  {r[0]} inst {f(r[ie]) / tot:.4f} stall {f(r[st]) / stot:.4f}  {r[src][:80]}")
