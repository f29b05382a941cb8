"""Per-source-line (CUDA line via -lineinfo) and per-SASS-opcode stall sampling of one kernel."""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, data = rows[1], rows[2:]
isrc, iall = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
by_op = collections.Counter()
by_reason = collections.Counter()
for r in data:
    if len(r) < len(h) or not r[iall].isdigit():
        continue
    op = r[isrc].split()[0] if r[isrc].split() else "?"
    if op.startswith("@"):
        op = r[isrc].split()[1]
    by_op[op.split(".")[0]] += int(r[iall] or 0)
    for i in stall_cols:
        try:
            by_reason[(op.split(".")[0], h[i])] += int(r[i] or 0)
        except ValueError:
            pass
tot = sum(by_op.values())
print("samples", tot)
for op, v in by_op.most_common(15):
    reasons = sorted(((by_reason[(op, h[i])], h[i]) for i in stall_cols), reverse=True)[:4]
    print(f"{op:10s} {v:8d} {100*v/tot:5.1f}%  " + ", ".join(f"{n.replace('stall_','')}={c}" for c, n in reasons))
