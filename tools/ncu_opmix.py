"""Executed-instruction mix of one kernel from an ncu report's source page (SASS), per opcode,
normalised per unit of work: python tools/ncu_opmix.py REPORT KERNEL_REGEX UNITS."""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, data = rows[1], rows[2:]
isrc, iex, ith = h.index("Source"), h.index("Instructions Executed"), h.index("Thread Instructions Executed")
warp = collections.Counter()
thread = collections.Counter()
for r in data:
    if len(r) < len(h) or not r[iex].replace(",", "").isdigit():
        continue
    toks = r[isrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    warp[op] += int(r[iex].replace(",", ""))
    thread[op] += int(r[ith].replace(",", ""))
tw, tt = sum(warp.values()), sum(thread.values())
print(f"warp instr {tw:.4g} ({tw / units:.1f}/unit), thread instr {tt:.4g} ({tt / units:.1f}/unit)")
for op, v in warp.most_common(30):
    print(f"{op:10s} warp {v / units:8.2f}/unit  thread {thread[op] / units:8.1f}/unit  {100 * v / tw:5.1f}%")
