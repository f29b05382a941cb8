"""Shared-memory wavefronts (actual / ideal) and global L1 requests per unit of work, by CUDA source line.
python tools/ncu_wavefronts.py REPORT KERNEL_REGEX UNITS"""
import csv
import subprocess
import sys

rep, kern, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source",
                      "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = []
for hi in [i for i, r in enumerate(rows) if r and r[0] == "Line No"]:
    h = rows[hi]
    fn = rows[hi - 2][1].split("/")[-1] if hi >= 2 else ""
    iw, ii, ig = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"), h.index("L1 Tag Requests Global")
    for r in rows[hi + 1:]:
        if not r or r[0] in ("File Path", "Function Name", "Line No"):
            break
        if len(r) <= iw or r[2] != "-":
            continue
        try:
            w, idl, g = int(r[iw] or 0), int(r[ii] or 0), int(r[ig] or 0)
        except ValueError:
            continue
        if w or g:
            res.append((w, idl, g, fn, r[0], r[1][:80]))
res.sort(reverse=True)
print(f"shared wavefronts/unit {sum(x[0] for x in res) / units:.2f} (ideal {sum(x[1] for x in res) / units:.2f}), "
      f"global L1 requests/unit {sum(x[2] for x in res) / units:.2f}")
for w, i, g, f, l, s in res[:20]:
    print(f"{w / units:6.2f} ideal {i / units:6.2f} glob {g / units:5.2f} {f[:16]:16s} {l:>5s} {s}")
