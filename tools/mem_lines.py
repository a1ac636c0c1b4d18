"""Shared-memory wavefronts (actual/ideal) and global sectors per source line: mem_lines.py REP [DIV] [N]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, cur = "", None, None
cols = ["L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal", "L2 Theoretical Sectors Global",
        "L2 Theoretical Sectors Global Ideal", "L1 Tag Requests Global", "Instructions Executed"]
agg = defaultdict(lambda: [0.0] * len(cols))
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; idx = [hdr.index(c) for c in cols]; continue
    if hdr is None or len(r) < len(hdr) or r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = (fname, r[0], r[1].strip()); continue
    for j, i in enumerate(idx):
        try:
            agg[cur][j] += float(r[i] or 0)
        except ValueError:
            pass
tot = [sum(v[j] for v in agg.values()) for j in range(len(cols))]
print("totals per unit:", {c: round(t / div, 1) for c, t in zip(cols, tot)})
for key, name in ((0, "shared wavefronts"), (2, "global L2 sectors"), (4, "global L1 tag requests")):
    print("==", name)
    for cur, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:N]:
        if v[key] <= 0: break
        print(f"  {v[key]/div:7.1f} (ideal {v[key+1]/div:6.1f}) {cur[0]}:{cur[1]} {cur[2][:70]}" if key < 4 else
              f"  {v[key]/div:7.1f} {cur[0]}:{cur[1]} {cur[2][:70]}")
