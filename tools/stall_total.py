"""Top source lines by all warp stall samples together: stall_total.py REP [N]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, cur = "", None, None
agg = defaultdict(lambda: [0, 0])
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r
        iS = hdr.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in hdr else None
        iI = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
        continue
    if hdr is None or len(r) < len(hdr) or r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = (fname, r[0], r[1].strip()[:90]); continue
    for j, i in enumerate((iS, iI)):
        if i is None:
            continue
        try:
            agg[cur][j] += float(r[i] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
print("total stall samples", tot)
for cur, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{100 * v[0] / tot:5.1f}%  inst {v[1] / 1e6:7.1f}M  {cur[0]}:{cur[1]} {cur[2]}")
