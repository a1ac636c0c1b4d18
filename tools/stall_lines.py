"""Top source lines per stall reason: stall_lines.py REP [N]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
reasons = ["short_scoreboard", "long_scoreboard", "wait", "barrier"]
mets = ",".join(f"smsp__pcsamp_warps_issue_stalled_{r}" for r in reasons)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--metrics", mets],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, cur = "", None, None
agg = defaultdict(lambda: [0] * len(reasons))
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; idx = [hdr.index(c) for c in hdr if c.startswith("stall_")]; names = [hdr[i] for i in idx]; continue
    if hdr is None or len(r) < len(hdr) or r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = (fname, r[0], r[1].strip()); continue
    for j, i in enumerate(idx):
        try:
            agg[cur][j] += int(r[i] or 0)
        except ValueError:
            pass
for j, nm in enumerate(names):
    tot = sum(v[j] for v in agg.values()) or 1
    print("==", nm, tot)
    for cur, v in sorted(agg.items(), key=lambda kv: -kv[1][j])[:N]:
        print(f"  {100*v[j]/tot:5.1f}% {cur[0]}:{cur[1]} {cur[2][:80]}")
