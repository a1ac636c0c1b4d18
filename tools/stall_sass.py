"""Top SASS instructions by a stall reason: stall_sass.py REP [reason ...]"""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]
reasons = sys.argv[2:] or ["short_scoreboard", "wait", "long_scoreboard", "barrier"]
mets = ",".join(f"smsp__pcsamp_warps_issue_stalled_{r}" for r in reasons)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--metrics", mets],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
for ci in range(2, len(hdr)):
    col = [(int(r[ci] or 0), r[1].strip()) for r in data if len(r) > ci]
    tot = sum(c for c, _ in col) or 1
    print(f"== {hdr[ci]} total {tot}")
    ops = Counter()
    for c, s in col:
        t = s.split()
        if t:
            ops[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += c
    print("   by opcode: " + "  ".join(f"{o}:{100*n/tot:.0f}%" for o, n in ops.most_common(10)))
