"""Opcode mix of the SASS executed for a source-line range: sass_mix.py REP FILE LO HI [DIV]"""
import csv, io, subprocess, sys
from collections import Counter
rep, fn, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
div = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
fname, hdr, cur = "", None, None
c = Counter(); tot = 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; iI = hdr.index("Instructions Executed"); continue
    if hdr is None or len(r) < 10 or r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = (fname, int(r[0])); continue
    if cur and (fn == "*" or cur[0] == fn) and lo <= cur[1] <= hi:
        try:
            n = int(float(r[iI]))
        except ValueError:
            n = 0
        t = r[3].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        c[op] += n; tot += n
print(f"total {tot/1e6:.2f}M  per-unit {tot/div:.1f}")
for op, n in c.most_common(45):
    print(f"  {op:28s} {100*n/tot:5.1f}%  {n/div:7.1f}")
