"""Summarise an ncu report of the tile kernel: key raw metrics, per-section and per-line
instruction counts and stall samples, SASS opcode mix.  Usage: ncu_summary.py REP [sections]"""
import csv, io, re, subprocess, sys
from collections import Counter, defaultdict

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
pat = (r"gpu__time_duration.sum|dram__bytes_(read|write).sum$|smsp__inst_executed.sum$|smsp__issue_active.avg.pct|"
       r"sm__warps_active.avg.pct|registers_per_thread$|pipe_fp64_cycles.*avg.*active$|"
       r"l1tex__data_pipe_lsu_wavefronts_mem_shared.sum$|warps_eligible.avg|occupancy_limit_(reg|shared)|"
       r"l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed|"
       r"l1tex__data_pipe_lsu_wavefronts_mem_shared_op_(ld|st).sum$|TriageCompute.l1tex__data_pipe_lsu_wavefronts.*avg$|"
       r"l1tex__t_sector_hit_rate.pct|memory_l1_wavefronts_shared(_ideal)?$|"
       r"smsp__pcsamp_warps_issue_stalled_[a-z_]*_not_issued$|shared_mem_per_block_dynamic|grid_size")
for k in sorted(d):
    if re.search(pat, k) and d[k] not in ("0", "0.0"):
        print(f"  {k} {d[k]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))

def num(x):
    try:
        return int(float(x))
    except ValueError:
        return 0

lines, sass = [], []
fname, hdr, cur = "", None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; iI = hdr.index("Instructions Executed"); iS = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) < 10 or r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = [fname, int(r[0]), r[1], num(r[iI]), num(r[iS])]; lines.append(cur)
    else:
        sass.append((r[3].strip(), num(r[iI])))
tot = sum(l[3] for l in lines) or 1
st = sum(l[4] for l in lines) or 1
print(f"total inst {tot/1e6:.2f}M  samples {st}")
secs = []
if len(sys.argv) > 2:
    secs = eval(sys.argv[2])
if secs:
    agg = defaultdict(lambda: [0, 0])
    for f, ln, _, n, s in lines:
        name = "other:" + f
        for nm, ff, lo, hi in secs:
            if f == ff and lo <= ln <= hi:
                name = nm; break
        agg[name][0] += n; agg[name][1] += s
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:22s} inst {v[0]/1e6:7.2f}M ({100*v[0]/tot:5.1f}%)  stall {100*v[1]/st:5.1f}%")
for f, ln, txt, n, s in sorted(lines, key=lambda l: -l[3])[:25]:
    print(f"  {f}:{ln:<5d} inst {100*n/tot:5.1f}% stall {100*s/st:5.1f}%  {txt.strip()[:80]}")
c = Counter()
for s, n in sass:
    t = s.split()
    if t:
        c[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += n
T = sum(c.values()) or 1
print("  " + "  ".join(f"{op}:{100*n/T:.1f}%" for op, n in c.most_common(24)))
