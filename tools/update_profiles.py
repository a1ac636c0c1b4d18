"""Copy one tools/round_artifacts.sh run (gpurun_out/TAG_*) into profiles/: bench lines,
reference line, cfg1 launch list, the ncu summary of the tile kernel, traffic.json.
Usage: python tools/update_profiles.py TAG [ROUND]"""
import csv, io, json, os, subprocess, sys

tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else "r01"
G = lambda n: os.path.join("gpurun_out", f"{tag}_{n}")
P = lambda n: os.path.join("profiles", f"{rnd}_{n}")


def last_json_line(path):
    lines = [l for l in open(path).read().splitlines() if l.strip().startswith("{")]
    return lines[-1] if lines else None


for c in (1, 2, 3, 4):
    line = last_json_line(G(f"bench_cfg{c}.json"))
    if line:
        open(P(f"bench_cfg{c}.json"), "w").write(line + "\n")
line = last_json_line(G("bench_reference.json"))
if line:
    open(P("bench_reference.log"), "w").write(line + "\n")


def csv_from(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    return lines[start:]


lines = csv_from(G("cfg1_launches.csv"))
open(P("cfg1_launches.csv"), "w").write("\n".join(lines) + "\n")


def metrics(lines):
    rows = list(csv.reader(lines))
    hdr = rows[0]
    iM, iV, iU = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}
    return {r[iM]: float(r[iV]) * scale.get(r[iU], 1) for r in rows[1:] if len(r) == len(hdr)}


t = {}
for c in (2, 4):
    m = metrics(csv_from(G(f"cfg{c}_tile_traffic.csv")))
    t[f"cfg{c}"] = int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
rep = G("cfg1_tile.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
t["cfg1"] = int(float(d["dram__bytes_read.sum"]) * sc[u["dram__bytes_read.sum"]] +
                float(d["dram__bytes_write.sum"]) * sc[u["dram__bytes_write.sum"]])
t["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of acopf_tile_kernel (the dominant kernel): "
              "cfg1 from one `ncu --set full` capture of `python bench.py --steps 1 --warmup 1 --no-cpu-baseline "
              "--no-e2e` (profiles/%s_cfg1_tile_kernel_ncu_full.txt); cfg2/cfg4 from `ncu --metrics "
              "dram__bytes_read.sum,dram__bytes_write.sum -k regex:acopf_tile_kernel -c 1` of `bench.py --config N`; "
              "the concurrent aux kernel adds ~2 MB" % rnd)
json.dump(dict(sorted(t.items())), open("profiles/traffic.json", "w"), indent=1)
secs = subprocess.run([sys.executable, "tools/secs.py"], capture_output=True, text=True).stdout
summ = subprocess.run([sys.executable, "tools/ncu_summary.py", rep, secs], capture_output=True, text=True).stdout
stalls = subprocess.run([sys.executable, "tools/stall_lines.py", rep, "6"], capture_output=True, text=True).stdout
with open(P("cfg1_tile_kernel_ncu_full.txt"), "w") as fh:
    fh.write("# ncu --set full --import-source on --clock-control none -k regex:acopf_tile_kernel -c 1 "
             "python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e\n")
    fh.write("# summary by tools/ncu_summary.py (sections from tools/secs.py) and tools/stall_lines.py\n")
    fh.write(summ)
    fh.write("--- stall attribution (top source lines per reason) ---\n")
    fh.write(stalls)
print(json.dumps(t, indent=1))
