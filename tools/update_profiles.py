"""Copy one tools/r02_cycle.sh run (gpurun_out/TAG_*) into profiles/: bench lines, the reference
line, the default command's launch list, ncu summaries of the tile kernel for every config,
traffic.json (DRAM bytes per tile-kernel launch from the full captures) and the parity report.
Usage: python tools/update_profiles.py TAG [ROUND]"""
import csv, io, json, os, shutil, subprocess, sys

tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else "r02"
G = lambda n: os.path.join("gpurun_out", f"{tag}_{n}")
P = lambda n: os.path.join("profiles", f"{rnd}_{n}")


def last_json_line(path):
    if not os.path.exists(path):
        return None
    lines = [l for l in open(path).read().splitlines() if l.strip().startswith("{")]
    return lines[-1] if lines else None


for name in ("bench_cfg4", "bench_cfg1", "bench_cfg2", "bench_cfg3", "bench_cfg4_sharded", "bench_reference"):
    line = last_json_line(G(name + ".json"))
    if line:
        open(P(name + ".json"), "w").write(line + "\n")


def csv_from(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    return lines[start:]


open(P("cfg4_launches.csv"), "w").write("\n".join(csv_from(G("cfg4_launches.csv"))) + "\n")
if os.path.exists(G("parity.json")):
    shutil.copy(G("parity.json"), P("parity_report.json"))

sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
t = {}
secs = subprocess.run([sys.executable, "tools/secs.py"], capture_output=True, text=True).stdout
for c in (4, 1, 2, 3):
    rep = G(f"cfg{c}_tile.ncu-rep")
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
    t[f"cfg{c}"] = int(float(d["dram__bytes_read.sum"]) * sc[u["dram__bytes_read.sum"]] +
                       float(d["dram__bytes_write.sum"]) * sc[u["dram__bytes_write.sum"]])
    summ = subprocess.run([sys.executable, "tools/ncu_summary.py", rep, secs], capture_output=True, text=True).stdout
    stalls = subprocess.run([sys.executable, "tools/stall_lines.py", rep, "6"], capture_output=True, text=True).stdout
    mem = subprocess.run([sys.executable, "tools/mem_lines.py", rep, "1", "20"], capture_output=True, text=True).stdout
    with open(P(f"cfg{c}_tile_kernel_ncu_full.txt"), "w") as fh:
        fh.write(f"# ncu --set full --import-source on --clock-control none -k regex:acopf_tile_kernel -c 1 "
                 f"python bench.py --config {c} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e\n")
        fh.write("# summary by tools/ncu_summary.py, tools/stall_lines.py, tools/mem_lines.py\n")
        fh.write(summ)
        fh.write("--- stall attribution (top source lines per reason) ---\n")
        fh.write(stalls)
        fh.write("--- memory attribution (shared wavefronts / global sectors per source line) ---\n")
        fh.write(mem)
t["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of acopf_tile_kernel (the dominant kernel), "
              f"from the `ncu --set full` capture of `python bench.py --config N --steps 1 --warmup 1` "
              f"(profiles/{rnd}_cfgN_tile_kernel_ncu_full.txt); the concurrent generator/coupling kernel and the "
              "interleave pre-pass are separate launches (profiles/%s_cfg4_launches.csv)" % rnd)
json.dump(dict(sorted(t.items())), open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(t, indent=1))
