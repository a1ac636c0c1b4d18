"""Throughput on a 70,000-bus synthetic network (ACTIVSg70k scale, beyond BASELINE's sizes):
20 points per step, device-resident inputs over two rotating sets, roofline as bench.py."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2203_10587_b200 import synthetic as syn, BatchEvaluator, _lib as L
from paper_2203_10587_b200.packer import PackedCase, Topology
from paper_2203_10587_b200.stage import stage_plan

points, steps = 20, 20
case = syn.make_case(70_000, 20_000, 10_000, seed=70)
topo = Topology(PackedCase(case))
ev = BatchEvaluator([stage_plan(topo) for _ in range(points)], device=0, layout="independent")
xl, xu, _ = topo.bounds()
kinds = syn.variable_kinds([(topo.nb, topo.ng)])
m1 = ev.m // points
sets = []
for r in range(2):
    xs, ms = zip(*[syn.random_point(kinds, xl, xu, m1, 1000 * r + i) for i in range(points)])
    sets.append((torch.from_numpy(np.concatenate(xs)).cuda(), torch.from_numpy(np.concatenate(ms)).cuda(), ev.alloc()))
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
for k in range(5):
    x, m, o = sets[k % 2]; ev.eval_device(x, m, 1.0, L.ALL, out=o, stream=st.cuda_stream)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for k in range(steps):
    x, m, o = sets[k % 2]; ev.eval_device(x, m, 1.0, L.ALL, out=o, stream=st.cuda_stream)
b.record(st)
torch.cuda.synchronize()
ms_step = a.elapsed_time(b) / steps
by = bench.algorithmic_bytes(ev)
peak = json.load(open(os.path.join(bench.HERE, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(bench.HERE, "MEASURED_PEAKS.json")) else bench.FALLBACK_HBM_GBS
gbs = by / (ms_step / 1000) / 1e9
print(json.dumps({"network": "70,000 buses, 90,000 branches, 10,000 generators", "points_per_step": points,
                  "ms_per_step": round(ms_step, 4), "evals_per_s": round(points / (ms_step / 1000), 1),
                  "algorithmic_bytes_per_step": by, "achieved_gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}))
