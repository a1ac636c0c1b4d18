"""Time the evaluation per callback family (what-mask) on config 1 (100 points)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
sys.argv = [sys.argv[0]]
import bench
from paper_2203_10587_b200 import _lib as L

run = bench.build_ours(1, 100, 0, seed0=5)
ev = run.ev
x = torch.from_numpy(run.x_h).cuda(); m = torch.from_numpy(run.m_h).cuda()
out = ev.alloc()
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
res = {}
for name, what in [("ALL", L.ALL), ("CONS", L.CONS), ("JAC", L.JAC), ("HESS", L.HESS), ("OBJ+GRAD", L.OBJ | L.GRAD), ("OBJ", L.OBJ), ("GRAD", L.GRAD),
                   ("CONS+JAC", L.CONS | L.JAC)]:
    for _ in range(3): ev.eval_device(x, m, 1.0, what, out=out, stream=s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s)
    for _ in range(10): ev.eval_device(x, m, 1.0, what, out=out, stream=s.cuda_stream)
    e1.record(s); torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 10
print(json.dumps(res))
from paper_2203_10587_b200 import solution as SOL
for _ in range(3): SOL.device_flows(ev, x, stream=s.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record(s)
for _ in range(10): SOL.device_flows(ev, x, stream=s.cuda_stream)
e1.record(s); torch.cuda.synchronize()
print(json.dumps({"FLOWS(+alloc)": e0.elapsed_time(e1) / 10}))
