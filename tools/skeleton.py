"""Run the config-1 batch with a given what-mask a few times (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
what = int(sys.argv[1]); sys.argv = [sys.argv[0]]
import torch, bench
from paper_2203_10587_b200 import _lib as L
run = bench.build_ours(1, 100, 0, seed0=5)
ev = run.ev
x = torch.from_numpy(run.x_h).cuda(); m = torch.from_numpy(run.m_h).cuda()
out = ev.alloc()
for _ in range(4): ev.eval_device(x, m, 1.0, what, out=out)
torch.cuda.synchronize()
