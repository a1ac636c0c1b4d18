"""How much the synthetic networks' random bus numbering costs: the cfg1 network as built,
and the same network with its buses renumbered in breadth-first order from the reference
bus (identical topology and parameters; only the order, hence tile membership and gather
locality, changes).  100 points per step, device-resident inputs, two rotating sets."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from collections import deque
from dataclasses import replace
import numpy as np
import torch
from paper_2203_10587_b200 import synthetic as syn, BatchEvaluator, _lib as L
from paper_2203_10587_b200.packer import PackedCase, Topology
from paper_2203_10587_b200.stage import stage_plan


def bfs_order(case):
    ids = [b.id for b in case.buses]
    pos = {b: i for i, b in enumerate(ids)}
    adj = [[] for _ in ids]
    for br in case.branches:
        if br.status:
            a, b = pos[br.fbus], pos[br.tbus]
            adj[a].append(b); adj[b].append(a)
    ref = next(i for i, b in enumerate(case.buses) if b.btype == 3)
    seen, order, q = {ref}, [], deque([ref])
    while q:
        u = q.popleft(); order.append(u)
        for v in sorted(adj[u], key=lambda v: len(adj[v])):
            if v not in seen:
                seen.add(v); q.append(v)
    order += [i for i in range(len(ids)) if i not in seen]
    return order


def run(case, points=100, steps=30):
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
    fo, to = np.asarray(topo.fo), np.asarray(topo.to)
    return a.elapsed_time(b) / steps, float(np.mean(np.abs(fo - to))), float(np.mean(fo // 47 == to // 47))


case = syn.config_case(1)
local = replace(case, buses=tuple(case.buses[i] for i in bfs_order(case)))
for name, c in (("as built", case), ("BFS-numbered", local)):
    ms, d, intra = run(c)
    print(f"{name:13s} {ms:.4f} ms per 100-point step; mean |f - t| {d:.0f} slots; intra-tile branches {intra:.3f}")
