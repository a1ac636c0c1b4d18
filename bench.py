#!/usr/bin/env python
"""Benchmark: ACOPF callback evaluations/sec on B200 (BASELINE.json metric).

Default workload = BASELINE config 1: the synthetic 10,000-bus network
(tree + 3,000 chords, 2,500 generators), 100 seeded evaluation points; one
step = one batched evaluation of objective + gradient + constraints +
Jacobian values + Lagrangian-Hessian values at all 100 points (one kernel
launch).  ``--config 2|3|4`` benches the composite configs instead (one step
= one evaluation of the whole composite).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) every rank evaluates its own 100-point batch on its
GPU (config 1 does not shard: replicas, weak scaling); the time is the max
over ranks of the device-measured time.  ``--impl reference`` times the
reference algorithm's CPU implementation (the numpy oracle port, bit-exact to
the reference) on all host cores instead.

Timing: W untimed warm-up steps; each timed step is bracketed by CUDA events
on the launching stream; a 256 MiB buffer is written between timed steps to
flush the 126 MB L2 (not timed).  nvidia-smi clocks are sampled during the
timed region.  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "ACOPF callback evals/sec (obj+grad+g+h+J+H), 1/2/4/8 GPU; % HBM roofline"
UNIT = "evals/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=1, choices=(1, 2, 3, 4))
    ap.add_argument("--points", type=int, default=100, help="evaluation points per step (config 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# workloads

def workload_desc(cfg: int, points: int) -> dict:
    return {
        1: dict(workload=f"cfg1: synthetic 10,000-bus network (tree + 3,000 chords, 12,999 branches, "
                         f"2,500 generators), {points} seeded points per step, batch=1 each"),
        2: dict(workload="cfg2: N-1 SCOPF composite, 2,000-bus network (tree + 600 chords, 500 gens), "
                         "base + 1,024 non-bridge branch contingencies (1,025 stages), corrective dc=0.1 pu"),
        3: dict(workload="cfg3: multiperiod composite, 2,000-bus network, 96 periods, seeded daily load "
                         "profile, ramp dt=0.05 Pmax"),
        4: dict(workload="cfg4: stochastic SCOPF composite, 25,000-bus network (tree + 8,000 chords, "
                         "6,000 gens), 32 scenarios x (base + 31 N-1) = 1,024 stages, 20% wind"),
    }[cfg]


def _composite_args(cfg: int):
    from paper_2203_10587_b200 import synthetic as syn
    from paper_2203_10587_b200.types import CouplingMode
    if cfg == 2:
        base, ctgs = syn.config2_inputs()
        return "scopf", (base, ctgs, CouplingMode()), None
    if cfg == 3:
        return "multiperiod", (syn.config3_periods(), 15.0), None
    base, scens, ctgs = syn.config4_inputs()
    per_scen = len(ctgs) + 1
    return "general", (scens, ctgs, [base], CouplingMode(), 30.0), per_scen


class Runner:
    """One benchmark step = one evaluation of the workload on this rank's GPU."""

    def __init__(self, ev, x_h, m_h, units, sharded=None):
        self.ev, self.x_h, self.m_h, self.units, self.sharded = ev, x_h, m_h, units, sharded


def build_ours(cfg: int, points: int, device: int, seed0: int, dist=None, rank=0, world=1):
    """Runner for config cfg on cuda:device (sharded over ranks for composites when world > 1)."""
    from paper_2203_10587_b200 import synthetic as syn
    from paper_2203_10587_b200 import BatchEvaluator, compose_general, compose_multiperiod, compose_scopf
    from paper_2203_10587_b200.packer import PackedCase, Topology
    from paper_2203_10587_b200.stage import stage_plan
    if cfg == 1:
        case = syn.config_case(1)
        topo = Topology(PackedCase(case))
        ev = BatchEvaluator([stage_plan(topo) for _ in range(points)], device=device, layout="independent")
        xl, xu, _ = topo.bounds()
        kinds = syn.variable_kinds([(topo.nb, topo.ng)])
        m1 = ev.m // points
        xs, ms = [], []
        for i in range(points):
            x, m = syn.random_point(kinds, xl, xu, m1, seed0 + i)
            xs.append(x)
            ms.append(m)
        return Runner(ev, np.concatenate(xs), np.concatenate(ms), points)
    kind, args, per_scen = _composite_args(cfg)
    if world > 1:
        from paper_2203_10587_b200.dispatch import ShardedComposite
        from paper_2203_10587_b200.lattice import composite_spec
        spec = composite_spec(kind, *args)
        align = None if per_scen is None else [k // per_scen for k in range(len(spec.plans))]
        sc = ShardedComposite(spec, dist, rank, world, device=f"cuda:{device}", align=align)
        kinds = syn.variable_kinds(spec.stage_dims[sc.plan.s0:sc.plan.s1])
        rng = np.random.default_rng(seed0)
        xl, xu = np.zeros(len(kinds)), np.ones(len(kinds))
        x, _ = syn.random_point(kinds, xl + 0.1, xu, 1, seed0)
        x = np.concatenate([x, np.zeros(sc.n_x - sc.plan.n_loc)])
        return Runner(sc.ev, x, rng.standard_normal(sc.ev.m), 1, sharded=sc)
    fn = {"scopf": compose_scopf, "multiperiod": compose_multiperiod, "general": compose_general}[kind]
    p, imap = fn(*args, device=device)
    ev = p.evaluator
    kinds = syn.variable_kinds([(pl.topo.nb, pl.topo.ng) for pl in ev.plans])
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, seed0)
    return Runner(ev, x, mult, 1)


def algorithmic_bytes(ev) -> int:
    """fp64 reads of x, mult, per-stage loads, topology once; writes of all outputs."""
    topo_bytes = sum(72 * t.nbr + 32 * t.nb + 28 * t.ng for t in ev.topos)
    load_sets = {(id(p.topo), p.load_key) for p in ev.plans}
    extra_loads = 16 * sum(ev.plans[0].topo.nb for _ in range(max(0, len(load_sets) - len(ev.topos))))
    reads = 8 * (ev.n + ev.m) + topo_bytes + extra_loads
    writes = 8 * (ev.n_obj + ev.n + ev.m + ev.nnz_j + ev.nnz_h)
    return int(reads + writes)


# ---------------------------------------------------------------------------
# clocks

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].isdigit():
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [int(r[1]) for r in rows]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": int(statistics.median(busy)), "sm_max_mhz": int(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3] not in ("", "[N/A]"))}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm (oracle port of the reference algorithm)

_ORACLE = {}


def _oracle_init(cfg):
    from paper_2203_10587_b200 import synthetic as syn
    from oracle.stage import StageOracle
    case = syn.config_case(1)
    o = StageOracle(case)
    kinds = syn.variable_kinds([(o.nb, o.ng)])
    _ORACLE["o"] = o
    _ORACLE["kinds"] = kinds


def _oracle_eval(seed):
    from paper_2203_10587_b200 import synthetic as syn
    o = _ORACLE["o"]
    x, mult = syn.random_point(_ORACLE["kinds"], o.xl, o.xu, o.m_eq + o.m_ineq, seed)
    t = time.perf_counter()
    o.objective(x)
    o.gradient(x)
    o.constraints(x)
    o.jacobian(x)
    o.lagrangian_hessian(x, 1.0, mult)
    return time.perf_counter() - t


def cpu_baseline_single(seconds: float = 12.0) -> dict:
    """1-core oracle port, bounded sample of config-1 points."""
    _oracle_init(1)
    _oracle_eval(0)
    spent, n = 0.0, 0
    while spent < seconds and n < 400:
        spent += _oracle_eval(1000 + n)
        n += 1
    return {"value": n / spent, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"cfg1 10k-bus network, {n} seeded points x (obj+grad+cons+jac+hess), "
                      f"numpy/scipy oracle port (bit-exact to the reference), 1 thread, {spent:.1f} s"}


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    ctx = mp.get_context("fork")
    per_step = 2 * cores
    with ctx.Pool(cores, initializer=_oracle_init, initargs=(1,)) as pool:
        for w in range(max(args.warmup, 1)):
            pool.map(_oracle_eval, range(per_step))
        times = []
        for k in range(args.steps):
            t = time.perf_counter()
            pool.map(_oracle_eval, range(10_000 + k * per_step, 10_000 + (k + 1) * per_step))
            times.append(time.perf_counter() - t)
    total = sum(times)
    value = per_step * args.steps / total
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": dict(workload_desc(1, per_step), points_per_step=per_step, parallelism=f"{cores} host processes"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{per_step} cfg1 points per step over {cores} worker processes "
                                   "(EMPAR-style pool, runner.py:305-312), numpy/scipy oracle port"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    run = build_ours(args.config, args.points, local, seed0=1_000_000 * (rank + 1), dist=dist if world > 1 else None,
                     rank=rank, world=world)
    ev, x_h, m_h, units, sc = run.ev, run.x_h, run.m_h, run.units, run.sharded
    x = torch.from_numpy(x_h).to(dev)
    mult = torch.from_numpy(m_h).to(dev)
    out = ev.alloc()
    # a dedicated (non-default) stream: the kernels, the events and the copies all live on it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    from paper_2203_10587_b200 import _lib as L

    def step():
        if sc is None:
            ev.eval_device(x, mult, 1.0, L.ALL, out=out, stream=sptr)
        else:
            sc.evaluate(x, mult, 1.0, L.ALL, out=out, stream=sptr)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches0 = ev.launches()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        for k in range(args.steps):
            flush.zero_()
            starts[k].record(stream)
            step()
            ends[k].record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    gpu_launches = ev.launches() - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(sum(step_ms))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    # config 1: every rank evaluates its own batch (weak); composites: one composite over all ranks (strong)
    value = (units * world if sc is None else units) * args.steps / (total_ms / 1000.0)

    # roofline of the (single) evaluation kernel
    bytes_step = algorithmic_bytes(ev)
    if world > 1 and sc is not None:
        b = torch.tensor([float(bytes_step)], dtype=torch.float64, device=dev)
        dist.all_reduce(b)              # the whole composite's bytes
        bytes_step = int(b.item())
    kernel_ms = statistics.mean(step_ms)
    peaks_path = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured"
    else:
        peak, peak_src = FALLBACK_HBM_GBS, "fallback"
    achieved = bytes_step / (kernel_ms / 1000.0) / 1e9 / (world if sc is not None else 1)
    traffic = None
    tpath = os.path.join(HERE, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"cfg{args.config}")

    # end to end through the C ABI with pinned host buffers (H2D + eval + D2H per step)
    e2e = None
    if not args.no_e2e and sc is None:
        xp = torch.from_numpy(x_h).pin_memory()
        mp_ = torch.from_numpy(m_h).pin_memory()
        hout = {k: torch.empty(v.numel(), dtype=torch.float64).pin_memory() for k, v in out.items()}
        sizes = dict(obj=ev.n_obj, grad=ev.n, cons=ev.m, jac=ev.nnz_j, hess=ev.nnz_h)
        hout = {k: hout[k][:sizes[k]] for k in hout}
        for _ in range(2):
            ev.eval_host_ptrs(xp.data_ptr(), mp_.data_ptr(), 1.0, L.ALL, hout, stream=sptr)
        e_steps = max(3, min(args.steps, 10))
        es = [torch.cuda.Event(enable_timing=True) for _ in range(e_steps)]
        ee = [torch.cuda.Event(enable_timing=True) for _ in range(e_steps)]
        for k in range(e_steps):
            es[k].record(stream)
            ev.eval_host_ptrs(xp.data_ptr(), mp_.data_ptr(), 1.0, L.ALL, hout, stream=sptr)
            ee[k].record(stream)
        torch.cuda.synchronize(dev)
        e_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(es, ee))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": units * world * e_steps / (float(e_ms.item()) / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": 8 * (ev.n + ev.m),
               "d2h_bytes_per_step": 8 * sum(sizes.values()),
               "path": "acopf_batch_eval_host (C ABI) on pinned host buffers"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config == 1:
        cpu = cpu_baseline_single()

    if rank == 0:
        cfg = workload_desc(args.config, args.points)
        cfg.update(points_per_step=units if args.config == 1 else None, stages_per_step=len(ev.plans),
                   l2="256 MiB buffer written between timed steps (untimed)",
                   parallelism=(f"replicas x{world}" if sc is None else f"stage shards x{world} (NCCL halo + objective)")
                   if world > 1 else "single GPU",
                   algorithmic_bytes_per_step=bytes_step)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if (args.config == 1 or world == 1) else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, SURVEY §8d)",
            "config": cfg,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "acopf_tile_kernel (one launch per step; the generator/objective kernel "
                                   "runs concurrently on a forked stream and is included in kernel_ms)",
                         "kernel_ms": kernel_ms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(gpu_launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
