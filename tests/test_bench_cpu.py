"""CPU checks of bench.py's host side: the reference arm's JSON line (the driver runs
``bench.py --impl reference``) and the roofline numerator (SURVEY §8(d) algorithmic bytes)
of the two small configs, planned without a GPU."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    """--impl reference on cfg3: one JSON line with the contract's keys, its own
    cpu_baseline, a zero-copy e2e and the same workload config as the GPU arm."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "3", "--steps", "1",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["kind"] == "port"
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.workload_config(3)


@pytest.mark.parametrize("cfg,expected", [(3, 87_598_032)])
def test_algorithmic_bytes(cfg, expected):
    """The roofline numerator of cfg3: reads of x and the stage multipliers, the
    varying loads and the topology once; writes of every output value."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2203_10587_b200 import compose_multiperiod
    kind, args, _ = bench._composite_args(cfg)
    p, imap = compose_multiperiod(*args)
    assert bench.algorithmic_bytes(p.evaluator, len(imap.coupling_rows)) == expected
