"""bench.py's JSON-line contract (the driver parses it) and the committed evidence it cites.

CPU: the ncu / DRAM-traffic lookups return the committed captures for the configs the bench
lines name.  GPU: one short default-config run prints exactly one JSON line with every key
the driver reads (metric, value, roofline with its live kernel time, e2e with copied bytes,
gpu_launches, clocks)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_committed_evidence_lookups():
    import bench
    for cfg in ("cfg2", "cfg3", "cfg3r2", "cfg4", "ns2000", "jd", "cfg3f", "pen_cfg2", "cfg5_batch"):
        e = bench.ncu_for(cfg, 1.0e6)
        assert e is not None, cfg
        assert 0.0 < e["issue_active"] <= 1.0 and e["warp_instructions"] > 0
        assert os.path.exists(os.path.join(ROOT, e["source"])), e["source"]
        assert e["lane_instructions_per_candidate"] > 0
    for cfg in ("cfg2", "cfg4", "cfg5_batch", "pen_cfg2", "jd"):
        t = bench.traffic_for(cfg)
        assert isinstance(t, int) and t > 0, cfg
    assert bench.ncu_for("no-such-config") is None


@pytest.mark.gpu
def test_default_line_contract():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                          "--no-cpu-baseline", "--no-per-op", "--no-north-star", "--no-row-shard"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 5 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "kernel_ms"):
        assert k in r, k
    assert 0.0 < r["frac"] < 1.0 and r["kernel_ms"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert "workload" in d["config"]
