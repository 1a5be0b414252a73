"""Per-step device times of a device-resident descent (L2 flushed before every step):
median, percentiles and the outlier steps (full relayouts show up here)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3r2")
ap.add_argument("--steps", type=int, default=300)
ap.add_argument("--slack", type=int, default=0)
ap.add_argument("--show", type=int, default=0, help="print the first SHOW step times")
a = ap.parse_args()
inst, sol = G.config(a.config)
gi = T.Instance.from_gen(inst, slack=a.slack) if a.slack else T.Instance.from_gen(inst)
gs = T.Solution(gi, sol)
mask = T.OP_STANDARD if inst.tw is None else T.OP_STANDARD & ~T.OP_2OPT
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
ms = gs.descent(mask, a.steps, l2_flush=flush, timed=True) * 1e3
_, applied = gs.device_stats()
med = float(np.median(ms))
out = [(i, round(float(m), 1)) for i, m in enumerate(ms) if m > 2 * med]
print(a.config, "slack", a.slack or "default", "steps", a.steps, "applied", applied,
      "us/step median %.1f p10 %.1f p90 %.1f mean %.1f" % (med, np.percentile(ms, 10), np.percentile(ms, 90), ms.mean()),
      "outliers (step, us):", out[:20], "n_out", len(out), "share of time %.2f" % (sum(m for _, m in out) / ms.sum()))
if a.show:
    print("first steps (us):", [round(float(m), 1) for m in ms[:a.show]])
