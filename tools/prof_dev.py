"""ncu driver: device-resident steps (tga_descent) on a config."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--config", default="cfg2")
ap.add_argument("--granular", type=int, default=0)
ap.add_argument("--score", default="feasible", choices=["feasible", "penalised"])
a = ap.parse_args()
inst, sol = G.config(a.config)
gi = T.Instance.from_gen(inst, granular_theta=a.granular, score_mode=1 if a.score == "penalised" else 0)
gs = T.Solution(gi, sol)
mask = T.OP_STANDARD if inst.tw is None else T.OP_STANDARD & ~T.OP_2OPT
ms = gs.descent(mask, a.steps, timed=True)
print("step ms", [round(float(x), 4) for x in ms])
