"""ncu driver: repeated tga_eval of one operator mask on a fixed solution (steady-state sweeps)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=6)
ap.add_argument("--config", default="ns2000")
ap.add_argument("--mask", default="ns", help="ns | all | inter | hex mask")
ap.add_argument("--score", type=int, default=0)
a = ap.parse_args()
inst, sol = G.config(a.config)
gs = T.Solution(T.Instance.from_gen(inst, score_mode=a.score), sol)
m = {"ns": T.OP_FUSED_NS, "all": T.OP_STANDARD if inst.tw is None else T.OP_STANDARD & ~T.OP_2OPT,
     "inter": T.OP_INTER}.get(a.mask) or int(a.mask, 16)
for _ in range(a.reps):
    gs.eval(m)
torch.cuda.synchronize()
print("keys", [hex(int(k)) for k in gs.keys()[:11]])
