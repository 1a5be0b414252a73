"""Short driver for ncu: N local-search steps on a config (no timing)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tga_gen as G
from paper_2506_17357_b200 import tga as T
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--config", default="cfg2")
ap.add_argument("--mask", default="all")
a = ap.parse_args()
inst, sol = G.config(a.config)
gi = T.Instance.from_gen(inst)
gs = T.Solution(gi, sol)
mask = {"all": T.OP_STANDARD if inst.tw is None else T.OP_STANDARD & ~T.OP_2OPT, "inter": T.OP_INTER,
        "ns": T.OP_FUSED_NS}[a.mask]
for _ in range(a.steps):
    gs.eval(mask & T.OP_INTER)
    gs.eval((mask & T.OP_INTRA) | T.EVAL_ACCUMULATE)
    ok, mv = gs.best_move(mask)
    if ok:
        gs.apply(mv)
print("done", T.launch_count())
