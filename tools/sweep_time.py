"""Steady-state time of one operator sweep: G back-to-back tga_eval of a mask captured
in a CUDA graph, replayed R times between two CUDA events (as bench.py's per-operator
block), plus the same with CUDA events around every sweep inside the graph."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="ns2000")
ap.add_argument("--mask", default="ns")
ap.add_argument("--sweeps", type=int, default=20)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
inst, sol = G.config(a.config)
gs = T.Solution(T.Instance.from_gen(inst), sol)
m = {"ns": T.OP_FUSED_NS, "inter": T.OP_INTER, "all": T.OP_STANDARD}.get(a.mask) or int(a.mask, 16)
st = torch.cuda.Stream()
gs.set_stream(st)
gs.eval(m, st)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for _ in range(a.sweeps):
        gs.eval(m, st)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    e0.record(st)
    for _ in range(a.reps):
        g.replay()
    e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (a.sweeps * a.reps)
c = gs.counts()
cand = sum(int(c[v]) for v in range(23) if (m >> v) & 1)
print(f"{a.config} mask {m:#x}: {us:.2f} us/sweep, {cand / us / 1e6:.3g} T moves/s ({cand} candidates)")
