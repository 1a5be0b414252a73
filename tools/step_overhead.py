"""Diagnostics: where the device step's time goes outside the kernels.
A: descent with per-step events, inter-kernel events and an L2 flush (bench.py's timed region)
B: per-step events + flush, no inter-kernel events
C: K steps in one graph, no events inside, no flush (warm L2), total / K
D: K steps round-robin over R replicas (working set > L2), stream-captured, total / K"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--replicas", type=int, default=24)
a = ap.parse_args()
inst, sol = G.config(a.config)
gi = T.Instance.from_gen(inst)
mask = T.OP_STANDARD if inst.tw is None else T.OP_STANDARD & ~T.OP_2OPT
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
K = a.steps

gs = T.Solution(gi, sol)
gs.descent(mask, 3); torch.cuda.synchronize()
gs.enable_timing(True)
ms = gs.descent(mask, K, l2_flush=flush, timed=True)
inter = gs.timings(); gs.enable_timing(False)
print("A events+inter events+flush: step %.2f us, inter %.2f us" % (1e3 * np.mean(ms[2:]), 1e3 * np.mean(inter[2:])))
gs = T.Solution(gi, sol)
gs.descent(mask, 3); torch.cuda.synchronize()
ms = gs.descent(mask, K, l2_flush=flush, timed=True)
print("B events+flush:              step %.2f us" % (1e3 * np.mean(ms[2:])))
gs = T.Solution(gi, sol)
gs.descent(mask, 3); torch.cuda.synchronize()
t0 = time.perf_counter(); gs.descent(mask, K); torch.cuda.synchronize(); t1 = time.perf_counter()
print("C one graph, warm, no events: step %.2f us (host wall incl. graph build)" % (1e6 * (t1 - t0) / K))
# D: replicas on one stream, captured into one graph, timed by two events
st = torch.cuda.Stream()
reps = [T.Solution(gi, G.perturb(sol, 10, 100 + k)) for k in range(a.replicas)]
for r in reps:
    r.set_stream(st)
for r in reps:
    r.step_async(mask)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for k in range(K):
        reps[k % a.replicas].step_async(mask)
g.replay(); torch.cuda.synchronize()
def timed(graph):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        graph.replay()
        e1.record(st)
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / K
print("D %d replicas round-robin, one graph: step %.2f us" % (a.replicas, timed(g)))
for r in reps:
    r.enable_timing(True)
g3 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g3, stream=st):
    for k in range(K):
        reps[k % a.replicas].step_async(mask)
with torch.cuda.stream(st):
    g3.replay()
torch.cuda.synchronize()
for r in reps:
    r.timings()
t = timed(g3)
inter = np.concatenate([r.timings() for r in reps])
print("F replicas + inter-kernel events: step %.2f us, inter %.2f us (n=%d)" % (t, 1e3 * np.mean(inter), len(inter)))
