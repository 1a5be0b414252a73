"""Workload for compute-sanitizer (tools/sanitize.sh): cfg1 and cfg2 in both score
modes through every entry point that launches kernels -- eval (fused fast path,
generic tile kernel incl. the reversed-segment variants, intra kernels, the north-star
sweep with its pipelined key resets), host step, device-resident steps (pick/update with
its grid barrier), reload, the candidate dump, a VRPSPDTW (pickup) instance and a small
population batch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tga_gen as G
from paper_2506_17357_b200 import tga as T

which = sys.argv[1] if len(sys.argv) > 1 else "all"
cases = []
if which in ("all", "cfg1"):
    cases += [("cfg1", *G.cvrp_small(0, spare=True))]
if which in ("all", "cfg2"):
    cases += [("cfg2", *G.config("cfg2"))]
if which in ("all", "vrptw"):
    cases += [("vrptw", *G.gh_like(1, n=120, kind="R2"))]
if which in ("all", "pd"):
    cases += [("pd", *G.jd_like(1, n=60))]
for name, inst, sol in cases:
    for mode in (0, 1):
        gi = T.Instance.from_gen(inst, score_mode=mode)
        mask = T.OP_ALL if inst.tw is None else T.OP_ALL & ~T.OP_2OPT
        a, b = T.Solution(gi, sol), T.Solution(gi, sol)
        a.eval(mask); a.keys()
        for _ in range(3):
            a.step(mask)
            b.step_async(mask)
        b.routes(); b.device_stats()
        a.reload(G.perturb(sol, 10, 1))
        a.eval(mask); a.best_move(mask)
        if inst.tw is None and mode == 0:   # the north-star sweep: an evaluation loop + device steps
            for _ in range(3):
                a.eval(T.OP_FUSED_NS)
            a.keys()
            b.step_async(T.OP_FUSED_NS); b.routes()
        if name != "cfg2":
            a.eval_dump(mask, 1); a.eval_dump(mask, 2)
        print(name, "mode", mode, "ok", flush=True)
if which in ("all", "ns2000"):
    inst, sol = G.config("ns2000")
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    for _ in range(3):
        gs.eval(T.OP_FUSED_NS)
    gs.keys(); gs.step_async(T.OP_FUSED_NS); gs.routes()
    print("ns2000 ok", flush=True)
if which in ("all", "batch"):
    inst, sols = G.population(0, n=60, n_sol=6)
    gi = T.Instance.from_gen(inst)
    bt = T.Batch(gi, sols)
    m = T.OP_ALL & ~T.OP_2OPT
    bt.eval(m); bt.keys()
    bt.step_async(m); bt.device_stats()
    print("batch ok", flush=True)
