import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import tga_gen as G
from paper_2506_17357_b200 import tga as T
inst, sols = G.population(0, n=200, n_sol=64)
gi = T.Instance.from_gen(inst)
b = T.Batch(gi, sols)
mask = T.OP_ALL & ~T.OP_2OPT
singles = [T.Solution(gi, s) for s in sols]
for it in range(6):
    b.eval(mask)
    status, moves = b.best_moves(mask)
    for k in range(len(sols)):
        singles[k].eval(mask)
        ok, mv = singles[k].best_move(mask)
        bm = moves[k]
        same = (ok == (status[k] == 0)) and (not ok or (mv.variant, mv.u, mv.v, mv.delta_i) == (bm.variant, bm.u, bm.v, bm.delta_i))
        if not same:
            print("it", it, "sol", k, "single", ok, mv.variant, mv.u, mv.v, mv.delta_i, "batch", status[k], bm.variant, bm.u, bm.v, bm.delta_i, bm.route_a, bm.pos_a, bm.route_b, bm.pos_b)
            bk = b.keys()[k]; sk = singles[k].keys()
            print(" keys differ at", [v for v in range(23) if bk[v] != sk[v]])
            sys.exit(1)
    try:
        b.apply(moves, apply_mask=(status == 0))
    except Exception as e:
        print("apply failed it", it, e); sys.exit(1)
    for k in range(len(sols)):
        if status[k] == 0:
            singles[k].apply(singles[k].best_move(mask)[1]) if False else None
    # re-sync singles with the batch routes
    singles = [T.Solution(gi, b.solution(k).routes()) for k in range(len(sols))]
print("batch consistent over 6 steps")
