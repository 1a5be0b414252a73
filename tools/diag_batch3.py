import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
inst, sols = G.population(0, n=200, n_sol=64)
gi = T.Instance.from_gen(inst)
mask = T.OP_ALL & ~T.OP_2OPT
# A: single solutions, many steps, check vs fresh every step
bad = 0
for k in [30, 5, 17]:
    s = T.Solution(gi, sols[k])
    for it in range(12):
        ok, mv = s.step(mask)
        fresh = T.Solution(gi, s.routes())
        a1, a2 = s.attributes(), fresh.attributes()
        diff = [key for key in a1 if not np.array_equal(a1[key], a2[key])]
        if diff:
            print("single sol", k, "it", it, "move", mv.variant, mv.route_a, mv.pos_a, mv.route_b, mv.pos_b, "diff", diff); bad += 1; break
        if not ok: break
print("single done, bad", bad)
# B: batch with a sync after every apply
b = T.Batch(gi, sols)
for it in range(6):
    b.eval(mask)
    status, moves = b.best_moves(mask)
    for k in range(len(sols)):
        if status[k] == 0:
            h = b.solution(k)
            h.apply(moves[k])
            torch.cuda.synchronize()
            fresh = T.Solution(gi, h.routes())
            a1, a2 = h.attributes(), fresh.attributes()
            diff = [key for key in a1 if not np.array_equal(a1[key], a2[key])]
            if diff:
                m = moves[k]
                print("batch-sync it", it, "sol", k, "move", m.variant, m.route_a, m.pos_a, m.route_b, m.pos_b, "diff", diff)
                sys.exit(1)
print("batch-sync ok")
