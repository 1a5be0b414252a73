import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import tga_gen as G
from paper_2506_17357_b200 import tga as T
inst, sols = G.population(0, n=200, n_sol=64)
gi = T.Instance.from_gen(inst)
b = T.Batch(gi, sols)
mask = T.OP_ALL & ~T.OP_2OPT
for it in range(6):
    b.eval(mask)
    bk = b.keys()
    status, moves = b.best_moves(mask)
    for k in range(len(sols)):
        h = b.solution(k)
        fresh = T.Solution(gi, h.routes())
        fresh.eval(mask)
        fk = fresh.keys()
        h.eval(mask)
        hk = h.keys()
        if not (np.array_equal(fk, bk[k]) and np.array_equal(fk, hk)):
            print("it", it, "sol", k, "batch==fresh", np.array_equal(fk, bk[k]), "borrowed==fresh", np.array_equal(fk, hk))
            a1, a2 = h.attributes(), fresh.attributes()
            for key in a1:
                if not np.array_equal(a1[key], a2[key]): print("  attr differs", key, np.nonzero(a1[key] != a2[key])[0][:10])
            R, N, Q, g = h.info(); print("  info", R, N, Q, g)
            sys.exit(1)
    b.eval(mask)
    status, moves = b.best_moves(mask)
    print("it", it, "applying", int((status == 0).sum()), [ (moves[k].variant, moves[k].route_a, moves[k].route_b) for k in range(len(sols)) if status[k]==0][:5])
    b.apply(moves, apply_mask=(status == 0))
print("ok")
