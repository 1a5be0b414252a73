import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, ctypes
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
inst, sols = G.population(0, n=200, n_sol=64)
gi = T.Instance.from_gen(inst)
mask = T.OP_ALL & ~T.OP_2OPT
b = T.Batch(gi, sols)
def same(h):
    fresh = T.Solution(gi, h.routes())
    a1, a2 = h.attributes(), fresh.attributes()
    return [key for key in a1 if not np.array_equal(a1[key], a2[key])]
for it in range(6):
    b.eval(mask)
    status, moves = b.best_moves(mask)
    for k in range(len(sols)):
        if status[k] == 0:
            h = b.solution(k)
            before = h.routes()
            pre = same(h)
            h.apply(moves[k])
            torch.cuda.synchronize()
            d = same(h)
            if d:
                m = moves[k]
                print("it", it, "sol", k, "pre-diff", pre, "move", m.variant, m.route_a, m.pos_a, m.route_b, m.pos_b, "diff", d)
                print("route lens before", [len(r) for r in before])
                s = T.Solution(gi, before)
                mm = T.Move(); ctypes.memmove(ctypes.byref(mm), ctypes.byref(m), ctypes.sizeof(mm))
                mm.generation = s.info()[3]
                s.apply(mm); torch.cuda.synchronize()
                print("single replay diff", same(s), "routes equal", s.routes() == h.routes())
                sys.exit(1)
print("ok")
