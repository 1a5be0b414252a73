import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tga_gen as G
from paper_2506_17357_b200 import tga as T
inst, sol = G.cvrp_small(0, spare=True)
gi = T.Instance.from_gen(inst)
gs = T.Solution(gi, sol)
print("loaded", gs.info(), flush=True)
print("cost", gs.cost(), flush=True)
for name, m in [("intra", T.OP_INTRA), ("2opt*", T.OP_2OPT_STAR), ("inter", T.OP_INTER)]:
    gs.eval(m)
    print(name, [hex(int(k)) for k in gs.keys()][:12], flush=True)
