import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tga_gen as G
from paper_2506_17357_b200 import tga as T
inst, sols = G.population(1, n=200, n_sol=8)
gi = T.Instance.from_gen(inst)
mask = T.OP_ALL & ~T.OP_2OPT
db = T.Batch(gi, sols)
for _ in range(3):
    db.step_async(mask)
print(db.device_stats())
