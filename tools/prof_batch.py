"""ncu driver: device-resident batch steps of config 5 (population)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
inst, sols = G.config("cfg5")
b = T.Batch(T.Instance.from_gen(inst), sols)
mask = T.OP_STANDARD & ~T.OP_2OPT
for _ in range(3):
    b.step_async(mask)
torch.cuda.synchronize()
print("ok")
