"""Diagnostics: per-CTA timeline of the north-star sweep kernel (TGA_NS_PROBE=1).
Stamps: 0 start, 1 first tile's data arrived, 2 tiles done, 3 end (after the fused argmin)."""
import argparse, ctypes as C, os, sys
os.environ["TGA_NS_PROBE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="ns2000")
ap.add_argument("--cold", type=int, default=0)
a = ap.parse_args()
inst, sol = G.config(a.config)
gs = T.Solution(T.Instance.from_gen(inst), sol)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
lib = T.lib()
lib.tga_debug_ns_probe.argtypes = [C.c_void_p, C.c_int32]
for rep in range(4):
    if a.cold:
        flush.fill_(rep)
    torch.cuda.synchronize()
    gs.eval(T.OP_FUSED_NS)
    torch.cuda.synchronize()
    buf = np.zeros(4 * 4096, dtype=np.uint64)
    lib.tga_debug_ns_probe(buf.ctypes.data, 4 * 4096)
    p = buf.reshape(4096, 4).astype(np.int64)
    t0 = p[:, 0][p[:, 0] > 0].min()
    p = p[p[:, 0] >= t0] - t0
    q = lambda c: np.percentile(p[:, c], [0, 50, 90, 100]).round(0).astype(int).tolist()
    print(f"{a.config} rep {rep} cold={a.cold}: CTAs {len(p)}; ns [min,50,90,max]: start {q(0)} data {q(1)} "
          f"tiles-done {q(2)} end {q(3)}; tile phase {np.percentile(p[:, 2] - p[:, 1], [0, 50, 90, 100]).round(0).astype(int).tolist()}")
