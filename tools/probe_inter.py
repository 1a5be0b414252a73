"""Diagnostics: per-CTA timeline of the fused inter kernel (TGA_INTER_PROBE=1).
Stamps: 0 start, 1 intra done, 2 first tile data arrived, 3 end; 4-7 intra warp 0: start, slot loads, keys, REDUX done."""
import argparse, ctypes as C, os, sys
os.environ["TGA_INTER_PROBE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--cold", type=int, default=1)
a = ap.parse_args()
inst, sol = G.config(a.config)
gs = T.Solution(T.Instance.from_gen(inst), sol)
ap2 = None
mask = {"ns": T.OP_FUSED_NS, "all": T.OP_STANDARD}.get(os.environ.get("PROBE_MASK", "all"), T.OP_STANDARD)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
lib = T.lib()
lib.tga_debug_inter_probe.argtypes = [C.c_void_p, C.c_int32]
for rep in range(3):
    if a.cold:
        flush.fill_(rep)
    torch.cuda.synchronize()
    gs.eval(mask)
    torch.cuda.synchronize()
    buf = np.zeros(8 * 4096, dtype=np.uint64)
    lib.tga_debug_inter_probe(buf.ctypes.data, 8 * 4096)
    p = buf.reshape(4096, 8).astype(np.int64)
    t0 = p[:, 0][p[:, 0] > 0].min()
    live = p[:, 0] >= t0
    p = p[live] - t0
    n = len(p)
    q = lambda c: np.percentile(p[:, c], [0, 50, 90, 100]).round(0).astype(int).tolist()
    print(f"{a.config} rep {rep}: CTAs {n}; ns percentiles [min,50,90,max]: start {q(0)} intra {q(1)} "
          f"first-data {q(2)} end {q(3)}")
    w = p[:, 4] > -t0 // 2   # CTAs whose warp 0 ran an intra slot in this launch
    if w.any():
        iw = p[w]
        qq = lambda c: np.percentile(iw[:, c] - iw[:, 4], [0, 50, 90, 100]).round(0).astype(int).tolist()
        print("   intra warp (from its start): slot loads", qq(5), "keys", qq(6), "redux", qq(7), "n", int(w.sum()))
    if w.any() and (~w).any():
        pe = lambda m: np.percentile(p[m][:, 3], [50, 90, 100]).round(0).astype(int).tolist()
        print("   end ns [50,90,max]: CTAs with an intra unit", pe(w), " without", pe(~w))
    d = p[:, 3] - p[:, 2]
    print("   per-CTA tile phase ns [min,50,90,max]", np.percentile(d, [0, 50, 90, 100]).round(0).astype(int).tolist(),
          " wait for first data", np.percentile(p[:, 2] - p[:, 1], [0, 50, 90, 100]).round(0).astype(int).tolist())
