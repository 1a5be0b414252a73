"""Diagnostics: clock64 phase stamps of the device-resident pick/update kernel.
phases: 0 start, 1 counts done, 2 pick decoded, 3 splice written, 4 barrier 1,
5 rows + scans, 6 barrier 2, 7 columns (block 0's view; cycles at ~1.9 GHz)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import tga_gen as G
from paper_2506_17357_b200 import tga as T
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--steps", type=int, default=12)
ap.add_argument("--replicas", type=int, default=20)
a = ap.parse_args()
inst, sol = G.config(a.config)
gi = T.Instance.from_gen(inst)
mask = T.OP_STANDARD if inst.tw is None else T.OP_STANDARD & ~T.OP_2OPT
# --replicas R: R copies stepped round-robin (the bench's regime: each step's data was
# evicted by the other replicas' steps, the kernels' code stays in L2); 0 = one solution
# with a 256 MB L2 flush before every step (data AND code cold)
reps = [T.Solution(gi, sol) for _ in range(max(1, a.replicas))]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda") if a.replicas == 0 else None
for r in reps:
    r.descent(mask, 3)
torch.cuda.synchronize()
rows = []
tls = []
gs = reps[0]
for k in range(a.steps):
    for r in reps[1:]:   # the other replicas' steps stream their data through L2
        r.step_async(mask)
    gs.debug_probe(True)
    if flush is not None:
        flush.fill_(k)
    ms = gs.descent(mask, 1, timed=True)
    p = gs.debug_probe(False).astype(np.int64)
    d = [int(p[i] - p[0]) if p[i] else -1 for i in range(8)]
    rows.append(d)
    tl = p[16:16 + 1024].reshape(512, 2).astype(np.int64)
    nb = int((tl[:, 0] > 0).sum())
    if nb:
        t0 = tl[:nb, 0].min()
        st, en = tl[:nb, 0] - t0, tl[:nb, 1] - t0
        late = np.argsort(-en)[:6]
        tls.append((st, en))
        print("   blocks %d: start max %d ns, end median %d max %d ns; block0 end %d; latest:" % (nb, st.max(), np.median(en), en.max(), en[0]),
              [(int(b), int(st[b]), int(en[b])) for b in late])
    print(a.config, "step %.1f us" % (1e3 * float(ms[0])), "phase cycles", d,
          "| scan ends (ns after block 0 decode):", [int(p[12 + q]) - int(p[11]) if p[12 + q] else None for q in range(2)],
          "block 0 end:", int(p[14]) - int(p[11]) if p[14] else None,
          "| route-0 scan ns: passes", int(p[9]) - int(p[8]) if p[8] else None, "records", int(p[10]) - int(p[9]) if p[9] else None,
          "start", int(p[8]) - int(p[11]) if p[8] else None,
          "staged gathers", int(p[15]) - int(p[8]) if p[15] and p[8] else None)
r = np.array(rows[2:], dtype=np.float64)
print("median phase (us @1.965GHz):", [round(x / 1965.0, 2) for x in np.median(r, axis=0)])
