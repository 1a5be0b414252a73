#!/usr/bin/env python
"""Benchmark of the TGA hot path on B200 (BASELINE.json metric: moves evaluated/s
and full-neighbourhood sweeps/s per operator).

A *step* is one best-improvement local-search iteration of the whole hot path
 on the BASELINE config-2 workload (Uchoa X-like
CVRP, 1000 customers, X-n1001-k43 shape + one spare route), entirely on the
device (tga_step_async):
    eval of all 23 variants (one fused inter+intra kernel)
    -> on-device best key, decode and splice of the changed routes
    -> Dp row/column refresh + re-scan of the changed routes (same kernel).
value = canonical candidates evaluated / device time of K steps (one CUDA graph
between two CUDA events).  The working set of one solution is smaller than L2,
so R replicas of it are stepped round-robin (inputs larger than L2 between two
steps of a replica); each replica follows the config's own descent.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tga|reference]
                    [--config cfg2|ns2000|cfg3|cfg3r2|cfg4|cfg5] [--shard replicas|rows]
Under torchrun (N>1) every rank runs its own descents (weak scaling, no
collective) or, with --shard rows, one solution's candidate rows are split
over the ranks and the packed keys are MIN-allreduced over NCCL inside tga_eval.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "moves evaluated/sec and neighbourhood sweeps/sec per operator at 1/2/4/8 B200"
UNIT = "moves/s"

# Algorithmic lane-operations per candidate: the
# arithmetic of the variant's delta / load / feasibility formulas plus the
# select + min of the fused argmin, CVRP integer path.  Row- or column-only
# terms (removal gains, route loads) are amortised and not counted.
ALG_OPS = {1: 10, 2: 11, 3: 11, 4: 11, 5: 18, 6: 18, 7: 18, 8: 18, 9: 18, 10: 18,
           0: 5, 11: 5, 12: 5, 13: 5}
for _v in range(14, 23):
    ALG_OPS[_v] = 9
# VRPTW TW-I fast path (inter variants): the CVRP terms plus, per new route
# F + seg + B, the Eq. 4 check in T_V = 0 form: 2-opt* two
# (add + compare) checks, relocate one 6-op check per direction, swap/cross two.
ALG_OPS_TW = {1: 14, 2: 17, 3: 17, 4: 17, 5: 30, 6: 30, 7: 30, 8: 30, 9: 30, 10: 30}
# penalised CVRP (score = dD + w_Q dL_V, Eq. 16a): the validity compare replaces the
# capacity compare, plus two clamped excesses, their sum and the weighted add (4 ops)
ALG_OPS_PEN = {v: (ALG_OPS[v] + 4 if 1 <= v <= 10 else ALG_OPS[v]) for v in ALG_OPS}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["tga", "reference"], default="tga")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-op", action="store_true")
    ap.add_argument("--score", choices=["feasible", "penalised"], default="feasible",
                    help="score mode (DESIGN.md reading 4): feasible-only or penalised dD + w_Q dL_V (+ w_T dT_V)")
    ap.add_argument("--granular", type=int, default=0,
                    help="theta > 0: edge-based neighbourhood (ETGA, P:390-401) with granularity threshold theta")
    ap.add_argument("--no-north-star", action="store_true",
                    help="skip the north-star sweep block (ns2000 fused 2-opt*+relocate+swap) of the default line")
    ap.add_argument("--no-row-shard", action="store_true",
                    help="skip the row-sharded cfg4 sweep block (SURVEY §8(e)) of the default line")
    ap.add_argument("--shard", choices=["replicas", "rows"], default="replicas",
                    help="N>1: independent descents per GPU (weak scaling, no collective) or one "
                         "solution's candidate rows split over the GPUs (NCCL MIN-allreduce of the keys)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"tga_clocks_{os.getpid()}.csv")

    def start(self):
        if os.environ.get("TGA_BENCH_NO_SMI"):   # diagnostics only: measure the sampler's own interference
            return
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for nm, val in zip(names, p[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if sm:
            out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                   "samples": len(sm)}
        return out


# ------------------------------------------------------------------ helpers
def load_for(fn, seconds):
    """Run fn repeatedly for about `seconds` (keeps the GPU loaded while clocks are sampled)."""
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        fn()
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def ncu_for(config: str, candidates: float | None = None):
    """The committed ncu page of a config's dominant kernel (profiles/ncu_evidence.json): issue
    activity beside the roofline fraction (the ALG_OPS fraction credits sharing
    between variants), and executed lane instructions per candidate when the count is known."""
    p = os.path.join(ROOT, "profiles", "ncu_evidence.json")
    if not os.path.exists(p):
        return None
    e = json.load(open(p)).get(config)
    if not e:
        return None
    out = {"issue_active": e["issue_active_pct"] / 100.0, "warp_instructions": e["warp_instructions"],
           "ncu_us_cold": e["ncu_us"], "source": e["source"]}
    if candidates:
        out["lane_instructions_per_candidate"] = e["warp_instructions"] * 32.0 / candidates
    return out


def traffic_for(config: str):
    """DRAM bytes per launch of the dominant kernel from one committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get(config)
    return None


def reduce_(t, op):
    """all_reduce through the process group (CPU staging under gloo)."""
    import torch.distributed as dist
    if dist.get_backend() == "gloo":
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op)
    return t


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def oracle_sweep_rate(inst, routes, budget_s=12.0, rows_frac=None, row_offset=0):
    """CPU oracle (single thread, as it stands) on all variants; returns
    (moves/s, candidates, seconds, sweeps)."""
    import oracle as O
    orc = O.Oracle.from_instance(inst)
    variants = [v for v in range(23) if not (inst.tw is not None and v == 0)]
    Q = O.canonical_q(routes)
    tot_c, tot_t, sweeps = 0, 0.0, 0
    while True:
        for v in variants:
            if rows_frac:
                span = max(1, int(Q * rows_frac))
                lo = (row_offset * span) % Q
                t0 = time.perf_counter()
                m = orc.best_move(routes, v, u_lo=lo, u_hi=min(Q, lo + span))
            else:
                t0 = time.perf_counter()
                m = orc.best_move(routes, v)
            tot_t += time.perf_counter() - t0
            tot_c += m.n_candidates
        sweeps += 1
        if tot_t >= budget_s or rows_frac:
            break
    return tot_c / tot_t, tot_c, tot_t, sweeps


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_all_cores_rate(inst, routes, budget_s=6.0):
    """The CPU oracle as it stands, process-parallel over canonical u-row chunks on every
    host core (ctypes releases the GIL for each C call, one thread per core):
    full sweeps of every standard variant; returns (moves/s, candidates, seconds, sweeps, cores)."""
    import oracle as O
    from concurrent.futures import ThreadPoolExecutor
    orc = O.Oracle.from_instance(inst)
    variants = [v for v in range(23) if not (inst.tw is not None and v == 0)]
    Q = O.canonical_q(routes)
    ptr_cust = orc._csr(routes)
    nw = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    k = max(1, min(Q, 4 * nw))
    jobs = [(v, Q * i // k, Q * (i + 1) // k) for v in variants for i in range(k) if Q * (i + 1) // k > Q * i // k]
    tot_c, sweeps = 0, 0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=nw) as ex:
        while True:
            for m in ex.map(lambda j: orc.best_move(ptr_cust, j[0], u_lo=j[1], u_hi=j[2]), jobs):
                tot_c += m.n_candidates
            sweeps += 1
            if time.perf_counter() - t0 >= budget_s:
                break
    dt = time.perf_counter() - t0
    return tot_c / dt, tot_c, dt, sweeps, nw


def concat_sweep_rate(inst, routes, budget_s=5.0):
    """The fast CPU evaluator (cpu_baseline/: O(1) concatenation per candidate,
    the paper's MA-N-style CPU move evaluation), single thread, full
    sweeps of every variant; returns (moves/s, candidates, seconds, sweeps)."""
    import cpu_baseline as CB
    cb = CB.ConcatCPU.from_instance(inst)
    variants = [v for v in range(23) if not (inst.tw is not None and v == 0)]
    tot_c, tot_t, sweeps = 0, 0.0, 0
    while tot_t < budget_s:
        for v in variants:
            t0 = time.perf_counter()
            _, _, _, _, n = cb.best_move(routes, v)
            tot_t += time.perf_counter() - t0
            tot_c += n
        sweeps += 1
    return tot_c / tot_t, tot_c, tot_t, sweeps


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    ws, rank, _ = dist_init(args)
    if rank != 0:
        return 0
    import tga_gen as G
    inst, sol = G.config(args.config, args.seed)
    routes = sol.routes
    frac = 1.0 / 16
    for w in range(args.warmup):
        oracle_sweep_rate(inst, routes, rows_frac=frac, row_offset=w)
    tot_c, tot_t = 0, 0.0
    for k in range(args.steps):
        _, c, t, _ = oracle_sweep_rate(inst, routes, rows_frac=frac, row_offset=args.warmup + k)
        tot_c += c
        tot_t += t
    v = tot_c / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {G.CONFIGS.get(args.config, args.config)}; "
                               "all 23 move variants", "seed": args.seed},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"each step = all 23 variants over 1/16 of the canonical u-rows "
                                   f"(rotating), single-threaded C oracle rebuilding every neighbour"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ tga arm
def run_population(args, ws, rank, local, dev):
    """BASELINE config 5: 1024 VRPTW solutions (200 customers) evaluated as one
    batch; N ranks split the population (each owns 1024/N solutions, no
    collective).  A step = batch eval of every variant + best moves + apply."""
    import torch
    import tga_gen as G
    from paper_2506_17357_b200 import tga as T
    inst, sols = G.config("cfg5", args.seed)
    lo, hi = T.shard_range(len(sols), rank, ws)
    mine = sols[lo:hi]
    stream = torch.cuda.Stream(device=dev)
    gi = T.Instance.from_gen(inst)
    b = T.Batch(gi, mine)
    b.set_stream(stream)
    mask = T.OP_STANDARD & ~T.OP_2OPT

    def counts_total():
        return sum(int(sum(int(x) for v, x in enumerate(b.solution(k).counts()) if (mask >> v) & 1))
                   for k in range(len(mine)))

    def step():
        b.step_async(mask)   # batch eval + on-device pick/splice + update for every solution
        return 0

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    b.device_stats()
    K = min(args.steps, 50)
    cand = 0
    sampler = ClockSampler(local)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    # clock samples under load (see run_tga): batch evals of a copy of the population
    lb = T.Batch(gi, mine)
    lb.set_stream(stream)
    sampler.start()
    load_for(lambda: (lb.eval(mask), torch.cuda.synchronize(dev)), 0.4)
    b.device_stats()
    launches0 = T.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    applied = 0
    tot_ms = 0.0
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(K):
            step()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    tot_ms = e0.elapsed_time(e1)   # K batch steps back to back on the batch stream (CUDA events)
    launches = T.launch_count() - launches0
    dc, applied = b.device_stats()
    cand = int(dc.sum())
    load_for(lambda: (lb.eval(mask), torch.cuda.synchronize(dev)), 0.4)
    clocks = sampler.stop()
    del lb
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([tot_ms, float(cand)], device=dev, dtype=torch.float64)
        tm = t.clone()
        reduce_(tm, dist.ReduceOp.MAX)
        reduce_(t, dist.ReduceOp.SUM)
        tot_ms, cand = float(tm[0].item()), float(t[1].item())
    # ---- roofline of the batch inter-route kernel: CUDA events around K batch evals of
    # the inter variants alone (each = a 184 B/solution key memset + k_inter_fast_batch)
    inter_mask = mask & T.OP_INTER
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    b.eval(inter_mask)
    with torch.cuda.stream(stream):
        for a_, z_ in evs:
            a_.record(stream)
            b.eval(inter_mask)
            z_.record(stream)
    torch.cuda.synchronize(dev)
    kern_ms = statistics.mean(a_.elapsed_time(z_) for a_, z_ in evs)
    cnt_all = np.zeros(T.N_VARIANTS, dtype=np.float64)   # closed-form counts, every variant
    for k in range(len(mine)):
        cnt_all += b.solution(k).counts().astype(np.float64)
    ops = float(sum(cnt_all[v] * ALG_OPS_TW[v] for v in range(1, 11)))
    pk, pk_src = peaks()
    alu_peak = 148 * 128 * float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    roof = {"bound": "alu", "achieved": ops / (kern_ms / 1e3) / 1e12, "peak": alu_peak / 1e12, "unit": "Tops/s",
            "frac": ops / (kern_ms / 1e3) / alu_peak, "traffic": traffic_for("cfg5_batch"),
            "ncu": ncu_for("cfg5_batch", float(cnt_all[1:11].sum())),
            "peak_source": f"148 SM x 128 lanes x {float(pk.get('sm_max_mhz', 1965.0)):.0f} MHz ({pk_src} sm_max_mhz)",
            "kernel": "k_inter_fast_batch<16, TW, all-inter> (+ key memset), CUDA events around each batch eval",
            "kernel_ms": kern_ms, "candidates_per_launch": float(cnt_all[1:11].sum()), "alg_ops_per_launch": ops}
    # ---- e2e through the C ABI with host buffers: every step reloads every solution of
    # the population from host CSR arrays, evaluates the batch and reads the best moves back
    e2e_steps = 3
    host = [s_.flat() for s_ in mine]
    t0 = time.perf_counter()
    e2e_c = 0
    for _ in range(e2e_steps):
        for k, (ptr_, cust_) in enumerate(host):
            b.solution(k).reload((ptr_, cust_))
        b.eval(mask)
        b.best_moves(mask)
        e2e_c += int(sum(int(x) for v, x in enumerate(cnt_all) if (mask >> v) & 1))
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t0
    h2d = sum(4 * (len(p_) + len(c_)) for p_, c_ in host)
    e2e = {"value": e2e_c / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(len(mine) * T.N_VARIANTS * 8),
           "step": "per-solution tga_solution_reload from host CSR + tga_batch_eval + tga_batch_best_moves; "
                   "host wall clock"}
    if rank != 0:
        return 0
    line = {"metric": METRIC, "value": cand / (tot_ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": K,
            "warmup": max(args.warmup, 3), "ms_per_step": tot_ms / K, "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f32 (integer-valued)",
            "data": "synthetic",
            "config": {"workload": "cfg5: population 1024 x VRPTW 200 customers (R1_2-like, TW-I); "
                                   "step = batch eval of 22 variants + best moves + apply",
                       "solutions": len(sols), "parallelism": f"population split x{ws}"},
            "applied_moves": applied, "gpu_launches": int(launches), "clocks": clocks,
            "roofline": roof, "cpu_baseline": None,
            "e2e": e2e}
    print(json.dumps(line, default=float), flush=True)
    return 0


def run_tga(args):
    import torch
    ws, rank, local = dist_init(args)
    # TGA_BENCH_SHARED_GPU=1: a multi-rank smoke run on a box with fewer GPUs than
    # ranks (ranks share devices; the process group then uses gloo, since NCCL
    # refuses two ranks on one GPU).  Never set for a measurement.
    shared = os.environ.get("TGA_BENCH_SHARED_GPU") == "1"
    if shared:
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    if args.config == "cfg5":
        return run_population(args, ws, rank, local, dev)
    import tga_gen as G
    from paper_2506_17357_b200 import tga as T

    inst, sol0 = G.config(args.config, args.seed)
    stream = torch.cuda.Stream(device=dev)
    score_mode = 1 if args.score == "penalised" else 0
    gi = T.Instance.from_gen(inst, granular_theta=args.granular, score_mode=score_mode)
    row_shard = ws > 1 and args.shard == "rows"
    # Cold-cache timing without flush nodes: R replicas of the workload's
    # solution (separate device state each) stepped round-robin, so that
    # between two steps of one replica > 1.5 x L2 of other replicas' data has
    # streamed through (the timing rule's "inputs larger than L2").  Each
    # replica runs exactly the single-solution descent of the config.
    probe = T.Solution(gi, sol0)
    R_, N_, _, _ = probe.info()
    pitch = -(-(N_ + 2 * R_ + 8 * R_) // 128) * 128
    ws_bytes = pitch * pitch * 4 + pitch * 400
    l2 = getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 * 2 ** 20) or 126 * 2 ** 20
    n_rep = 1 if row_shard else max(1, min(64, -(-int(1.5 * l2) // ws_bytes)))
    probe.close()
    reps = [T.Solution(gi, sol0) for _ in range(n_rep)]
    for r in reps:
        r.set_stream(stream)
    gs = reps[0]
    if row_shard:
        import torch.distributed as dist
        obj = [T.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        gs.comm_init(rank, ws, obj[0])
    mask_all = T.OP_STANDARD if inst.tw is None else (T.OP_STANDARD & ~T.OP_2OPT)
    K = args.steps
    W = max(args.warmup, 3)

    def capture_steps(sols=None):
        sols = sols or reps
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for k in range(K):
                sols[k % len(sols)].step_async(mask_all)   # eval -> on-device pick/splice -> update
        return g

    def replay(g, timed=False):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            # a ~0.1 ms spin kernel ahead of the start event keeps the device busy while the host
            # submits the graph, so the device-timed region holds the K steps and not the host's
            # submission latency of a graph of 2K nodes (measured ~70 us per launch otherwise)
            torch.cuda._sleep(200_000)
            e0.record(stream)
            g.replay()
            e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1)

    # ---------------- warm-up: W device steps of every replica, then one replay of the graph.
    # Replica i takes i extra warm-up steps: identical replicas descending in lockstep would
    # all reach a full relayout (a route outgrowing its spare slots, ~20 us) at the same step,
    # so whether the timed window holds n_rep relayouts or none would depend on K; staggered,
    # the window sees them at the descent's own rate.
    for _ in range(W):
        for r in reps:
            r.step_async(mask_all)
    for i, r in enumerate(reps):
        for _ in range(i):
            r.step_async(mask_all)
    torch.cuda.synchronize(dev)
    launches0 = T.launch_count()
    g_val = capture_steps()
    launches = T.launch_count() - launches0      # kernels in the K captured steps
    replay(g_val)
    # clock-sampling load: the same steps on separate copies (the timed replicas' state
    # and keys stay untouched)
    load_reps = [T.Solution(gi, sol0) for _ in range(min(n_rep, 4))]
    for r in load_reps:
        r.set_stream(stream)
        r.step_async(mask_all)
    g_load = capture_steps(load_reps)
    replay(g_load)

    # ---------------- timed region: the K steps, one graph launch between two events
    for r in reps:
        r.device_stats()   # clear the on-device counters of the warm-up
    sampler = ClockSampler(local)
    # nvidia-smi samples every 100 ms but K steps take ~1 ms: the same graph is replayed
    # for ~0.4 s before and after the timed replay so the clock samples see the load
    sampler.start()
    load_for(lambda: replay(g_load), 0.4)
    for r in reps:
        r.device_stats()   # count only the timed replay's steps
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    tot_ms = replay(g_val, timed=True)
    dev_counts = np.zeros(T.N_VARIANTS, dtype=np.uint64)
    applied = 0
    for r in reps:
        c, a_ = r.device_stats()   # exact candidate counts of the K evaluated neighbourhoods
        dev_counts += c
        applied += a_
    # K-dependence of the line: the same steps as a graph of 2K, so the per-step
    # cost without any fixed cost of one graph replay is (T(2K) - T(K)) / K
    g_2k = None
    try:
        g_2k = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_2k, stream=stream):
            for k in range(2 * K):
                reps[k % len(reps)].step_async(mask_all)
        replay(g_2k)
        t2k_ms = replay(g_2k)
        step_marginal_ms = max(0.0, (t2k_ms - tot_ms) / K)
        graph_fixed_ms = max(0.0, tot_ms - K * step_marginal_ms)
    except Exception:   # pragma: no cover - capture failure must not cost the line
        step_marginal_ms, graph_fixed_ms = None, None
    del g_2k
    for r in reps:
        r.device_stats()
    load_for(lambda: replay(g_load), 0.4)
    clocks = sampler.stop()
    del g_load, load_reps
    cand_total = float(dev_counts.sum())
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        reduce_(t, dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        if not row_shard:   # independent descents: every rank's candidates count
            c = torch.tensor([cand_total], device=dev, dtype=torch.float64)
            reduce_(c, dist.ReduceOp.SUM)
            cand_total = float(c.item())
        dist.barrier()
    value = cand_total / (tot_ms / 1e3)

    # ---------------- kernel timing pass: the same K steps again with CUDA events
    # around every inter-route launch (recorded by the library on its stream).
    # Event nodes cost several us each inside a graph, so the value pass has none.
    for r in reps:
        r.enable_timing(True)
    g_ker = capture_steps()
    replay(g_ker)
    replay(g_ker)   # the library's events keep the records of this (second) replay
    inter_ms = []
    for r in reps:
        inter_ms.extend(float(x) for x in r.timings())
        r.enable_timing(False)
    for r in reps:
        r.device_stats()
    del g_ker

    # ---------------- roofline of the dominant kernel (inter-route eval), live events
    pk, pk_src = peaks()
    inter_avg_s = statistics.mean(inter_ms) / 1e3
    R, N, Qc, _ = gs.info()
    Qp = N + 2 * R
    # the CVRP fast path evaluates inter AND intra candidates in the one timed launch
    inter_sel = [v for v in range(23) if (mask_all >> v) & 1] if inst.tw is None else list(range(1, 11))
    shard_div = ws if row_shard else 1   # a launch evaluates 1/N of the rows when row-sharded
    inter_cands = float(sum(int(dev_counts[v]) for v in inter_sel)) / K / shard_div
    alg_bytes = (Qp * Qp / 2.0) * 4.0 / shard_div       # Dp upper triangle, int32
    if args.granular:
        # ETGA: per evaluated cell its 5x5 Dp neighbourhood and the two slot records
        # (+ the two time-window records) are gathered -- cells = customer pairs of the
        # edge mask + (customer, start depot) + (start depot, start depot) pairs
        # bytes GATHERED per cell (served by L2 or HBM): customer-pair cells read the ~20
        # distinct Dp values of all streams, cells with a start depot the 6 of 2-opt* and
        # relocate, both the two slot records (+ two time-window records)
        _, _, n_pairs = gi.info()
        recs = 2 * 80 + (2 * 64 if inst.tw is not None else 0)
        alg_bytes = (n_pairs * (20 * 4 + recs) + (N * R + R * (R - 1) / 2.0) * (6 * 4 + recs)) / shard_div
    ops_tab = (ALG_OPS_PEN if score_mode else ALG_OPS) if inst.tw is None else ALG_OPS_TW
    alg_ops = float(sum(int(dev_counts[v]) * ops_tab[v] for v in inter_sel)) / K / shard_div
    sm_mhz_peak = float(pk.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 128 * sm_mhz_peak * 1e6            # lane-ops/s (4 SMSP x 32 lanes x 1 issue/clk)
    hbm_peak = float(pk["hbm_gbs"]) * 1e9
    t_hbm = alg_bytes / hbm_peak
    t_alu = alg_ops / alu_peak
    # captures are per kernel: the edge-based and the penalised instantiations have their own
    traffic_key = ("etga_" if args.granular else "") + ("pen_" if score_mode else "") + args.config
    hbm_view = {"bound": "hbm", "achieved": alg_bytes / inter_avg_s / 1e9, "peak": hbm_peak / 1e9,
                "unit": "GB/s", "frac": (alg_bytes / inter_avg_s) / hbm_peak,
                "traffic": traffic_for(traffic_key), "peak_source": pk_src}
    alu_view = {"bound": "alu", "achieved": alg_ops / inter_avg_s / 1e12, "peak": alu_peak / 1e12,
                "unit": "Tops/s", "frac": (alg_ops / inter_avg_s) / alu_peak,
                "traffic": traffic_for(traffic_key),
                "peak_source": f"148 SM x 128 lanes x {sm_mhz_peak:.0f} MHz ({pk_src} sm_max_mhz)"}
    primary, alt = (alu_view, hbm_view) if t_alu >= t_hbm else (hbm_view, alu_view)
    if args.granular:
        kname = ("k_etga<" + ("TW, " if inst.tw is not None else "") + "all-inter> (+ k_slot_of after a host "
                 "layout): the edge-mask cells; intra variants in their own kernels")
    elif getattr(inst, "pickup", None) is not None:
        kname = ("k_inter<TW, all-inter> (VRPSPDTW: generic tile kernel with the Eq. 3a-d load records; "
                 "intra in its own kernel)")
    elif getattr(inst, "mode", None) == G.MODE_TWF:
        kname = ("k_inter<float, TW, all-inter> (TW-F: generic tile kernel, real-valued Eq. 4 times; "
                 "intra in its own kernel)")
    elif inst.tw is not None and score_mode:
        kname = "k_inter<TW, all-inter> (penalised VRPTW: generic tile kernel; intra in its own kernel)"
    elif inst.tw is None:
        kname = "k_inter_fast<all-inter> (CVRP: inter tiles + intra warps in one launch)"
    else:
        kname = "k_inter_fast<TW, all-inter> (VRPTW inter tiles; intra in its own kernel)"
    primary = dict(primary, kernel=kname + ", live CUDA events",
                   kernel_ms=inter_avg_s * 1e3, candidates_per_launch=inter_cands,
                   alg_bytes_per_launch=alg_bytes, alg_ops_per_launch=alg_ops)
    if not args.granular and shard_div == 1:
        primary["ncu"] = ncu_for(("pen_" if score_mode else "") + args.config, inter_cands)

    # ---------------- steady state per operator: CUDA-graph replay of back-to-back sweeps
    per_op = {}
    if not args.no_per_op and not args.granular:   # per-op counts are full-neighbourhood closed forms
        cnt_now = gs.counts().astype(np.int64)
        groups = dict(T.OPERATORS)
        groups["fused 2-opt*+relocate+swap"] = T.OP_FUSED_NS
        groups["all inter"] = T.OP_INTER
        groups["all"] = mask_all
        for name, m in groups.items():
            m &= mask_all | T.OP_REVERSED   # (the reversed-segment variants: per-operator lines only)
            if not m:
                continue
            G_SWEEPS, REPS = 20, 10
            gs.eval(m, stream)
            torch.cuda.synchronize(dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(G_SWEEPS):
                    gs.eval(m, stream)
            g.replay()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for _ in range(REPS):
                    g.replay()
                e1.record(stream)
            torch.cuda.synchronize(dev)
            per_sweep_s = e0.elapsed_time(e1) / 1e3 / (G_SWEEPS * REPS)
            c = int(sum(cnt_now[v] for v in range(T.N_VARIANTS) if (m >> v) & 1))
            per_op[name] = {"moves_per_s": c / per_sweep_s, "sweeps_per_s": 1.0 / per_sweep_s,
                            "us_per_sweep": per_sweep_s * 1e6, "candidates": c}
            del g

    # ---------------- row-sharded large sweep: cfg4's candidate rows over the
    # ranks, keys MIN-allreduced over NCCL inside every tga_eval (one collective per sweep)
    row_block = None
    if not args.no_row_shard and not row_shard and args.config != "cfg4":
        row_block = row_shard_block(args, ws, rank, local, dev, stream)
    ns_block = None
    if rank == 0 and not args.no_north_star and not row_shard:
        ns_block = north_star_block(args, dev, stream)
    if rank != 0:
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---------------- e2e through the C ABI with host buffers
    # each step: tga_solution_reload(host CSR routes of a new solution: H2D of
    # the routes + slot layout, Dp rebuild, full attribute scan) -> tga_eval(all)
    # -> tga_best_move (D2H of 8 B per variant); host wall clock, instance resident
    import tga_gen as G2
    e2e_sols = [G2.perturb(sol0, 20, 7000 + k).flat() for k in range(8)]
    e2e_steps = min(K, 40)
    s2 = T.Solution(gi, sol0)
    for k in range(3):
        s2.reload(e2e_sols[k % 8]); s2.eval(mask_all); s2.best_move(mask_all)
    torch.cuda.synchronize(dev)
    e2e_c = 0
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        s2.reload(e2e_sols[k % 8])
        s2.eval(mask_all)
        s2.best_move(mask_all)
        e2e_c += int(sum(int(x) for v, x in enumerate(s2.counts()) if (mask_all >> v) & 1))
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t0
    s2.close()
    ptr, cust = sol0.flat()
    h2d = 4 * (len(ptr) + len(cust)) + 5 * 4 * (N + 2 * R) + 8 * R
    e2e = {"value": e2e_c / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": 23 * 8,
           "step": "tga_solution_reload(host CSR routes) + tga_eval(all) + tga_best_move; "
                   "host wall clock, instance resident"}

    # ---------------- CPU oracle baseline (rank 0, N=1 only)
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        rate, c, t, sw = oracle_sweep_rate(inst, sol0.routes, budget_s=12.0)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{sw} full sweep(s) of all variants on state A ({c} candidates, {t:.1f} s), "
                         "single-threaded C oracle that rebuilds every neighbour route"}
    cpu_all = None
    if ws == 1 and not args.no_cpu_baseline:
        rate, c, t, sw, nw = oracle_all_cores_rate(inst, sol0.routes)
        cpu_all = {"value": rate, "unit": UNIT, "cores": nw, "kind": "oracle, all host cores",
                   "cpu": cpu_model(),
                   "sample": f"{sw} full sweep(s) of all variants on state A ({c} candidates, {t:.1f} s), the "
                             f"C oracle over canonical u-row chunks on {nw} threads (one per core)"}
        if cpu:
            cpu["cpu"] = cpu_model()
    cpu_fast = None
    if ws == 1 and not args.no_cpu_baseline:
        rate, c, t, sw = concat_sweep_rate(inst, sol0.routes, budget_s=5.0)
        cpu_fast = {"value": rate, "unit": UNIT, "cores": 1, "kind": "concat (O(1) per candidate, MA-N-style)",
                    "sample": f"{sw} full sweep(s) of all variants on state A ({c} candidates, {t:.1f} s), "
                              "single-threaded C, prefix/suffix records + Eq. 2-4 concatenation",
                    "gpu_over_cpu": None}

    sweeps_per_s = (K if row_shard else K * ws) / (tot_ms / 1e3)
    if cpu_fast:
        cpu_fast["gpu_over_cpu"] = value / cpu_fast["value"]   # cf. the paper's gamma_s, not the target
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K,
        "warmup": max(args.warmup, 3), "ms_per_step": tot_ms / K, "higher_is_better": True,
        "scaling": "strong" if row_shard else "weak", "vs_baseline": None,
        "dtype": ("int32" if inst.tw is None else
                  "f32 (real-valued TW-F distances and times)" if getattr(inst, "mode", None) == G.MODE_TWF else
                  "f32 (integer-valued TW-I times; int32 loads)"),
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {G.CONFIGS.get(args.config, args.config)}; "
                               + (f"edge-based neighbourhood (ETGA) theta={args.granular}; " if args.granular else "")
                               + ("penalised score dD + 10 dL_V (+ 10 dT_V); " if score_mode else "")
                               + "step = eval all variants + best move + apply",
                   "customers": N, "routes": R, "canonical_slots": Qc, "seed": args.seed,
                   "l2": (f"inputs larger than L2: {n_rep} replicas of the solution stepped round-robin "
                          f"({n_rep * ws_bytes / 2**20:.0f} MB of Dp + records vs {l2 / 2**20:.0f} MB L2)"
                          if n_rep > 1 else "Dp larger than L2"),
                   "replicas": n_rep,
                   "parallelism": (f"row-shard x{ws} (NCCL MIN-allreduce)" if row_shard else
                                   f"independent descents x{ws}" if ws > 1 else "1 GPU")},
        "sweeps_per_s": sweeps_per_s, "applied_moves": int(applied),
        "us_per_step_marginal": None if step_marginal_ms is None else step_marginal_ms * 1e3,
        "graph_launch_fixed_us": None if graph_fixed_ms is None else graph_fixed_ms * 1e3,
        "step": "tga_step_async: eval all variants -> on-device best move + splice -> update kernel; "
                "K steps captured in one CUDA graph, timed by two CUDA events",
        "kernel_timing": "second pass of the same K-step graph with CUDA events around every "
                         "inter-route launch (event nodes add several us per step)",
        "candidates_per_step": cand_total / K,
        "roofline": primary, "roofline_alt": alt,
        "per_operator_steady_state": per_op,
        "cpu_baseline": cpu, "cpu_baseline_all_cores": cpu_all, "cpu_baseline_concat": cpu_fast,
        "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
    }
    if row_block is not None:
        line["row_shard"] = row_block
    if ns_block is not None:
        line["north_star"] = ns_block
    print(json.dumps(line, default=float), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def north_star_block(args, dev, stream):
    """BASELINE.json north_star: the 2000-customer full 2-opt*+relocate+swap sweep
    (X-like CVRP, 2000 customers, 87 routes + spare; one solution, L2-warm steady
    state).  us_per_sweep: S back-to-back tga_eval(OP_FUSED_NS) -- key
    reset + the k_ns_sweep launch -- in one CUDA graph, CUDA events around R replays; the
    solution does not change between them, so each reset is a programmatic dependent of
    the previous sweep that releases the next sweep at once, and consecutive sweeps
    overlap (the tail of one with the loads and compute of the next).  kernel_us:
    accumulating evals (no reset, plain launches): one sweep at a time, launch gap
    included.
    Fractions: algorithmic lane-ops (ALG_OPS x exact candidate counts) over the
    148 x 128 x f_max issue peak, and the Dp upper triangle (Qp^2 / 2 int32) over the
    measured HBM copy bandwidth."""
    import torch
    import tga_gen as G
    from paper_2506_17357_b200 import tga as T
    inst, sol = G.config("ns2000", args.seed)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    gs.set_stream(stream)
    m = T.OP_FUSED_NS
    S, REPS = 20, 10

    def graph():
        for _ in range(3):
            gs.eval(m, stream)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(S):
                gs.eval(m, stream)
        g.replay()
        torch.cuda.synchronize(dev)
        return g

    g = graph()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(REPS):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    per_s = e0.elapsed_time(e1) / 1e3 / (S * REPS)
    del g
    # kernel-only stream: accumulating evals need no key reset, so the graph holds S
    # back-to-back k_ns_sweep launches (the same sweep; keys stay the minimum)
    gs.eval(m, stream)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(S):
            gs.eval(m | T.EVAL_ACCUMULATE, stream)
    g.replay()
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(REPS):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    kern_s = e0.elapsed_time(e1) / 1e3 / (S * REPS)
    del g
    c = gs.counts()
    R, N, Qc, _ = gs.info()
    cand = int(c[1]) + int(c[2]) + int(c[5])
    ops = float(int(c[1]) * ALG_OPS[1] + int(c[2]) * ALG_OPS[2] + int(c[5]) * ALG_OPS[5])
    Qp = N + 4 * R      # physical slots (2 spare slots per route)
    tri = Qp * Qp / 2.0 * 4.0
    pk, pk_src = peaks()
    alu_peak = 148 * 128 * float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    hbm_peak = float(pk["hbm_gbs"]) * 1e9
    gs.close()
    return {"workload": "ns2000: " + G.CONFIGS["ns2000"] + "; fused 2-opt*+relocate+swap sweep (k_ns_sweep)",
            "candidates": cand, "us_per_sweep": per_s * 1e6, "sweeps_per_s": 1.0 / per_s,
            "moves_per_s": cand / per_s, "kernel_us": kern_s * 1e6,
            "alu_frac_kernel": ops / kern_s / alu_peak, "alu_frac_sweep": ops / per_s / alu_peak,
            "hbm_frac_kernel": tri / kern_s / hbm_peak, "hbm_frac_sweep": tri / per_s / hbm_peak,
            "alg_ops": ops, "alg_bytes": tri, "alu_peak_tops": alu_peak / 1e12, "hbm_peak_gbs": hbm_peak / 1e9,
            "peak_source": pk_src, "target": "sweep >= 0.6 of the binding roofline (ALU issue: <= 4.6 us)",
            "target_met": bool(ops / per_s / alu_peak >= 0.6),
            "ncu": dict(ncu_for("ns_sweep_ns2000", cand) or {},
                        note="one cold sweep in isolation under ncu (no overlap with a neighbouring sweep)")}


def row_shard_block(args, ws, rank, local, dev, stream):
    """BASELINE config 4 (10^4 customers) with its candidate rows split over the N ranks
    (DESIGN.md §9): every rank evaluates 1/N of the tile plan, the 23
    packed keys are MIN-allreduced over NCCL inside tga_eval (ncclAllReduce on the
    solution's stream), all ranks hold identical keys.  Timed: S back-to-back sweeps
    (eval + allreduce) in one CUDA graph, CUDA events, max over ranks (strong scaling:
    the same neighbourhood at every N).  At N = 1 the same sweep without a collective."""
    import torch
    import tga_gen as G
    from paper_2506_17357_b200 import tga as T
    inst, sol = G.config("cfg4", args.seed)
    gi = T.Instance.from_gen(inst)
    gs = T.Solution(gi, sol)
    gs.set_stream(stream)
    if ws > 1:
        import torch.distributed as dist
        if os.environ.get("TGA_BENCH_SHARED_GPU") == "1":
            # ranks sharing one GPU (a smoke run of the multi-rank flow): NCCL refuses two ranks
            # on one device, so the shards run without the collective (keys per shard)
            gs.set_shard(rank, ws)
        else:
            obj = [T.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            gs.comm_init(rank, ws, obj[0])
    out = {"workload": "cfg4: " + G.CONFIGS["cfg4"] + f"; candidate rows over {ws} rank(s), keys "
                       "MIN-allreduced over NCCL per sweep" if ws > 1 else "cfg4 on 1 GPU (no collective)",
           "scaling": "strong", "n_gpus": ws}
    full = gs.counts()
    for name, m in (("all inter", T.OP_INTER), ("fused 2-opt*+relocate+swap", T.OP_FUSED_NS)):
        S, REPS = 10, 3
        for _ in range(3):
            gs.eval(m, stream)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(S):
                gs.eval(m, stream)
        g.replay()
        torch.cuda.synchronize(dev)
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(REPS):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        if ws > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            reduce_(t, dist.ReduceOp.MAX)
            ms = float(t.item())
        keys = gs.keys()
        per = ms / 1e3 / (S * REPS)
        cand = int(sum(int(full[v]) for v in range(23) if (m >> v) & 1))   # whole neighbourhood
        out[name] = {"us_per_sweep": per * 1e6, "sweeps_per_s": 1.0 / per, "moves_per_s": cand / per,
                     "candidates": cand, "keys_head": [hex(int(k)) for k in keys[1:3]]}
        del g
    gs.close()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_tga(args)


if __name__ == "__main__":
    sys.exit(main())
