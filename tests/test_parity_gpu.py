"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element on the same seeded inputs.

Bar (BASELINE.json north_star): integer distances (CVRP nint, VRPTW integer
tenths) -> best-move keys bit-exact per variant (score and canonical index);
real-valued time windows -> scores within 1e-4 relative and identical masks
outside the ambiguity band (reading 13).
"""
import numpy as np
import pytest

import oracle as O
import tga_gen as G
from tests import brute
from tests import par_oracle
from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu

if gpu_available():
    from paper_2506_17357_b200 import tga as T
else:  # pragma: no cover - collected on CPU boxes, skipped by the marker filter
    T = None


def _need_gpu():
    if not gpu_available():
        pytest.skip("no CUDA device")


INTER = [1, 2, 3, 4, 5, 6, 7, 8, 9, 10]
INTRA_TW = list(range(11, 23))
ALLV = list(range(23))


def oracle_key(m: O.Move, Q: int):
    if not m.found:
        return None
    return (m.score, m.u * Q + m.v)


def gpu_keys(sol, integer=True):
    ks = sol.keys()
    out = {}
    for v in range(T.N_VARIANTS):
        k = int(ks[v])
        out[v] = None if k == 0xFFFFFFFFFFFFFFFF else T.decode_key(k, integer)
    return out


def check_exact(inst, routes, variants, mode=0, label=""):
    orc = O.Oracle.from_instance(inst)
    gi = T.Instance.from_gen(inst, score_mode=mode)
    gs = T.Solution(gi, routes)
    mask = sum(1 << v for v in variants)
    gs.eval(mask)
    got = gpu_keys(gs, integer=True)
    Q = O.canonical_q(routes)
    for v in variants:
        m = orc.best_move(routes, v, mode=mode)
        exp = oracle_key(m, Q)
        assert got[v] == exp, f"{label} variant {v} ({T.VARIANT_NAMES[v]}): gpu {got[v]} oracle {exp}"
    return gi, gs, orc


# ---------------------------------------------------------------- cfg1: 20 customers, 4 routes
@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("spare", [False, True])
@pytest.mark.parametrize("mode", [0, 1])
def test_cfg1_all_variants_exact(seed, spare, mode):
    _need_gpu()
    inst, sol = G.cvrp_small(seed, spare=spare)
    check_exact(inst, sol, ALLV, mode, f"cfg1 s{seed}")


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("spare", [False, True])
@pytest.mark.parametrize("mode", [0, 1])
def test_cfg1_gpu_vs_brute_force(seed, spare, mode):
    """BASELINE config 1 as its row states it: "full 2-opt/2-opt*/relocate/swap
    sweep vs brute force" -- the GPU keys of every variant against the
    independent brute-force generator (tests/brute.py, no oracle involved):
    lowest (score, canonical index) of every neighbour it builds by list surgery."""
    _need_gpu()
    inst, sol = G.cvrp_small(seed, spare=spare)
    gs = T.Solution(T.Instance.from_gen(inst, score_mode=mode), sol)
    gs.eval(T.OP_STANDARD)
    got = gpu_keys(gs, integer=True)
    Q = O.canonical_q(sol)
    d, dem = inst.dist.tolist(), inst.demand.tolist()
    for op, n1, n2, var in BRUTE_OPS:
        exp = brute.best(brute.scores(d, dem, None, inst.capacity, sol.routes, op, n1, n2, mode,
                                      with_index=True), Q)
        assert got[var] == exp, (seed, spare, mode, op, n1, n2, got[var], exp)


BRUTE_OPS = ([("2opt*", 1, 1, 1), ("2opt", 1, 1, 0)]
             + [("relocate", n, 1, v) for n, v in O.V_RELOC.items()]
             + [("swap", a, b, v) for (a, b), v in O.V_SWAP.items()]
             + [("intra_relocate", n, 1, v) for n, v in O.V_IRELOC.items()]
             + [("intra_swap", a, b, v) for (a, b), v in O.V_ISWAP.items()])


@pytest.mark.parametrize("seed", range(12))
def test_cfg1_random_partitions_exact(seed):
    """Feasible and infeasible random partitions, ragged + empty routes."""
    _need_gpu()
    inst, _ = G.cvrp_small(seed)
    sol = G.random_partition(20, 3 + seed % 4, 900 + seed, allow_empty=True)
    for mode in (0, 1):
        check_exact(inst, sol, ALLV, mode, f"cfg1-rand s{seed}")


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("mode", [0, 1])
def test_small_vrptw_exact(seed, mode):
    """TW-I (integer tenths in fp32 on the GPU): bit-exact keys."""
    _need_gpu()
    inst, sol = G.gh_like(seed, n=60, kind="R1" if seed % 2 == 0 else "R2")
    if seed >= 3:
        sol = G.perturb(sol, 12, seed)  # infeasible states too
    check_exact(inst, sol, INTER + INTRA_TW, mode, f"vrptw s{seed}")


def test_long_routes_chunked_scan():
    """Routes longer than one warp (L > 32) exercise the scan carries."""
    _need_gpu()
    inst, sol = G.gh_like(5, n=300, kind="R2")
    long_sol = G.Solution([sum(sol.routes[:4], [])] + sol.routes[4:])
    for mode in (0, 1):
        check_exact(inst, long_sol, INTER + INTRA_TW, mode, "long")
    inst2, sol2 = G.x_like(3, n=300, target_routes=3)
    check_exact(inst2, sol2, ALLV, 1, "long-cvrp")


# ---------------------------------------------------------------- attributes (a2)
@pytest.mark.parametrize("name", ["cfg1", "vrptw"])
def test_attribute_rebuild_matches_full_rebuild(name):
    _need_gpu()
    if name == "cfg1":
        inst, sol = G.cvrp_small(1, spare=True)
    else:
        inst, sol = G.gh_like(2, n=200, kind="R2")
        sol = G.perturb(sol, 30, 5)
    orc = O.Oracle.from_instance(inst)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    a, b = gs.attributes(), orc.attributes(sol)
    for k in ("pre_L", "suf_L", "pre_D", "suf_D", "pre_TV", "suf_TV"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    if inst.tw is not None:
        np.testing.assert_array_equal(a["start"], b["start"])
    D, LV, TV = orc.cost(sol)
    di, df, le, te = gs.cost()
    assert di == D and le == LV and te == TV


def test_counts_match_oracle_enumeration():
    _need_gpu()
    inst, _ = G.cvrp_small(2)
    sol = G.random_partition(20, 5, 77, allow_empty=True)
    orc = O.Oracle.from_instance(inst)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    c = gs.counts()
    for v in ALLV:
        assert int(c[v]) == orc.best_move(sol, v).n_candidates


# ---------------------------------------------------------------- lockstep trajectories (a7, a8)
@pytest.mark.parametrize("name", ["cvrp", "vrptw"])
def test_lockstep_descent(name):
    """Identical search trajectories: best move over all variants,
    applied on both sides, keys equal at every step; delta == cost change."""
    _need_gpu()
    if name == "cvrp":
        inst, sol = G.x_like(4, n=150, target_routes=8)
        variants = ALLV
    else:
        inst, sol = G.gh_like(4, n=150, kind="R2")
        variants = INTER + INTRA_TW
    orc = O.Oracle.from_instance(inst)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    mask = sum(1 << v for v in variants)
    routes = [list(r) for r in sol.routes]
    D0 = orc.cost(routes)[0]
    for step in range(25):
        gs.eval(mask)
        improving, mv = gs.best_move(mask)
        ob = orc.best_over(routes, variants)
        if ob is None or not ob.score < 0:
            assert not improving
            break
        assert improving
        Q = O.canonical_q(routes)
        assert (mv.variant, mv.delta_i, mv.u, mv.v) == (ob.variant, ob.score, ob.u, ob.v), step
        assert (mv.route_a, mv.pos_a, mv.route_b, mv.pos_b) == (ob.route_a, ob.pos_a, ob.route_b, ob.pos_b)
        gs.apply(mv)
        routes = orc.apply(routes, ob.variant, ob.route_a, ob.pos_a, ob.route_b, ob.pos_b)
        assert gs.routes() == routes
        D1 = orc.cost(routes)[0]
        assert D1 - D0 == mv.delta_i
        assert gs.cost()[0] == D1
        D0 = D1
    # the incremental state equals a fresh load of the final routes
    fresh = T.Solution(gs.inst, routes)
    fresh.eval(mask)
    gs.eval(mask)
    np.testing.assert_array_equal(fresh.keys(), gs.keys())


def test_stale_move_rejected():
    _need_gpu()
    inst, sol = G.x_like(5, n=80, target_routes=5)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    gs.eval(T.OP_INTER)
    ok, mv = gs.best_move(T.OP_INTER)
    assert ok
    gs.apply(mv)
    with pytest.raises(T.TgaError) as e:
        gs.apply(mv)
    assert e.value.code == -3


def test_two_opt_with_time_windows_unsupported():
    _need_gpu()
    inst, sol = G.gh_like(0, n=40, kind="R1")
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    with pytest.raises(T.TgaError) as e:
        gs.eval(T.OP_2OPT)
    assert e.value.code == -4


# ---------------------------------------------------------------- sharding (a6)
@pytest.mark.parametrize("n_shards", [2, 3, 8])
def test_virtual_shards_equal_unsharded(n_shards):
    """Row shards evaluated one after another, keys min-combined on the host:
    equal to the unsharded keys (the exact combine of the NCCL allreduce)."""
    _need_gpu()
    inst, sol = G.x_like(6, n=400, target_routes=17)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    gs.eval(T.OP_STANDARD)
    full = gs.keys()
    comb = np.full(T.N_VARIANTS, np.iinfo(np.uint64).max, dtype=np.uint64)
    for s in range(n_shards):
        gs.set_shard(s, n_shards)
        gs.eval(T.OP_STANDARD)
        comb = np.minimum(comb, gs.keys())
    np.testing.assert_array_equal(comb, full)


# ---------------------------------------------------------------- full-size configs
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg3r2"])
def test_full_size_configs_exact(name):
    """BASELINE configs 2-3 at full size, the launch configuration bench.py
    times: every variant's key vs the oracle's full enumeration."""
    _need_gpu()
    inst, sol = G.config(name)
    variants = ALLV if inst.tw is None else INTER + INTRA_TW
    check_exact(inst, sol, variants, 0, name)


def test_cfg2_state_b_after_descent():
    """'State B' (after accepted moves) at full size: sampled candidates
    scored one by one by the oracle agree with the GPU keys."""
    _need_gpu()
    inst, sol = G.config("cfg2")
    orc = O.Oracle.from_instance(inst)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    for _ in range(30):
        gs.eval(T.OP_STANDARD)
        ok, mv = gs.best_move(T.OP_STANDARD)
        if not ok:
            break
        gs.apply(mv)
    routes = gs.routes()
    check_exact(inst, routes, ALLV, 0, "cfg2-B")


# ---------------------------------------------------------------- TW-F (real-valued)
def test_real_valued_time_windows_tolerance():
    """TW-F: fp32 GPU vs fp64 oracle.  The GPU's best score within 1e-4 relative of the
    oracle's; the candidate it picks is, in the oracle's enumeration, feasible and
    within the same bar of the optimum; when the oracle's best is separated from the
    runner-up by more than twice the bar, the index must match (readings 13, 17)."""
    _need_gpu()
    inst, sol = G.gh_like(1, n=200, kind="R2", mode="twf")
    orc = O.Oracle.from_instance(inst)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    mask = sum(1 << v for v in INTER + INTRA_TW)
    gs.eval(mask)
    got = gpu_keys(gs, integer=False)
    Q = O.canonical_q(sol)
    for v in INTER + INTRA_TW:
        sc, us, vs, best = orc.enumerate(sol, v)
        if not best.found:
            assert got[v] is None
            continue
        assert got[v] is not None
        s_gpu, idx_gpu = got[v]
        tol = 1e-4 * max(1.0, abs(best.score))          # the north star's 1e-4 relative bar
        assert abs(s_gpu - best.score) <= tol, (v, s_gpu, best.score)
        # the GPU's chosen candidate, looked up in the oracle's enumeration: feasible, and
        # scored by the oracle within the bar of the optimum
        at = np.nonzero((us.astype(np.int64) * Q + vs) == idx_gpu)[0]
        assert len(at) == 1, (v, idx_gpu)
        assert np.isfinite(sc[at[0]]) and abs(sc[at[0]] - best.score) <= tol, (v, sc[at[0]], best.score)
        order = np.sort(sc[np.isfinite(sc)])
        if len(order) > 1 and order[1] - order[0] > 2 * tol:
            assert idx_gpu == best.u * Q + best.v, v


# ---------------------------------------------------------------- step / reload / timing ABI
def test_step_reload_and_timing():
    """tga_step == eval + best_move + apply; tga_solution_reload == a fresh load;
    live timings are recorded for the inter-route launch."""
    _need_gpu()
    inst, sol = G.x_like(8, n=200, target_routes=9)
    gi = T.Instance.from_gen(inst)
    a = T.Solution(gi, sol)
    b = T.Solution(gi, sol)
    a.enable_timing(True)
    for _ in range(10):
        a.eval(T.OP_STANDARD)
        ok, mv = a.best_move(T.OP_STANDARD)
        applied, mv2 = b.step(T.OP_STANDARD)
        assert ok == applied and (mv.variant, mv.u, mv.v, mv.delta_i) == (mv2.variant, mv2.u, mv2.v, mv2.delta_i)
        if ok:
            a.apply(mv)
    assert a.routes() == b.routes()
    t = a.timings()
    assert len(t) == 10 and (t > 0).all()
    other = G.perturb(sol, 15, 3)
    b.reload(other)
    fresh = T.Solution(gi, other)
    b.eval(T.OP_STANDARD)
    fresh.eval(T.OP_STANDARD)
    np.testing.assert_array_equal(b.keys(), fresh.keys())
    assert b.routes() == fresh.routes()


# ---------------------------------------------------------------- population batch (config 5)
@pytest.mark.parametrize("mode", [0, 1])
def test_batch_population_exact(mode):
    """BASELINE config 5 shape (R1_2-like VRPTW, 200 customers) at reduced
    population: every solution's 22 keys (2-opt is CVRP-only) == oracle."""
    _need_gpu()
    inst, sols = G.population(0, n=200, n_sol=24)
    gi = T.Instance.from_gen(inst, score_mode=mode)
    b = T.Batch(gi, sols)
    mask = T.OP_STANDARD & ~T.OP_2OPT
    b.eval(mask)
    keys = b.keys()
    orc = O.Oracle.from_instance(inst)
    for k, sol in enumerate(sols):
        Q = O.canonical_q(sol)
        for v in INTER + INTRA_TW:
            m = orc.best_move(sol, v, mode=mode)
            exp = oracle_key(m, Q)
            kk = int(keys[k, v])
            got = None if kk == 0xFFFFFFFFFFFFFFFF else T.decode_key(kk)
            assert got == exp, (k, v, got, exp)


def test_batch_full_population_1024():
    """Full config 5 (1024 solutions): batch keys == single-solution keys for
    every solution, a seeded sample of 32 == oracle; one batch step of
    best moves + apply keeps every solution consistent with a fresh load."""
    _need_gpu()
    inst, sols = G.config("cfg5")
    assert len(sols) == 1024
    gi = T.Instance.from_gen(inst)
    b = T.Batch(gi, sols)
    mask = T.OP_STANDARD & ~T.OP_2OPT
    b.eval(mask)
    keys = b.keys()
    rng = np.random.default_rng(5)
    orc = O.Oracle.from_instance(inst)
    for k in rng.choice(1024, size=32, replace=False):
        sol = sols[int(k)]
        Q = O.canonical_q(sol)
        for v in INTER + INTRA_TW:
            m = orc.best_move(sol, v)
            exp = oracle_key(m, Q)
            kk = int(keys[k, v])
            got = None if kk == 0xFFFFFFFFFFFFFFFF else T.decode_key(kk)
            assert got == exp, (int(k), v, got, exp)
    for k in range(0, 1024, 97):
        single = T.Solution(gi, sols[k])
        single.eval(mask)
        np.testing.assert_array_equal(single.keys(), keys[k])
    status, moves = b.best_moves(mask)
    b.apply(moves, apply_mask=(status == 0))
    b.eval(mask)
    keys2 = b.keys()
    for k in range(0, 1024, 131):
        routes = b.solution(k).routes()
        fresh = T.Solution(gi, routes)
        fresh.eval(mask)
        np.testing.assert_array_equal(fresh.keys(), keys2[k])


# ---------------------------------------------------------------- large CVRP (config 4)
def check_exact_parallel(inst, routes, variants, mode=0, label="", gs=None, wQ=10, wT=10):
    """GPU keys of every variant == the oracle's GLOBAL best over the whole
    neighbourhood, enumerated row-parallel on every host core (tests/par_oracle)."""
    if gs is None:
        gs = T.Solution(T.Instance.from_gen(inst, score_mode=mode, w_load=wQ, w_tw=wT), routes)
    gs.eval(sum(1 << v for v in variants))
    got = gpu_keys(gs, integer=True)
    orc = O.Oracle.from_instance(inst)
    exp, count = par_oracle.best_keys(orc, routes, variants, mode, wQ=float(wQ), wT=float(wT))
    c = gs.counts()
    for v in variants:
        assert got[v] == exp[v], f"{label} variant {v} ({T.VARIANT_NAMES[v]}): gpu {got[v]} oracle {exp[v]}"
        assert int(c[v]) == count[v], (label, v, int(c[v]), count[v])
    return gs


@pytest.mark.parametrize("name", ["cfg4", "cfg4s"])
def test_cfg4_large_global_exact(name):
    """BASELINE config 4 at full size (10^4 customers; mean route length 100 or
    23; 7.6-7.8e8 candidates): every variant's GPU key (score and canonical
    index) == the oracle's global argmin, enumerated on all host cores -- not a
    window around the GPU's own answer.  Row shards of the same launch
    configuration min-combine to the unsharded keys."""
    _need_gpu()
    inst, sol = G.config(name)
    gs = check_exact_parallel(inst, sol.routes, ALLV, 0, name)
    full = gs.keys()
    comb = np.full(T.N_VARIANTS, np.iinfo(np.uint64).max, dtype=np.uint64)
    for sh in range(4):
        gs.set_shard(sh, 4)
        gs.eval(T.OP_STANDARD)
        comb = np.minimum(comb, gs.keys())
    np.testing.assert_array_equal(comb, full)


def test_ns2000_full_size_exact():
    """The north-star workload (X-like CVRP, 2000 customers, 87 routes + spare) at
    full size, the launch configuration bench.py times: every variant == the
    oracle's global best (all host cores), and the fused 2-opt*+relocate+swap
    sweep alone gives the same three keys."""
    _need_gpu()
    inst, sol = G.config("ns2000")
    gs = check_exact_parallel(inst, sol.routes, ALLV, 0, "ns2000")
    ref = gs.keys()
    gs.eval(T.OP_FUSED_NS)
    ns = gs.keys()
    for v in (1, 2, 5):
        assert ns[v] == ref[v], v


def test_cfg4_shape_reduced_exact():
    """Config-4 shape (clustered, long routes ~100) at n=2000: full oracle parity."""
    _need_gpu()
    inst, sol = G.large_cvrp(1, n=2000, mean_len=100)
    check_exact(inst, sol, ALLV, 0, "cfg4-2000")


# ---------------------------------------------------------------- device-resident step (NEXT #1)
@pytest.mark.parametrize("name", ["cvrp", "vrptw", "cfg2"])
def test_device_resident_step_matches_host_step(name):
    """tga_step_async (pick + splice + update on the device) follows exactly
    the trajectory of the host-driven tga_step; its on-device candidate
    counts equal the closed forms of the host."""
    _need_gpu()
    if name == "cvrp":
        inst, sol = G.x_like(9, n=200, target_routes=9)
    elif name == "vrptw":
        inst, sol = G.gh_like(9, n=200, kind="R2")
    else:
        inst, sol = G.config("cfg2")
    mask = T.OP_STANDARD if inst.tw is None else T.OP_STANDARD & ~T.OP_2OPT
    gi = T.Instance.from_gen(inst)
    host = T.Solution(gi, sol)
    dev = T.Solution(gi, sol)
    exp_counts = np.zeros(T.N_VARIANTS, dtype=np.uint64)
    applied = 0
    for k in range(40):
        c = host.counts()
        for v in range(T.N_VARIANTS):
            if (mask >> v) & 1:
                exp_counts[v] += c[v]
        ok, _ = host.step(mask)
        applied += int(ok)
        dev.step_async(mask)
        if k % 10 == 9:
            assert dev.routes() == host.routes(), k
    counts, app = dev.device_stats()
    assert app == applied
    np.testing.assert_array_equal(counts, exp_counts)
    assert dev.routes() == host.routes()
    host.eval(mask)
    dev.eval(mask)
    np.testing.assert_array_equal(dev.keys(), host.keys())
    # host-side calls after device steps: apply a host move on the device-stepped object
    ok, mv = dev.best_move(mask)
    if ok:
        dev.apply(mv)
        fresh = T.Solution(gi, dev.routes())
        fresh.eval(mask)
        dev.eval(mask)
        np.testing.assert_array_equal(dev.keys(), fresh.keys())


def test_batch_device_step_matches_host_batch():
    _need_gpu()
    inst, sols = G.population(1, n=200, n_sol=64)
    gi = T.Instance.from_gen(inst)
    mask = T.OP_STANDARD & ~T.OP_2OPT
    hb = T.Batch(gi, sols)
    db = T.Batch(gi, sols)
    for _ in range(5):
        hb.eval(mask)
        status, moves = hb.best_moves(mask)
        hb.apply(moves, apply_mask=(status == 0))
        db.step_async(mask)
    for k in range(64):
        assert db.solution(k).routes() == hb.solution(k).routes(), k
    counts, applied = db.device_stats()
    assert applied > 0


@pytest.mark.parametrize("mode", [0, 1])
def test_vrptw_intra_warp_kernel_long_routes(mode):
    """Warp-parallel VRPTW intra kernel (mean route length >= 16): chunked
    scans across 32-lane boundaries (routes of 31..70 customers), both modes,
    feasible and perturbed (warping) states."""
    _need_gpu()
    inst, sol = G.gh_like(7, n=240, kind="R2")
    routes = [r for r in sol.routes]
    merged = G.Solution([routes[0] + routes[1], routes[2] + routes[3][:10]] + [routes[3][10:]] + routes[4:])
    for s in (merged, G.perturb(merged, 20, 3)):
        assert sum(len(r) for r in s.routes) >= 16 * len(s.routes)
        check_exact(inst, s, INTRA_TW + INTER, mode, "tw-warp")


@pytest.mark.parametrize("slack", [-1, 1, 5])
def test_slack_layouts_lockstep(slack):
    """Spare slots per route (0 = none, 1 = frequent relayouts, 5): host-driven
    and device-resident descents follow the oracle's trajectory; keys equal a
    fresh load after every few moves (the partial refresh touches only the two
    changed routes unless one outgrows its slots)."""
    _need_gpu()
    inst, sol = G.x_like(12, n=160, target_routes=8)
    orc = O.Oracle.from_instance(inst)
    gi = T.Instance.from_gen(inst, slack=slack)
    host = T.Solution(gi, sol)
    dev = T.Solution(gi, sol)
    routes = [list(r) for r in sol.routes]
    for step in range(30):
        ob = orc.best_over(routes, ALLV)
        if ob is None or not ob.score < 0:
            break
        ok, mv = host.step(T.OP_STANDARD)
        assert ok and (mv.variant, mv.u, mv.v, mv.delta_i) == (ob.variant, ob.u, ob.v, ob.score)
        dev.step_async(T.OP_STANDARD)
        routes = orc.apply(routes, ob.variant, ob.route_a, ob.pos_a, ob.route_b, ob.pos_b)
        if step % 7 == 6:
            assert host.routes() == routes and dev.routes() == routes
            fresh = T.Solution(gi, routes)
            for s in (host, dev, fresh):
                s.eval(T.OP_STANDARD)
            np.testing.assert_array_equal(host.keys(), fresh.keys())
            np.testing.assert_array_equal(dev.keys(), fresh.keys())
    assert dev.routes() == routes


@pytest.mark.parametrize("name", ["cvrp3000", "vrptw_r1", "vrptw_r1_penalised"])
def test_device_step_column_paths_and_short_tw_routes(name):
    """Device-resident steps where the update copies the changed Dp columns
    from the refreshed rows behind a grid barrier (Q_p > 2560), and on short
    VRPTW routes (R1 shape, warp-parallel intra kernel): lockstep with the
    host-driven step, and keys equal a fresh load of the resulting routes."""
    _need_gpu()
    mode = 0
    if name == "cvrp3000":
        inst, sol = G.large_cvrp(3, n=3000, mean_len=60)
        mask = T.OP_STANDARD
    else:
        inst, sol = G.gh_like(4, n=300, kind="R1")
        mask = T.OP_STANDARD & ~T.OP_2OPT
        mode = 1 if name.endswith("penalised") else 0
    gi = T.Instance.from_gen(inst, score_mode=mode)
    host = T.Solution(gi, sol)
    dev = T.Solution(gi, sol)
    R, N, _, _ = dev.info()
    if name == "cvrp3000":
        assert N + 4 * R > 2560
    for k in range(16):
        host.step(mask)
        dev.step_async(mask)
        if k % 8 == 7:
            assert dev.routes() == host.routes(), k
    fresh = T.Solution(gi, dev.routes())
    for s in (host, dev, fresh):
        s.eval(mask)
    np.testing.assert_array_equal(dev.keys(), fresh.keys())
    np.testing.assert_array_equal(host.keys(), fresh.keys())


# ---------------------------------------------------------------- edge-based neighbourhood (ETGA, NEXT #3)
def _etga_check(inst, routes, theta, variants, label):
    """keys of every variant == the masked oracle; the device's evaluated
    inter-route candidate counts == the masked oracle's counts."""
    orc = O.Oracle.from_instance(inst)
    M = O.granular_mask(inst.dist, theta)
    gi = T.Instance.from_gen(inst, granular_theta=theta)
    gs = T.Solution(gi, routes)
    gs.device_stats()
    gs.eval(sum(1 << v for v in variants))
    got = gpu_keys(gs, integer=True)
    counts, _ = gs.device_stats()
    Q = O.canonical_q(routes)
    for v in variants:
        m = orc.best_move(routes, v, mask=M)
        assert got[v] == oracle_key(m, Q), (label, theta, v, got[v], oracle_key(m, Q))
        if v in INTER:
            assert int(counts[v]) == m.n_candidates, (label, theta, v, int(counts[v]), m.n_candidates)


@pytest.mark.parametrize("theta", [1, 3, 8])
@pytest.mark.parametrize("seed", range(3))
def test_etga_small_exact(theta, seed):
    _need_gpu()
    inst, sol = G.cvrp_small(seed, spare=True)
    _etga_check(inst, sol.routes, theta, ALLV, f"cfg1-{seed}")
    inst, sol = G.gh_like(seed, n=60, kind="R1")
    _etga_check(inst, sol.routes, theta, INTER + INTRA_TW, f"vrptw-{seed}")
    for k in range(3):
        part = G.random_partition(20, 3 + k, 900 + 10 * seed + k)
        inst, _ = G.cvrp_small(seed, spare=False)
        _etga_check(inst, part.routes, theta, ALLV, f"partition-{k}")


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_etga_full_size_exact(name):
    """Full-size configs at the paper's granularity thresholds (X: 20, GH: 100; Table params)."""
    _need_gpu()
    inst, sol = G.config(name)
    theta = 20 if name == "cfg2" else 100
    _etga_check(inst, sol.routes, theta, INTER, name)


def test_etga_theta_all_is_full_neighbourhood():
    _need_gpu()
    inst, sol = G.x_like(3, n=150, target_routes=7)
    full = T.Solution(T.Instance.from_gen(inst), sol)
    edge = T.Solution(T.Instance.from_gen(inst, granular_theta=inst.dist.shape[0]), sol)
    for s in (full, edge):
        s.eval(T.OP_STANDARD)
    np.testing.assert_array_equal(full.keys(), edge.keys())


@pytest.mark.parametrize("name", ["cvrp", "vrptw"])
def test_etga_device_step_lockstep(name):
    """Device-resident ETGA steps follow the host-driven ETGA trajectory and the
    masked oracle's best move at every step."""
    _need_gpu()
    if name == "cvrp":
        inst, sol = G.x_like(6, n=200, target_routes=9)
        mask, theta = T.OP_STANDARD, 10
    else:
        inst, sol = G.gh_like(6, n=200, kind="R2")
        mask, theta = T.OP_STANDARD & ~T.OP_2OPT, 20
    orc = O.Oracle.from_instance(inst)
    M = O.granular_mask(inst.dist, theta)
    gi = T.Instance.from_gen(inst, granular_theta=theta)
    host = T.Solution(gi, sol)
    dev = T.Solution(gi, sol)
    routes = [list(r) for r in sol.routes]
    variants = [v for v in ALLV if (mask >> v) & 1]
    for step in range(15):
        best = None
        for v in variants:
            m = orc.best_move(routes, v, mask=M)
            if m.found and (best is None or m.score < best.score):
                best = m
        if best is None or not best.score < 0:
            break
        ok, mv = host.step(mask)
        assert ok and (mv.variant, mv.u, mv.v, mv.delta_i) == (best.variant, best.u, best.v, best.score), step
        dev.step_async(mask)
        routes = orc.apply(routes, best.variant, best.route_a, best.pos_a, best.route_b, best.pos_b)
    assert host.routes() == routes and dev.routes() == routes


# ---------------------------------------------------------------- degenerate shapes
def _degenerate_cases():
    """(name, instance, routes): one customer; all customers in one route among
    empty routes; routes of exactly 1, 2, 3 customers (the or-opt / cross
    segment-length boundaries); an overloaded route (feasible-only: nothing
    improving out of it unless it becomes feasible)."""
    base, _ = G.cvrp_small(11, n=12, n_routes=3)
    yield "one-customer", G.Instance("one", base.mode, base.coords[:2], base.dist[:2, :2].copy(),
                                     base.demand[:2].copy(), base.capacity), [[1], []]
    yield "single-route+empties", base, [list(range(1, 13)), [], [], []]
    yield "lengths-1-2-3", base, [[1], [2, 3], [4, 5, 6], [7, 8, 9, 10, 11, 12], []]
    tight = G.Instance("tight", base.mode, base.coords, base.dist, base.demand, int(base.demand.max()) * 3)
    yield "overloaded", tight, [list(range(1, 9)), [9], [10, 11], [12], []]
    tw_inst, tw_sol = G.gh_like(12, n=12, kind="R1")
    yield "tw-lengths", tw_inst, [[1], [2, 3], [4, 5, 6], [7, 8, 9, 10, 11, 12], []]


@pytest.mark.parametrize("mode", [0, 1])
def test_degenerate_shapes_exact(mode):
    """Every variant's key == the oracle on degenerate solutions, and one device
    step from each agrees with the host step."""
    _need_gpu()
    for name, inst, routes in _degenerate_cases():
        variants = ALLV if inst.tw is None else INTER + INTRA_TW
        check_exact(inst, routes, variants, mode, name)
        gi = T.Instance.from_gen(inst, score_mode=mode)
        host, dev = T.Solution(gi, routes), T.Solution(gi, routes)
        m = sum(1 << v for v in variants)
        host.step(m)
        dev.step_async(m)
        assert dev.routes() == host.routes(), name


@pytest.mark.parametrize("n_shards", [2, 3, 8])
def test_etga_virtual_shards_equal_unsharded(n_shards):
    """ETGA cell shards (the row-shard plan of a multi-GPU run) min-combined on the
    host == the unsharded keys; their evaluated-candidate counts add up."""
    _need_gpu()
    inst, sol = G.x_like(7, n=400, target_routes=17)
    gs = T.Solution(T.Instance.from_gen(inst, granular_theta=12), sol)
    gs.device_stats()
    gs.eval(T.OP_STANDARD)
    full = gs.keys()
    full_counts, _ = gs.device_stats()
    comb = np.full(T.N_VARIANTS, np.iinfo(np.uint64).max, dtype=np.uint64)
    tot = np.zeros(T.N_VARIANTS, dtype=np.uint64)
    for s in range(n_shards):
        gs.set_shard(s, n_shards)
        gs.eval(T.OP_STANDARD)
        comb = np.minimum(comb, gs.keys())
        c, _ = gs.device_stats()
        tot += c
    np.testing.assert_array_equal(comb, full)
    np.testing.assert_array_equal(tot[1:11], full_counts[1:11])


@pytest.mark.parametrize("force", ["0", "1"])
def test_vrptw_intra_kernels_forced(force):
    """Both VRPTW intra kernels on every route length: by default the route-length threshold picks
    the walk (short routes) or the warp-scan kernel (long routes); TGA_WARP_TW forces one, read
    once per process, so the small and full-size VRPTW parity tests rerun in a subprocess."""
    _need_gpu()
    import os
    import subprocess
    import sys
    env = dict(os.environ, TGA_WARP_TW=force)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.abspath(__file__), "-q", "-m", "gpu", "-p",
                        "no:cacheprovider", "-k", "test_small_vrptw_exact or test_full_size_configs_exact"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


# ---------------------------------------------------------------- ABI guards (advisor findings)
def test_physical_pitch_overflow_rejected():
    """Keys pack u * pitch + v over PHYSICAL slots in 32 bits: a layout whose
    padded pitch^2 exceeds 2^32 is rejected at load even when the canonical
    Q^2 fits (here N + R = 1044, but 2 + slack spare slots per route blow the
    pitch up)."""
    _need_gpu()
    inst, sol = G.x_like(0, n=1000)
    gi = T.Instance.from_gen(inst, slack=100000)
    with pytest.raises(T.TgaError) as e:
        T.Solution(gi, sol)
    assert e.value.code == -1 and "pitch" in str(e.value)


def test_mixed_grid_device_steps_share_the_barrier():
    """Device steps of the same solutions through the population batch (small
    grids per solution) and one by one (one block per SM) alternate: the grid
    barrier and arrival counters reset every launch, so the trajectories equal
    the host-driven steps."""
    _need_gpu()
    inst, sols = G.population(2, n=200, n_sol=4)
    gi = T.Instance.from_gen(inst)
    mask = T.OP_STANDARD & ~T.OP_2OPT
    db = T.Batch(gi, sols)
    host = [T.Solution(gi, s) for s in sols]
    for it in range(12):
        if it % 3 == 2:
            for k in range(4):
                db.solution(k).step_async(mask)
        else:
            db.step_async(mask)
        for h in host:
            h.step(mask)
    for k in range(4):
        assert db.solution(k).routes() == host[k].routes(), k


def test_integer_score_range_guard():
    """Integer scores are packed as 32-bit order-preserving images: distances or
    penalty weights whose candidate scores could overflow int32 are rejected at
    instance creation (TGA_F32 stays available)."""
    _need_gpu()
    inst, sol = G.cvrp_small(0)
    big = (inst.dist.astype(np.int64) * (2 ** 26)).astype(np.int32)
    with pytest.raises(T.TgaError) as e:
        T.Instance(big, inst.demand, inst.capacity)
    assert e.value.code == -1
    with pytest.raises(T.TgaError):
        T.Instance(inst.dist, inst.demand, inst.capacity, score_mode=T.SCORE_PENALISED, w_load=2 ** 28)
    T.Instance(inst.dist.astype(np.float32) * 2.0 ** 26, inst.demand, inst.capacity)   # float path accepted


# ---------------------------------------------------------------- penalised score (Eq. 16a) at full size
@pytest.mark.parametrize("name", ["cfg2", "ns2000", "cfg3"])
def test_penalised_full_size_exact(name):
    """Penalised mode (score = dD + w_Q dL_V (+ w_T dT_V), Eq. 16a, DESIGN.md
    reading 4) at full size: CVRP on the fused fast path (penalised records),
    VRPTW on the generic tile kernel; every variant == the oracle's global best."""
    _need_gpu()
    inst, sol = G.config(name)
    variants = ALLV if inst.tw is None else INTER + INTRA_TW
    check_exact_parallel(inst, sol.routes, variants, 1, f"{name}-pen")
    # an infeasible state (overloaded routes) makes the penalty terms bite
    check_exact_parallel(inst, G.perturb(sol, 60, 11).routes, variants, 1, f"{name}-pen-perturbed")


def test_penalised_generic_multi_tile():
    """The generic tile kernel (penalised VRPTW) with more tiles than resident
    CTAs, so its double-buffered persistent tile loop runs (n = 3000, R2 shape)."""
    _need_gpu()
    inst, sol = G.gh_like(8, n=3000, kind="R2")
    sol = G.perturb(sol, 40, 8)
    # w_T = 1: with 3000 customers the int32 score-range guard rejects w_T = 10
    gs = T.Solution(T.Instance.from_gen(inst, score_mode=1, w_load=10, w_tw=1), sol)
    R, N, _, _ = gs.info()
    assert (N + 4 * R) // 32 * ((N + 4 * R) // 64) // 2 > 4 * 148, "must exceed one tile per CTA"
    check_exact_parallel(inst, sol.routes, INTER + INTRA_TW, 1, "tw-pen-3000", gs=gs, wQ=10, wT=1)


@pytest.mark.parametrize("name", ["cvrp", "cvrp-slack0"])
def test_penalised_device_steps_lockstep(name):
    """Penalised CVRP: device-resident steps (fast path + on-device pick/update)
    follow the host-driven steps; keys equal a fresh load afterwards."""
    _need_gpu()
    inst, sol = G.x_like(13, n=400, target_routes=17)
    sol = G.perturb(sol, 30, 13)
    gi = T.Instance.from_gen(inst, score_mode=1, slack=-1 if name.endswith("0") else 0)
    host, dev = T.Solution(gi, sol), T.Solution(gi, sol)
    for k in range(30):
        host.step(T.OP_STANDARD)
        dev.step_async(T.OP_STANDARD)
        if k % 10 == 9:
            assert dev.routes() == host.routes(), k
    fresh = T.Solution(gi, dev.routes())
    for s in (dev, fresh):
        s.eval(T.OP_STANDARD)
    np.testing.assert_array_equal(dev.keys(), fresh.keys())
