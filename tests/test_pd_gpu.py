"""GPU parity of the VRPSPDTW loads (Eq. 3a-d):
customers with a delivery d_i and a pickup p_i, the capacity test on the
largest load a route carries.  The CUDA path keeps prefix / suffix (L_I, L_O, L_M)
records from a segmented warp scan of the Eq. 3 concatenation and concatenates
them per candidate; the oracle re-simulates every neighbour's load profile.

Bar: integer data (TW-I times, integer loads) -> load records, every candidate's
score and feasibility, and every best-move key bit-exact; trajectories identical."""
import numpy as np
import pytest

import oracle as O
import tga_gen as G
from tests import par_oracle
from tests.conftest import gpu_available
from tests.test_fields_gpu import compare_fields

pytestmark = pytest.mark.gpu

if gpu_available():
    from paper_2506_17357_b200 import tga as T
else:  # pragma: no cover
    T = None

VARIANTS = list(range(1, 23))   # every variant but 2-opt (CVRP only)


def _need_gpu():
    if not gpu_available():
        pytest.skip("no CUDA device")


def keys_vs_oracle(inst, routes, mode=0, label="", parallel=False):
    gs = T.Solution(T.Instance.from_gen(inst, score_mode=mode), routes)
    gs.eval(sum(1 << v for v in VARIANTS))
    ks = gs.keys()
    orc = O.Oracle.from_instance(inst)
    Q = O.canonical_q(routes)
    if parallel:
        exp, _ = par_oracle.best_keys(orc, routes, VARIANTS, mode)
    else:
        exp = {}
        for v in VARIANTS:
            m = orc.best_move(routes, v, mode=mode)
            exp[v] = (m.score, m.u * Q + m.v) if m.found else None
    for v in VARIANTS:
        k = int(ks[v])
        got = None if k == 0xFFFFFFFFFFFFFFFF else T.decode_key(k)
        assert got == exp[v], f"{label} variant {v}: gpu {got} oracle {exp[v]}"
    return gs


@pytest.mark.parametrize("seed", range(3))
def test_load_records_match_definition(seed):
    """Prefix / suffix records of every canonical slot: L_I and L_O are the delivery and
    pickup sums, L_M the oracle's simulated largest load of that subsequence."""
    _need_gpu()
    inst, sol = G.jd_like(seed, n=200)
    orc = O.Oracle.from_instance(inst)
    for routes in (sol.routes, G.perturb(sol, 30, seed).routes):
        gs = T.Solution(T.Instance.from_gen(inst), routes)
        pre, suf = gs.load_records()
        c = 0
        for r in routes:
            nodes = [0] + list(r) + [0]
            for p in range(len(r) + 1):
                head, tail = nodes[:p + 1], nodes[p:]
                assert tuple(pre[c]) == (int(inst.demand[head].sum()), int(inst.pickup[head].sum()),
                                         orc.seq_lmax(head)), (c, "prefix")
                assert tuple(suf[c]) == (int(inst.demand[tail].sum()), int(inst.pickup[tail].sum()),
                                         orc.seq_lmax(tail)), (c, "suffix")
                c += 1


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("seed", range(4))
def test_small_pd_keys_exact(seed, mode):
    """60-customer JD-like instances, start state + a perturbed (overloaded, warping)
    state + random partitions: every variant's key == the oracle's."""
    _need_gpu()
    inst, sol = G.jd_like(seed, n=60)
    keys_vs_oracle(inst, sol.routes, mode, f"jd60 s{seed}")
    keys_vs_oracle(inst, G.perturb(sol, 15, 10 + seed).routes, mode, f"jd60-perturbed s{seed}")
    keys_vs_oracle(inst, G.random_partition(60, 8, 20 + seed).routes, mode, f"jd60-rand s{seed}")


@pytest.mark.parametrize("mode", [0, 1])
def test_pd_fields_exact(mode):
    """Every candidate of every variant (jd200, start and perturbed): score bit-exact,
    feasibility mask identical (the DUMP instantiations of the generic kernels)."""
    _need_gpu()
    inst, sol = G.config("jd200")
    for routes in (sol.routes, G.perturb(sol, 25, 7).routes):
        n, _ = compare_fields(inst, routes, VARIANTS, mode, flags=2, label="jd200")
        assert n > 0


def test_pd_full_size_global_exact():
    """The JD-like 1000-customer instance at full size: every variant's key == the
    oracle's global argmin (row-parallel on every host core), counts exact."""
    _need_gpu()
    inst, sol = G.config("jd")
    keys_vs_oracle(inst, sol.routes, 0, "jd", parallel=True)


def test_pd_device_descent_lockstep():
    """Device-resident best-improvement steps follow the oracle's trajectory; the
    incremental records equal a fresh load's at the end."""
    _need_gpu()
    inst, sol = G.jd_like(5, n=150)
    orc = O.Oracle.from_instance(inst)
    gi = T.Instance.from_gen(inst)
    dev = T.Solution(gi, sol)
    mask = sum(1 << v for v in VARIANTS)
    routes = [list(r) for r in sol.routes]
    moves = 0
    for step in range(25):
        ob = orc.best_over(routes, VARIANTS)
        dev.step_async(mask)
        if ob is None or not ob.score < 0:
            break
        routes = orc.apply(routes, ob.variant, ob.route_a, ob.pos_a, ob.route_b, ob.pos_b)
        moves += 1
        assert dev.routes() == routes, step
    assert dev.device_stats()[1] == moves
    fresh = T.Solution(gi, routes)
    np.testing.assert_array_equal(np.stack(dev.load_records()), np.stack(fresh.load_records()))
    dev.eval(mask)
    fresh.eval(mask)
    np.testing.assert_array_equal(dev.keys(), fresh.keys())


def test_pd_host_apply_lockstep():
    """Host-driven eval -> best move -> apply with the incremental update kernel."""
    _need_gpu()
    inst, sol = G.jd_like(6, n=120)
    orc = O.Oracle.from_instance(inst)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    mask = sum(1 << v for v in VARIANTS)
    routes = [list(r) for r in sol.routes]
    for step in range(15):
        gs.eval(mask)
        ok, mv = gs.best_move(mask)
        ob = orc.best_over(routes, VARIANTS)
        if ob is None or not ob.score < 0:
            assert not ok
            break
        assert (mv.variant, mv.delta_i, mv.route_a, mv.pos_a, mv.route_b, mv.pos_b) == \
            (ob.variant, ob.score, ob.route_a, ob.pos_a, ob.route_b, ob.pos_b), step
        gs.apply(mv)
        routes = orc.apply(routes, ob.variant, ob.route_a, ob.pos_a, ob.route_b, ob.pos_b)
        assert gs.routes() == routes


def test_pd_batch_matches_single_solutions():
    _need_gpu()
    inst, sol = G.jd_like(7, n=100)
    sols = [sol] + [G.perturb(sol, 5 + k, 300 + k) for k in range(7)]
    gi = T.Instance.from_gen(inst)
    b = T.Batch(gi, sols)
    mask = sum(1 << v for v in VARIANTS)
    b.eval(mask)
    bk = b.keys()
    for k, s in enumerate(sols):
        one = T.Solution(gi, s)
        one.eval(mask)
        np.testing.assert_array_equal(bk[k], one.keys())


def test_pd_rejections():
    """2-opt with pickups is unsupported; pickups cannot change under loaded solutions."""
    _need_gpu()
    inst, sol = G.jd_like(0, n=40)
    gi = T.Instance.from_gen(inst)
    gs = T.Solution(gi, sol)
    with pytest.raises(T.TgaError) as e:
        gs.eval(T.OP_2OPT)
    assert e.value.code == -4
    import ctypes as C
    p = np.ascontiguousarray(inst.pickup, dtype=np.int32)
    assert T.lib().tga_instance_set_pickup(gi._h, p.ctypes.data_as(C.c_void_p)) == -1
