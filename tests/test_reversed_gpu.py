"""GPU parity of the reversed-segment variants (P:677:
"Relocate and Swap can incorporate reversed subsequences by exchanging the first
and last node index tensors, as in 2-opt"): or-opt N=2,3 with the moved segment
inserted reversed (variants 23, 24) and cross (N,N), N=2,3, with both segments
reversed (25, 26).  They run in the generic tile kernel (also beside the CVRP fast
path), with the reversed segment's Eq. 4 / Eq. 3 records concatenated from its
nodes in reverse order.

Bar: integer data -> every candidate's score and feasibility and every key
bit-exact against the oracle's explicit splice; trajectories identical."""
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

REV = [23, 24, 25, 26]


def _need_gpu():
    if not gpu_available():
        pytest.skip("no CUDA device")


def rev_keys(inst, routes, mode=0, label="", extra=0, parallel=False):
    gs = T.Solution(T.Instance.from_gen(inst, score_mode=mode), routes)
    gs.eval(T.OP_REVERSED | extra)
    ks = gs.keys()
    orc = O.Oracle.from_instance(inst)
    Q = O.canonical_q(routes)
    if parallel:
        exp, count = par_oracle.best_keys(orc, routes, REV, mode)
        c = gs.counts()
        for v in REV:
            assert int(c[v]) == count[v], (label, v)
    else:
        exp = {}
        for v in REV:
            m = orc.best_move(routes, v, mode=mode)
            exp[v] = (m.score, m.u * Q + m.v) if m.found else None
    for v in REV:
        k = int(ks[v])
        got = None if k == 0xFFFFFFFFFFFFFFFF else T.decode_key(k)
        assert got == exp[v], f"{label} variant {v}: gpu {got} oracle {exp[v]}"
    return gs


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("seed", range(4))
def test_reversed_cfg1_exact(seed, mode):
    """Config 1 (with the spare route) and ragged random partitions; alone and beside
    the fused CVRP fast path (OP_ALL)."""
    _need_gpu()
    inst, sol = G.cvrp_small(seed, spare=True)
    rev_keys(inst, sol.routes, mode, f"cfg1 s{seed}")
    rev_keys(inst, sol.routes, mode, f"cfg1+all s{seed}", extra=T.OP_STANDARD)
    for k in range(2):
        part = G.random_partition(20, 4 + k, 800 + 10 * seed + k, allow_empty=True)
        rev_keys(inst, part.routes, mode, f"cfg1-rand s{seed}/{k}")


@pytest.mark.parametrize("kind", ["R1", "R2"])
def test_reversed_vrptw_exact(kind):
    _need_gpu()
    inst, sol = G.gh_like(2, n=150, kind=kind)
    rev_keys(inst, sol.routes, 0, kind)
    rev_keys(inst, G.perturb(sol, 20, 3).routes, 1, kind + "-perturbed-penalised")


def test_reversed_pickup_delivery_exact():
    _need_gpu()
    inst, sol = G.jd_like(3, n=80)
    rev_keys(inst, sol.routes, 0, "jd80")
    rev_keys(inst, G.perturb(sol, 10, 4).routes, 1, "jd80-perturbed-penalised")


@pytest.mark.parametrize("name", ["cvrp", "vrptw", "pd"])
def test_reversed_fields_exact(name):
    """Every candidate of the four reversed variants: score bit-exact, mask identical."""
    _need_gpu()
    if name == "cvrp":
        inst, sol = G.cvrp_small(2, spare=True)
    elif name == "vrptw":
        inst, sol = G.gh_like(5, n=200, kind="R1")
    else:
        inst, sol = G.config("jd200")
    for mode in (0, 1):
        n, _ = compare_fields(inst, sol.routes, REV, mode, flags=2, label=f"rev {name}")
        assert n > 0


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_reversed_full_size_global_exact(name):
    _need_gpu()
    inst, sol = G.config(name)
    rev_keys(inst, sol.routes, 0, name, parallel=True)


@pytest.mark.parametrize("name", ["cvrp", "vrptw"])
def test_reversed_device_descent_lockstep(name):
    """Device-resident steps over every variant (the 23 standard + the 4 reversed; the
    on-device splice walks the reversed pieces backwards) follow the oracle."""
    _need_gpu()
    if name == "cvrp":
        inst, sol = G.x_like(7, n=160, target_routes=8)
        variants = list(range(T.N_VARIANTS))
        mask = T.OP_ALL
    else:
        inst, sol = G.gh_like(7, n=160, kind="R2")
        variants = [v for v in range(T.N_VARIANTS) if v != 0]
        mask = T.OP_ALL & ~T.OP_2OPT
    orc = O.Oracle.from_instance(inst)
    dev = T.Solution(T.Instance.from_gen(inst), sol)
    routes = [list(r) for r in sol.routes]
    moves, rev_moves = 0, 0
    for step in range(30):
        ob = orc.best_over(routes, variants)
        dev.step_async(mask)
        if ob is None or not ob.score < 0:
            break
        routes = orc.apply(routes, ob.variant, ob.route_a, ob.pos_a, ob.route_b, ob.pos_b)
        moves += 1
        rev_moves += ob.variant in REV
        assert dev.routes() == routes, step
    assert dev.device_stats()[1] == moves


def test_reversed_host_apply_lockstep():
    """Only the reversed variants: host eval -> best move -> apply, the oracle's moves."""
    _need_gpu()
    inst, sol = G.x_like(8, n=200, target_routes=9)
    orc = O.Oracle.from_instance(inst)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    routes = [list(r) for r in sol.routes]
    applied = 0
    for step in range(12):
        gs.eval(T.OP_REVERSED)
        ok, mv = gs.best_move(T.OP_REVERSED)
        ob = orc.best_over(routes, REV)
        if ob is None or not ob.score < 0:
            assert not ok
            break
        assert (mv.variant, mv.delta_i, mv.route_a, mv.pos_a, mv.route_b, mv.pos_b) == \
            (ob.variant, ob.score, ob.route_a, ob.pos_a, ob.route_b, ob.pos_b), step
        gs.apply(mv)
        routes = orc.apply(routes, ob.variant, ob.route_a, ob.pos_a, ob.route_b, ob.pos_b)
        assert gs.routes() == routes
        applied += 1
    assert applied > 0


def test_reversed_batch_matches_single_solutions():
    _need_gpu()
    inst, sol = G.gh_like(9, n=120, kind="R1")
    sols = [sol] + [G.perturb(sol, 4 + k, 600 + k) for k in range(5)]
    gi = T.Instance.from_gen(inst)
    b = T.Batch(gi, sols)
    mask = T.OP_ALL & ~T.OP_2OPT
    b.eval(mask)
    bk = b.keys()
    for k, s in enumerate(sols):
        one = T.Solution(gi, s)
        one.eval(mask)
        np.testing.assert_array_equal(bk[k], one.keys())


def test_reversed_with_edge_based_neighbourhood_unsupported():
    _need_gpu()
    inst, sol = G.x_like(1, n=100, target_routes=5)
    gs = T.Solution(T.Instance.from_gen(inst, granular_theta=10), sol)
    with pytest.raises(T.TgaError) as e:
        gs.eval(T.OP_REVERSED)
    assert e.value.code == -4
