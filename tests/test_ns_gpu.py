"""GPU parity of the north-star sweep kernel (tga_ns.cu): an evaluation whose
inter-route part is exactly {2-opt*, relocate, swap (1,1)} (BASELINE.json
north_star "2-opt*+relocate+swap sweep") runs k_ns_sweep, a kernel of its own.

Bar (north_star; readings 4, 5): integer CVRP -> every candidate's
score and feasibility bit-exact (per-candidate DUMP instantiation vs the
oracle's canonical enumeration), best-move keys bit-exact against the oracle's
global argmin, trajectories identical.
"""
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

NS = [1, 2, 5]


def _need_gpu():
    if not gpu_available():
        pytest.skip("no CUDA device")


def ns_keys_vs_oracle(inst, routes, label, parallel=False):
    gs = T.Solution(T.Instance.from_gen(inst), routes)
    gs.eval(T.OP_FUSED_NS)
    ks = gs.keys()
    got = {v: (None if int(ks[v]) == 0xFFFFFFFFFFFFFFFF else T.decode_key(int(ks[v]))) for v in NS}
    orc = O.Oracle.from_instance(inst)
    Q = O.canonical_q(routes)
    if parallel:
        exp, count = par_oracle.best_keys(orc, routes, NS)
        c = gs.counts()
        for v in NS:
            assert int(c[v]) == count[v], (label, v)
    else:
        exp = {}
        for v in NS:
            m = orc.best_move(routes, v)
            exp[v] = (m.score, m.u * Q + m.v) if m.found else None
    for v in NS:
        assert got[v] == exp[v], f"{label} variant {v}: gpu {got[v]} oracle {exp[v]}"
    # variants outside the sweep stay untouched
    for v in range(T.N_VARIANTS):
        if v not in NS:
            assert int(ks[v]) == 0xFFFFFFFFFFFFFFFF, (label, v)
    return gs


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("spare", [False, True])
def test_ns_cfg1_exact(seed, spare):
    _need_gpu()
    inst, sol = G.cvrp_small(seed, spare=spare)
    ns_keys_vs_oracle(inst, sol.routes, f"cfg1 s{seed}")
    for k in range(3):   # ragged, empty, infeasible routes
        part = G.random_partition(20, 4 + k, 500 + 10 * seed + k, allow_empty=True)
        ns_keys_vs_oracle(inst, part.routes, f"cfg1-rand s{seed}/{k}")


@pytest.mark.parametrize("seed", range(3))
def test_ns_cfg1_fields_exact(seed):
    """Every candidate of the three variants: score bit-exact, mask identical, no
    extra candidate (the DUMP instantiation of k_ns_sweep)."""
    _need_gpu()
    inst, sol = G.cvrp_small(seed, spare=True)
    n, _ = compare_fields(inst, sol.routes, NS, 0, label=f"ns cfg1 s{seed}")
    assert n > 0
    part = G.random_partition(20, 5, 700 + seed, allow_empty=True)
    compare_fields(inst, part.routes, NS, 0, label=f"ns cfg1-rand s{seed}")


@pytest.mark.parametrize("name", ["cfg2", "ns2000"])
def test_ns_full_size_fields_exact(name):
    """Full-size per-candidate parity (cfg2: 3.7 M candidates, ns2000: 8.3 M): the
    tile plan's every diagonal / full tile and the partial last column band."""
    _need_gpu()
    inst, sol = G.config(name)
    n, _ = compare_fields(inst, sol.routes, NS, 0, label=f"ns {name}")
    assert n > 0


@pytest.mark.parametrize("name", ["cfg2", "ns2000"])
def test_ns_full_size_global_exact(name):
    _need_gpu()
    inst, sol = G.config(name)
    ns_keys_vs_oracle(inst, sol.routes, name, parallel=True)


def test_ns_cfg4_multi_tile_matches_all_variant_kernel():
    """n = 10^4: 1.3e4 tiles over the resident grid, so every CTA walks several
    tiles (the re-armed mbarrier path); the three keys equal the all-variant
    kernel's (which test_cfg4_large_global_exact pins to the oracle), and row
    shards min-combine to them."""
    _need_gpu()
    inst, sol = G.config("cfg4")
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    gs.eval(T.OP_INTER)
    ref = gs.keys()
    gs.eval(T.OP_FUSED_NS)
    ns = gs.keys()
    for v in NS:
        assert ns[v] == ref[v], v
    comb = np.full(T.N_VARIANTS, np.iinfo(np.uint64).max, dtype=np.uint64)
    for sh in range(3):
        gs.set_shard(sh, 3)
        gs.eval(T.OP_FUSED_NS)
        comb = np.minimum(comb, gs.keys())
    for v in NS:
        assert comb[v] == ref[v], v


def test_ns_with_intra_variants():
    """NS + intra-route variants in one eval: the sweep kernel, then the intra kernel."""
    _need_gpu()
    inst, sol = G.x_like(3, n=300, target_routes=13)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    mask = T.OP_FUSED_NS | T.OP_INTRA
    gs.eval(mask)
    got = gs.keys()
    orc = O.Oracle.from_instance(inst)
    Q = O.canonical_q(sol.routes)
    for v in NS + [0] + list(range(11, 23)):
        m = orc.best_move(sol.routes, v)
        exp = None if not m.found else (m.score, m.u * Q + m.v)
        k = int(got[v])
        assert (None if k == 0xFFFFFFFFFFFFFFFF else T.decode_key(k)) == exp, v


def test_ns_device_descent_lockstep():
    """Device-resident steps with the north-star mask (eval by k_ns_sweep, on-device
    pick + apply) follow the oracle's best-improvement trajectory move for move."""
    _need_gpu()
    inst, sol = G.x_like(8, n=250, target_routes=11)
    orc = O.Oracle.from_instance(inst)
    gi = T.Instance.from_gen(inst)
    dev = T.Solution(gi, sol)
    routes = [list(r) for r in sol.routes]
    moves = 0
    for step in range(30):
        ob = orc.best_over(routes, NS)
        dev.step_async(T.OP_FUSED_NS)
        if ob is None or not ob.score < 0:
            break
        routes = orc.apply(routes, ob.variant, ob.route_a, ob.pos_a, ob.route_b, ob.pos_b)
        moves += 1
        assert dev.routes() == routes, step
    _, applied = dev.device_stats()
    assert applied == moves


def test_ns_publish_accumulate_and_reset():
    """The sweep kernel publishes its keys itself (no reset node): a plain eval resets
    every other variant's key, an accumulating eval (TGA_EVAL_ACCUMULATE) keeps the
    keys of an earlier eval of other variants, and back-to-back evals (captured or
    not) give the same keys every time."""
    _need_gpu()
    inst, sol = G.x_like(2, n=400, target_routes=17)
    gs = T.Solution(T.Instance.from_gen(inst), sol)
    gs.eval(T.OP_STANDARD)
    ref = gs.keys()
    gs.eval(T.OP_OR_OPT | T.OP_CROSS | T.OP_INTRA)
    gs.eval(T.OP_FUSED_NS | T.EVAL_ACCUMULATE)
    np.testing.assert_array_equal(gs.keys(), ref)
    for _ in range(5):
        gs.eval(T.OP_FUSED_NS)
    ks = gs.keys()
    for v in range(T.N_VARIANTS):
        assert ks[v] == (ref[v] if v in NS else np.uint64(0xFFFFFFFFFFFFFFFF)), v


@pytest.mark.parametrize("rw", [4, 8, 16])
def test_ns_rows_per_warp_instantiations_exact(rw, monkeypatch):
    """Each rows-per-warp instantiation of the sweep (tiles of 16 / 32 / 64 rows; the
    load picks one by plan size, TGA_NS_RW forces it): every candidate bit-exact on a
    ragged 20-customer partition and on cfg2, and the keys equal the oracle's."""
    _need_gpu()
    monkeypatch.setenv("TGA_NS_RW", str(rw))
    inst, sol = G.cvrp_small(1, spare=True)
    compare_fields(inst, G.random_partition(20, 5, 900 + rw, allow_empty=True).routes, NS, 0, label=f"rw{rw} cfg1")
    inst, sol = G.config("cfg2")
    n, _ = compare_fields(inst, sol.routes, NS, 0, label=f"rw{rw} cfg2")
    assert n > 0
    ns_keys_vs_oracle(inst, sol.routes, f"rw{rw} cfg2", parallel=True)
