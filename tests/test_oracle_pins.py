"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names the passage it checks.  P:n = PAPER.md line n (the paper is
not read at run time; the citation is for the reader).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import tga_gen as G
from tests import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _orc(coords, demand, capacity, tw=None):
    dist = G.euclid_nint(np.asarray(coords))
    return O.Oracle(dist, np.asarray(demand), capacity, tw), dist


# ---------------------------------------------------------------- hand-worked
@pytest.mark.parametrize("ex", json.load(open(os.path.join(GOLD, "hand_worked.json")))["examples"],
                         ids=lambda e: e["name"])
def test_hand_worked_deltas(ex):
    """SURVEY §8(c) hand-worked deltas (2-opt, relocate, 2-opt*, swap)."""
    orc, _ = _orc(ex["coords"], ex["demand"], ex["capacity"])
    assert orc.cost(ex["routes"])[0] == ex["cost_before"]
    m = orc.score_candidate(ex["routes"], ex["variant"], ex["ra"], ex["pa"], ex["rb"], ex["pb"])
    assert m.found and m.feasible and m.dD == ex["delta"] and m.score == ex["delta"]
    # canonical slot ids worked by hand (golden "u", "v", "Q")
    assert (m.u, m.v) == (ex["u"], ex["v"]) and O.canonical_q(ex["routes"]) == ex["Q"]
    sc, us, vs, _ = orc.enumerate(ex["routes"], ex["variant"])
    assert (ex["delta"], ex["u"], ex["v"]) in set(zip(sc.tolist(), us.tolist(), vs.tolist()))
    new = orc.apply(ex["routes"], ex["variant"], ex["ra"], ex["pa"], ex["rb"], ex["pb"])
    assert new == ex["routes_after"]
    assert orc.cost(new)[0] == ex["cost_after"]
    # the operator's best move can only be at least as good
    best = orc.best_move(ex["routes"], ex["variant"])
    assert best.score <= ex["delta"]


@pytest.mark.parametrize("ex", json.load(open(os.path.join(GOLD, "time_windows.json")))["examples"],
                         ids=lambda e: e["name"])
def test_hand_worked_schedules(ex):
    """P:49-51 arrival/wait/service; time warp P:211; SPEC S:135 corrected."""
    dist = np.asarray(ex["dist"], dtype=np.float64)
    n = dist.shape[0]
    orc = O.Oracle(dist, np.zeros(n, dtype=np.int64), 100, np.asarray(ex["tw"], dtype=np.float64))
    D, L, TV, arr, st = orc.route_eval(ex["route"])
    assert D == ex["D"] and TV == ex["TV"]
    assert list(arr) == ex["arrival"] and list(st) == ex["start"]


# ---------------------------------------------------------------- closed forms
def _closed_counts(lengths):
    """Closed-form neighbourhood sizes (SPEC S:282 form)."""
    R = len(lengths)
    c = {}
    pairs = [(a, b) for a in range(R) for b in range(R) if a != b]
    c[O.V_2OPT_STAR] = sum((lengths[a] + 1) * (lengths[b] + 1) for a, b in pairs if a < b)
    for n, v in O.V_RELOC.items():
        c[v] = sum(max(lengths[a] - n + 1, 0) * (lengths[b] + 1) for a, b in pairs)
    for (n1, n2), v in O.V_SWAP.items():
        c[v] = sum(max(lengths[a] - n1 + 1, 0) * max(lengths[b] - n2 + 1, 0)
                   for a, b in pairs if (a < b or n1 != n2))
    c[O.V_2OPT] = sum(L * (L - 1) // 2 for L in lengths)
    for n, v in O.V_IRELOC.items():
        c[v] = sum(max(L - n + 1, 0) * max(L - n, 0) for L in lengths)
    for (n1, n2), v in O.V_ISWAP.items():
        tot = 0
        for L in lengths:
            M = L - n1 - n2 + 1
            tot += M * (M + 1) // 2 if M >= 1 else 0
        c[v] = tot
    # reversed segments: the same candidate spaces as or-opt N and cross (N, N)
    for n, v in O.V_RELOC_REV.items():
        c[v] = c[O.V_RELOC[n]]
    for n, v in O.V_CROSS_REV.items():
        c[v] = c[O.V_SWAP[(n, n)]]
    return c


def test_counts_cfg1_table():
    """SURVEY §8(a) 'Neighbourhood sizes' row cfg1 (n=20, R=4, equal routes)."""
    inst, sol = G.cvrp_small(0)
    sol = G.Solution([list(range(1 + 5 * r, 6 + 5 * r)) for r in range(4)])
    orc = O.Oracle.from_instance(inst)
    cnt = {v: orc.best_move(sol, v).n_candidates for v in range(O.N_VARIANTS)}
    assert cnt[O.V_2OPT_STAR] == 216
    assert cnt[O.V_RELOC[1]] == 360
    assert cnt[O.V_SWAP[(1, 1)]] == 150
    inter = [O.V_2OPT_STAR] + list(O.V_RELOC.values()) + list(O.V_SWAP.values())
    assert sum(cnt[v] for v in inter) == 1944
    intra = [O.V_2OPT] + list(O.V_IRELOC.values()) + [O.V_ISWAP[(1, 1)]]
    assert sum(cnt[v] for v in intra) == 232


@pytest.mark.parametrize("seed", range(6))
def test_counts_closed_form_random(seed):
    """Candidate counts == closed forms for ragged routes incl. empty ones."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(6, 14))
    inst, _ = G.cvrp_small(seed, n=n)
    sol = G.random_partition(n, int(rng.integers(2, 5)), seed, allow_empty=True)
    orc = O.Oracle.from_instance(inst)
    closed = _closed_counts([len(r) for r in sol.routes])
    for v in range(O.N_VARIANTS):
        assert orc.best_move(sol, v).n_candidates == closed[v], v


# ---------------------------------------------------------------- brute force
BRUTE_OPS = ([("2opt*", 1, 1, O.V_2OPT_STAR), ("2opt", 1, 1, O.V_2OPT)]
             + [("relocate", n, 1, v) for n, v in O.V_RELOC.items()]
             + [("swap", a, b, v) for (a, b), v in O.V_SWAP.items()]
             + [("intra_relocate", n, 1, v) for n, v in O.V_IRELOC.items()]
             + [("intra_swap", a, b, v) for (a, b), v in O.V_ISWAP.items()]
             + [("relocate_rev", n, 1, v) for n, v in O.V_RELOC_REV.items()]
             + [("swap_rev", n, n, v) for n, v in O.V_CROSS_REV.items()])


def _tiny(seed, tw):
    rng = np.random.default_rng(77 + seed)
    n = int(rng.integers(4, 9))
    coords = np.vstack([[50, 50], rng.integers(0, 101, size=(n, 2))])
    dist = G.euclid_nint(coords)
    demand = np.concatenate([[0], rng.integers(1, 21, size=n)]).astype(np.int32)
    twa = None
    if tw:
        twa = np.zeros((n + 1, 3))
        twa[0] = (0, 600, 0)
        e = rng.integers(0, 200, size=n)
        twa[1:, 0] = e
        twa[1:, 1] = e + rng.integers(20, 300, size=n)
        twa[1:, 2] = 10
    sol = G.random_partition(n, int(rng.integers(2, 4)), 500 + seed, allow_empty=True)
    cap = int(rng.integers(30, 90))
    return dist, demand, twa, cap, sol


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("tw", [False, True])
@pytest.mark.parametrize("mode", [0, 1])
def test_brute_force_neighbourhood(seed, tw, mode):
    """Every operator: multiset of scores == brute force; best == min."""
    dist, demand, twa, cap, sol = _tiny(seed, tw)
    orc = O.Oracle(dist, demand, cap, twa)
    d = dist.tolist()
    t = None if twa is None else twa.tolist()
    _brute_vs_oracle(orc, d, demand.tolist(), t, cap, sol.routes, mode)


def _brute_vs_oracle(orc, d, demand, t, cap, routes, mode):
    """Every variant: the multiset of (score, u, v) triples of the oracle's canonical
    enumeration == the brute-force neighbours with their canonical slot pair named
    from the definition (brute.slot_id); the oracle's best == the lowest (score,
    u * Q + v) of the brute force (reading 5)."""
    Q = O.canonical_q(routes)
    for op, n1, n2, var in BRUTE_OPS:
        bt = brute.scores(d, demand, t, cap, routes, op, n1, n2, mode, with_index=True)
        sc, us, vs, best = orc.enumerate(routes, var, mode)
        got = sorted(zip(sc.tolist(), us.tolist(), vs.tolist()))
        assert sorted(bt) == got, (op, n1, n2)
        bb = brute.best(bt, Q)
        assert best.found == (bb is not None), (op, n1, n2)
        if bb is not None:
            assert (best.score, best.u * Q + best.v) == bb, (op, n1, n2)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("spare", [False, True])
@pytest.mark.parametrize("mode", [0, 1])
def test_cfg1_oracle_vs_brute_force(seed, spare, mode):
    """BASELINE config 1 ("full 2-opt/2-opt*/relocate/swap sweep vs brute force"):
    20 customers, 4 routes, Q=100 -- every variant of the oracle against the
    independent brute force, scores AND canonical indices."""
    inst, sol = G.cvrp_small(seed, spare=spare)
    orc = O.Oracle.from_instance(inst)
    _brute_vs_oracle(orc, inst.dist.tolist(), inst.demand.tolist(), None, inst.capacity, sol.routes, mode)


@pytest.mark.parametrize("seed", range(3))
def test_cfg1_random_partitions_vs_brute_force(seed):
    """Config-1 instances with ragged, empty and overloaded routes (both modes)."""
    inst, _ = G.cvrp_small(seed)
    sol = G.random_partition(20, 3 + seed, 900 + seed, allow_empty=True)
    orc = O.Oracle.from_instance(inst)
    for mode in (0, 1):
        _brute_vs_oracle(orc, inst.dist.tolist(), inst.demand.tolist(), None, inst.capacity, sol.routes, mode)


@pytest.mark.parametrize("seed", range(5))
def test_tie_break_order_independent(seed):
    """Reading 5: lowest (score, index); shuffling enumeration order changes nothing."""
    inst, sol = G.cvrp_small(seed)
    # many ties: unit grid distances
    orc = O.Oracle.from_instance(inst)
    Q = O.canonical_q(sol)
    rng = np.random.default_rng(seed)
    for var in range(O.N_VARIANTS):
        sc, us, vs, best = orc.enumerate(sol, var, mode=1)
        if not len(sc):
            continue
        keys = [(s, u * Q + v) for s, u, v in zip(sc, us, vs)]
        perm = rng.permutation(len(keys))
        shuffled = min(keys[i] for i in perm)
        assert shuffled == (best.score, best.u * Q + best.v)
        assert all(k1[1] < k2[1] for k1, k2 in zip(keys, keys[1:])), "canonical order"


# ---------------------------------------------------------------- textbook reductions
def test_two_opt_is_tsp_formula():
    """R=1, Q=inf, no TW: 2-opt delta == c(a,c)+c(b,d)-c(a,b)-c(c,d)."""
    rng = np.random.default_rng(3)
    coords = rng.integers(0, 1000, size=(13, 2))
    dist = G.euclid_nint(coords)
    orc = O.Oracle(dist, np.ones(13, dtype=np.int64), 10 ** 9)
    route = list(rng.permutation(np.arange(1, 13)))
    nodes = [0] + route + [0]
    for i in range(1, 13):
        for j in range(i + 1, 13):
            m = orc.score_candidate([route], O.V_2OPT, 0, i, 0, j)
            a, b, c, d = nodes[i - 1], nodes[i], nodes[j], nodes[j + 1]
            assert m.dD == dist[a, c] + dist[b, d] - dist[a, b] - dist[c, d]


def test_intra_relocate_is_insertion_formula():
    """R=1: relocating one node = removal gain + classic insertion cost."""
    rng = np.random.default_rng(4)
    coords = rng.integers(0, 1000, size=(10, 2))
    dist = G.euclid_nint(coords)
    orc = O.Oracle(dist, np.ones(10, dtype=np.int64), 10 ** 9)
    route = list(rng.permutation(np.arange(1, 10)))
    nodes = [0] + route + [0]
    L = len(route)
    for u in range(1, L + 1):
        for v in range(0, L + 1):
            if u - 1 <= v <= u:
                continue
            m = orc.score_candidate([route], O.V_IRELOC[1], 0, u, 0, v)
            x = nodes[u]
            rem = dist[nodes[u - 1], nodes[u + 1]] - dist[nodes[u - 1], x] - dist[x, nodes[u + 1]]
            ins = dist[nodes[v], x] + dist[x, nodes[v + 1]] - dist[nodes[v], nodes[v + 1]]
            assert m.dD == rem + ins


def test_two_opt_star_is_edge_exchange():
    """Two routes, no capacity/TW: 2-opt* delta == c(u,v+1)+c(v,u+1)-c(u,u+1)-c(v,v+1)."""
    rng = np.random.default_rng(5)
    coords = rng.integers(0, 1000, size=(11, 2))
    dist = G.euclid_nint(coords)
    orc = O.Oracle(dist, np.ones(11, dtype=np.int64), 10 ** 9)
    ra, rb = [1, 2, 3, 4, 5], [6, 7, 8, 9, 10]
    na, nb = [0] + ra + [0], [0] + rb + [0]
    for u in range(0, 6):
        for v in range(0, 6):
            m = orc.score_candidate([ra, rb], O.V_2OPT_STAR, 0, u, 1, v)
            exp = dist[na[u], nb[v + 1]] + dist[nb[v], na[u + 1]] - dist[na[u], na[u + 1]] \
                - dist[nb[v], nb[v + 1]]
            assert m.dD == exp


# ---------------------------------------------------------------- TW special cases
def test_unbounded_windows_never_warp():
    """All windows [0, inf) => TV == 0."""
    inst, sol = G.x_like(0, n=60, target_routes=5)
    tw = np.zeros((61, 3))
    tw[:, 1] = 1e12
    tw[1:, 2] = 7
    orc = O.Oracle(inst.dist, inst.demand, inst.capacity, tw)
    for r in sol.routes:
        assert orc.route_eval([0] + r + [0])[2] == 0.0


def test_appointment_windows_closed_form():
    """l_i = e_i (appointments): start_k = e_k, warp_k = max(a_k - e_k, 0)."""
    rng = np.random.default_rng(9)
    n = 12
    dist = rng.integers(1, 50, size=(n + 1, n + 1)).astype(np.float64)
    dist = np.floor((dist + dist.T) / 2)
    np.fill_diagonal(dist, 0)
    tw = np.zeros((n + 1, 3))
    tw[0] = (0, 10 ** 6, 0)
    tw[1:, 0] = tw[1:, 1] = np.sort(rng.integers(0, 400, size=n))
    tw[1:, 2] = 5
    orc = O.Oracle(dist, np.zeros(n + 1, dtype=np.int64), 100, tw)
    route = list(range(1, n + 1))
    D, L, TV, arr, st = orc.route_eval([0] + route + [0])
    exp_tv, prev, tprev = 0.0, 0, 0.0
    for k, c in enumerate(route, start=1):
        a = tprev + tw[prev, 2] + dist[prev, c]
        assert arr[k] == a and st[k] == tw[c, 0]
        exp_tv += max(a - tw[c, 0], 0.0)
        prev, tprev = c, tw[c, 0]
    assert TV == exp_tv


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("name", ["cvrp", "twi"])
def test_descent_invariants(name):
    """Apply best moves: delta == cost change (exact), coverage, capacity
    (Alg. A2)."""
    if name == "cvrp":
        inst, sol = G.x_like(1, n=80, target_routes=6)
    else:
        inst, sol = G.gh_like(1, n=80, kind="R1")
    orc = O.Oracle.from_instance(inst)
    routes = sol.routes
    D0, LV0, TV0 = orc.cost(routes)
    assert LV0 == 0 and TV0 == 0, "state A is feasible by construction"
    variants = [v for v in range(O.N_VARIANTS) if not (inst.tw is not None and v == O.V_2OPT)]
    for _ in range(6):
        best = orc.best_over(routes, variants)
        if best is None or not best.score < 0:
            break
        new = orc.apply(routes, best.variant, best.route_a, best.pos_a, best.route_b, best.pos_b)
        D1, LV1, TV1 = orc.cost(new)
        assert D1 - D0 == best.dD == best.score
        assert LV1 == 0 and TV1 == 0
        assert sorted(c for r in new for c in r) == list(range(1, inst.n_nodes))
        assert len(new) == len(routes)
        routes, D0 = new, D1


@pytest.mark.parametrize("ex", json.load(open(os.path.join(GOLD, "attributes.json")))["examples"],
                         ids=lambda e: e["name"])
def test_attributes_hand_worked(ex):
    """orc_attributes against hand-worked prefix / suffix records (golden
    attributes.json): D, L and T_V of every prefix [0..p] and suffix [p..L+1]
    (the suffix simulated from e of its first node), and the service starts."""
    dist = np.asarray(ex["dist"], dtype=np.float64)
    orc = O.Oracle(dist, np.asarray(ex["demand"], dtype=np.int64), 100, np.asarray(ex["tw"], dtype=np.float64))
    at = orc.attributes(ex["routes"])
    for k in ("pre_D", "pre_L", "pre_TV", "suf_D", "suf_L", "suf_TV", "start"):
        assert at[k].tolist() == ex[k], k


def test_attributes_prefix_suffix():
    """Prefix/suffix records: D/L additive, full-route values match route_eval."""
    inst, sol = G.gh_like(2, n=60, kind="R2")
    orc = O.Oracle.from_instance(inst)
    at = orc.attributes(sol)
    q = 0
    for r in sol.routes:
        nodes = [0] + r + [0]
        D, L, TV, arr, st = orc.route_eval(nodes)
        assert at["pre_D"][q] == 0 and at["suf_D"][q] == D and at["suf_L"][q] == L
        for p in range(len(r) + 1):
            assert at["pre_D"][q + p] + (at["suf_D"][q + p]) == D
            assert at["start"][q + p] == st[p]
        q += len(r) + 1


# ---------------------------------------------------------------- edge-based (ETGA) neighbourhood
def _mask_by_definition(dist, theta):
    """Reading 21 retyped independently of oracle.granular_mask: rank the other
    customers of i by (distance, id) with numpy's stable lexsort."""
    n = dist.shape[0]
    M = np.zeros((n, n), dtype=bool)
    for i in range(1, n):
        js = np.array([j for j in range(1, n) if j != i])
        order = np.lexsort((js, dist[i, js]))
        for j in js[order[:theta]]:
            M[i, j] = M[j, i] = True
    M[0, :] = M[:, 0] = True
    return M


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("tw", [False, True])
@pytest.mark.parametrize("theta", [1, 2])
def test_edge_based_neighbourhood_brute_force(seed, tw, theta):
    """ETGA: the masked oracle's best score and candidate count equal
    the brute-force neighbours whose key node pair the mask keeps; the mask
    equals its definition; intra-route variants are unmasked."""
    dist, demand, twa, cap, sol = _tiny(seed, tw)
    M = O.granular_mask(dist, theta)
    np.testing.assert_array_equal(M.astype(bool), _mask_by_definition(dist, theta))
    orc = O.Oracle(dist, demand, cap, twa)
    d = dist.tolist()
    t = None if twa is None else twa.tolist()
    for op, n1, n2, var in BRUTE_OPS:
        for mode in (0, 1):
            bs = brute.scores(d, demand.tolist(), t, cap, sol.routes, op, n1, n2, mode, mask=M)
            m = orc.best_move(sol, var, mode, mask=M)
            assert m.n_candidates == len(bs), (op, n1, n2, mode)
            finite = [x for x in bs if x != float("inf")]
            assert m.found == bool(finite), (op, n1, n2, mode)
            if finite:
                assert m.score == min(finite), (op, n1, n2, mode)


def test_edge_based_full_mask_is_the_full_neighbourhood():
    """theta >= n - 1 keeps every pair: ETGA == NTGA, index included."""
    inst, sol = G.cvrp_small(2, spare=True)
    orc = O.Oracle.from_instance(inst)
    M = O.granular_mask(inst.dist, inst.dist.shape[0])
    assert M.all() or (M | np.eye(M.shape[0], dtype=np.uint8)).all()
    for v in range(O.N_VARIANTS):
        a, b = orc.best_move(sol, v), orc.best_move(sol, v, mask=M)
        assert (a.found, a.score, a.u, a.v, a.n_candidates) == (b.found, b.score, b.u, b.v, b.n_candidates)


# ---------------------------------------------------------------- row-parallel driver
@pytest.mark.parametrize("tw", [False, True])
def test_parallel_oracle_equals_serial(tw):
    """tests/par_oracle (row chunks on a thread pool, min over chunk argmins) ==
    one serial canonical enumeration: same best key and candidate count for every
    variant, including uneven chunkings (SURVEY §8(d) all-core oracle)."""
    from tests import par_oracle
    if tw:
        inst, sol = G.gh_like(3, n=90, kind="R1")
        sol = G.perturb(sol, 10, 3)
    else:
        inst, sol = G.x_like(2, n=120, target_routes=6)
    orc = O.Oracle.from_instance(inst)
    Q = O.canonical_q(sol)
    variants = [v for v in range(O.N_VARIANTS) if not (tw and v == O.V_2OPT)]
    for mode in (0, 1):
        for chunks in (None, 7, Q):
            best, count = par_oracle.best_keys(orc, sol.routes, variants, mode, chunks_per_variant=chunks)
            for v in variants:
                m = orc.best_move(sol, v, mode)
                assert count[v] == m.n_candidates
                assert best[v] == ((m.score, m.u * Q + m.v) if m.found else None), (v, mode, chunks)


@pytest.mark.parametrize("seed", range(6))
def test_enumerate_full_feasibility_and_band(seed):
    """orc_enumerate_full's per-candidate feasibility flag and ambiguity-band flag
    (reading 13) == the brute force's own simulation of every neighbour,
    on windows whose deadlines coincide with reference starts (band cases occur)."""
    dist, demand, twa, cap, sol = _tiny(seed, True)
    # pull some deadlines onto the earliest starts of the current routes (exact ties)
    orc0 = O.Oracle(dist, demand, cap, twa)
    for r in [max(sol.routes, key=len)]:
        _, _, _, _, st = orc0.route_eval([0] + r + [0])
        for k, c in enumerate(r, start=1):
            if k % 2:
                twa[c, 1] = st[k]
    orc = O.Oracle(dist, demand, cap, twa)
    d, t = dist.tolist(), twa.tolist()
    nb = 0
    for op, n1, n2, var in BRUTE_OPS:
        for mode in (0, 1):
            bt = brute.scores(d, demand.tolist(), t, cap, sol.routes, op, n1, n2, mode, with_index="full")
            sc, us, vs, fe, bd, _ = orc.enumerate_full(sol, var, mode)
            got = sorted(zip(sc.tolist(), us.tolist(), vs.tolist(), fe.tolist(), bd.tolist()))
            assert sorted(bt) == got, (op, n1, n2, mode)
            nb += int(bd.sum())
    assert nb > 0, "the instance must exercise the band"


# ---------------------------------------------------------------- VRPSPDTW loads
PD_GOLD = json.load(open(os.path.join(GOLD, "pickup_delivery.json")))["examples"]


@pytest.mark.parametrize("ex", PD_GOLD, ids=lambda e: e["name"])
def test_pickup_delivery_hand_worked(ex):
    """Hand-worked maximum loads (golden, P:49-50 and Eq. 3a-d): the
    oracle's L_M of the route, and through it the capacity test: feasible iff
    L_M <= Q (the 'capacity-order' pair: the same customers, one order over Q = 16,
    the other within it)."""
    n = len(ex["demand"])
    coords = [[50, 50]] + [[10 * k, 5 * k] for k in range(1, n)]
    dist = G.euclid_nint(np.asarray(coords))
    orc = O.Oracle(dist, np.asarray(ex["demand"]), 16, None, np.asarray(ex["pickup"]))
    assert orc.seq_lmax([0] + ex["route"] + [0]) == ex["lmax"]
    assert max(ex["loads"]) == ex["lmax"]
    D, L, TV = None, None, None
    cost = orc.cost([ex["route"]])
    assert cost[1] == max(ex["lmax"] - 16, 0)       # load excess of the single route


def _pd_tiny(seed, tw=True):
    rng = np.random.default_rng(900 + seed)
    dist, demand, twa, cap, sol = _tiny(seed, tw)
    n = len(demand) - 1
    pickup = np.concatenate([[0], rng.integers(0, 21, size=n)]).astype(np.int32)
    demand = demand.copy()
    demand[1:] = rng.integers(0, 21, size=n)
    return dist, demand, pickup, twa, cap, sol


@pytest.mark.parametrize("seed", range(6))
def test_pickup_delivery_closed_forms(seed):
    """seq_lmax against three closed forms (no running simulation): without
    pickups it is the delivery sum (Eq. 3e-f); without deliveries the pickup sum;
    in general max over k of (deliveries of the customers after the first k +
    pickups of the first k)."""
    dist, demand, pickup, twa, cap, sol = _pd_tiny(seed)
    rng = np.random.default_rng(seed)
    for r in sol.routes + [list(rng.permutation(np.arange(1, len(demand))))]:
        r = [int(c) for c in r]
        nodes = [0] + r + [0]
        zero = np.zeros_like(pickup)
        assert O.Oracle(dist, demand, cap, None, zero).seq_lmax(nodes) == sum(int(demand[c]) for c in r)
        assert O.Oracle(dist, zero, cap, None, pickup).seq_lmax(nodes) == sum(int(pickup[c]) for c in r)
        exp = max(sum(int(demand[c]) for c in r[k:]) + sum(int(pickup[c]) for c in r[:k]) for k in range(len(r) + 1))
        assert O.Oracle(dist, demand, cap, None, pickup).seq_lmax(nodes) == exp


@pytest.mark.parametrize("seed", range(6))
def test_pickup_delivery_concatenation_rule(seed):
    """Eq. 3a-d -- the method's O(1) concatenation of (L_I, L_O, L_M),
    written here from the paper -- reaches the oracle's simulated L_M for every
    split of random sequences into two and three parts (the associativity the
    prefix / suffix records rely on)."""
    dist, demand, pickup, twa, cap, sol = _pd_tiny(seed)
    orc = O.Oracle(dist, demand, cap, None, pickup)
    rng = np.random.default_rng(50 + seed)

    def single(k):
        return (int(demand[k]), int(pickup[k]), max(int(demand[k]), int(pickup[k])))   # Eq. 3a

    def cat(a, b):   # Eq. 3b-d
        return (a[0] + b[0], a[1] + b[1], max(a[2] + b[0], a[1] + b[2]))

    def rec(seq):
        r = single(seq[0])
        for k in seq[1:]:
            r = cat(r, single(k))
        return r

    for _ in range(20):
        seq = [int(x) for x in rng.permutation(np.arange(1, len(demand)))[: int(rng.integers(1, len(demand)))]]
        full = rec(seq)
        assert full[2] == orc.seq_lmax(seq)
        for i in range(1, len(seq)):
            assert cat(rec(seq[:i]), rec(seq[i:]))[2] == orc.seq_lmax(seq)
            for j in range(i + 1, len(seq)):
                assert cat(cat(rec(seq[:i]), rec(seq[i:j])), rec(seq[j:]))[2] == orc.seq_lmax(seq)


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("mode", [0, 1])
def test_pickup_delivery_brute_force_neighbourhood(seed, mode):
    """VRPSPDTW (pickups + time windows): every variant's (score, u, v) multiset ==
    the brute force, whose load is the max-over-k closed form; best == min.
    2-opt is excluded: the paper applies it to the CVRP only."""
    dist, demand, pickup, twa, cap, sol = _pd_tiny(seed, tw=True)
    orc = O.Oracle(dist, demand, cap, twa, pickup)
    Q = O.canonical_q(sol.routes)
    for op, n1, n2, var in BRUTE_OPS:
        if var == O.V_2OPT:
            continue
        bt = brute.scores(dist.tolist(), demand.tolist(), twa.tolist(), cap, sol.routes, op, n1, n2, mode,
                          with_index=True, pickup=pickup.tolist())
        sc, us, vs, best = orc.enumerate(sol.routes, var, mode)
        assert sorted(bt) == sorted(zip(sc.tolist(), us.tolist(), vs.tolist())), (op, n1, n2)
        bb = brute.best(bt, Q)
        assert best.found == (bb is not None)
        if bb is not None:
            assert (best.score, best.u * Q + best.v) == bb, (op, n1, n2)


def test_pickup_delivery_changes_feasibility():
    """The pickups matter: on a JD-like instance some candidates that are feasible
    with the deliveries alone (CVRP / VRPTW loads) are infeasible with the pickups,
    and the counts of feasible candidates differ."""
    inst, sol = G.jd_like(1, n=60)
    with_p = O.Oracle.from_instance(inst)
    without = O.Oracle(inst.dist, inst.demand, inst.capacity, inst.tw)
    diff = 0
    for v in (O.V_2OPT_STAR, O.V_RELOC[1], O.V_SWAP[(1, 1)]):
        a = np.isfinite(with_p.enumerate(sol.routes, v)[0]).sum()
        b = np.isfinite(without.enumerate(sol.routes, v)[0]).sum()
        assert a <= b
        diff += b - a
    assert diff > 0
