"""GPU parity of every candidate's score and feasibility, not only the argmin.

tga_debug_eval_dump runs one evaluation with the DUMP instantiations of the
same kernels (the fused tile body / cell formulas, the generic tile kernel, the
three intra-route kernels) that also store each evaluated candidate's packed
key; the oracle's canonical enumeration (orc_enumerate_full: score, feasibility
and the TW-F ambiguity band of every candidate) is compared element by element.

Bars (BASELINE.json north_star; readings 4, 13):
  * integer (CVRP nint, VRPTW TW-I): every candidate's score bit-exact, the
    feasibility mask (Eq. 16b) identical, no extra candidate;
  * TW-F (real distances and times in fp32 vs the oracle's fp64): masks
    identical outside the oracle's ambiguity band, scores within the fp32
    summation bound of DESIGN.md reading 13, service starts within 1e-4
    relative; full-size cfg3f: the GPU's chosen candidate, looked up in the
    oracle, is optimal within the bound.
"""
import math

import numpy as np
import pytest

import oracle as O
import tga_gen as G
from tests import par_oracle
from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu

if gpu_available():
    from paper_2506_17357_b200 import tga as T
else:  # pragma: no cover
    T = None

NOKEY = np.uint64(0xFFFFFFFFFFFFFFFF)
INTER = list(range(1, 11))
INTRA_TW = list(range(11, 23))


def _need_gpu():
    if not gpu_available():
        pytest.skip("no CUDA device")


def decode_scores(keys, integer):
    """Vectorised score part of packed keys (order-preserving u32 image << 32)."""
    o = (np.asarray(keys, dtype=np.uint64) >> np.uint64(32)).astype(np.uint32)
    if integer:
        return (o ^ np.uint32(0x80000000)).view(np.int32).astype(np.float64)
    u = np.where(o & np.uint32(0x80000000), o ^ np.uint32(0x80000000), ~o).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def fp32_sum_bound(inst):
    """Largest fp32 rounding error of a candidate's distance delta: at most 8
    distances (Eq. 2: 4 new + 4 removed edges), each an fp32 value <= max c, are
    summed in fp32 -- 7 roundings of partial sums <= 8 max c, each <= 2^-24 of it
    (reading 13).  The operands are the same fp32 values on both sides."""
    return 7 * 2.0 ** -24 * 8 * float(np.max(inst.dist))


def compare_fields(inst, routes, variants, mode, flags=0, label=""):
    integer = np.issubdtype(np.asarray(inst.dist).dtype, np.integer)
    gi = T.Instance.from_gen(inst, score_mode=mode)
    gs = T.Solution(gi, routes)
    dump = gs.eval_dump(sum(1 << v for v in variants), flags)
    orc = O.Oracle.from_instance(inst)
    Q = O.canonical_q(routes)
    tol = fp32_sum_bound(inst)
    n_band = n_cmp = 0
    for v in variants:
        sc, us, vs, fe, band, _ = orc.enumerate_full(routes, v, mode)
        g = dump[v]
        got = g[us, vs]
        assert (got != 0).all(), f"{label} v{v}: {int((got == 0).sum())} candidates not evaluated"
        finite = np.isfinite(sc)
        gfin = got != NOKEY
        if integer or mode == 1:
            # mask: exactly the oracle's (feasible-only) / every candidate valid (penalised)
            assert (gfin == finite).all(), f"{label} v{v}: mask differs at {int((gfin != finite).sum())} candidates"
        else:
            ok = band | (gfin == finite)
            assert ok.all(), f"{label} v{v}: {int((~ok).sum())} mask flips outside the ambiguity band"
            n_band += int(band.sum())
        # no candidate outside the canonical space carries a valid key
        assert int((g != 0).sum() - (g == NOKEY).sum()) == int(gfin.sum()), f"{label} v{v}: extra candidates"
        both = gfin & finite
        gsc = decode_scores(got[both], integer)
        if integer:
            np.testing.assert_array_equal(gsc, sc[both], err_msg=f"{label} v{v}")
        else:
            assert np.abs(gsc - sc[both]).max(initial=0) <= tol, f"{label} v{v}: score beyond the fp32 bound"
        n_cmp += int(both.sum())
    return n_cmp, n_band


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("seed", range(3))
def test_cfg1_fields_exact(seed, mode):
    """Config 1 (CVRP, 20 customers, spare route): every candidate of all 23
    variants -- fused tile kernel + intra warps (feasible-only) or the generic
    tile kernel + intra kernel (penalised)."""
    _need_gpu()
    inst, sol = G.cvrp_small(seed, spare=True)
    n, _ = compare_fields(inst, sol.routes, list(range(23)), mode, label=f"cfg1 s{seed}")
    assert n > 0
    part = G.random_partition(20, 4, 300 + seed, allow_empty=True)   # infeasible / empty routes
    compare_fields(inst, part.routes, list(range(23)), mode, label=f"cfg1-rand s{seed}")


@pytest.mark.parametrize("flags", [1, 2])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("kind", ["R1", "R2"])
def test_vrptw200_twi_fields_exact(kind, mode, flags):
    """200-customer VRPTW, TW-I: every candidate of the 22 variants, with the
    warp-scan (flags 1) and the walking (flags 2) intra kernel; a perturbed
    (warping, overloaded) state too."""
    _need_gpu()
    inst, sol = G.gh_like(3, n=200, kind=kind)
    variants = INTER + INTRA_TW
    compare_fields(inst, sol.routes, variants, mode, flags, f"{kind}")
    compare_fields(inst, G.perturb(sol, 25, 4).routes, variants, mode, flags, f"{kind}-perturbed")


@pytest.mark.parametrize("flags", [1, 2])
@pytest.mark.parametrize("kind", ["R1", "R2"])
def test_vrptw200_twf_masks_and_scores(kind, flags):
    """TW-F (fp32 GPU, fp64 oracle), feasible-only: masks identical outside the
    oracle-computed ambiguity band (counted), scores within the fp32 summation
    bound, for every candidate."""
    _need_gpu()
    inst, sol = G.gh_like(4, n=200, kind=kind, mode="twf")
    for routes in (sol.routes, G.perturb(sol, 25, 5).routes):
        n, nb = compare_fields(inst, routes, INTER + INTRA_TW, 0, flags, f"twf {kind}")
        assert n > 0
        print(f"twf {kind} flags {flags}: {n} feasible candidates compared, {nb} in the band")


@pytest.mark.parametrize("kind", ["R1", "R2"])
def test_twf_service_starts_and_warps(kind):
    """TW-F attribute records: the service start at every slot (derived from the
    prefix record, start = T_E + T_D - T_V - s) within 1e-4 relative of the
    oracle's fp64 simulation; prefix / suffix time warps and loads likewise
    (loads exact)."""
    _need_gpu()
    inst, sol = G.gh_like(6, n=200, kind=kind, mode="twf")
    for routes in (sol.routes, G.perturb(sol, 30, 6).routes):
        gs = T.Solution(T.Instance.from_gen(inst), routes)
        a, b = gs.attributes(), O.Oracle.from_instance(inst).attributes(routes)
        for k in ("pre_L", "suf_L"):
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)
        for k in ("start", "pre_TV", "suf_TV", "pre_D", "suf_D"):
            np.testing.assert_allclose(a[k], b[k], rtol=1e-4, atol=1e-4, err_msg=k)


def test_cfg3f_full_size_best_moves():
    """Full-size TW-F (cfg3f: GH R1-like, 1000 customers, real distances): for every
    variant the candidate the GPU picks is, scored by the oracle, feasible and
    optimal within the fp32 bound; the GPU's score equals the oracle's at that
    index within the bound; when the oracle's best is separated from every other
    candidate by more than twice the bound, the index is the oracle's."""
    _need_gpu()
    inst, sol = G.config("cfg3f")
    routes = sol.routes
    gs = T.Solution(T.Instance.from_gen(inst), routes)
    variants = INTER + INTRA_TW
    gs.eval(sum(1 << v for v in variants))
    keys = gs.keys()
    orc = O.Oracle.from_instance(inst)
    Q = O.canonical_q(routes)
    tol = fp32_sum_bound(inst)
    R = len(routes)
    off = np.concatenate([[0], np.cumsum([len(r) + 1 for r in routes])])
    for v in variants:
        sc, us, vs, best = orc.enumerate(routes, v)
        if not best.found:
            assert int(keys[v]) == int(NOKEY), v
            continue
        s_gpu, idx = T.decode_key(int(keys[v]), False)
        u, w = idx // Q, idx % Q
        ra = int(np.searchsorted(off, u, side="right") - 1)
        rb = int(np.searchsorted(off, w, side="right") - 1)
        at = orc.score_candidate(routes, v, ra, u - off[ra], rb, w - off[rb])
        assert at.found and math.isfinite(at.score), (v, "GPU choice infeasible for the oracle")
        assert abs(at.score - best.score) <= tol, (v, at.score, best.score)
        assert abs(s_gpu - at.score) <= tol, (v, s_gpu, at.score)
        fin = np.sort(sc[np.isfinite(sc)])
        if len(fin) > 1 and fin[1] - fin[0] > 2 * tol:
            assert idx == best.u * Q + best.v, v
