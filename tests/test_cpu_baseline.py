"""The fast CPU baseline (cpu_baseline/, O(1) concatenation per candidate) is
pinned to the oracle: same best (score, canonical index) and the same number of
candidates for every variant, CVRP and VRPTW (TW-I), both score modes."""
import numpy as np
import pytest

import cpu_baseline as CB
import oracle as O
import tga_gen as G


def _cases():
    for seed in range(3):
        inst, sol = G.cvrp_small(seed, spare=True)
        yield f"cfg1-{seed}", inst, [sol.routes]
    inst, sol = G.cvrp_small(5, spare=False)
    rng = np.random.default_rng(7)
    yield "cfg1-partitions", inst, [G.random_partition(20, 4 + k % 3, 100 + k).routes for k in range(3)]
    inst, sol = G.gh_like(2, n=60, kind="R1")
    yield "vrptw-r1", inst, [sol.routes]
    inst, sol = G.gh_like(3, n=80, kind="R2")
    yield "vrptw-r2", inst, [sol.routes, G.perturb(sol, 10, 5).routes]


@pytest.mark.parametrize("mode", [0, 1])
def test_concat_baseline_equals_oracle(mode):
    for name, inst, sols in _cases():
        orc = O.Oracle.from_instance(inst)
        cb = CB.ConcatCPU.from_instance(inst)
        for routes in sols:
            Q = O.canonical_q(routes)
            for v in range(23):
                if v == 0 and inst.tw is not None:
                    continue
                m = orc.best_move(routes, v, mode=mode)
                found, score, u, vv, n = cb.best_move(routes, v, mode=mode)
                assert n == m.n_candidates, (name, v, n, m.n_candidates)
                assert found == m.found, (name, v)
                if found:
                    assert (score, u * Q + vv) == (m.score, m.u * Q + m.v), (name, v, score, u, vv, m)


def test_concat_baseline_row_restriction():
    inst, sol = G.cvrp_small(1, spare=True)
    cb = CB.ConcatCPU.from_instance(inst)
    Q = O.canonical_q(sol.routes)
    for v in (1, 2, 5, 11, 14):
        full = cb.best_move(sol.routes, v)
        parts = [cb.best_move(sol.routes, v, u_lo=lo, u_hi=min(Q, lo + 7)) for lo in range(0, Q, 7)]
        assert sum(p[4] for p in parts) == full[4]
        best = min(((p[1], p[2] * Q + p[3]) for p in parts if p[0]), default=None)
        assert best == ((full[1], full[2] * Q + full[3]) if full[0] else None)
