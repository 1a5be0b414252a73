"""Row-parallel driver of the CPU oracle (test infrastructure, SURVEY.md §8(d):
"process-parallel over u-row chunks on all host cores ... the full all-core run
provides the parity keys").

The oracle itself is unchanged: every job is one ``orc_best_move`` call over the
canonical rows [u_lo, u_hi) of one variant, run on a thread pool (ctypes releases
the GIL for the duration of the C call).  The canonical-order argmin over the
whole neighbourhood equals the lowest (score, u * Q + v) over the chunk argmins,
because each chunk keeps its first strictly smaller score in canonical order
(reading 5) -- the min is exact and order independent.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import oracle as O


def n_workers() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))


def best_keys(orc: O.Oracle, routes, variants, mode=0, chunks_per_variant=None, mask=None, wQ=10.0, wT=10.0):
    """{variant: (score, u * Q + v) or None, ...} over the full neighbourhood,
    plus {variant: total candidates}."""
    Q = O.canonical_q(routes)
    ptr_cust = orc._csr(routes)
    nw = n_workers()
    k = chunks_per_variant or max(1, min(Q, 4 * nw))
    bounds = [(Q * i // k, Q * (i + 1) // k) for i in range(k)]
    jobs = [(v, lo, hi) for v in variants for lo, hi in bounds if hi > lo]

    def run(job):
        v, lo, hi = job
        return v, orc.best_move(ptr_cust, v, mode=mode, wQ=wQ, wT=wT, u_lo=lo, u_hi=hi, mask=mask)

    best = {v: None for v in variants}
    count = {v: 0 for v in variants}
    with ThreadPoolExecutor(max_workers=nw) as ex:
        for v, m in ex.map(run, jobs):
            count[v] += m.n_candidates
            if m.found:
                key = (m.score, m.u * Q + m.v)
                if best[v] is None or key < best[v]:
                    best[v] = key
    return best, count
