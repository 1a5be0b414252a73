"""CPU oracle for full-neighbourhood VRP move evaluation -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2506_17357_b200``) never imports it and shares no code with it.

``tga_oracle.c`` is the plain C definition (see its header); this module is
the ctypes marshalling around it plus a tiny driver for lockstep runs.
Parity status of every function is listed in DESIGN.md ("Oracle pins").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tga_oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")

# variant ids (tie-break rank); mirrored from the C enum, checked against the
# ABI's table by tests/test_abi_load.py
V_2OPT, V_2OPT_STAR = 0, 1
V_RELOC = {1: 2, 2: 3, 3: 4}
V_SWAP = {(1, 1): 5, (1, 2): 6, (1, 3): 7, (2, 2): 8, (2, 3): 9, (3, 3): 10}
V_IRELOC = {1: 11, 2: 12, 3: 13}
V_ISWAP = {(a, b): 14 + 3 * (a - 1) + (b - 1) for a in (1, 2, 3) for b in (1, 2, 3)}
# reversed-segment variants, ranked after the standard 23
V_RELOC_REV = {2: 23, 3: 24}
V_CROSS_REV = {2: 25, 3: 26}
N_VARIANTS = 27
N_STANDARD = 23
INTRA = {V_2OPT} | set(V_IRELOC.values()) | set(V_ISWAP.values())


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no OpenMP, single-threaded)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB,
                               _SRC, "-lm"])
    return _LIB


class _Inst(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("C", C.POINTER(C.c_double)),
                ("demand", C.POINTER(C.c_int64)), ("e", C.POINTER(C.c_double)),
                ("l", C.POINTER(C.c_double)), ("s", C.POINTER(C.c_double)),
                ("Q", C.c_int64), ("pickup", C.POINTER(C.c_int64))]


class _Move(C.Structure):
    _fields_ = [("score", C.c_double), ("dD", C.c_double), ("dLV", C.c_double),
                ("dTV", C.c_double), ("variant", C.c_int32), ("u", C.c_int32),
                ("v", C.c_int32), ("route_a", C.c_int32), ("pos_a", C.c_int32),
                ("route_b", C.c_int32), ("pos_b", C.c_int32), ("found", C.c_int32),
                ("feasible", C.c_int32), ("n_candidates", C.c_int64)]


@dataclass
class Move:
    variant: int
    score: float
    dD: float
    dLV: float
    dTV: float
    u: int
    v: int
    route_a: int
    pos_a: int
    route_b: int
    pos_b: int
    found: bool
    feasible: bool
    n_candidates: int


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        _lib.orc_best_move.argtypes = [P(_Inst), C.c_int32, P(C.c_int32), P(C.c_int32),
                                       C.c_int32, C.c_int32, C.c_double, C.c_double,
                                       C.c_int32, C.c_int32, P(_Move)]
        _lib.orc_best_move_masked.argtypes = [P(_Inst), C.c_int32, P(C.c_int32), P(C.c_int32),
                                              C.c_int32, C.c_int32, C.c_double, C.c_double,
                                              C.c_int32, C.c_int32, P(C.c_uint8), P(_Move)]
        _lib.orc_enumerate.argtypes = [P(_Inst), C.c_int32, P(C.c_int32), P(C.c_int32),
                                       C.c_int32, C.c_int32, C.c_double, C.c_double,
                                       P(C.c_double), P(C.c_int32), P(C.c_int32), C.c_int64,
                                       P(_Move)]
        _lib.orc_enumerate_full.argtypes = [P(_Inst), C.c_int32, P(C.c_int32), P(C.c_int32),
                                            C.c_int32, C.c_int32, C.c_double, C.c_double,
                                            P(C.c_double), P(C.c_int32), P(C.c_int32), P(C.c_int8),
                                            P(C.c_int8), C.c_double, C.c_int64, P(_Move)]
        _lib.orc_score_candidate.argtypes = [P(_Inst), C.c_int32, P(C.c_int32), P(C.c_int32),
                                             C.c_int32, C.c_int32, C.c_double, C.c_double,
                                             C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(_Move)]
        _lib.orc_apply.argtypes = [P(_Inst), C.c_int32, P(C.c_int32), P(C.c_int32), C.c_int32,
                                   C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                   P(C.c_int32), P(C.c_int32)]
        _lib.orc_route_eval.argtypes = [P(_Inst), P(C.c_int32), C.c_int32, P(C.c_double),
                                        P(C.c_int64), P(C.c_double), P(C.c_double),
                                        P(C.c_double)]
        _lib.orc_attributes.argtypes = [P(_Inst), C.c_int32, P(C.c_int32), P(C.c_int32)] + \
            [P(C.c_double), P(C.c_int64), P(C.c_double)] * 2 + [P(C.c_double)]
        _lib.orc_solution_cost.argtypes = [P(_Inst), C.c_int32, P(C.c_int32), P(C.c_int32),
                                           P(C.c_double), P(C.c_double), P(C.c_double)]
        _lib.orc_seq_lmax.argtypes = [P(_Inst), P(C.c_int32), C.c_int32]
        _lib.orc_seq_lmax.restype = C.c_int64
    return _lib


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class Oracle:
    """Holds one instance (fp64 copies) and evaluates solutions given as
    CSR route arrays (route_ptr int32[R+1], customers int32[N])."""

    def __init__(self, dist, demand, capacity, tw=None, pickup=None):
        self.dist = np.ascontiguousarray(dist, dtype=np.float64)
        self.demand = np.ascontiguousarray(demand, dtype=np.int64)
        # VRPSPDTW pickup demands p_i; None => CVRP / VRPTW
        self.pickup = None if pickup is None else np.ascontiguousarray(pickup, dtype=np.int64)
        self.n = self.dist.shape[0]
        self.tw = None if tw is None else np.ascontiguousarray(tw, dtype=np.float64)
        if self.tw is not None:
            self.e = np.ascontiguousarray(self.tw[:, 0])
            self.l = np.ascontiguousarray(self.tw[:, 1])
            self.s = np.ascontiguousarray(self.tw[:, 2])
        self.capacity = int(capacity)
        self._inst = _Inst()
        self._inst.n_nodes = self.n
        self._inst.C = _ptr(self.dist, C.c_double)
        self._inst.demand = _ptr(self.demand, C.c_int64)
        if self.tw is not None:
            self._inst.e = _ptr(self.e, C.c_double)
            self._inst.l = _ptr(self.l, C.c_double)
            self._inst.s = _ptr(self.s, C.c_double)
        self._inst.Q = self.capacity
        if self.pickup is not None:
            self._inst.pickup = _ptr(self.pickup, C.c_int64)
        lib()

    @classmethod
    def from_instance(cls, inst):
        return cls(inst.dist, inst.demand, inst.capacity, inst.tw, getattr(inst, "pickup", None))

    def seq_lmax(self, nodes) -> int:
        """The largest load carried along a node sequence served in order (seq_lmax in
        tga_oracle.c; the delivery sum when the instance has no pickups)."""
        nd = np.ascontiguousarray(nodes, dtype=np.int32)
        return int(lib().orc_seq_lmax(C.byref(self._inst), _ptr(nd, C.c_int32), len(nd)))

    @staticmethod
    def _csr(routes):
        if isinstance(routes, tuple):
            ptr, cust = routes
        else:
            rr = routes.routes if hasattr(routes, "routes") else routes
            ptr = np.zeros(len(rr) + 1, dtype=np.int32)
            for i, r in enumerate(rr):
                ptr[i + 1] = ptr[i] + len(r)
            cust = np.array([c for r in rr for c in r], dtype=np.int32)
        return (np.ascontiguousarray(ptr, dtype=np.int32),
                np.ascontiguousarray(cust, dtype=np.int32))

    @staticmethod
    def _move(m: _Move) -> Move:
        return Move(m.variant, m.score, m.dD, m.dLV, m.dTV, m.u, m.v, m.route_a,
                    m.pos_a, m.route_b, m.pos_b, bool(m.found), bool(m.feasible),
                    int(m.n_candidates))

    def best_move(self, routes, variant: int, mode: int = 0, wQ: float = 10.0,
                  wT: float = 10.0, u_lo: int = 0, u_hi: int = -1, mask=None) -> Move:
        """mask: None (full neighbourhood, NTGA) or the n x n uint8 edge mask M of the
        edge-based neighbourhood (ETGA), e.g. granular_mask(dist, theta)."""
        ptr, cust = self._csr(routes)
        m = _Move()
        if mask is not None:
            mk = np.ascontiguousarray(mask, dtype=np.uint8)
            assert mk.shape == (self.n, self.n)
            rc = lib().orc_best_move_masked(C.byref(self._inst), len(ptr) - 1, _ptr(ptr, C.c_int32),
                                            _ptr(cust, C.c_int32), variant, mode, wQ, wT, u_lo, u_hi,
                                            _ptr(mk, C.c_uint8), C.byref(m))
            if rc != 0:
                raise ValueError(f"orc_best_move_masked failed: {rc}")
            return self._move(m)
        rc = lib().orc_best_move(C.byref(self._inst), len(ptr) - 1, _ptr(ptr, C.c_int32),
                                 _ptr(cust, C.c_int32), variant, mode, wQ, wT, u_lo, u_hi,
                                 C.byref(m))
        if rc != 0:
            raise ValueError(f"orc_best_move failed: {rc}")
        return self._move(m)

    def enumerate(self, routes, variant: int, mode: int = 0, wQ: float = 10.0,
                  wT: float = 10.0):
        """All candidates of a variant in canonical order: (scores, u, v, best)."""
        ptr, cust = self._csr(routes)
        m = _Move()
        lib().orc_best_move(C.byref(self._inst), len(ptr) - 1, _ptr(ptr, C.c_int32),
                            _ptr(cust, C.c_int32), variant, mode, wQ, wT, 0, -1, C.byref(m))
        n = int(m.n_candidates)
        sc = np.zeros(max(n, 1))
        us = np.zeros(max(n, 1), dtype=np.int32)
        vs = np.zeros(max(n, 1), dtype=np.int32)
        lib().orc_enumerate(C.byref(self._inst), len(ptr) - 1, _ptr(ptr, C.c_int32),
                            _ptr(cust, C.c_int32), variant, mode, wQ, wT,
                            _ptr(sc, C.c_double), _ptr(us, C.c_int32), _ptr(vs, C.c_int32),
                            n, C.byref(m))
        return sc[:n], us[:n], vs[:n], self._move(m)

    def enumerate_full(self, routes, variant: int, mode: int = 0, wQ: float = 10.0, wT: float = 10.0,
                       band_tol: float = 1e-4):
        """All candidates of a variant in canonical order with, per candidate, the
        feasibility of the changed routes and the TW-F ambiguity-band flag:
        (scores, u, v, feasible, band, best)."""
        ptr, cust = self._csr(routes)
        m = _Move()
        lib().orc_best_move(C.byref(self._inst), len(ptr) - 1, _ptr(ptr, C.c_int32),
                            _ptr(cust, C.c_int32), variant, mode, wQ, wT, 0, -1, C.byref(m))
        n = int(m.n_candidates)
        sc = np.zeros(max(n, 1))
        us = np.zeros(max(n, 1), dtype=np.int32)
        vs = np.zeros(max(n, 1), dtype=np.int32)
        fe = np.zeros(max(n, 1), dtype=np.int8)
        bd = np.zeros(max(n, 1), dtype=np.int8)
        lib().orc_enumerate_full(C.byref(self._inst), len(ptr) - 1, _ptr(ptr, C.c_int32),
                                 _ptr(cust, C.c_int32), variant, mode, wQ, wT,
                                 _ptr(sc, C.c_double), _ptr(us, C.c_int32), _ptr(vs, C.c_int32),
                                 _ptr(fe, C.c_int8), _ptr(bd, C.c_int8), band_tol, n, C.byref(m))
        return sc[:n], us[:n], vs[:n], fe[:n].astype(bool), bd[:n].astype(bool), self._move(m)

    def score_candidate(self, routes, variant, ra, pa, rb, pb, mode=0, wQ=10.0, wT=10.0):
        ptr, cust = self._csr(routes)
        m = _Move()
        lib().orc_score_candidate(C.byref(self._inst), len(ptr) - 1, _ptr(ptr, C.c_int32),
                                  _ptr(cust, C.c_int32), variant, mode, wQ, wT, ra, pa, rb,
                                  pb, C.byref(m))
        return self._move(m)

    def apply(self, routes, variant, ra, pa, rb, pb):
        ptr, cust = self._csr(routes)
        optr = np.zeros_like(ptr)
        ocust = np.zeros_like(cust)
        rc = lib().orc_apply(C.byref(self._inst), len(ptr) - 1, _ptr(ptr, C.c_int32),
                             _ptr(cust, C.c_int32), variant, ra, pa, rb, pb,
                             _ptr(optr, C.c_int32), _ptr(ocust, C.c_int32))
        if rc != 0:
            raise ValueError(f"orc_apply failed: {rc}")
        return [list(map(int, ocust[optr[i]:optr[i + 1]])) for i in range(len(optr) - 1)]

    def route_eval(self, nodes):
        """nodes include both depots; returns (D, L, TV, arrival, start)."""
        nodes = np.ascontiguousarray(nodes, dtype=np.int32)
        D, TV = C.c_double(), C.c_double()
        L = C.c_int64()
        arr = np.zeros(len(nodes))
        st = np.zeros(len(nodes))
        lib().orc_route_eval(C.byref(self._inst), _ptr(nodes, C.c_int32), len(nodes),
                             C.byref(D), C.byref(L), C.byref(TV), _ptr(arr, C.c_double),
                             _ptr(st, C.c_double))
        return D.value, L.value, TV.value, arr, st

    def attributes(self, routes):
        ptr, cust = self._csr(routes)
        Q = len(cust) + len(ptr) - 1
        out = {k: np.zeros(Q) for k in ("pre_D", "pre_TV", "suf_D", "suf_TV", "start")}
        out["pre_L"] = np.zeros(Q, dtype=np.int64)
        out["suf_L"] = np.zeros(Q, dtype=np.int64)
        lib().orc_attributes(C.byref(self._inst), len(ptr) - 1, _ptr(ptr, C.c_int32),
                             _ptr(cust, C.c_int32),
                             _ptr(out["pre_D"], C.c_double), _ptr(out["pre_L"], C.c_int64),
                             _ptr(out["pre_TV"], C.c_double), _ptr(out["suf_D"], C.c_double),
                             _ptr(out["suf_L"], C.c_int64), _ptr(out["suf_TV"], C.c_double),
                             _ptr(out["start"], C.c_double))
        return out

    def cost(self, routes):
        ptr, cust = self._csr(routes)
        D, LV, TV = C.c_double(), C.c_double(), C.c_double()
        lib().orc_solution_cost(C.byref(self._inst), len(ptr) - 1, _ptr(ptr, C.c_int32),
                                _ptr(cust, C.c_int32), C.byref(D), C.byref(LV), C.byref(TV))
        return D.value, LV.value, TV.value

    def best_over(self, routes, variants: List[int], mode=0, wQ=10.0, wT=10.0) -> Optional[Move]:
        """Best over several variants: lowest (score, variant rank, index)."""
        best = None
        for v in sorted(variants):
            m = self.best_move(routes, v, mode, wQ, wT)
            if m.found and (best is None or m.score < best.score):
                best = m
        return best


def granular_mask(dist, theta: int) -> np.ndarray:
    """Edge mask M of the granular neighbourhood (theta = granularity
    threshold, Table `params` P:528-529; reading 21), written out:
    NN(i) = the theta customers j != i with the smallest (c_ij, j);
    M_ij = 1 iff j in NN(i) or i in NN(j); every pair with the depot (node 0) is kept."""
    dist = np.asarray(dist, dtype=np.float64)
    n = dist.shape[0]
    M = np.zeros((n, n), dtype=np.uint8)
    for i in range(1, n):
        cand = [(dist[i, j], j) for j in range(1, n) if j != i]
        cand.sort()
        for _, j in cand[:theta]:
            M[i, j] = 1
            M[j, i] = 1
    M[0, :] = 1
    M[:, 0] = 1
    return M


def canonical_q(routes) -> int:
    """Q = N + R canonical slots."""
    rr = routes.routes if hasattr(routes, "routes") else routes
    return sum(len(r) for r in rr) + len(rr)
