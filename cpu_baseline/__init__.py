"""Fast CPU move evaluator (O(1) concatenation per candidate) -- a measured
BASELINE for bench.py only (the paper's MA-N CPU
evaluator, against which gamma_s of P:550 is taken).

Not the oracle (``oracle/`` re-simulates every neighbour) and not the product
path (``paper_2506_17357_b200/``); shares no code with either.  Its keys are
pinned to the oracle by ``tests/test_cpu_baseline.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tga_concat.c")
_LIB = os.path.join(_HERE, "libtcc.so")


def build(force: bool = False) -> str:
    """gcc -O2, single-threaded (no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Inst(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("C", C.POINTER(C.c_double)),
                ("demand", C.POINTER(C.c_int64)), ("e", C.POINTER(C.c_double)),
                ("l", C.POINTER(C.c_double)), ("s", C.POINTER(C.c_double)), ("Q", C.c_int64)]


class _Move(C.Structure):
    _fields_ = [("score", C.c_double), ("variant", C.c_int32), ("u", C.c_int32), ("v", C.c_int32),
                ("found", C.c_int32), ("n_candidates", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        _lib.tcc_best_move.argtypes = [P(_Inst), C.c_int32, P(C.c_int32), P(C.c_int32), C.c_int32,
                                       C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_int32, P(_Move)]
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class ConcatCPU:
    """One instance (fp64 copies); solutions as route lists or (ptr, cust) CSR."""

    def __init__(self, dist, demand, capacity, tw=None):
        self.dist = np.ascontiguousarray(dist, dtype=np.float64)
        self.demand = np.ascontiguousarray(demand, dtype=np.int64)
        self._i = _Inst()
        self._i.n_nodes = self.dist.shape[0]
        self._i.C = _p(self.dist, C.c_double)
        self._i.demand = _p(self.demand, C.c_int64)
        if tw is not None:
            tw = np.asarray(tw, dtype=np.float64)
            self.e, self.l, self.s = (np.ascontiguousarray(tw[:, k]) for k in range(3))
            self._i.e, self._i.l, self._i.s = (_p(x, C.c_double) for x in (self.e, self.l, self.s))
        self._i.Q = int(capacity)
        lib()

    @classmethod
    def from_instance(cls, inst):
        return cls(inst.dist, inst.demand, inst.capacity, inst.tw)

    @staticmethod
    def _csr(routes):
        rr = routes.routes if hasattr(routes, "routes") else routes
        ptr = np.zeros(len(rr) + 1, dtype=np.int32)
        for i, r in enumerate(rr):
            ptr[i + 1] = ptr[i] + len(r)
        cust = np.array([c for r in rr for c in r], dtype=np.int32)
        return ptr, np.ascontiguousarray(cust)

    def best_move(self, routes, variant, mode=0, wQ=10.0, wT=10.0, u_lo=0, u_hi=-1):
        """(found, score, u, v, n_candidates) over canonical rows [u_lo, u_hi)."""
        ptr, cust = self._csr(routes)
        m = _Move()
        rc = lib().tcc_best_move(C.byref(self._i), len(ptr) - 1, _p(ptr, C.c_int32), _p(cust, C.c_int32),
                                 variant, mode, wQ, wT, u_lo, u_hi, C.byref(m))
        if rc != 0:
            raise ValueError(f"tcc_best_move({variant}) failed: {rc}")
        return bool(m.found), m.score, m.u, m.v, int(m.n_candidates)
