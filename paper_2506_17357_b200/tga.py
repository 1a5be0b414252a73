"""Thin ctypes binding of libtga.so (include/tga.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module converts numpy arrays / torch streams to pointers and status codes to
exceptions.  There is no CPU fallback: if libtga.so is missing or a CUDA
device is unavailable the calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TGA_LIB: diagnostics only (A/B timing of two builds of the same sources in one GPU session)
LIB_PATH = os.environ.get("TGA_LIB") or os.path.join(_HERE, "libtga.so")

# ---------------------------------------------------------------- constants (include/tga.h)
OK, NO_IMPROVING_MOVE = 0, 1
ERR = {-1: "INVALID_ARGUMENT", -2: "STRUCTURE", -3: "STALE", -4: "UNSUPPORTED", -5: "CUDA",
       -6: "NCCL", -7: "OOM"}
I32, F32 = 0, 1
SCORE_FEASIBLE, SCORE_PENALISED = 0, 1
N_VARIANTS = 27
V_2OPT, V_2OPT_STAR = 0, 1
V_RELOCATE = {1: 2, 2: 3, 3: 4}
V_SWAP = {(1, 1): 5, (1, 2): 6, (1, 3): 7, (2, 2): 8, (2, 3): 9, (3, 3): 10}
V_IRELOCATE = {1: 11, 2: 12, 3: 13}
V_ISWAP = {(a, b): 14 + 3 * (a - 1) + (b - 1) for a in (1, 2, 3) for b in (1, 2, 3)}
# reversed-segment variants: or-opt N=2,3 and cross (N,N) N=2,3 with reversed segments
V_OROPT_REV = {2: 23, 3: 24}
V_CROSS_REV = {2: 25, 3: 26}
VARIANT_NAMES = (["2opt", "2opt*", "relocate", "or-opt2", "or-opt3", "swap11", "cross12", "cross13",
                  "cross22", "cross23", "cross33", "irelocate1", "irelocate2", "irelocate3"]
                 + [f"iswap{a}{b}" for a in (1, 2, 3) for b in (1, 2, 3)]
                 + ["or-opt2r", "or-opt3r", "cross22r", "cross33r"])
OP_2OPT = 1 << 0
OP_2OPT_STAR = 1 << 1
OP_RELOCATE = 1 << 2
OP_OR_OPT = (1 << 3) | (1 << 4)
OP_SWAP = 1 << 5
OP_CROSS = 0x1F << 6
OP_INTRA_RELOCATE = 0x7 << 11
OP_INTRA_SWAP = 0x1FF << 14
OP_INTER = 0x7FE
OP_INTRA = OP_2OPT | OP_INTRA_RELOCATE | OP_INTRA_SWAP
OP_REVERSED = 0xF << 23
OP_STANDARD = (1 << 23) - 1      # the 23 standard variants (the benchmarked neighbourhood)
OP_ALL = (1 << N_VARIANTS) - 1
OP_FUSED_NS = OP_2OPT_STAR | OP_RELOCATE | OP_SWAP
EVAL_ACCUMULATE = 1 << 31
OPERATORS = {"2opt": OP_2OPT, "2opt*": OP_2OPT_STAR, "relocate": OP_RELOCATE, "or-opt": OP_OR_OPT,
             "swap": OP_SWAP, "cross": OP_CROSS, "intra-relocate": OP_INTRA_RELOCATE,
             "intra-swap": OP_INTRA_SWAP, "or-opt reversed": 0x3 << 23, "cross reversed": 0x3 << 25}


class TgaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"tga error {code} ({ERR.get(code, '?')}): {msg}")
        self.code = code


class _Options(C.Structure):
    _fields_ = [("score_mode", C.c_int32), ("w_load", C.c_int32), ("w_tw", C.c_int32),
                ("device", C.c_int32), ("slack", C.c_int32), ("granular_theta", C.c_int32),
                ("reserved", C.c_int32 * 10)]


class Move(C.Structure):
    """tga_move (include/tga.h)."""
    _fields_ = [("variant", C.c_int32), ("n1", C.c_int32), ("n2", C.c_int32),
                ("route_a", C.c_int32), ("pos_a", C.c_int32), ("route_b", C.c_int32),
                ("pos_b", C.c_int32), ("u", C.c_int32), ("v", C.c_int32),
                ("feasible", C.c_int32), ("delta_i", C.c_int64), ("delta_f", C.c_double),
                ("key", C.c_uint64), ("generation", C.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None
_SYMBOLS = {
    "tga_instance_create": (C.c_int32, [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "tga_instance_destroy": (C.c_int32, [C.c_void_p]),
    "tga_solution_load": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tga_solution_destroy": (C.c_int32, [C.c_void_p]),
    "tga_eval": (C.c_int32, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "tga_best_move": (C.c_int32, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "tga_apply_move": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "tga_solution_keys": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "tga_solution_counts": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "tga_solution_cost": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tga_solution_routes": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "tga_solution_info": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tga_solution_attributes": (C.c_int32, [C.c_void_p] + [C.c_void_p] * 7),
    "tga_solution_set_shard": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32]),
    "tga_solution_set_stream": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "tga_step": (C.c_int32, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "tga_solution_reload": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "tga_solution_enable_timing": (C.c_int32, [C.c_void_p, C.c_int32]),
    "tga_solution_timings": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "tga_shard_range": (C.c_int32, [C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "tga_nccl_unique_id": (C.c_int32, [C.c_void_p]),
    "tga_comm_init": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "tga_instance_set_pickup": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "tga_solution_load_records": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "tga_batch_load": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]),
    "tga_batch_destroy": (C.c_int32, [C.c_void_p]),
    "tga_batch_size": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "tga_batch_solution": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p]),
    "tga_batch_eval": (C.c_int32, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "tga_batch_keys": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "tga_batch_best_moves": (C.c_int32, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "tga_batch_apply_moves": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "tga_step_async": (C.c_int32, [C.c_void_p, C.c_uint32]),
    "tga_solution_device_stats": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "tga_instance_info": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tga_solution_debug_probe": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p]),
    "tga_descent": (C.c_int32, [C.c_void_p, C.c_uint32, C.c_int32, C.c_void_p, C.c_uint64, C.c_void_p]),
    "tga_batch_step_async": (C.c_int32, [C.c_void_p, C.c_uint32]),
    "tga_batch_set_stream": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "tga_batch_device_stats": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "tga_debug_eval_dump": (C.c_int32, [C.c_void_p, C.c_uint32, C.c_int32, C.c_void_p, C.c_int64]),
    "tga_last_error": (C.c_char_p, []),
    "tga_version": (C.c_char_p, []),
    "tga_launch_count": (C.c_uint64, []),
}


def lib() -> C.CDLL:
    """Load libtga.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run paper_2506_17357_b200/build.py "
                              "(or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SYMBOLS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int, allow=(OK,)) -> int:
    if rc in allow:
        return rc
    msg = lib().tga_last_error().decode(errors="replace")
    raise TgaError(rc, msg)


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(getattr(stream, "cuda_stream"))  # torch.cuda.Stream


def version() -> str:
    return lib().tga_version().decode()


def launch_count() -> int:
    return int(lib().tga_launch_count())


def shard_range(n_items: int, shard: int, n_shards: int):
    """The library's row-shard plan: [lo, hi) of n_items for this shard."""
    lo, hi = C.c_int64(), C.c_int64()
    _check(lib().tga_shard_range(n_items, shard, n_shards, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().tga_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


class Instance:
    """tga_instance_create(dist, demand, tw, capacity)."""

    def __init__(self, dist, demand, capacity: int, tw=None, score_mode: int = SCORE_FEASIBLE,
                 w_load: int = 10, w_tw: int = 10, device: int = -1, slack: int = 0,
                 granular_theta: int = 0, pickup=None):
        dist = np.asarray(dist)
        if np.issubdtype(dist.dtype, np.integer):
            self.dist = np.ascontiguousarray(dist, dtype=np.int32)
            self.dtype = I32
        else:
            self.dist = np.ascontiguousarray(dist, dtype=np.float32)
            self.dtype = F32
        self.n = int(self.dist.shape[0])
        self.demand = np.ascontiguousarray(demand, dtype=np.int32)
        self.tw = None if tw is None else np.ascontiguousarray(tw, dtype=np.float32)
        self.capacity = int(capacity)
        opt = _Options()
        opt.score_mode, opt.w_load, opt.w_tw, opt.device = score_mode, w_load, w_tw, device
        opt.slack = slack
        opt.granular_theta = granular_theta   # > 0: edge-based neighbourhood (ETGA)
        self.score_mode = score_mode
        self.granular_theta = granular_theta
        h = C.c_void_p()
        _check(lib().tga_instance_create(self.n, _p(self.dist), self.dtype, None, _p(self.demand),
                                         _p(self.tw), self.capacity, C.byref(opt), C.byref(h)))
        self._h = h
        self.pickup = None
        if pickup is not None:   # VRPSPDTW
            self.pickup = np.ascontiguousarray(pickup, dtype=np.int32)
            _check(lib().tga_instance_set_pickup(self._h, _p(self.pickup)))

    @classmethod
    def from_gen(cls, inst, **kw):
        return cls(inst.dist, inst.demand, inst.capacity, inst.tw, pickup=getattr(inst, "pickup", None), **kw)

    def info(self):
        """(n_nodes, granular theta, unordered customer pairs kept by the edge mask)."""
        n, th, p = C.c_int32(), C.c_int32(), C.c_int64()
        _check(lib().tga_instance_info(self._h, C.byref(n), C.byref(th), C.byref(p)))
        return n.value, th.value, p.value

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().tga_instance_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _csr(routes):
    if isinstance(routes, tuple):
        ptr, cust = routes
    else:
        rr = routes.routes if hasattr(routes, "routes") else routes
        ptr = np.zeros(len(rr) + 1, dtype=np.int32)
        for i, r in enumerate(rr):
            ptr[i + 1] = ptr[i] + len(r)
        cust = np.array([c for r in rr for c in r], dtype=np.int32)
    return np.ascontiguousarray(ptr, dtype=np.int32), np.ascontiguousarray(cust, dtype=np.int32)


class Solution:
    """tga_solution_load(routes) + eval / best_move / apply_move."""

    def __init__(self, inst: Instance, routes):
        self.inst = inst
        ptr, cust = _csr(routes)
        h = C.c_void_p()
        _check(lib().tga_solution_load(inst.handle, len(ptr) - 1, _p(ptr), _p(cust), C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().tga_solution_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- hot path
    def eval(self, op_mask: int = OP_ALL, stream=None) -> None:
        _check(lib().tga_eval(self._h, op_mask, _stream_ptr(stream)))

    def best_move(self, op_mask: int = OP_ALL):
        """(improving: bool, Move).  Move.variant == -1 when no candidate was valid."""
        m = Move()
        rc = _check(lib().tga_best_move(self._h, op_mask, C.byref(m)), allow=(OK, NO_IMPROVING_MOVE))
        return rc == OK, m

    def apply(self, move: Move) -> None:
        _check(lib().tga_apply_move(self._h, C.byref(move)))

    def step(self, op_mask: int = OP_ALL):
        """eval + best_move + apply (if improving) in one call: (applied, Move)."""
        m = Move()
        rc = _check(lib().tga_step(self._h, op_mask, C.byref(m)), allow=(OK, NO_IMPROVING_MOVE))
        return rc == OK, m

    def step_async(self, op_mask: int = OP_ALL) -> None:
        """Device-resident step: eval + pick + apply + update, no host round trip."""
        _check(lib().tga_step_async(self._h, op_mask))

    def descent(self, op_mask: int, n_steps: int, l2_flush=None, timed: bool = False):
        """n device-resident steps enqueued from C; per-step device ms when timed.
        l2_flush: a torch CUDA tensor overwritten before every step (outside the timing)."""
        ms = np.zeros(max(n_steps, 1), dtype=np.float32) if timed else None
        fp, fb = (None, 0) if l2_flush is None else (l2_flush.data_ptr(), l2_flush.numel() * l2_flush.element_size())
        _check(lib().tga_descent(self._h, op_mask, n_steps, fp, fb, _p(ms)))
        return ms[:n_steps] if timed else None

    def eval_dump(self, op_mask: int = OP_ALL, flags: int = 0) -> np.ndarray:
        """Test-only: every candidate's packed key, [variant, Q, Q] over canonical
        slots (0 = not evaluated, ~0 = infeasible / invalid); see tga_debug_eval_dump."""
        _, _, Q, _ = self.info()
        out = np.zeros((N_VARIANTS, Q, Q), dtype=np.uint64)
        _check(lib().tga_debug_eval_dump(self._h, op_mask, flags, _p(out), out.size))
        return out

    def debug_probe(self, enable: bool = True):
        """Diagnostics: clock64 phase stamps of the last device step (16 u64) followed by the
        per-block (start, end) globaltimer pairs of its pick/update launch (512 x 2), then (re)arm."""
        out = np.zeros(16 + 1024, dtype=np.uint64)
        _check(lib().tga_solution_debug_probe(self._h, int(enable), _p(out)))
        return out

    def device_stats(self):
        """(counts per variant, applied moves) accumulated by step_async; clears them."""
        c = np.zeros(N_VARIANTS, dtype=np.uint64)
        a = C.c_uint64()
        _check(lib().tga_solution_device_stats(self._h, _p(c), C.byref(a)))
        return c, a.value

    def reload(self, routes) -> None:
        """Load another solution (same route count) into this object, asynchronously."""
        ptr, cust = _csr(routes)
        _check(lib().tga_solution_reload(self._h, len(ptr) - 1, _p(ptr), _p(cust)))

    def enable_timing(self, on: bool = True) -> None:
        _check(lib().tga_solution_enable_timing(self._h, int(on)))

    def timings(self) -> np.ndarray:
        """Durations (ms) of the inter-route launches recorded since the last call."""
        buf = np.zeros(8192, dtype=np.float32)
        n = C.c_int32()
        _check(lib().tga_solution_timings(self._h, _p(buf), len(buf), C.byref(n)))
        return buf[:n.value].copy()

    # ---- queries
    def keys(self) -> np.ndarray:
        k = np.zeros(N_VARIANTS, dtype=np.uint64)
        _check(lib().tga_solution_keys(self._h, _p(k)))
        return k

    def load_records(self):
        """VRPSPDTW prefix / suffix (L_I, L_O, L_M) records per canonical slot (Eq. 3a-d)."""
        R, N, _, _ = self.info()
        pre = np.zeros((N + R, 3), dtype=np.int32)
        suf = np.zeros((N + R, 3), dtype=np.int32)
        _check(lib().tga_solution_load_records(self._h, _p(pre), _p(suf)))
        return pre, suf

    def counts(self) -> np.ndarray:
        c = np.zeros(N_VARIANTS, dtype=np.uint64)
        _check(lib().tga_solution_counts(self._h, _p(c)))
        return c

    def info(self):
        R, N, Q, g = C.c_int32(), C.c_int32(), C.c_int32(), C.c_uint64()
        _check(lib().tga_solution_info(self._h, C.byref(R), C.byref(N), C.byref(Q), C.byref(g)))
        return R.value, N.value, Q.value, g.value

    def routes(self):
        R, N, _, _ = self.info()
        ptr = np.zeros(R + 1, dtype=np.int32)
        cust = np.zeros(max(N, 1), dtype=np.int32)
        _check(lib().tga_solution_routes(self._h, _p(ptr), _p(cust)))
        return [list(map(int, cust[ptr[i]:ptr[i + 1]])) for i in range(R)]

    def cost(self):
        di, df, le, te = C.c_int64(), C.c_double(), C.c_int64(), C.c_double()
        _check(lib().tga_solution_cost(self._h, C.byref(di), C.byref(df), C.byref(le), C.byref(te)))
        return di.value, df.value, le.value, te.value

    def attributes(self):
        _, _, Q, _ = self.info()
        out = {k: np.zeros(Q) for k in ("pre_D", "suf_D", "pre_TV", "suf_TV", "start")}
        out["pre_L"] = np.zeros(Q, dtype=np.int64)
        out["suf_L"] = np.zeros(Q, dtype=np.int64)
        _check(lib().tga_solution_attributes(self._h, _p(out["pre_L"]), _p(out["suf_L"]),
                                             _p(out["pre_D"]), _p(out["suf_D"]), _p(out["pre_TV"]),
                                             _p(out["suf_TV"]), _p(out["start"])))
        return out

    def set_stream(self, stream) -> None:
        """Use this cudaStream_t / torch.cuda.Stream for every later call."""
        _check(lib().tga_solution_set_stream(self._h, _stream_ptr(stream)))

    # ---- multi-GPU
    def set_shard(self, shard: int, n_shards: int) -> None:
        _check(lib().tga_solution_set_shard(self._h, shard, n_shards))

    def comm_init(self, rank: int, world: int, uid: bytes) -> None:
        buf = (C.c_char * 128).from_buffer_copy(uid)
        _check(lib().tga_comm_init(self._h, rank, world, C.cast(buf, C.c_void_p)))


class _Borrowed(Solution):
    """A solution owned by a Batch (not destroyed by Python)."""

    def __init__(self, inst, handle):
        self.inst = inst
        self._h = handle

    def close(self):
        self._h = None


class Batch:
    """tga_batch_*: a population of solutions of one instance evaluated together
    (BASELINE config 5)."""

    def __init__(self, inst: Instance, solutions):
        self.inst = inst
        n_routes, ptrs, custs = [], [], []
        for sol in solutions:
            ptr, cust = _csr(sol)
            n_routes.append(len(ptr) - 1)
            ptrs.append(ptr)
            custs.append(cust)
        self.n = len(n_routes)
        nr = np.array(n_routes, dtype=np.int32)
        ptr_all = np.ascontiguousarray(np.concatenate(ptrs), dtype=np.int32)
        cust_all = np.ascontiguousarray(np.concatenate(custs), dtype=np.int32)
        h = C.c_void_p()
        _check(lib().tga_batch_load(inst.handle, self.n, _p(nr), _p(ptr_all), _p(cust_all), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().tga_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solution(self, i: int) -> Solution:
        h = C.c_void_p()
        _check(lib().tga_batch_solution(self._h, i, C.byref(h)))
        return _Borrowed(self.inst, h)

    def eval(self, op_mask: int = OP_ALL, stream=None) -> None:
        _check(lib().tga_batch_eval(self._h, op_mask, _stream_ptr(stream)))

    def keys(self) -> np.ndarray:
        k = np.zeros((self.n, N_VARIANTS), dtype=np.uint64)
        _check(lib().tga_batch_keys(self._h, _p(k)))
        return k

    def best_moves(self, op_mask: int = OP_ALL):
        moves = (Move * self.n)()
        status = np.zeros(self.n, dtype=np.int32)
        _check(lib().tga_batch_best_moves(self._h, op_mask, C.cast(moves, C.c_void_p), _p(status)))
        return status, moves

    def step_async(self, op_mask: int = OP_ALL) -> None:
        _check(lib().tga_batch_step_async(self._h, op_mask))

    def set_stream(self, stream) -> None:
        _check(lib().tga_batch_set_stream(self._h, _stream_ptr(stream)))

    def device_stats(self):
        c = np.zeros(N_VARIANTS, dtype=np.uint64)
        a = C.c_uint64()
        _check(lib().tga_batch_device_stats(self._h, _p(c), C.byref(a)))
        return c, a.value

    def apply(self, moves, apply_mask=None) -> None:
        am = None if apply_mask is None else np.ascontiguousarray(apply_mask, dtype=np.int32)
        _check(lib().tga_batch_apply_moves(self._h, C.cast(moves, C.c_void_p), _p(am)))


def decode_key(key: int, integer: bool = True):
    """(score, flat index) of a packed key (order-preserving score << 32 | index)."""
    key = int(key)
    ordv, idx = key >> 32, key & 0xFFFFFFFF
    if integer:
        s = (ordv ^ 0x80000000)
        s = s - (1 << 32) if s >= 1 << 31 else s
        return s, idx
    u = (ordv ^ 0x80000000) if (ordv & 0x80000000) else (~ordv & 0xFFFFFFFF)
    return float(np.array([u], dtype=np.uint32).view(np.float32)[0]), idx
