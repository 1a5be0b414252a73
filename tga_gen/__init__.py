"""Seeded synthetic VRP inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no concatenation, no move
evaluation, no cost deltas).  It only draws instances (coordinates, demands,
time windows, distance matrices) and start solutions (customer partitions
into routes), with the shapes of the paper's benchmark families:

* configs come from BASELINE.json ``configs`` and SURVEY.md §8(d);
* X (CVRP, Uchoa et al.) shape: "100 X benchmark instances ... 100 to
  1000 customers"; X-n1001-k43 has M=43 routes;
* GH (VRPTW, Gehring-Homberger) shape: P:514; R1-like routes of ~10,
  R2-like routes of ~40-50;
* distances: CVRPLIB round-nearest integers; the
  VRPTW "TW-I" mode uses integer tenths floor(10*euclid) so fp32 on the GPU is
  exact; "TW-F" uses real distances that are exactly representable in fp32
  (so both sides start from the same numbers and only arithmetic precision
  differs).

The time windows of a VRPTW instance are drawn around a reference schedule of
the constructed start solution (no waiting: customer i is reached at a_i and
its window is placed to contain a_i), so the start solution ("state A") is
feasible by construction.  That schedule is a plain cumulative sum of travel
and service times along the reference routes - instance construction, not
the method.

Everything is a pure function of its seed.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

__all__ = [
    "Instance", "Solution", "euclid_nint", "euclid_tenths", "euclid_f32",
    "cvrp_small", "x_like", "gh_like", "large_cvrp", "population",
    "random_partition", "perturb", "config", "CONFIGS", "jd_like",
]

MODE_CVRP = "cvrp"   # integer distances, no time windows
MODE_TWI = "twi"     # integer-tenths distances/times, time windows
MODE_TWF = "twf"     # real (fp32-representable) distances/times, time windows


@dataclasses.dataclass
class Instance:
    """A VRP instance.  Node 0 is the depot.

    dist:     (n+1, n+1) int32 (cvrp/twi) or float64 holding fp32 values (twf)
    demand:   (n+1,) int32, demand[0] == 0
    tw:       (n+1, 3) float64 [e, l, s] or None (CVRP); travel time == dist
    capacity: vehicle capacity Q
    pickup:   (n+1,) int32 pickup demands p_i (VRPSPDTW), pickup[0] == 0;
              None for CVRP / VRPTW (p_i = 0)
    """
    name: str
    mode: str
    coords: np.ndarray
    dist: np.ndarray
    demand: np.ndarray
    capacity: int
    tw: Optional[np.ndarray] = None
    pickup: Optional[np.ndarray] = None

    @property
    def n_nodes(self) -> int:
        return int(self.dist.shape[0])

    @property
    def n_customers(self) -> int:
        return self.n_nodes - 1


@dataclasses.dataclass
class Solution:
    """Routes as customer lists (depots implicit at both ends).  Empty routes
    are allowed and kept."""
    routes: List[List[int]]

    def flat(self):
        """(route_ptr int32[R+1], customers int32[N]) CSR form used by the ABI."""
        ptr = np.zeros(len(self.routes) + 1, dtype=np.int32)
        for i, r in enumerate(self.routes):
            ptr[i + 1] = ptr[i] + len(r)
        cust = np.array([c for r in self.routes for c in r], dtype=np.int32)
        return ptr, cust

    def copy(self) -> "Solution":
        return Solution([list(r) for r in self.routes])


# ---------------------------------------------------------------- distances
def _euclid(coords: np.ndarray) -> np.ndarray:
    d = coords[:, None, :] - coords[None, :, :]
    return np.sqrt((d.astype(np.float64) ** 2).sum(-1))


def euclid_nint(coords: np.ndarray) -> np.ndarray:
    """CVRPLIB convention: nint(sqrt(dx^2+dy^2))."""
    return np.floor(_euclid(coords) + 0.5).astype(np.int32)


def euclid_tenths(coords: np.ndarray) -> np.ndarray:
    """TW-I convention: floor(10*sqrt(dx^2+dy^2)) integer tenths."""
    return np.floor(10.0 * _euclid(coords) + 1e-9).astype(np.int32)


def euclid_f32(coords: np.ndarray) -> np.ndarray:
    """TW-F convention: real distances rounded to fp32 (held as float64)."""
    return _euclid(coords).astype(np.float32).astype(np.float64)


def _dist_for_mode(coords, mode):
    if mode == MODE_CVRP:
        return euclid_nint(coords)
    if mode == MODE_TWI:
        return euclid_tenths(coords)
    if mode == MODE_TWF:
        return euclid_f32(coords)
    raise ValueError(mode)


# ---------------------------------------------------------------- solutions
def _sweep_split(coords, demand, capacity, depot=0, n_routes=None, rng=None, max_len=None):
    """Angular sweep around the depot, cut when the capacity would be
    exceeded (or into n_routes equal-count sectors when given)."""
    n = coords.shape[0] - 1
    c = coords[1:] - coords[depot]
    ang = np.arctan2(c[:, 1], c[:, 0])
    off = 0.0 if rng is None else rng.uniform(-math.pi, math.pi)
    ang = np.mod(ang - off, 2 * math.pi)
    order = np.argsort(ang, kind="stable") + 1
    routes: List[List[int]] = []
    if n_routes is not None:
        for chunk in np.array_split(order, n_routes):
            routes.append([int(x) for x in chunk])
        return routes
    cur: List[int] = []
    load = 0
    for i in order:
        if cur and (load + int(demand[i]) > capacity or (max_len and len(cur) >= max_len)):
            routes.append(cur)
            cur, load = [], 0
        cur.append(int(i))
        load += int(demand[i])
    if cur:
        routes.append(cur)
    return routes


def random_partition(n_customers: int, n_routes: int, seed: int,
                     allow_empty: bool = True) -> Solution:
    """A uniformly random assignment + order of customers into n_routes."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(np.arange(1, n_customers + 1))
    if allow_empty:
        cuts = np.sort(rng.integers(0, n_customers + 1, size=n_routes - 1))
    else:
        cuts = np.sort(rng.choice(np.arange(1, n_customers), size=n_routes - 1,
                                  replace=False))
    parts = np.split(perm, cuts)
    return Solution([[int(x) for x in p] for p in parts])


def perturb(sol: Solution, n_moves: int, seed: int) -> Solution:
    """Random relocations of single customers (keeps an exact partition)."""
    rng = np.random.default_rng(seed)
    s = sol.copy()
    for _ in range(n_moves):
        nonempty = [i for i, r in enumerate(s.routes) if r]
        a = int(rng.choice(nonempty))
        x = s.routes[a].pop(int(rng.integers(0, len(s.routes[a]))))
        b = int(rng.integers(0, len(s.routes)))
        s.routes[b].insert(int(rng.integers(0, len(s.routes[b]) + 1)), x)
    return s


# ---------------------------------------------------------------- configs
def cvrp_small(seed: int = 0, n: int = 20, n_routes: int = 4,
               capacity: int = 100, spare: bool = False):
    """BASELINE config 1: 20 customers, 4 routes, Q=100, integer Euclidean.
    Depot (50,50); customers uniform integer in [0,100]^2; d ~ U{1..20}."""
    rng = np.random.default_rng(1000 + seed)
    coords = np.empty((n + 1, 2), dtype=np.int64)
    coords[0] = (50, 50)
    coords[1:] = rng.integers(0, 101, size=(n, 2))
    demand = np.zeros(n + 1, dtype=np.int32)
    demand[1:] = rng.integers(1, 21, size=n)
    inst = Instance(f"cvrp{n}-s{seed}", MODE_CVRP, coords, euclid_nint(coords),
                    demand, capacity)
    routes = _sweep_split(coords, demand, capacity, n_routes=n_routes)
    if spare:
        routes.append([])
    return inst, Solution(routes)


def _uchoa_coords(rng, n, grid, depot_kind, cust_kind):
    if depot_kind == "central":
        depot = np.array([grid // 2, grid // 2])
    elif depot_kind == "eccentric":
        depot = np.array([0, 0])
    else:
        depot = rng.integers(0, grid + 1, size=2)
    pts = []
    if cust_kind in ("clustered", "random-clustered"):
        n_clu = n // 2 if cust_kind == "random-clustered" else n
        n_seeds = int(rng.integers(3, 9))
        seeds = rng.integers(0, grid + 1, size=(n_seeds, 2))
        while len(pts) < n_clu:
            s = seeds[int(rng.integers(0, n_seeds))]
            p = np.rint(s + rng.normal(0, grid / 25.0, size=2)).astype(np.int64)
            if 0 <= p[0] <= grid and 0 <= p[1] <= grid:
                pts.append(p)
    while len(pts) < n:
        pts.append(rng.integers(0, grid + 1, size=2))
    coords = np.vstack([depot[None, :], np.array(pts[:n])]).astype(np.int64)
    return coords


def _uchoa_demand(rng, n, kind, coords):
    if kind == "unitary":
        d = np.ones(n, dtype=np.int64)
    elif kind == "small-large-var":      # U[1,10] / U[5,10] / U[1,100] / U[50,100]
        d = rng.integers(1, 101, size=n)
    elif kind == "u1-10":
        d = rng.integers(1, 11, size=n)
    elif kind == "u5-10":
        d = rng.integers(5, 11, size=n)
    elif kind == "u50-100":
        d = rng.integers(50, 101, size=n)
    elif kind == "quadrant":
        c = coords[1:]
        mid = (coords[1:].max() + 1) // 2
        odd = ((c[:, 0] >= mid) ^ (c[:, 1] >= mid)).astype(bool)
        d = np.where(odd, rng.integers(51, 101, size=n), rng.integers(1, 51, size=n))
    else:  # many small, few large
        big = rng.random(n) < 0.1
        d = np.where(big, rng.integers(50, 101, size=n), rng.integers(1, 11, size=n))
    out = np.zeros(n + 1, dtype=np.int32)
    out[1:] = d
    return out


def x_like(seed: int = 0, n: int = 1000, target_routes: int = 43,
           depot_kind: str = "central", cust_kind: str = "random-clustered",
           demand_kind: str = "small-large-var", spare: int = 1):
    """BASELINE config 2: Uchoa X-like CVRP (X-n1001-k43 shape): [0,1000]^2,
    Q chosen so the mean route has n/target_routes customers (P:1017 M=43)."""
    rng = np.random.default_rng(2000 + seed)
    coords = _uchoa_coords(rng, n, 1000, depot_kind, cust_kind)
    demand = _uchoa_demand(rng, n, demand_kind, coords)
    r = n / float(target_routes)
    capacity = int(math.ceil(r * demand[1:].sum() / n * 1.04))
    capacity = max(capacity, int(demand.max()))
    inst = Instance(f"X-like-n{n}-s{seed}", MODE_CVRP, coords, euclid_nint(coords),
                    demand, capacity)
    routes = _sweep_split(coords, demand, capacity, rng=rng)
    routes += [[] for _ in range(spare)]
    return inst, Solution(routes)


def large_cvrp(seed: int = 0, n: int = 10000, mean_len: int = 100, spare: int = 1):
    """BASELINE config 4: Arnold/Belgium-like 10^4 customers, clustered around a
    central depot on [0,10^4]^2; mean route length 100 (R~100) or 23 (R~435)."""
    rng = np.random.default_rng(4000 + seed)
    coords = _uchoa_coords(rng, n, 10000, "central", "random-clustered")
    demand = np.zeros(n + 1, dtype=np.int32)
    demand[1:] = rng.integers(1, 11, size=n)
    capacity = int(math.ceil(mean_len * demand[1:].sum() / n * 1.03))
    inst = Instance(f"L-n{n}-len{mean_len}-s{seed}", MODE_CVRP, coords,
                    euclid_nint(coords), demand, capacity)
    routes = _sweep_split(coords, demand, capacity, rng=rng)
    routes += [[] for _ in range(spare)]
    return inst, Solution(routes)


def _tw_around_schedule(rng, inst_dist, routes, service, density, width_lo, width_hi,
                        n_nodes, horizon_slack, integer):
    """Windows [e_i, l_i] containing the no-wait reference arrival a_i of each
    customer on its reference route (plain cumulative travel+service times)."""
    tw = np.zeros((n_nodes, 3), dtype=np.float64)
    arrival = np.zeros(n_nodes, dtype=np.float64)
    ret = 0.0
    for r in routes:
        t, prev = 0.0, 0
        for c in r:
            t = t + (service if prev else 0.0) + float(inst_dist[prev, c])
            arrival[c] = t
            prev = c
        if r:
            ret = max(ret, t + service + float(inst_dist[prev, 0]))
    horizon = float(math.ceil(ret * horizon_slack))
    tw[0] = (0.0, horizon, 0.0)
    for i in range(1, n_nodes):
        a = arrival[i]
        latest = horizon - service - float(inst_dist[i, 0])
        if rng.random() < density:
            w = rng.uniform(width_lo, width_hi)
            lo = max(0.0, a - rng.uniform(0.0, 1.0) * w)
            hi = min(max(a, lo + w), latest)
        else:
            lo, hi = 0.0, latest
        if integer:
            lo, hi = math.floor(lo), math.ceil(hi)
            hi = min(hi, math.floor(latest))
        else:
            lo = float(np.float32(lo))
            hi = float(np.float32(hi))
        # the reference arrival must stay inside its window (feasible state A)
        lo = min(lo, math.floor(a)) if integer else min(lo, a)
        hi = max(hi, math.ceil(a)) if integer else max(hi, float(np.float32(a)))
        tw[i] = (lo, hi, service)
    return tw


def gh_like(seed: int = 0, n: int = 1000, kind: str = "R1", density: float = 1.0,
            mode: str = MODE_TWI, spare: int = 1):
    """BASELINE config 3: Gehring-Homberger-like VRPTW.

    R1-like: short horizon, narrow windows, Q=200, routes of ~10 customers.
    R2-like: long horizon, wide windows, Q=1000, routes of ~40-50.
    Service time 10 (R) as in Solomon/GH; times in tenths for TW-I."""
    rng = np.random.default_rng(3000 + seed + (0 if kind == "R1" else 77))
    grid = 500 if n >= 600 else 250
    coords = _uchoa_coords(rng, n, grid, "central", "random")
    demand = np.zeros(n + 1, dtype=np.int32)
    demand[1:] = rng.integers(1, 31, size=n)
    if kind == "R1":
        capacity, route_len, width, slack = 200, 10, (100.0, 300.0), 1.15
    else:
        capacity, route_len, width, slack = 1000, 45, (1500.0, 4000.0), 1.10
    scale = 10.0 if mode == MODE_TWI else 1.0
    dist = _dist_for_mode(coords, mode)
    # routes: sweep with both a capacity cut and a length cap (reference tour)
    routes = _sweep_split(coords, demand, capacity, rng=rng, max_len=route_len)
    service = 10.0 * scale
    tw = _tw_around_schedule(rng, dist, routes, service, density,
                             width[0] * scale, width[1] * scale, n + 1, slack,
                             integer=(mode == MODE_TWI))
    inst = Instance(f"GH-{kind}-n{n}-{mode}-s{seed}", mode, coords, dist, demand,
                    capacity, tw)
    routes += [[] for _ in range(spare)]
    return inst, Solution(routes)


def _max_load(route, demand, pickup):
    """Largest load carried along a route (instance construction only): after the
    first k customers the vehicle holds the deliveries of the rest and the pickups
    of these."""
    return max(int(demand[route[k:]].sum()) + int(pickup[route[:k]].sum()) for k in range(len(route) + 1))


def jd_like(seed: int = 0, n: int = 1000, mode: str = MODE_TWI, spare: int = 1,
            route_len: int = 14, capacity: int = 200):
    """VRPSPDTW shaped like the JD benchmark ("20 JD benchmark instances ...
    based on real-world JD Logistics data with 200, 400, 600, 800, and 1000
    customers"; Liu et al. 2021; the data is not in the reference): random-clustered
    customers around a central depot, every customer with a delivery d_i and a
    pickup p_i, GH-like time windows placed around a reference schedule
    (so the start solution is time-feasible), service 10.  The reference routes are
    an angular sweep cut where the route's largest load would exceed Q (so the start
    is capacity-feasible and loads are tight) or at route_len customers."""
    rng = np.random.default_rng(6000 + seed)
    grid = 500 if n >= 600 else 250
    coords = _uchoa_coords(rng, n, grid, "central", "random-clustered")
    demand = np.zeros(n + 1, dtype=np.int32)
    pickup = np.zeros(n + 1, dtype=np.int32)
    demand[1:] = rng.integers(0, 41, size=n)
    pickup[1:] = rng.integers(0, 41, size=n)
    scale = 10.0 if mode == MODE_TWI else 1.0
    dist = _dist_for_mode(coords, mode)
    c = coords[1:] - coords[0]
    ang = np.mod(np.arctan2(c[:, 1], c[:, 0]) - rng.uniform(-math.pi, math.pi), 2 * math.pi)
    routes: List[List[int]] = []
    cur: List[int] = []
    for i in (np.argsort(ang, kind="stable") + 1):
        trial = np.array(cur + [int(i)], dtype=np.int64)
        if cur and (len(cur) >= route_len or _max_load(trial, demand, pickup) > capacity):
            routes.append(cur)
            cur = []
        cur.append(int(i))
    if cur:
        routes.append(cur)
    service = 10.0 * scale
    tw = _tw_around_schedule(rng, dist, routes, service, 1.0, 100.0 * scale, 300.0 * scale,
                             n + 1, 1.15, integer=(mode == MODE_TWI))
    inst = Instance(f"JD-like-n{n}-{mode}-s{seed}", mode, coords, dist, demand, capacity, tw,
                    pickup=pickup)
    routes += [[] for _ in range(spare)]
    return inst, Solution(routes)


def population(seed: int = 0, n: int = 200, n_sol: int = 1024, mode: str = MODE_TWI):
    """BASELINE config 5: one R1_2-like instance (200 customers, Q=200,
    ~18-23 routes) and n_sol solutions: the reference construction plus
    independent seeded random perturbations."""
    inst, base = gh_like(seed, n=n, kind="R1", mode=mode, spare=1)
    sols = [base]
    for k in range(1, n_sol):
        sols.append(perturb(base, n_moves=5 + (k % 11), seed=50_000 + 97 * seed + k))
    return inst, sols


CONFIGS = {
    "cfg1": "synthetic CVRP, 20 customers, 4 routes, capacity 100",
    "cfg2": "Uchoa X-like CVRP, 1000 customers, X-n1001-k43 shape",
    "cfg3": "Gehring-Homberger-like VRPTW, 1000 customers (R1-like, TW-I)",
    "cfg3r2": "Gehring-Homberger-like VRPTW, 1000 customers (R2-like, TW-I)",
    "cfg4": "large CVRP 10000 customers, mean route length 100",
    "cfg4s": "large CVRP 10000 customers, mean route length 23",
    "ns2000": "X-like CVRP, 2000 customers, 87 routes (north-star sweep)",
    "cfg5": "population 1024 x VRPTW 200 customers (R1_2-like, TW-I)",
    "jd": "JD-like VRPSPDTW, 1000 customers (delivery + pickup, time windows, TW-I)",
    "jd200": "JD-like VRPSPDTW, 200 customers (delivery + pickup, time windows, TW-I)",
}


def config(name: str, seed: int = 0):
    """(Instance, Solution) for a named configuration (cfg5 -> list)."""
    if name == "cfg1":
        return cvrp_small(seed)
    if name == "cfg2":
        return x_like(seed, n=1000, target_routes=43)
    if name == "ns2000":
        return x_like(seed, n=2000, target_routes=87)
    if name == "cfg3":
        return gh_like(seed, n=1000, kind="R1")
    if name == "cfg3r2":
        return gh_like(seed, n=1000, kind="R2")
    if name == "cfg3f":
        return gh_like(seed, n=1000, kind="R1", mode=MODE_TWF)
    if name == "cfg4":
        return large_cvrp(seed, n=10000, mean_len=100)
    if name == "cfg4s":
        return large_cvrp(seed, n=10000, mean_len=23)
    if name == "cfg5":
        return population(seed)
    if name == "jd":
        return jd_like(seed, n=1000)
    if name == "jd200":
        return jd_like(seed, n=200)
    raise KeyError(name)
