"""Independent brute-force neighbourhood generator (pure Python, tiny inputs).

Pins the oracle's operator semantics and best move (SURVEY.md §8(c) "What pins
each part": "An independent generator produces every solution reachable by one
move ... scores it ... and compares the best score and the set of scores with
the canonical enumerator").  It works on plain customer lists with Python list
surgery and no shared code with oracle/; the canonical (u, v) of a move is named
from the definition of the candidate space (slot_id), so the multiset of
(score, u, v) triples pins the oracle's index map as well as its scores.

Operators (PAPER.md Fig. `operators` P:107-146; segment lengths per SURVEY
§8(c) item 7): relocate/or-opt (segment of N consecutive customers moved to
another route), swap/cross (exchange of an N1-segment and an N2-segment between
two routes), 2-opt* (exchange of tails), 2-opt (reverse a block of one route),
intra relocate (segment moved elsewhere in its own route), intra swap
(exchange two disjoint segments of one route, first of length N1).
"""
from __future__ import annotations

import math
from typing import Dict, List, Tuple


def simulate(dist, demand, tw, route, pickup=None):
    """Event simulation of one route given as customers only (depot implicit).
    Returns (distance, load, time_warp).  load = the delivery sum (CVRP / VRPTW) or,
    with pickups (VRPSPDTW), the largest load carried: after serving the
    first k customers the vehicle holds the deliveries of the others and the pickups
    of these, max over k = 0..L (a closed form, not the oracle's running simulation)."""
    nodes = [0] + list(route) + [0]
    D = sum(dist[nodes[k]][nodes[k + 1]] for k in range(len(nodes) - 1))
    if pickup is None:
        L = sum(demand[c] for c in route)
    else:
        L = max(sum(demand[c] for c in route[k:]) + sum(pickup[c] for c in route[:k])
                for k in range(len(route) + 1))
    TV = 0.0
    if tw is not None:
        t = tw[0][0]
        for k in range(1, len(nodes)):
            p, q = nodes[k - 1], nodes[k]
            arr = t + tw[p][2] + dist[p][q]
            st = max(arr, tw[q][0])
            if st > tw[q][1]:
                TV += st - tw[q][1]
                st = tw[q][1]
            t = st
    return D, L, TV


def in_band(dist, tw, route, tol=1e-4):
    """Some stop's service would start within tol * max(1, |l|) of its deadline l
    (the TW-F ambiguity band, reading 13), simulated as in simulate()."""
    if tw is None:
        return False
    nodes = [0] + list(route) + [0]
    t = tw[0][0]
    for k in range(1, len(nodes)):
        p, q = nodes[k - 1], nodes[k]
        st = max(t + tw[p][2] + dist[p][q], tw[q][0])
        if abs(st - tw[q][1]) < tol * max(1.0, abs(tw[q][1])):
            return True
        t = min(st, tw[q][1])
    return False


def segments(route, n):
    return [(i, route[i:i + n]) for i in range(0, len(route) - n + 1)]


def slot_id(routes, r, p):
    """Canonical slot id of position p (0 = start depot) of route r, written from
    its definition (SURVEY.md §8(c) "Canonical candidate space and index"; one
    depot slot per route, Q = N + R): id = sum_{r' < r} (L_r' + 1) + p."""
    return sum(len(routes[q]) + 1 for q in range(r)) + p


def neighbours(routes: List[List[int]], op: str, n1: int = 1, n2: int = 1, keyed: bool = False,
               indexed: bool = False):
    """Yield (changed_route_ids, new_routes_for_them) for one operator/variant;
    keyed=True appends, for inter-route moves, the node pair the move is keyed
    on (moved segment's first customer / cut node, insertion or cut node of the
    other route; 0 = the depot) -- the pair an edge mask filters (ETGA);
    indexed=True appends the canonical (u, v) slot pair of the move, named from
    the SURVEY §8(c) operator table through slot_id: u = the first slot of the
    moved / first segment or the cut slot of route a, v = the insertion-after,
    second-segment or cut slot (intra relocate: the slot the insertion node
    occupied in the ORIGINAL route)."""
    R = len(routes)

    def out(ids, news, pair=None, uv=None):
        t = (ids, news)
        if keyed:
            t = t + (pair,)
        if indexed:
            t = t + (uv,)
        return t

    S = lambda r, p: slot_id(routes, r, p)

    if op == "relocate":
        for a in range(R):
            for i, seg in segments(routes[a], n1):
                rest = routes[a][:i] + routes[a][i + n1:]
                for b in range(R):
                    if b == a:
                        continue
                    for k in range(len(routes[b]) + 1):
                        after = routes[b][k - 1] if k > 0 else 0
                        yield out((a, b), (rest, routes[b][:k] + seg + routes[b][k:]), (seg[0], after),
                                  (S(a, i + 1), S(b, k)))
    elif op == "relocate_rev":   # the moved segment inserted reversed
        for a in range(R):
            for i, seg in segments(routes[a], n1):
                rest = routes[a][:i] + routes[a][i + n1:]
                for b in range(R):
                    if b == a:
                        continue
                    for k in range(len(routes[b]) + 1):
                        after = routes[b][k - 1] if k > 0 else 0
                        yield out((a, b), (rest, routes[b][:k] + seg[::-1] + routes[b][k:]), (seg[0], after),
                                  (S(a, i + 1), S(b, k)))
    elif op == "swap_rev":   # both exchanged segments inserted reversed, n1 == n2
        for a in range(R):
            for b in range(a + 1, R):
                for i, sa in segments(routes[a], n1):
                    for j, sb in segments(routes[b], n2):
                        yield out((a, b), (routes[a][:i] + sb[::-1] + routes[a][i + n1:],
                                           routes[b][:j] + sa[::-1] + routes[b][j + n2:]), (sa[0], sb[0]),
                                  (S(a, i + 1), S(b, j + 1)))
    elif op == "swap":
        for a in range(R):
            for b in range(R):
                if a == b or (n1 == n2 and b < a):
                    continue
                for i, sa in segments(routes[a], n1):
                    for j, sb in segments(routes[b], n2):
                        yield out((a, b), (routes[a][:i] + sb + routes[a][i + n1:],
                                           routes[b][:j] + sa + routes[b][j + n2:]), (sa[0], sb[0]),
                                  (S(a, i + 1), S(b, j + 1)))
    elif op == "2opt*":
        for a in range(R):
            for b in range(a + 1, R):
                for i in range(len(routes[a]) + 1):
                    for j in range(len(routes[b]) + 1):
                        ca = routes[a][i - 1] if i > 0 else 0
                        cb = routes[b][j - 1] if j > 0 else 0
                        yield out((a, b), (routes[a][:i] + routes[b][j:],
                                           routes[b][:j] + routes[a][i:]), (ca, cb), (S(a, i), S(b, j)))
    elif op == "2opt":
        for a in range(R):
            r = routes[a]
            for i in range(len(r)):
                for j in range(i + 1, len(r)):
                    yield out((a,), (r[:i] + r[i:j + 1][::-1] + r[j + 1:],), None, (S(a, i + 1), S(a, j + 1)))
    elif op == "intra_relocate":
        for a in range(R):
            r = routes[a]
            for i, seg in segments(r, n1):
                rest = r[:i] + r[i + n1:]
                for k in range(len(rest) + 1):
                    if k == i:
                        continue  # the identity placement
                    # inserted after rest[k-1]: original position k (before the segment)
                    # or k + n1 (after it); k = 0 is the start depot
                    p_orig = k if k <= i else k + n1
                    yield out((a,), (rest[:k] + seg + rest[k:],), None, (S(a, i + 1), S(a, p_orig)))
    elif op == "intra_swap":
        for a in range(R):
            r = routes[a]
            for i in range(len(r)):
                for j in range(i + n1, len(r) - n2 + 1):
                    if i + n1 > len(r):
                        continue
                    new = r[:i] + r[j:j + n2] + r[i + n1:j] + r[i:i + n1] + r[j + n2:]
                    yield out((a,), (new,), None, (S(a, i + 1), S(a, j + 1)))
    else:
        raise ValueError(op)


def scores(dist, demand, tw, capacity, routes, op, n1=1, n2=1, mode=0, wQ=10.0, wT=10.0, mask=None,
           with_index=False, pickup=None):
    """List of scores of every neighbour (feasible-only: inf if infeasible).
    mask: inter-route neighbours only where mask[pair] is set (edge-based, ETGA).
    with_index: (score, u, v) triples with the canonical slot pair of each move."""
    cur = {}
    for idx, r in enumerate(routes):
        cur[idx] = simulate(dist, demand, tw, r, pickup)
    out = []
    for item in neighbours(routes, op, n1, n2, keyed=True, indexed=True):
        ids, news, pair, uv = item
        if mask is not None and pair is not None and not mask[pair[0]][pair[1]]:
            continue
        dD = dLV = dTV = 0.0
        feas = True
        for rid, nr in zip(ids, news):
            D, L, TV = simulate(dist, demand, tw, nr, pickup)
            D0, L0, TV0 = cur[rid]
            dD += D - D0
            dLV += max(L - capacity, 0) - max(L0 - capacity, 0)
            dTV += TV - TV0
            feas = feas and L <= capacity and TV == 0
        sc = (dD if feas else math.inf) if mode == 0 else dD + wQ * dLV + wT * dTV
        if with_index == "full":
            out.append((sc, uv[0], uv[1], feas, any(in_band(dist, tw, nr) for nr in news)))
        else:
            out.append((sc, uv[0], uv[1]) if with_index else sc)
    return out


def best(triples, Q):
    """Lowest (score, u * Q + v) over finite scores (reading 5), or None."""
    fin = [(s, u * Q + v) for s, u, v in triples if s != math.inf]
    return min(fin) if fin else None
