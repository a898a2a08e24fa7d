"""Contraction-tree search for large circuit networks (plan producer; see
plans/sycamore_plan.py). Recursive balanced bisection of the tensor graph
(spectral split + Fiduccia-Mattheyses refinement, randomised), greedy
pairing inside small parts, greedy slicing, and rotation-based local search
(the paper's local transformations) on the exact
multi-amplitude objective.

Leg sets are Python ints (bitmasks over the closed legs); a tree is a list of
merges (a, b) over tensor ids (leaves 0..n-1, merge i -> id n + i).
"""
from __future__ import annotations

import math
import random
from typing import List, Sequence, Tuple

import numpy as np


def kappa(q: int, k: int) -> float:
    """Expected distinct q-bit tuples among k uniform random bitstrings."""
    if k <= 1:
        return 1.0
    if q >= 62:
        return float(k)
    m = float(1 << q)
    return m * -math.expm1(-k / m) if k < 40 * m else m


class Network:
    def __init__(self, legs: Sequence[int], qubits: Sequence[int], k: int):
        self.legs = list(legs)
        self.q = list(qubits)
        self.n = len(self.legs)
        self.k = k
        # leg -> holders
        self.holders = {}
        for i, l in enumerate(self.legs):
            x = l
            while x:
                b = x & -x
                self.holders.setdefault(b, []).append(i)
                x ^= b
        # adjacency with multiplicity
        self.adj = [dict() for _ in range(self.n)]
        for b, hs in self.holders.items():
            if len(hs) == 2:
                u, v = hs
                self.adj[u][v] = self.adj[u].get(v, 0) + 1
                self.adj[v][u] = self.adj[v].get(u, 0) + 1


# ---- bisection -------------------------------------------------------------------


def _boundary(net: Network, part: Sequence[int]) -> int:
    x = 0
    for i in part:
        x ^= net.legs[i]
    return x


def _fm_refine(net: Network, vs: List[int], side: dict, ext: dict, lo: int, hi: int, rng, passes=4):
    """Fiduccia-Mattheyses on the cut within `vs` plus each vertex's external
    legs charged to... (external legs count toward both parts' boundaries
    equally, so only internal cut edges matter). Balance: |A| in [lo, hi]."""
    cnt = [0, 0]
    for v in vs:
        cnt[side[v]] += 1

    def gain(v):
        s = side[v]
        g = 0
        for u, w in net.adj[v].items():
            if u in side:
                g += w if side[u] != s else -w
        return g

    for _ in range(passes):
        moved = set()
        best_cut_delta, cur_delta, best_len = 0, 0, 0
        seq = []
        for _step in range(len(vs)):
            cand, cg = None, None
            for v in vs:
                if v in moved:
                    continue
                s = side[v]
                if s == 0 and cnt[0] - 1 < lo:
                    continue
                if s == 1 and cnt[0] + 1 > hi:
                    continue
                g = gain(v) + rng.random() * 0.01
                if cg is None or g > cg:
                    cand, cg = v, g
            if cand is None:
                break
            s = side[cand]
            side[cand] = 1 - s
            cnt[s] -= 1
            cnt[1 - s] += 1
            moved.add(cand)
            cur_delta -= int(round(cg))
            seq.append(cand)
            if cur_delta < best_cut_delta:
                best_cut_delta, best_len = cur_delta, len(seq)
        # roll back past the best prefix
        for v in seq[best_len:]:
            s = side[v]
            side[v] = 1 - s
            cnt[s] -= 1
            cnt[1 - s] += 1
        if best_len == 0:
            break


def bisect(net: Network, vs: List[int], rng: random.Random, imbalance: float, noise: float) -> Tuple[List[int], List[int]]:
    n = len(vs)
    idx = {v: i for i, v in enumerate(vs)}
    L = np.zeros((n, n))
    for v in vs:
        for u, w in net.adj[v].items():
            if u in idx:
                ww = w * (1.0 + noise * rng.random())
                L[idx[v], idx[u]] -= ww
                L[idx[v], idx[v]] += ww
    L += np.eye(n) * 1e-9
    try:
        w, V = np.linalg.eigh(L)
        f = V[:, 1] if n > 1 else np.zeros(1)
    except np.linalg.LinAlgError:
        f = np.array([rng.random() for _ in range(n)])
    f = f + noise * 1e-3 * np.array([rng.random() for _ in range(n)])
    order = [vs[i] for i in np.argsort(f)]
    lo = max(1, int(math.floor(n * (0.5 - imbalance))))
    hi = min(n - 1, int(math.ceil(n * (0.5 + imbalance))))
    # sweep for the smallest internal cut among balanced prefixes
    side = {v: 1 for v in vs}
    cut = 0
    best_cut, best_k = None, lo
    inside = set()
    for kk, v in enumerate(order[:hi], start=1):
        for u, ww in net.adj[v].items():
            if u in idx:
                cut += -ww if u in inside else ww
        inside.add(v)
        if kk >= lo and (best_cut is None or cut < best_cut):
            best_cut, best_k = cut, kk
    for v in order[:best_k]:
        side[v] = 0
    _fm_refine(net, vs, side, None, lo, hi, rng)
    a = [v for v in vs if side[v] == 0]
    b = [v for v in vs if side[v] == 1]
    if not a or not b:
        a, b = order[: n // 2], order[n // 2:]
    return a, b


def greedy_merge(net: Network, ids: List[int], legs: dict, qs: dict, rng, temp: float, merges: list, next_id: list):
    """Greedy pairing of the given subtree ids (legs/qs dicts updated)."""
    alive = list(ids)
    while len(alive) > 1:
        best, bs = None, None
        for i in range(len(alive)):
            for j in range(i + 1, len(alive)):
                a, b = alive[i], alive[j]
                shared = legs[a] & legs[b]
                out = legs[a] ^ legs[b]
                s = (1 << out.bit_count()) - (1 << legs[a].bit_count()) - (1 << legs[b].bit_count())
                s = math.copysign(math.log1p(abs(s)), s) - (0.5 if shared else -2.0)
                if temp > 0:
                    s -= temp * math.log(-math.log(rng.random() or 1e-300))
                if bs is None or s < bs:
                    best, bs = (a, b), s
        a, b = best
        n = next_id[0]
        next_id[0] += 1
        legs[n] = legs[a] ^ legs[b]
        qs[n] = qs[a] + qs[b]
        merges.append((a, b))
        alive.remove(a)
        alive.remove(b)
        alive.append(n)
    return alive[0]


def bisection_tree(net: Network, rng: random.Random, cutoff: int = 8, imbalance: float = 0.15,
                   noise: float = 0.3, temp: float = 0.1):
    legs = {i: net.legs[i] for i in range(net.n)}
    qs = {i: net.q[i] for i in range(net.n)}
    merges: List[Tuple[int, int]] = []
    next_id = [net.n]

    def rec(vs: List[int]) -> int:
        if len(vs) <= cutoff:
            return greedy_merge(net, vs, legs, qs, rng, temp, merges, next_id)
        a, b = bisect(net, vs, rng, imbalance * (0.5 + rng.random()), noise)
        ra, rb = rec(a), rec(b)
        n = next_id[0]
        next_id[0] += 1
        legs[n] = legs[ra] ^ legs[rb]
        qs[n] = qs[ra] + qs[rb]
        merges.append((ra, rb))
        return n

    rec(list(range(net.n)))
    return merges


# ---- costs -----------------------------------------------------------------------


def evaluate(net: Network, merges, sliced: int = 0, chunk: int = 0):
    """(total MACs, largest memo table, largest order). chunk > 0: memo
    streaming — request-dependent nodes evaluated per chunk of `chunk`
    requests, tables holding one chunk's distinct tuples."""
    legs = [l & ~sliced for l in net.legs]
    qs = list(net.q)
    b = chunk if 0 < chunk < net.k else net.k
    n_chunks = math.ceil(net.k / b)
    tot = 0.0
    big = 0.0
    order = 0
    for a_, b_ in merges:
        la, lb = legs[a_], legs[b_]
        q = qs[a_] + qs[b_]
        kt = kappa(q, b) if q else 1.0
        ev = kt * n_chunks if q else 1.0
        tot += ev * (1 << (la | lb).bit_count())
        out = la ^ lb
        legs.append(out)
        qs.append(q)
        big = max(big, kt * (1 << out.bit_count()))
        order = max(order, out.bit_count())
    return tot * (1 << sliced.bit_count()), big, order


def node_legs(net: Network, merges, sliced: int = 0):
    legs = [l & ~sliced for l in net.legs]
    qs = list(net.q)
    for a, b in merges:
        legs.append(legs[a] ^ legs[b])
        qs.append(qs[a] + qs[b])
    return legs, qs


def slice_greedy(net: Network, merges, max_table: float, max_slices: int, min_slices: int = 0,
                 cand_frac: float = 0.25):
    sliced = 0
    for _ in range(max_slices):
        cost, big, _ = evaluate(net, merges, sliced)
        if big <= max_table and sliced.bit_count() >= min_slices:
            break
        legs, qs = node_legs(net, merges, sliced)
        tabs = [(kappa(qs[i], net.k) * (1 << legs[i].bit_count()), legs[i]) for i in range(net.n, len(legs))]
        top = max(t for t, _ in tabs)
        cand = 0
        for t, l in tabs:
            if t >= top * cand_frac:
                cand |= l
        best, bk = None, None
        x = cand
        while x:
            bit = x & -x
            x ^= bit
            c, bg, _ = evaluate(net, merges, sliced | bit)
            key = (max(bg, max_table), c)
            if bk is None or key < bk:
                best, bk = bit, key
        if best is None:
            break
        sliced |= best
    return sliced


# ---- local search: subtree rotations ----------------------------------------------


def to_children(net: Network, merges):
    n = net.n
    ch = {}
    for i, (a, b) in enumerate(merges):
        ch[n + i] = [a, b]
    return ch, n + len(merges) - 1


def from_children(net: Network, ch, root) -> list:
    merges = []
    remap = {}
    nxt = [net.n]

    def rec(v):
        if v < net.n:
            return v
        a, b = ch[v]
        ra, rb = rec(a), rec(b)
        merges.append((ra, rb))
        i = nxt[0]
        nxt[0] += 1
        return i

    import sys

    sys.setrecursionlimit(100000)
    rec(root)
    return merges


def anneal(net: Network, merges, sliced: int, steps: int, rng: random.Random, t0: float = 0.5,
           t1: float = 0.01, max_table: float = float("inf"), penalty: float = 8.0):
    """Simulated annealing over the paper's rotations (a*b)*c -> (a*c)*b /
    (c*b)*a on log2(cost) + penalty * log2(max(table / max_table, 1)),
    evaluated exactly (O(nodes) per step)."""
    ch, root = to_children(net, merges)

    def objective(chd):
        m = from_children(net, chd, root)
        c, big, _ = evaluate(net, m, sliced)
        return math.log2(c) + penalty * max(0.0, math.log2(big / max_table)) if c > 0 else 0.0, m

    cur, cur_m = objective(ch)
    best, best_m = cur, cur_m
    internal = [v for v in ch]
    for step in range(steps):
        temp = t0 * (t1 / t0) ** (step / max(1, steps - 1))
        v = rng.choice(internal)
        a, b = ch[v]
        # pick a child that is internal to rotate with
        kids = [x for x in (a, b) if x in ch]
        if not kids:
            continue
        u = rng.choice(kids)
        other = b if u == a else a
        x, y = ch[u]
        # (x*y)*other -> (x*other)*y or (y*other)*x
        if rng.random() < 0.5:
            new_u, new_other = [x, other], y
        else:
            new_u, new_other = [y, other], x
        old_v, old_u = ch[v], ch[u]
        ch[u] = new_u
        ch[v] = [u, new_other]
        val, m = objective(ch)
        if val <= cur or rng.random() < math.exp((cur - val) / max(temp, 1e-9)):
            cur, cur_m = val, m
            if val < best:
                best, best_m = val, m
        else:
            ch[v] = old_v
            ch[u] = old_u
    return best_m


def greedy_tree(net: Network, rng: random.Random, temp: float = 0.0, alpha: float = 1.0):
    """opt_einsum-style greedy: repeatedly contract the pair sharing a leg
    with the smallest size(out) - alpha (size(a) + size(b)), k-weighted
    (k_T 2^r), with Gumbel noise of scale `temp` on log2 scores."""
    import heapq

    legs = list(net.legs)
    qs = list(net.q)
    alive = set(range(net.n))
    holders = {}
    for i, l in enumerate(legs):
        x = l
        while x:
            b = x & -x
            holders.setdefault(b, set()).add(i)
            x ^= b

    def size(i):
        return kappa(qs[i], net.k) * (1 << legs[i].bit_count())

    def score(a, b):
        out = legs[a] ^ legs[b]
        s = kappa(qs[a] + qs[b], net.k) * (1 << out.bit_count()) - alpha * (size(a) + size(b))
        if temp > 0:
            g = -math.log(-math.log(rng.random() or 1e-300))
            s = s - temp * g * abs(s) if s != 0 else -temp * g
        return s

    heap = []
    for b, hs in holders.items():
        hl = sorted(hs)
        for x in range(len(hl)):
            for y in range(x + 1, len(hl)):
                heapq.heappush(heap, (score(hl[x], hl[y]), hl[x], hl[y]))
    merges = []
    while len(alive) > 1:
        if not heap:
            hl = sorted(alive, key=size)
            a, b = hl[0], hl[1]
        else:
            s, a, b = heapq.heappop(heap)
            if a not in alive or b not in alive:
                continue
        n = len(legs)
        legs.append(legs[a] ^ legs[b])
        qs.append(qs[a] + qs[b])
        merges.append((a, b))
        alive.discard(a)
        alive.discard(b)
        for i in (a, b):
            x = legs[i]
            while x:
                bb = x & -x
                holders[bb].discard(i)
                x ^= bb
        x = legs[n]
        nbrs = set()
        while x:
            bb = x & -x
            holders.setdefault(bb, set()).add(n)
            nbrs |= holders[bb]
            x ^= bb
        nbrs.discard(n)
        for j in nbrs:
            heapq.heappush(heap, (score(min(j, n), max(j, n)) if True else 0, min(j, n), max(j, n)))
        alive.add(n)
    return merges
