"""Definition-level oracles for tiny cases -- TEST INFRASTRUCTURE ONLY.

Independent restatements of the reference's slow references
(pkg/src/semimat/oracle.py) working on dense lists of Python ints, which
cannot overflow.  Nothing here shares code with the C oracle or the product.
"""

from __future__ import annotations

import heapq
import itertools


def _dims(a, b):
    if len(a[0]) != len(b):
        raise ValueError("inner dimensions disagree")
    return len(a), len(b), len(b[0])


def bool_product(a, b):
    """OR over k of AND terms (restates oracle.py:19-31)."""
    rows, inner, cols = _dims(a, b)
    return [[int(any(a[i][k] and b[k][j] for k in range(inner))) for j in range(cols)]
            for i in range(rows)]


def antidist_product(a, b, limit):
    """max over k of max(a + b - S, 0) (restates oracle.py:34-46)."""
    rows, inner, cols = _dims(a, b)
    return [[max([0] + [a[i][k] + b[k][j] - limit for k in range(inner)])
             for j in range(cols)] for i in range(rows)]


def dist_product(a, b, limit):
    """min over k of min(a + b, S) (the min-plus dual, scalars.py:60-68)."""
    rows, inner, cols = _dims(a, b)
    return [[min([limit] + [a[i][k] + b[k][j] for k in range(inner)])
             for j in range(cols)] for i in range(rows)]


def closure_by_squaring(a, limit=None):
    """a * (I | a)^(2^m) squared to a fixpoint (restates oracle.py:49-74).

    limit None = Boolean semiring, otherwise anti-distance saturating at limit.
    """
    n = len(a)
    if limit is None:
        mul, one = bool_product, 1
    else:
        mul, one = (lambda x, y: antidist_product(x, y, limit)), limit
    power = [[max(a[i][j], one) if i == j else a[i][j] for j in range(n)] for i in range(n)]
    while True:
        nxt = mul(power, power)
        if nxt == power:
            break
        power = nxt
    return mul(a, power)


def apsp_antidist(n, edges, limit):
    """Per-source Dijkstra, paths of >= 1 edge, distances >= S collapse to 0.

    Restates oracle.py:77-103 (anti-distance output: S - d for d < S).
    """
    adj = [[] for _ in range(n)]
    for u, v, w in edges:
        adj[u].append((v, w))
    out = []
    for s in range(n):
        dist = {}
        frontier = [(w, v) for v, w in adj[s]]
        heapq.heapify(frontier)
        while frontier:
            d, v = heapq.heappop(frontier)
            if v in dist:
                continue
            dist[v] = d
            for t, w in adj[v]:
                if t not in dist:
                    heapq.heappush(frontier, (d + w, t))
        out.append([limit - dist[v] if v in dist and dist[v] < limit else 0
                    for v in range(n)])
    return out


def walk_closure(a):
    """Boolean closure by enumerating every walk of 1..n edges, n <= 6
    (restates oracle.py:106-128)."""
    n = len(a)
    if n > 6:
        raise ValueError("walk enumeration supports at most 6 vertices")
    out = [[0] * n for _ in range(n)]
    for length in range(1, n + 1):
        for start in range(n):
            for walk in itertools.product(range(n), repeat=length):
                prev, ok = start, True
                for v in walk:
                    if not a[prev][v]:
                        ok = False
                        break
                    prev = v
                if ok:
                    out[start][walk[-1]] = 1
    return out
