"""Deterministic instance generators for the BASELINE configs.

The random families reproduce the reference test helpers bit for bit
(proj/tests/helpers.hpp:12-80): ``std::mt19937(seed)`` drawn once per vertex
pair u < v in row-major order and compared against ``uint64(p * 2^32)``.
Graphs are returned as adjacency rows (Python ints, bit u of rows[v] set for
every edge) and can be rendered as PACE .gr text for etw_graph_parse.
"""
from __future__ import annotations

from typing import List, Sequence


class MT19937:
    """32-bit Mersenne Twister with std::mt19937's init_genrand seeding."""

    def __init__(self, seed: int):
        mt = [0] * 624
        mt[0] = seed & 0xFFFFFFFF
        for i in range(1, 624):
            mt[i] = (1812433253 * (mt[i - 1] ^ (mt[i - 1] >> 30)) + i) & 0xFFFFFFFF
        self.mt, self.idx = mt, 624

    def _twist(self):
        mt = self.mt
        for i in range(624):
            y = (mt[i] & 0x80000000) | (mt[(i + 1) % 624] & 0x7FFFFFFF)
            mt[i] = mt[(i + 397) % 624] ^ (y >> 1) ^ (0x9908B0DF if y & 1 else 0)
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 624:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= y >> 11
        y ^= (y << 7) & 0x9D2C5680
        y ^= (y << 15) & 0xEFC60000
        y ^= y >> 18
        return y & 0xFFFFFFFF


def _rows(n: int, edges) -> List[int]:
    rows = [0] * n
    for u, v in edges:
        if u != v:
            rows[u] |= 1 << v
            rows[v] |= 1 << u
    return rows


def random_graph(seed: int, n: int, density: float, connected: bool = False) -> List[int]:
    """helpers.hpp:12-20 (random_graph) / :23-32 (random_connected_graph)."""
    rng = MT19937(seed)
    threshold = int(density * 4294967296.0)
    edges = [(v, v + 1) for v in range(n - 1)] if connected else []
    for u in range(n):
        for v in range(u + 1, n):
            if rng() < threshold:
                edges.append((u, v))
    return _rows(n, edges)


def complete_graph(n: int) -> List[int]:
    return _rows(n, [(u, v) for u in range(n) for v in range(u + 1, n)])


def cycle_graph(n: int) -> List[int]:
    return _rows(n, [(v, (v + 1) % n) for v in range(n)])


def path_graph(n: int) -> List[int]:
    return _rows(n, [(v, v + 1) for v in range(n - 1)])


def biclique(a: int, b: int) -> List[int]:
    return _rows(a + b, [(u, a + v) for u in range(a) for v in range(b)])


def grid_graph(r: int, c: int) -> List[int]:
    e = []
    for i in range(r):
        for j in range(c):
            if j + 1 < c:
                e.append((i * c + j, i * c + j + 1))
            if i + 1 < r:
                e.append((i * c + j, (i + 1) * c + j))
    return _rows(r * c, e)


def petersen_graph() -> List[int]:
    e = []
    for v in range(5):
        e += [(v, (v + 1) % 5), (5 + v, 5 + (v + 2) % 5), (v, 5 + v)]
    return _rows(10, e)


def grid_with_chords(r: int, c: int, chords: int, seed: int) -> List[int]:
    """BASELINE cfg 5: grid_graph(r, c) plus `chords` random extra edges,
    endpoints drawn as (rng() % n, rng() % n) from std::mt19937(seed),
    skipping u == v and pairs already present (cfg 5a/5b)."""
    n = r * c
    rows = grid_graph(r, c)
    rng = MT19937(seed)
    added = 0
    while added < chords:
        u, v = rng() % n, rng() % n
        if u == v or (rows[u] >> v) & 1:
            continue
        rows[u] |= 1 << v
        rows[v] |= 1 << u
        added += 1
    return rows


def myciel(i: int) -> List[int]:
    """DIMACS myciel<i>: the Mycielski construction applied i-1 times to K2
    (myciel3 = Groetzsch, 11 vertices; myciel4 = 23 vertices, identical to
    proj/tests/instances/myciel4.gr with the standard numbering)."""
    n, edges = 2, [(0, 1)]
    for _ in range(i - 1):
        new = list(edges)
        for u, v in edges:
            new += [(u, n + v), (v, n + u)]
        new += [(n + i, 2 * n) for i in range(n)]
        edges, n = new, 2 * n + 1
    return _rows(n, edges)


def queen_graph(r: int, c: int) -> List[int]:
    """Row-major queen graph (queen5_5 / queen6_6 instances)."""
    e = []
    cells = [(i, j) for i in range(r) for j in range(c)]
    for a, (i1, j1) in enumerate(cells):
        for b in range(a + 1, len(cells)):
            i2, j2 = cells[b]
            if i1 == i2 or j1 == j2 or abs(i1 - i2) == abs(j1 - j2):
                e.append((a, b))
    return _rows(r * c, e)


def to_gr(rows: Sequence[int]) -> str:
    n = len(rows)
    edges = [(u, v) for u in range(n) for v in range(u + 1, n) if (rows[u] >> v) & 1]
    return f"p tw {n} {len(edges)}\n" + "".join(f"{u + 1} {v + 1}\n" for u, v in edges)


def edge_count(rows: Sequence[int]) -> int:
    return sum(bin(r).count("1") for r in rows) // 2
