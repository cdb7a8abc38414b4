// Minor-min-width contraction loop shared by the host (one-off root bound,
// solver.cpp:31) and the oracle-parity MMW traces; the device prune runs
// mmw_child (wave_device.cuh) on an explicit minor instead. Restates
// run_mmw / contract_step / adjacent_roots (proj/src/mmw.cpp:49-140) over a
// byte-per-vertex DSU and degree array, walking the original graph through
// eliminated vertices and same-class members instead of building the minor.
#pragma once

#include "vset.hpp"

namespace etw {

template <int W>
struct MinorState {
    const Set<W>* adj;  // original adjacency
    Set<W> elim;        // eliminated vertices
    Set<W> alive;       // alive class roots
    unsigned char* parent;
    unsigned char* degree;
};

template <int W>
ETW_HD int minor_find(MinorState<W>& m, int x) {
    while (m.parent[x] != x) {
        m.parent[x] = m.parent[m.parent[x]];
        x = m.parent[x];
    }
    return x;
}

// Alive class roots adjacent to the class of root r (mmw.cpp:49-71).
template <int W>
ETW_HD Set<W> minor_adjacent_roots(MinorState<W>& m, int r) {
    Set<W> roots = Set<W>::zero();
    Set<W> seen = Set<W>::bit(r);
    Set<W> frontier = seen;
    while (frontier.any()) {
        int x = frontier.pop();
        Set<W> nb = m.adj[x] - seen;
        seen |= nb;
        frontier |= nb & m.elim;
        Set<W> live = nb - m.elim;
        while (live.any()) {
            int y = live.pop();
            int ry = minor_find<W>(m, y);
            if (ry == r) frontier.add(y);
            else if (m.alive.has(ry)) roots.add(ry);
        }
    }
    return roots;
}

// max over steps of the second-smallest alive degree, stopping once it
// exceeds cap (run_mmw, mmw.cpp:120-140; contract_step, mmw.cpp:81-116)
template <int W>
ETW_HD int minor_min_width(MinorState<W>& m, int cap) {
    int bound = 0;
    while (m.alive.count() >= 2) {
        int d1 = 1 << 30, d2 = 1 << 30, v = -1;
        Set<W> it = m.alive;
        while (it.any()) {
            int x = it.pop();
            int d = m.degree[x];
            if (d < d1) {
                d2 = d1;
                d1 = d;
                v = x;
            } else if (d < d2) {
                d2 = d;
            }
        }
        if (d2 > bound) bound = d2;
        if (bound > cap) return bound;
        if (d1 == 0) {  // isolated class: drop it
            m.alive.del(v);
            continue;
        }
        Set<W> adj_v = minor_adjacent_roots<W>(m, v);
        int u = -1, du = 1 << 30;
        Set<W> it2 = adj_v;
        while (it2.any()) {
            int x = it2.pop();
            if (m.degree[x] < du) {
                du = m.degree[x];
                u = x;
            }
        }
        Set<W> common = adj_v & minor_adjacent_roots<W>(m, u);
        common.del(v);
        common.del(u);
        int c = common.count();
        m.parent[u] = static_cast<unsigned char>(v);
        m.alive.del(u);
        m.degree[v] = static_cast<unsigned char>(m.degree[v] + m.degree[u] - c - 2);
        while (common.any()) --m.degree[common.pop()];
    }
    return bound;
}

}  // namespace etw
