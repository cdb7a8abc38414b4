#include "preprocess.hpp"

#include <algorithm>
#include <array>
#include <functional>

namespace etw {

namespace {

// Sub-instance over `keep` (ascending original ids), cut given in original ids.
SubInstance induced(const Graph& g, const HostSet& keep, int cut_original) {
    SubInstance sub;
    std::array<int, kMaxVertices> local{};
    for (int v : members(keep)) {
        local[v] = static_cast<int>(sub.to_original.size());
        sub.to_original.push_back(v);
    }
    std::vector<std::pair<int, int>> edges;
    for (int v : members(keep))
        for (int u : members(g.neighbors(v) & keep))
            if (u > v) edges.emplace_back(local[v], local[u]);
    sub.graph = Graph::from_edges(static_cast<int>(sub.to_original.size()), edges);
    sub.parent_cut = cut_original < 0 ? -1 : local[cut_original];
    return sub;
}

// Components in order of their smallest vertex (preprocess.cpp:26-44).
std::vector<HostSet> components(const Graph& g) {
    std::vector<HostSet> out;
    HostSet covered = HostSet::zero();
    for (int r = 0; r < g.vertex_count(); ++r) {
        if (covered.has(r)) continue;
        HostSet comp = HostSet::bit(r), frontier = HostSet::bit(r);
        while (frontier.any()) {
            int v = frontier.pop();
            HostSet fresh = g.neighbors(v) - comp;
            comp |= fresh;
            frontier |= fresh;
        }
        covered |= comp;
        out.push_back(comp);
    }
    return out;
}

// Hopcroft-Tarjan biconnected blocks of the component containing `root`,
// iterative, visiting neighbours in ascending order; blocks are recorded in
// the order their articulation test fires (same as preprocess.cpp:47-82).
std::vector<HostSet> blocks_from(const Graph& g, int root) {
    struct Frame {
        int u, parent;
        size_t next;
    };
    std::vector<int> disc(g.vertex_count(), 0), low(g.vertex_count(), 0);
    std::vector<std::pair<int, int>> edge_stack;
    std::vector<Frame> stack;
    std::vector<HostSet> blocks;
    int clock = 0;
    disc[root] = low[root] = ++clock;
    stack.push_back({root, -1, 0});
    while (!stack.empty()) {
        Frame& f = stack.back();
        const std::vector<int>& nb = g.neighbor_list(f.u);
        if (f.next < nb.size()) {
            int u = f.u;
            int v = nb[f.next++];
            if (v == f.parent) continue;
            if (disc[v] == 0) {
                edge_stack.emplace_back(u, v);
                disc[v] = low[v] = ++clock;
                stack.push_back({v, u, 0});
            } else if (disc[v] < disc[u]) {
                edge_stack.emplace_back(u, v);
                low[u] = std::min(low[u], disc[v]);
            }
            continue;
        }
        int child = f.u;
        stack.pop_back();
        if (stack.empty()) break;
        int u = stack.back().u;
        low[u] = std::min(low[u], low[child]);
        if (low[child] >= disc[u]) {
            HostSet block = HostSet::zero();
            for (;;) {
                auto e = edge_stack.back();
                edge_stack.pop_back();
                block.add(e.first);
                block.add(e.second);
                if (e.first == u && e.second == child) break;
            }
            blocks.push_back(block);
        }
    }
    return blocks;
}

std::vector<int> as_list(const HostSet& s) {
    std::vector<int> v;
    for (int x : members(s)) v.push_back(x);
    return v;
}

// Post-order walk of the block-cut tree, rooted at the block with the
// lexicographically smallest vertex list (preprocess.cpp:87-112).
void emit_post_order(const Graph& g, const std::vector<HostSet>& blocks,
                     std::vector<SubInstance>& out) {
    std::vector<size_t> lex(blocks.size());
    for (size_t i = 0; i < lex.size(); ++i) lex[i] = i;
    std::sort(lex.begin(), lex.end(),
              [&](size_t a, size_t b) { return as_list(blocks[a]) < as_list(blocks[b]); });
    std::array<int, kMaxVertices> owners{};
    for (const HostSet& b : blocks)
        for (int v : members(b)) ++owners[v];
    std::vector<char> done(blocks.size(), 0);
    std::function<void(size_t, int)> visit = [&](size_t b, int cut) {
        done[b] = 1;
        for (int c : members(blocks[b])) {
            if (owners[c] < 2 || c == cut) continue;
            for (size_t other : lex)
                if (!done[other] && blocks[other].has(c)) visit(other, c);
        }
        out.push_back(induced(g, blocks[b], cut));
    };
    visit(lex.front(), -1);
}

// Lexicographic branch and bound for the maximum clique
// (preprocess.cpp:171-184): candidates are taken smallest first, ties in
// size resolved towards the lexicographically smaller list.
void grow_clique(const Graph& g, std::vector<int>& cur, HostSet cand, std::vector<int>& best) {
    if (cand.none()) {
        if (cur.size() > best.size() || (cur.size() == best.size() && cur < best)) best = cur;
        return;
    }
    while (cand.any()) {
        if (cur.size() + static_cast<size_t>(cand.count()) < best.size()) return;
        int v = cand.pop();
        cur.push_back(v);
        grow_clique(g, cur, cand & g.neighbors(v), best);
        cur.pop_back();
    }
}

// Maximum number of internally vertex-disjoint s-t paths (s, t
// non-adjacent), by augmenting paths in the vertex-split residual graph.
// The residual arcs are derived from bitsets instead of an arc list:
//   out(u) -> in(w)  for every edge uw (infinite capacity),
//   out(u) -> in(u)  when u carries a path (reverse of the vertex arc),
//   in(v)  -> out(v) when v is still free,
//   in(v)  -> out(u) when a path enters v from u (reverse flow arc).
// The value is a max-flow value, hence independent of the augmentation
// order (the reference runs Dinic on an explicit network, preprocess.cpp:
// 115-169, 218-243).
class MengerFlow {
public:
    explicit MengerFlow(const Graph& g) : g_(g), n_(g.vertex_count()), into_(n_), par_in_(n_), par_out_(n_) {}

    int paths(int s, int t) {
        used_ = HostSet::zero();
        for (HostSet& x : into_) x = HostSet::zero();
        int flow = 0;
        while (augment(s, t)) ++flow;
        return flow;
    }

private:
    bool augment(int s, int t) {
        HostSet seen_in = HostSet::zero(), seen_out = HostSet::bit(s);
        HostSet frontier_out = seen_out;
        for (;;) {
            HostSet reached_in = HostSet::zero();
            for (int u : members(frontier_out)) {
                HostSet c = g_.neighbors(u);
                if (used_.has(u)) c.add(u);
                c = c - seen_in;
                for (int v : members(c)) par_in_[v] = u;
                seen_in |= c;
                reached_in |= c;
            }
            if (seen_in.has(t)) break;
            HostSet reached_out = HostSet::zero();
            for (int v : members(reached_in)) {
                HostSet c = into_[v];
                if (!used_.has(v)) c.add(v);
                c = c - seen_out;
                for (int x : members(c)) par_out_[x] = v;
                seen_out |= c;
                reached_out |= c;
            }
            if (reached_out.none()) return false;
            frontier_out = reached_out;
        }
        // walk the path back from in(t), updating the flow
        int x_in = t;
        for (;;) {
            const int u = par_in_[x_in];  // arc out(u) -> in(x_in)
            if (u == x_in) used_.del(u);  // reverse vertex arc: u is freed
            else into_[x_in].add(u);      // forward edge arc
            if (u == s) break;
            const int v = par_out_[u];    // arc in(v) -> out(u)
            if (v == u) used_.add(u);     // forward vertex arc: u now carries a path
            else into_[v].del(u);         // reverse flow arc: cancels u -> v
            x_in = v;
        }
        return true;
    }

    const Graph& g_;
    int n_;
    HostSet used_ = HostSet::zero();
    std::vector<HostSet> into_;  // into_[v] = vertices u with a path arc u -> v
    std::vector<int> par_in_, par_out_;
};

}  // namespace

std::vector<SubInstance> split_instance(const Graph& g, SplitMode mode) {
    std::vector<SubInstance> out;
    if (mode == SplitMode::none) {
        out.push_back(induced(g, g.vertices(), -1));
        return out;
    }
    for (const HostSet& comp : components(g)) {
        if (mode == SplitMode::connected || comp.count() == 1) {
            out.push_back(induced(g, comp, -1));
            continue;
        }
        emit_post_order(g, blocks_from(g, comp.lowest()), out);
    }
    return out;
}

HostSet max_clique(const Graph& g) {
    std::vector<int> cur, best;
    grow_clique(g, cur, g.vertices(), best);
    HostSet c = HostSet::zero();
    for (int v : best) c.add(v);
    return c;
}

PathCounts disjoint_path_counts(const Graph& g, int need) {
    int n = g.vertex_count();
    PathCounts pc;
    pc.n = n;
    pc.counts.assign(static_cast<size_t>(n) * n, 0);
    MengerFlow flow(g);
    for (int s = 0; s < n; ++s)
        for (int t = s + 1; t < n; ++t) {
            // at most min(deg s, deg t) paths: below `need` that bound decides
            const int bound = std::min(g.neighbors(s).count(), g.neighbors(t).count());
            int c = g.adjacent(s, t) ? PathCounts::kAdjacent
                                     : (bound < need ? bound : flow.paths(s, t));
            pc.counts[static_cast<size_t>(s) * n + t] = static_cast<uint8_t>(c);
            pc.counts[static_cast<size_t>(t) * n + s] = static_cast<uint8_t>(c);
        }
    return pc;
}

Graph improve_graph(const Graph& g, int k, const PathCounts& paths) {
    int n = g.vertex_count();
    std::vector<HostSet> rows = g.rows();
    for (int u = 0; u < n; ++u)
        for (int v = u + 1; v < n; ++v)
            if (!g.adjacent(u, v) && paths.at(u, v) >= k + 1) {
                rows[u].add(v);
                rows[v].add(u);
            }
    return Graph::from_rows(n, std::move(rows));
}

}  // namespace etw
