#include "preprocess.hpp"

#include <algorithm>
#include <array>
#include <deque>
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
// non-adjacent): unit vertex capacities via the usual in/out split, BFS
// augmenting paths. The value is a max-flow value, hence independent of the
// augmentation order (the reference uses Dinic, preprocess.cpp:115-169).
class VertexFlow {
public:
    explicit VertexFlow(const Graph& g) : g_(g), n_(g.vertex_count()) {
        // node 2v = in(v), 2v+1 = out(v)
        int nodes = 2 * n_;
        head_.assign(nodes, -1);
        for (int v = 0; v < n_; ++v) add_arc(2 * v, 2 * v + 1, 1);
        for (int v = 0; v < n_; ++v)
            for (int u : g.neighbor_list(v)) add_arc(2 * v + 1, 2 * u, kBig);
        base_cap_ = cap_;
    }

    int paths(int s, int t) {
        cap_ = base_cap_;
        int src = 2 * s + 1, dst = 2 * t;
        int flow = 0;
        std::vector<int> via(2 * n_);
        for (;;) {
            std::fill(via.begin(), via.end(), -2);
            std::deque<int> q{src};
            via[src] = -1;
            while (!q.empty() && via[dst] == -2) {
                int x = q.front();
                q.pop_front();
                for (int a = head_[x]; a >= 0; a = next_[a]) {
                    int y = to_[a];
                    if (cap_[a] > 0 && via[y] == -2) {
                        via[y] = a;
                        q.push_back(y);
                    }
                }
            }
            if (via[dst] == -2) return flow;
            for (int y = dst; y != src;) {
                int a = via[y];
                cap_[a] -= 1;
                cap_[a ^ 1] += 1;
                y = to_[a ^ 1];
            }
            ++flow;
        }
    }

private:
    static constexpr int kBig = 1 << 20;
    void add_arc(int a, int b, int c) {
        to_.push_back(b);
        cap_.push_back(c);
        next_.push_back(head_[a]);
        head_[a] = static_cast<int>(to_.size()) - 1;
        to_.push_back(a);
        cap_.push_back(0);
        next_.push_back(head_[b]);
        head_[b] = static_cast<int>(to_.size()) - 1;
    }
    const Graph& g_;
    int n_;
    std::vector<int> head_, next_, to_, cap_, base_cap_;
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

PathCounts disjoint_path_counts(const Graph& g) {
    int n = g.vertex_count();
    PathCounts pc;
    pc.n = n;
    pc.counts.assign(static_cast<size_t>(n) * n, 0);
    VertexFlow flow(g);
    for (int s = 0; s < n; ++s)
        for (int t = s + 1; t < n; ++t) {
            int c = g.adjacent(s, t) ? PathCounts::kAdjacent : flow.paths(s, t);
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
