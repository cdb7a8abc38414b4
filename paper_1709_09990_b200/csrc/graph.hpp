// Host graph model, parsers and order checks.
//
// Mirrors the reference's Graph / parse_graph / detect_format / q_set /
// eliminate_all / verify_order (proj/src/graph.hpp:24-89, graph.cpp:9-205)
// with identical parse semantics and error messages, widened from 64 to 128
// vertices (the reference rejects n > 64 at graph.cpp:111-113).
#pragma once

#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "vset.hpp"

namespace etw {

struct ParseError : std::runtime_error {
    int line;
    ParseError(int line_, const std::string& msg)
        : std::runtime_error("line " + std::to_string(line_) + ": " + msg), line(line_) {}
};

enum class GraphFormat { pace_gr, dimacs_col };

class Graph {
public:
    Graph() = default;
    static Graph from_edges(int n, const std::vector<std::pair<int, int>>& edges);
    static Graph from_rows(int n, std::vector<HostSet> rows);

    int vertex_count() const { return n_; }
    long long edge_count() const { return m_; }
    HostSet vertices() const { return HostSet::prefix(n_); }
    const HostSet& neighbors(int v) const { return rows_[v]; }
    const std::vector<int>& neighbor_list(int v) const { return lists_[v]; }
    bool adjacent(int u, int v) const { return rows_[u].has(v); }
    const std::vector<HostSet>& rows() const { return rows_; }
    bool operator==(const Graph& o) const { return n_ == o.n_ && rows_ == o.rows_; }

private:
    int n_ = 0;
    long long m_ = 0;
    std::vector<HostSet> rows_;
    std::vector<std::vector<int>> lists_;
};

Graph parse_graph(std::string_view text, GraphFormat format);
GraphFormat detect_format(std::string_view text);
std::string serialize_gr(const Graph& g);

// Q(S,v) on the host (graph.hpp:61-78): vertices outside s, other than v,
// reachable from v through s. Used for verification and the one-off root
// MMW bound; the per-round evaluations run on the device.
HostSet reach_outside(const Graph& g, const HostSet& s, int v);

Graph eliminate_all(const Graph& g, const HostSet& s);

using EliminationOrder = std::vector<int>;
bool is_permutation(const Graph& g, const EliminationOrder& pi);
// max_i |Q(prefix_i, pi[i])|; throws std::invalid_argument for non-permutations
int order_width(const Graph& g, const EliminationOrder& pi);

}  // namespace etw
