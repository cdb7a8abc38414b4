// Host-side preprocessing that runs once per block (or once per k):
// connected / biconnected splitting with post-ordered blocks, the exact
// maximum clique (forbidden suffix), pairwise vertex-disjoint path counts
// and the improvement edges. Contract: identical outputs to the reference
// (proj/src/preprocess.hpp:12-46, preprocess.cpp:1-260), since every layer
// the device produces depends on the clique and the improved graph.
#pragma once

#include <cstdint>
#include <vector>

#include "graph.hpp"

namespace etw {

enum class SplitMode { none = 0, connected = 1, biconnected = 2 };

struct SubInstance {
    Graph graph;
    std::vector<int> to_original;  // local id -> original id
    int parent_cut = -1;           // local id of the cut shared with the parent block
};

// Blocks are emitted in post-order over the block-cut tree so a stitched
// order can defer each cut vertex to its parent (preprocess.cpp:87-112).
std::vector<SubInstance> split_instance(const Graph& g, SplitMode mode);

// Maximum clique, lexicographically smallest vertex list among the maximum
// ones (preprocess.cpp:171-184, 210-216).
HostSet max_clique(const Graph& g);

// counts[u*n+v] = number of internally vertex-disjoint u-v paths; 255 for
// adjacent pairs (never consulted). preprocess.cpp:218-243.
struct PathCounts {
    static constexpr int kAdjacent = 255;
    int n = 0;
    std::vector<uint8_t> counts;
    int at(int u, int v) const { return counts[static_cast<size_t>(u) * n + v]; }
};
// Pairs whose degree bound min(deg u, deg v) is below `need` get that bound
// instead of the exact count (enough for improve_graph at any k >= need-1).
PathCounts disjoint_path_counts(const Graph& g, int need = 0);

// Adds every non-edge {u,v} joined by >= k+1 disjoint paths
// (preprocess.cpp:245-258).
Graph improve_graph(const Graph& g, int k, const PathCounts& paths);

}  // namespace etw
