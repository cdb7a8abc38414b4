// Tree decomposition induced by an elimination order, and its validation
// (reference: proj/src/treedec.hpp:10-30, treedec.cpp:8-120). Host-only; used
// by etw_check_order to validate device-produced orders.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "graph.hpp"

namespace etw {

struct TreeDecomposition {
    std::vector<HostSet> bags;               // bag(v) = {v} + Q(prefix before v, v)
    std::vector<std::pair<int, int>> edges;  // v -> earliest-eliminated member of Q
    int width = -1;
};

TreeDecomposition decomposition_from_order(const Graph& g, const EliminationOrder& order);

// Vertex coverage, edge coverage, running intersection, recorded width.
bool validate_decomposition(const Graph& g, const TreeDecomposition& td, std::string* why);

}  // namespace etw
