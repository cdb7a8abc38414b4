// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A thin extern "C" harness around the *unmodified* reference elimtw core
// (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libetwref.so). It lets the Python tests and bench.py's
// cpu_baseline / --impl reference legs drive the reference's own
// `decide` (proj/src/dp.cpp:167-194), `expand_layer` (dp.cpp:73-165),
// `solve` (proj/src/solver.cpp:149-196), Bloom hashing (proj/src/bloom.cpp:
// 27-70), MMW (proj/src/mmw.cpp:20-161) and preprocess
// (proj/src/preprocess.cpp:188-258) with plain pointers, so every golden
// vector in tests/golden/ comes from the reference itself.
//
// All symbols are prefixed ref_ and everything else in the .so is hidden,
// so the reference's own etw_* never interposes on the product library.

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "bloom.hpp"
#include "dp.hpp"
#include "graph.hpp"
#include "mmw.hpp"
#include "preprocess.hpp"
#include "solver.hpp"
#include "treedec.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

using namespace elimtw;

namespace {

Graph graph_from_rows(int n, const uint64_t* rows) {
    std::vector<VertexSet> r(n);
    for (int v = 0; v < n; ++v) r[v].w[0] = rows[v];
    return Graph::from_rows(n, r);
}

struct RefRun {
    Outcome outcome = Outcome::infeasible;
    SearchState witness;
    bool overflowed = false;
    std::vector<LayerStats> rounds;
    std::vector<std::vector<SearchState>> layers;
    std::string error;
};

DpConfig make_cfg(int dedup, int mmw, int threads, uint64_t cap, int bpe, int hashes) {
    DpConfig cfg;
    cfg.dedup = dedup ? DedupMode::exact_set : DedupMode::bloom;
    cfg.use_mmw = mmw != 0;
    cfg.thread_count = threads;
    cfg.max_layer_states = cap;
    cfg.bloom.bits_per_element = bpe;
    cfg.bloom.num_hashes = hashes;
    return cfg;
}

}  // namespace

// ---- Bloom / Murmur (bloom.cpp) ----------------------------------------
REF_API uint32_t ref_murmur3_x86_32(const void* data, size_t len, uint32_t seed) {
    return murmur3_x86_32(data, len, seed);
}

REF_API void ref_hash_pair(uint64_t key, uint32_t* h1, uint32_t* h2) {
    auto p = ConcurrentBloom::hash_pair(key);
    *h1 = p.first;
    *h2 = p.second;
}

// Inserts `count` keys in order into a fresh filter sized for
// `expected` elements and writes the novel flag of each insert.
REF_API uint64_t ref_bloom_insert_seq(uint64_t expected, int bpe, int hashes,
                                      const uint64_t* keys, size_t count,
                                      uint8_t* novel_out) {
    ConcurrentBloom f(expected, BloomParams{bpe, hashes});
    for (size_t i = 0; i < count; ++i) novel_out[i] = f.insert_and_check(keys[i]) ? 1 : 0;
    return f.bit_count();
}

REF_API double ref_bloom_expected_fp(uint64_t expected, int bpe, int hashes,
                                     uint64_t inserted) {
    ConcurrentBloom f(expected, BloomParams{bpe, hashes});
    return f.expected_false_positive_rate(inserted);
}

// ---- graph / q_set (graph.hpp:61-78) ------------------------------------
REF_API uint64_t ref_q_set(int n, const uint64_t* rows, uint64_t s, int v) {
    Graph g = graph_from_rows(n, rows);
    VertexSet vs;
    vs.w[0] = s;
    return q_set(g, vs, v).w[0];
}

// ---- DP engine (dp.cpp) ------------------------------------------------
// Returns a handle; every finished layer is captured through the
// reference's own DpConfig::observer seam (dp.hpp:31-32) when keep_layers.
REF_API void* ref_decide(int n, const uint64_t* rows, int k, uint64_t forbidden,
                         int dedup, int mmw, int threads, uint64_t cap, int bpe,
                         int hashes, int rounds, int keep_layers) {
    auto* run = new RefRun;
    try {
        Graph g = graph_from_rows(n, rows);
        DpConfig cfg = make_cfg(dedup, mmw, threads, cap, bpe, hashes);
        if (keep_layers) {
            cfg.observer = [run](int, int, const std::vector<SearchState>& st) {
                run->layers.push_back(st);
            };
        }
        VertexSet f;
        f.w[0] = forbidden;
        DecideResult r = decide(g, k, f, cfg, rounds);
        run->outcome = r.outcome;
        run->witness = r.witness;
        run->overflowed = r.overflowed;
        run->rounds = r.rounds;
    } catch (const std::exception& e) {
        run->error = e.what();
    }
    return run;
}

// Runs expand_layer once on an explicit input list (test_dp.cpp:66-143).
REF_API void* ref_expand_layer(int n, const uint64_t* rows, int k, uint64_t forbidden,
                               const uint64_t* in_sets, const uint32_t* in_hist,
                               size_t in_count, int dedup, int mmw, int threads,
                               uint64_t cap, int bpe, int hashes) {
    auto* run = new RefRun;
    try {
        Graph g = graph_from_rows(n, rows);
        DpConfig cfg = make_cfg(dedup, mmw, threads, cap, bpe, hashes);
        std::vector<SearchState> in(in_count);
        for (size_t i = 0; i < in_count; ++i) in[i] = {in_sets[i], in_hist[i]};
        VertexSet f;
        f.w[0] = forbidden;
        LayerStats st;
        LayerList out = expand_layer(g, k, f, in, cfg, st);
        run->rounds.push_back(st);
        run->overflowed = out.overflowed;
        run->layers.push_back(std::move(out.states));
    } catch (const std::exception& e) {
        run->error = e.what();
    }
    return run;
}

REF_API const char* ref_run_error(void* h) {
    return static_cast<RefRun*>(h)->error.c_str();
}

REF_API int ref_run_outcome(void* h) { return static_cast<int>(static_cast<RefRun*>(h)->outcome); }
REF_API int ref_run_overflowed(void* h) { return static_cast<RefRun*>(h)->overflowed ? 1 : 0; }
REF_API uint64_t ref_run_witness_set(void* h) { return static_cast<RefRun*>(h)->witness.set; }
REF_API uint32_t ref_run_witness_hist(void* h) { return static_cast<RefRun*>(h)->witness.history; }
REF_API int ref_run_round_count(void* h) { return static_cast<int>(static_cast<RefRun*>(h)->rounds.size()); }

// stats: 6 u64 per round: k, round, expanded, emitted, duplicates, mmw_pruned;
// overflowed flags go to ovf.
REF_API void ref_run_rounds(void* h, uint64_t* stats, uint8_t* ovf) {
    auto* run = static_cast<RefRun*>(h);
    for (size_t i = 0; i < run->rounds.size(); ++i) {
        const LayerStats& s = run->rounds[i];
        stats[6 * i + 0] = static_cast<uint64_t>(s.k);
        stats[6 * i + 1] = static_cast<uint64_t>(s.round);
        stats[6 * i + 2] = s.expanded;
        stats[6 * i + 3] = s.emitted;
        stats[6 * i + 4] = s.duplicates;
        stats[6 * i + 5] = s.mmw_pruned;
        ovf[i] = s.overflowed ? 1 : 0;
    }
}

REF_API int ref_run_layer_count(void* h) { return static_cast<int>(static_cast<RefRun*>(h)->layers.size()); }
REF_API uint64_t ref_run_layer_size(void* h, int i) {
    return static_cast<RefRun*>(h)->layers[i].size();
}
REF_API void ref_run_layer(void* h, int i, uint64_t* sets, uint32_t* hist) {
    const auto& L = static_cast<RefRun*>(h)->layers[i];
    for (size_t j = 0; j < L.size(); ++j) {
        sets[j] = L[j].set;
        hist[j] = L[j].history;
    }
}
REF_API void ref_run_free(void* h) { delete static_cast<RefRun*>(h); }

// ---- MMW (mmw.cpp) -----------------------------------------------------
REF_API int ref_mmw_lower_bound(int n, const uint64_t* rows, uint64_t s, int cap) {
    Graph g = graph_from_rows(n, rows);
    VertexSet vs;
    vs.w[0] = s;
    return mmw_lower_bound(g, vs, cap);
}

// Trace rows of 5 ints: v, u, common, min_degree_after, bound_after.
REF_API int ref_mmw_trace(int n, const uint64_t* rows, uint64_t s, int cap, int* out,
                          int max_steps, int* bound_out) {
    Graph g = graph_from_rows(n, rows);
    VertexSet vs;
    vs.w[0] = s;
    auto steps = mmw_trace(g, vs, cap, bound_out);
    int m = static_cast<int>(steps.size());
    for (int i = 0; i < m && i < max_steps; ++i) {
        out[5 * i + 0] = steps[i].step.v;
        out[5 * i + 1] = steps[i].step.u;
        out[5 * i + 2] = steps[i].step.common;
        out[5 * i + 3] = steps[i].step.min_degree_after;
        out[5 * i + 4] = steps[i].bound_after;
    }
    return m;
}

// Degrees of the derived child view (mmw.cpp:20-43), 0 for non-alive.
REF_API void ref_mmw_child_degrees(int n, const uint64_t* rows, uint64_t s, int v,
                                   uint8_t* deg_out) {
    Graph g = graph_from_rows(n, rows);
    VertexSet vs;
    vs.w[0] = s;
    VertexSet r[kMaxVertices];
    for (int w = 0; w < n; ++w)
        if (!vs.contains(w)) r[w] = q_set(g, vs, w);
    MinorView view = init_view_after(g, vs, v, r);
    for (int w = 0; w < n; ++w) deg_out[w] = view.alive.contains(w) ? view.degree[w] : 0;
}

// ---- preprocess (preprocess.cpp) ---------------------------------------
REF_API uint64_t ref_max_clique(int n, const uint64_t* rows) {
    return max_clique(graph_from_rows(n, rows)).w[0];
}

REF_API void ref_disjoint_paths(int n, const uint64_t* rows, uint8_t* out) {
    DisjointPathsMatrix m = vertex_disjoint_paths(graph_from_rows(n, rows));
    std::memcpy(out, m.counts.data(), m.counts.size());
}

// Writes, per sub-instance, its vertex list (original ids) into verts
// (concatenated), sizes into sizes, and parent cut (local id) into cuts.
REF_API int ref_split(int n, const uint64_t* rows, int mode, int* verts, int* sizes,
                      int* cuts) {
    auto subs = split_instance(graph_from_rows(n, rows), static_cast<SplitMode>(mode));
    int off = 0;
    for (size_t i = 0; i < subs.size(); ++i) {
        sizes[i] = static_cast<int>(subs[i].to_original.size());
        cuts[i] = subs[i].parent_cut;
        for (int v : subs[i].to_original) verts[off++] = v;
    }
    return static_cast<int>(subs.size());
}

// ---- full solve (solver.cpp) -------------------------------------------
// Options mirror etw_options (elimtw.h:51-63). Returns 0 on success and
// copies the stats JSON (stats_json, solver.cpp:198-297) into json_buf.
REF_API int ref_solve(int n, const uint64_t* rows, int dedup, int split, int use_mmw,
                      int use_clique, int use_improvement, int threads, uint64_t cap,
                      int bpe, int hashes, int start_k, int emit_order, int* kind,
                      int* value, int* order, size_t* order_len, char* json_buf,
                      size_t json_len, char* err, size_t err_len) {
    try {
        Graph g = graph_from_rows(n, rows);
        SolveOptions o;
        o.dp = make_cfg(dedup, use_mmw, threads, cap, bpe, hashes);
        o.split = static_cast<SplitMode>(split);
        o.use_clique = use_clique != 0;
        o.use_improvement = use_improvement != 0;
        if (start_k >= 0) o.starting_k = start_k;
        o.emit_order = emit_order != 0;
        SolveResult r = solve(g, o);
        *kind = r.kind == ResultKind::exact ? 0 : 1;
        *value = r.value;
        *order_len = r.order.size();
        for (size_t i = 0; i < r.order.size(); ++i) order[i] = r.order[i];
        if (json_buf && json_len) {
            std::string js = stats_json(g, o, r);
            std::snprintf(json_buf, json_len, "%s", js.c_str());
        }
        return 0;
    } catch (const std::exception& e) {
        if (err && err_len) std::snprintf(err, err_len, "%s", e.what());
        return 1;
    }
}

REF_API int ref_verify_order(int n, const uint64_t* rows, const int* order, int len) {
    Graph g = graph_from_rows(n, rows);
    return verify_order(g, EliminationOrder(order, order + len));
}

// ---- deterministic generators (proj/tests/helpers.hpp:12-80) -------------
#include "helpers.hpp"

// kind: 0 random_graph(seed,n,p), 1 random_connected_graph(seed,n,p),
// 2 grid_graph(a,b), 3 complete(a), 4 cycle(a), 5 path(a), 6 biclique(a,b),
// 7 petersen. Returns n and fills rows (n <= 64).
REF_API int ref_generate(int kind, uint32_t seed, int a, int b, double p, uint64_t* rows) {
    Graph g;
    switch (kind) {
        case 0: g = test::random_graph(seed, a, p); break;
        case 1: g = test::random_connected_graph(seed, a, p); break;
        case 2: g = test::grid_graph(a, b); break;
        case 3: g = test::complete_graph(a); break;
        case 4: g = test::cycle_graph(a); break;
        case 5: g = test::path_graph(a); break;
        case 6: g = test::biclique(a, b); break;
        default: g = test::petersen_graph(); break;
    }
    for (int v = 0; v < g.vertex_count(); ++v) rows[v] = g.neighbors(v).w[0];
    return g.vertex_count();
}

REF_API int ref_parse(const char* text, size_t len, int* n_out, uint64_t* rows,
                      char* err, size_t err_len) {
    try {
        std::string body(text, len);
        Graph g = parse_graph(body, detect_format(body));
        *n_out = g.vertex_count();
        for (int v = 0; v < g.vertex_count(); ++v) rows[v] = g.neighbors(v).w[0];
        return 0;
    } catch (const std::exception& e) {
        if (err && err_len) std::snprintf(err, err_len, "%s", e.what());
        return 1;
    }
}

// improve_graph(g, k, vertex_disjoint_paths(g)) (preprocess.cpp:218-258)
REF_API void ref_improve_graph(int n, const uint64_t* rows, int k, uint64_t* out_rows) {
    Graph g = graph_from_rows(n, rows);
    Graph h = improve_graph(g, k, vertex_disjoint_paths(g));
    for (int v = 0; v < n; ++v) out_rows[v] = h.neighbors(v).w[0];
}

// Full solve with the DpConfig::observer seam capturing every layer the
// search phase and reconstruction produce, in call order (k in stats[0]).
REF_API void* ref_solve_layers(int n, const uint64_t* rows, int dedup, int split, int use_mmw,
                               int use_clique, int use_improvement, uint64_t cap,
                               int start_k) {
    auto* run = new RefRun;
    try {
        Graph g = graph_from_rows(n, rows);
        SolveOptions o;
        o.dp = make_cfg(dedup, use_mmw, 1, cap, 24, 17);
        o.split = static_cast<SplitMode>(split);
        o.use_clique = use_clique != 0;
        o.use_improvement = use_improvement != 0;
        if (start_k >= 0) o.starting_k = start_k;
        o.emit_order = false;
        o.dp.observer = [run](int k, int round, const std::vector<SearchState>& st) {
            LayerStats s;
            s.k = k;
            s.round = round;
            s.emitted = st.size();
            run->rounds.push_back(s);
            run->layers.push_back(st);
        };
        (void)solve(g, o);
    } catch (const std::exception& e) {
        run->error = e.what();
    }
    return run;
}
