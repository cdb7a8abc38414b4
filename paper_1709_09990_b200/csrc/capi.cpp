// C ABI of libelimtw.so.1: the reference's 14 etw_* entry points
// (proj/include/elimtw.h:66-99, proj/src/capi.cpp:72-200) plus the additive
// etwg_* device seam (include/elimtw_gpu.h). Exceptions never cross the ABI:
// ParseError -> ETW_ERROR_PARSE, std::invalid_argument ->
// ETW_ERROR_INVALID_ARGUMENT, everything else (CUDA failures, missing device)
// -> ETW_ERROR_INTERNAL with the message in the caller's buffer.
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "elimtw.h"
#include "elimtw_gpu.h"
#include "engine.hpp"
#include "graph.hpp"
#include "preprocess.hpp"
#include "solver.hpp"
#include "treedec.hpp"

using namespace etw;

struct etw_graph {
    Graph g;
};

struct etw_result {
    SolveResult result;
    Graph graph;
    SolveOptions opts;
    std::string stats;
};

struct etwg_run {
    Outcome outcome = Outcome::infeasible;
    State witness;
    bool overflowed = false;
    std::vector<LayerStats> rounds;
    std::vector<std::vector<State>> layers;
    std::vector<std::pair<int, int>> tags;
};

namespace {

void write_error(char* err, size_t len, const char* msg) {
    if (err && len) std::snprintf(err, len, "%s", msg);
}

etw_status status_of_current_exception(char* err, size_t len) {
    try {
        throw;
    } catch (const ParseError& e) {
        write_error(err, len, e.what());
        return ETW_ERROR_PARSE;
    } catch (const std::invalid_argument& e) {
        write_error(err, len, e.what());
        return ETW_ERROR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        write_error(err, len, e.what());
        return ETW_ERROR_INTERNAL;
    } catch (...) {
        write_error(err, len, "unknown error");
        return ETW_ERROR_INTERNAL;
    }
}

// capi.cpp:48-66
SolveOptions options_from(const etw_options& o) {
    SolveOptions s;
    s.dp.dedup = o.dedup == ETW_DEDUP_EXACT ? DedupMode::exact_set : DedupMode::bloom;
    s.dp.use_mmw = o.use_mmw != 0;
    s.dp.thread_count = o.thread_count;
    s.dp.max_layer_states = o.max_layer_states;
    s.dp.bloom_bits_per_element = o.bloom_bits_per_element;
    s.dp.bloom_hashes = o.bloom_hashes;
    s.split = o.split == ETW_SPLIT_NONE
                  ? SplitMode::none
                  : (o.split == ETW_SPLIT_CONNECTED ? SplitMode::connected : SplitMode::biconnected);
    s.use_clique = o.use_clique != 0;
    s.use_improvement = o.use_improvement != 0;
    if (o.start_k >= 0) s.starting_k = o.start_k;
    s.emit_order = o.emit_order != 0;
    return s;
}

Graph graph_from_words(int n, const uint64_t* rows) {
    if (n < 0 || n > kMaxVertices) throw std::invalid_argument("vertex count out of range");
    std::vector<HostSet> r(n);
    for (int v = 0; v < n; ++v) {
        r[v].w[0] = rows[2 * v];
        r[v].w[1] = rows[2 * v + 1];
    }
    return Graph::from_rows(n, std::move(r));
}

HostSet set_from_words(const uint64_t* w) {
    HostSet s = HostSet::zero();
    if (w) {
        s.w[0] = w[0];
        s.w[1] = w[1];
    }
    return s;
}

DpConfig dp_from(int dedup, int use_mmw, uint64_t cap, int bpe, int hashes) {
    DpConfig c;
    c.dedup = dedup == ETW_DEDUP_EXACT ? DedupMode::exact_set : DedupMode::bloom;
    c.use_mmw = use_mmw != 0;
    c.max_layer_states = cap;
    c.bloom_bits_per_element = bpe;
    c.bloom_hashes = hashes;
    return c;
}

}  // namespace

extern "C" {

void etw_options_init(etw_options* o) {
    if (!o) return;
    o->dedup = ETW_DEDUP_BLOOM;
    o->split = ETW_SPLIT_BICONNECTED;
    o->use_mmw = 0;
    o->use_clique = 1;
    o->use_improvement = 1;
    o->thread_count = 1;
    o->max_layer_states = 10000000;
    o->bloom_bits_per_element = 24;
    o->bloom_hashes = 17;
    o->start_k = -1;
    o->emit_order = 0;
}

etw_status etw_graph_parse(const char* text, size_t len, etw_format format, etw_graph** out,
                           char* err, size_t err_len) {
    if (!out) return ETW_ERROR_INVALID_ARGUMENT;
    *out = nullptr;
    if (!text) {
        write_error(err, err_len, "text is null");
        return ETW_ERROR_INVALID_ARGUMENT;
    }
    try {
        std::string body(text, len);
        GraphFormat f = format == ETW_FORMAT_DIMACS ? GraphFormat::dimacs_col : GraphFormat::pace_gr;
        if (format == ETW_FORMAT_AUTO) f = detect_format(body);
        *out = new etw_graph{parse_graph(body, f)};
        return ETW_OK;
    } catch (...) {
        return status_of_current_exception(err, err_len);
    }
}

void etw_graph_free(etw_graph* g) { delete g; }

int etw_graph_vertex_count(const etw_graph* g) { return g ? g->g.vertex_count() : 0; }

long long etw_graph_edge_count(const etw_graph* g) { return g ? g->g.edge_count() : 0; }

etw_status etw_solve(const etw_graph* g, const etw_options* opts, etw_result** out, char* err,
                     size_t err_len) {
    if (!out) return ETW_ERROR_INVALID_ARGUMENT;
    *out = nullptr;
    if (!g || !opts) {
        write_error(err, err_len, "graph or options is null");
        return ETW_ERROR_INVALID_ARGUMENT;
    }
    try {
        auto* r = new etw_result;
        try {
            r->graph = g->g;
            r->opts = options_from(*opts);
            r->result = solve(g->g, r->opts);
        } catch (...) {
            delete r;
            throw;
        }
        *out = r;
        return ETW_OK;
    } catch (...) {
        return status_of_current_exception(err, err_len);
    }
}

void etw_result_free(etw_result* r) { delete r; }

etw_result_kind etw_result_kind_of(const etw_result* r) {
    return r && r->result.kind == ResultKind::lower_bound_only ? ETW_RESULT_LOWER_BOUND
                                                               : ETW_RESULT_EXACT;
}

int etw_result_value(const etw_result* r) { return r ? r->result.value : 0; }

size_t etw_result_order_len(const etw_result* r) { return r ? r->result.order.size() : 0; }

const int* etw_result_order(const etw_result* r) {
    return r && !r->result.order.empty() ? r->result.order.data() : nullptr;
}

const char* etw_result_stats_json(etw_result* r) {
    if (!r) return "";
    if (r->stats.empty()) {
        try {
            r->stats = stats_json(r->graph, r->opts, r->result);
        } catch (...) {
            return "";
        }
    }
    return r->stats.c_str();
}

etw_status etw_check_order(const etw_graph* g, const int* order, size_t len, int* width_out,
                           int* valid_out, char* err, size_t err_len) {
    if (!g || (!order && len > 0)) {
        write_error(err, err_len, "graph or order is null");
        return ETW_ERROR_INVALID_ARGUMENT;
    }
    try {
        EliminationOrder pi(order, order + len);
        if (!is_permutation(g->g, pi)) {
            write_error(err, err_len, "order is not a permutation of the vertices");
            return ETW_ERROR_INVALID_ARGUMENT;
        }
        const int width = order_width(g->g, pi);
        if (width_out) *width_out = width;
        if (valid_out) {
            TreeDecomposition td = decomposition_from_order(g->g, pi);
            std::string why;
            *valid_out = td.width == width && validate_decomposition(g->g, td, &why) ? 1 : 0;
        }
        return ETW_OK;
    } catch (...) {
        return status_of_current_exception(err, err_len);
    }
}

const char* etw_version(void) { return "1.0.0"; }

// ---------------------------------------------------------------------------
// additive device seam

int etwg_device_info(int* device, int* sm_count, char* name, size_t name_len) {
    try {
        DeviceInfo info;
        if (!device_available(&info)) return 0;
        if (device) *device = info.device;
        if (sm_count) *sm_count = info.sm_count;
        if (name && name_len) std::snprintf(name, name_len, "%s", info.name);
        return 1;
    } catch (...) {
        return 0;
    }
}

etw_status etwg_decide(int n, const uint64_t* rows, int k, const uint64_t* forbidden, int dedup,
                       int use_mmw, uint64_t cap, int bpe, int hashes, int rounds, int keep_layers,
                       etwg_run** out, char* err, size_t err_len) {
    if (!out) return ETW_ERROR_INVALID_ARGUMENT;
    *out = nullptr;
    try {
        Graph g = graph_from_words(n, rows);
        auto* run = new etwg_run;
        LayerObserver obs = [run](int kk, int round, const std::vector<State>& layer) {
            run->layers.push_back(layer);
            run->tags.emplace_back(kk, round);
        };
        try {
            DecideResult r = device_decide(g, k, set_from_words(forbidden),
                                           dp_from(dedup, use_mmw, cap, bpe, hashes), rounds,
                                           keep_layers ? &obs : nullptr);
            run->outcome = r.outcome;
            run->witness = r.witness;
            run->overflowed = r.overflowed;
            run->rounds = std::move(r.rounds);
        } catch (...) {
            delete run;
            throw;
        }
        *out = run;
        return ETW_OK;
    } catch (...) {
        return status_of_current_exception(err, err_len);
    }
}

etw_status etwg_expand_layer(int n, const uint64_t* rows, int k, const uint64_t* forbidden,
                             const uint64_t* sets, const uint32_t* hist, size_t count, int dedup,
                             int use_mmw, uint64_t cap, int bpe, int hashes, etwg_run** out,
                             char* err, size_t err_len) {
    if (!out) return ETW_ERROR_INVALID_ARGUMENT;
    *out = nullptr;
    try {
        Graph g = graph_from_words(n, rows);
        std::vector<State> in(count);
        for (size_t i = 0; i < count; ++i) {
            in[i].set = set_from_words(sets + 2 * i);
            in[i].history = hist[i];
        }
        LayerStats st;
        st.k = k;
        ExpandResult r = device_expand_layer(g, k, set_from_words(forbidden), in,
                                             dp_from(dedup, use_mmw, cap, bpe, hashes), st);
        auto* run = new etwg_run;
        run->overflowed = r.overflowed;
        run->rounds.push_back(st);
        run->layers.push_back(std::move(r.states));
        run->tags.emplace_back(k, 0);
        *out = run;
        return ETW_OK;
    } catch (...) {
        return status_of_current_exception(err, err_len);
    }
}

etw_status etwg_solve_layers(const etw_graph* g, const etw_options* opts, etwg_run** out,
                             char* err, size_t err_len) {
    if (!out) return ETW_ERROR_INVALID_ARGUMENT;
    *out = nullptr;
    if (!g || !opts) {
        write_error(err, err_len, "graph or options is null");
        return ETW_ERROR_INVALID_ARGUMENT;
    }
    try {
        auto* run = new etwg_run;
        try {
            SolveOptions so = options_from(*opts);
            so.emit_order = false;
            so.observer = [run](int kk, int round, const std::vector<State>& layer) {
                run->layers.push_back(layer);
                run->tags.emplace_back(kk, round);
            };
            SolveResult res = solve(g->g, so);
            run->outcome = res.kind == ResultKind::exact ? Outcome::feasible : Outcome::indeterminate;
            for (const ComponentReport& c : res.components)
                for (const AttemptReport& a : c.attempts)
                    for (const LayerStats& l : a.layers) run->rounds.push_back(l);
        } catch (...) {
            delete run;
            throw;
        }
        *out = run;
        return ETW_OK;
    } catch (...) {
        return status_of_current_exception(err, err_len);
    }
}

int etwg_run_outcome(const etwg_run* r) { return r ? static_cast<int>(r->outcome) : 1; }
int etwg_run_overflowed(const etwg_run* r) { return r && r->overflowed ? 1 : 0; }
void etwg_run_witness(const etwg_run* r, uint64_t* set2, uint32_t* hist) {
    if (!r) return;
    if (set2) {
        set2[0] = r->witness.set.w[0];
        set2[1] = r->witness.set.w[1];
    }
    if (hist) *hist = r->witness.history;
}
int etwg_run_round_count(const etwg_run* r) { return r ? static_cast<int>(r->rounds.size()) : 0; }
void etwg_run_rounds(const etwg_run* r, uint64_t* stats, uint8_t* ovf) {
    if (!r) return;
    for (size_t i = 0; i < r->rounds.size(); ++i) {
        const LayerStats& s = r->rounds[i];
        uint64_t* o = stats + 6 * i;
        o[0] = static_cast<uint64_t>(s.k);
        o[1] = static_cast<uint64_t>(s.round);
        o[2] = s.expanded;
        o[3] = s.emitted;
        o[4] = s.duplicates;
        o[5] = s.mmw_pruned;
        if (ovf) ovf[i] = s.overflowed ? 1 : 0;
    }
}
int etwg_run_layer_count(const etwg_run* r) { return r ? static_cast<int>(r->layers.size()) : 0; }
uint64_t etwg_run_layer_size(const etwg_run* r, int i) { return r ? r->layers[i].size() : 0; }
void etwg_run_layer_tag(const etwg_run* r, int i, int* k, int* round) {
    if (!r) return;
    if (k) *k = r->tags[i].first;
    if (round) *round = r->tags[i].second;
}
void etwg_run_layer(const etwg_run* r, int i, uint64_t* sets2, uint32_t* hist) {
    if (!r) return;
    const std::vector<State>& L = r->layers[i];
    for (size_t j = 0; j < L.size(); ++j) {
        sets2[2 * j] = L[j].set.w[0];
        sets2[2 * j + 1] = L[j].set.w[1];
        hist[j] = L[j].history;
    }
}
void etwg_run_free(etwg_run* r) { delete r; }

uint64_t etwg_bloom_insert(uint64_t expected, int bpe, int hashes, const uint64_t* keys, int words,
                           size_t count, uint8_t* novel_out, uint32_t* bits_out, size_t bits_words) {
    try {
        std::vector<uint64_t> k(keys, keys + static_cast<size_t>(words) * count);
        std::vector<uint8_t> novel;
        std::vector<uint32_t> bits;
        uint64_t m = device_bloom_insert(expected, bpe, hashes, k, words, novel,
                                         bits_out ? &bits : nullptr);
        if (novel_out) std::memcpy(novel_out, novel.data(), novel.size());
        if (bits_out) std::memcpy(bits_out, bits.data(), std::min(bits_words, bits.size()) * 4);
        return m;
    } catch (...) {
        return 0;
    }
}

int etwg_times(double* out, int len) {
    KernelTimes t = engine_times();
    const double v[] = {t.decide_ms,
                        t.expand_ms,
                        t.insert_ms,
                        t.append_ms,
                        t.clear_ms,
                        t.fused_ms,
                        static_cast<double>(t.expand_launches),
                        static_cast<double>(t.insert_launches),
                        static_cast<double>(t.append_launches),
                        static_cast<double>(t.clear_launches),
                        static_cast<double>(t.fused_launches),
                        static_cast<double>(t.kernel_launches),
                        t.layer_bytes,
                        t.dedup_bytes,
                        static_cast<double>(t.expanded),
                        static_cast<double>(t.h2d_bytes),
                        static_cast<double>(t.d2h_bytes),
                        t.exchange_bytes,
                        static_cast<double>(t.reruns),
                        t.expand_bytes,
                        t.insert_bytes,
                        t.append_bytes,
                        static_cast<double>(t.offered),
                        static_cast<double>(t.unique),
                        static_cast<double>(t.bloom_probed),
                        static_cast<double>(t.bloom_fp),
                        t.records};
    int n = static_cast<int>(sizeof v / sizeof v[0]);
    if (len < n) n = len;
    for (int i = 0; i < n; ++i) out[i] = v[i];
    return n;
}

etw_status etwg_set_virtual_shards(int shards, char* err, size_t err_len) {
    try {
        shard_set_virtual(shards);
        return ETW_OK;
    } catch (...) {
        return status_of_current_exception(err, err_len);
    }
}

etw_status etwg_nccl_unique_id(uint8_t* id128, char* err, size_t err_len) {
    if (!id128) return ETW_ERROR_INVALID_ARGUMENT;
    try {
        shard_unique_id(id128);
        return ETW_OK;
    } catch (...) {
        return status_of_current_exception(err, err_len);
    }
}

etw_status etwg_shard_init(const uint8_t* id128, int rank, int world, int device, char* err,
                           size_t err_len) {
    if (!id128) return ETW_ERROR_INVALID_ARGUMENT;
    try {
        shard_init_nccl(id128, rank, world, device);
        return ETW_OK;
    } catch (...) {
        return status_of_current_exception(err, err_len);
    }
}

void etwg_shard_release(void) {
    try {
        shard_release();
    } catch (...) {
    }
}

void etwg_set_shard_mode(int emitter) {
    try {
        shard_set_mode(emitter);
    } catch (...) {
    }
}

void etwg_set_shard_handoff(uint64_t states) {
    try {
        shard_set_handoff(states);
    } catch (...) {
    }
}

int etwg_shard_exchange_p2p(void) {
    try {
        return shard_p2p();
    } catch (...) {
        return 0;
    }
}

void etwg_shard_info(int* world, int* rank, int* is_virtual) {
    try {
        shard_info(world, rank, is_virtual);
    } catch (...) {
        if (world) *world = 1;
        if (rank) *rank = 0;
        if (is_virtual) *is_virtual = 0;
    }
}

void etwg_set_profiling(int on) { engine_set_profiling(on != 0); }
void etwg_timer_begin(void) {
    try {
        engine_timer_begin();
    } catch (...) {
    }
}
double etwg_timer_end(void) {
    try {
        return engine_timer_end();
    } catch (...) {
        return -1.0;
    }
}
void etwg_reset_times(void) { engine_reset_times(); }

void etwg_graph_rows(const etw_graph* g, uint64_t* rows) {
    if (!g) return;
    for (int v = 0; v < g->g.vertex_count(); ++v) {
        rows[2 * v] = g->g.neighbors(v).w[0];
        rows[2 * v + 1] = g->g.neighbors(v).w[1];
    }
}

// Host preprocessing entry points: no exception crosses the ABI. The void
// ones return ETW_OK / ETW_ERROR_INVALID_ARGUMENT / ETW_ERROR_INTERNAL, the
// counting ones -1 on any failure (bad n, allocation failure).
static etw_status prep_status(const std::exception_ptr& e) {
    try {
        std::rethrow_exception(e);
    } catch (const std::invalid_argument&) {
        return ETW_ERROR_INVALID_ARGUMENT;
    } catch (...) {
        return ETW_ERROR_INTERNAL;
    }
}

etw_status etwg_max_clique(int n, const uint64_t* rows, uint64_t* out2) {
    if (!rows || !out2) return ETW_ERROR_INVALID_ARGUMENT;
    try {
        HostSet c = max_clique(graph_from_words(n, rows));
        out2[0] = c.w[0];
        out2[1] = c.w[1];
        return ETW_OK;
    } catch (...) {
        return prep_status(std::current_exception());
    }
}

etw_status etwg_disjoint_paths(int n, const uint64_t* rows, uint8_t* out) {
    if (!rows || !out) return ETW_ERROR_INVALID_ARGUMENT;
    try {
        PathCounts pc = disjoint_path_counts(graph_from_words(n, rows));
        std::memcpy(out, pc.counts.data(), pc.counts.size());
        return ETW_OK;
    } catch (...) {
        return prep_status(std::current_exception());
    }
}

etw_status etwg_improve_graph(int n, const uint64_t* rows, int k, uint64_t* out_rows) {
    if (!rows || !out_rows) return ETW_ERROR_INVALID_ARGUMENT;
    try {
        Graph g = graph_from_words(n, rows);
        Graph h = improve_graph(g, k, disjoint_path_counts(g));
        for (int v = 0; v < n; ++v) {
            out_rows[2 * v] = h.neighbors(v).w[0];
            out_rows[2 * v + 1] = h.neighbors(v).w[1];
        }
        return ETW_OK;
    } catch (...) {
        return prep_status(std::current_exception());
    }
}

int etwg_mmw_lower_bound(int n, const uint64_t* rows, const uint64_t* s, int cap) {
    if (!rows || !s) return -1;
    try {
        return mmw_lower_bound(graph_from_words(n, rows), set_from_words(s), cap);
    } catch (...) {
        return -1;
    }
}

int etwg_split(int n, const uint64_t* rows, int mode, int* verts, int* sizes, int* cuts) {
    if (!rows || !verts || !sizes || !cuts) return -1;
    try {
        std::vector<SubInstance> subs =
            split_instance(graph_from_words(n, rows), static_cast<SplitMode>(mode));
        int off = 0;
        for (size_t i = 0; i < subs.size(); ++i) {
            sizes[i] = static_cast<int>(subs[i].to_original.size());
            cuts[i] = subs[i].parent_cut;
            for (int v : subs[i].to_original) verts[off++] = v;
        }
        return static_cast<int>(subs.size());
    } catch (...) {
        return -1;
    }
}

}  // extern "C"
