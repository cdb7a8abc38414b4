// The device seam. `device_decide` replaces the reference's CPU `decide`
// (proj/src/dp.hpp:78-79, dp.cpp:167-194) wholesale and `device_expand_layer`
// its per-round unit `expand_layer` (dp.hpp:68-70, dp.cpp:73-165): the layer
// lives in HBM across rounds, every round runs as sm_100a kernels
// (wavefront.cu), and only per-round counters plus the witness come back to
// the host. There is no CPU fallback: without a CUDA device these throw
// DeviceError, which the C ABI maps to ETW_ERROR_INTERNAL.
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "graph.hpp"

#include <cstdio>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges are free unless a profiler attaches

namespace etw {

struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum class DedupMode { bloom = 0, exact_set = 1 };

// dp.hpp:25-33 (thread_count is validated but the device ignores it)
struct DpConfig {
    uint64_t max_layer_states = 10'000'000;
    DedupMode dedup = DedupMode::bloom;
    int bloom_bits_per_element = 24;
    int bloom_hashes = 17;
    bool use_mmw = false;
    int thread_count = 1;
};

// dp.hpp:14-21: eliminated prefix + last four eliminations, newest low byte
struct State {
    HostSet set = HostSet::zero();
    uint32_t history = 0xFFFFFFFFu;
};

inline uint32_t push_history(uint32_t h, int v) { return (h << 8) | static_cast<uint32_t>(v & 0xFF); }

// dp.hpp:35-43
struct LayerStats {
    int k = 0;
    int round = 0;
    uint64_t expanded = 0;
    uint64_t emitted = 0;
    uint64_t duplicates = 0;
    uint64_t mmw_pruned = 0;
    bool overflowed = false;
};

enum class Outcome { feasible, infeasible, indeterminate };

// dp.hpp:52-57
struct DecideResult {
    Outcome outcome = Outcome::infeasible;
    State witness;
    bool overflowed = false;
    std::vector<LayerStats> rounds;
};

// Test-only seam (dp.hpp:31-32): called with every finished layer. Setting
// it forces a device->host copy of every layer.
using LayerObserver = std::function<void(int k, int round, const std::vector<State>&)>;

DecideResult device_decide(const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg,
                           int rounds = -1, const LayerObserver* observer = nullptr);

// Replicated prefix of an owner-sharded decide: the single-device engine runs
// the decide until a layer exceeds `handoff_above` states (small layers are
// cheaper to expand redundantly on every GPU than to route). When it stops
// there, `handed` is set and the layer (device pointers, valid until the
// engine's next call) is left for the shards; the result holds the rounds run.
struct EngineLayer {
    const void* keys = nullptr;      // u64[W] per state
    const unsigned* hist = nullptr;  // u32 per state
    uint64_t count = 0;
    int W = 1;
    int rounds_done = 0;
    bool handed = false;
};
DecideResult device_decide_prefix(const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg,
                                  int rounds, const LayerObserver* observer, uint64_t handoff_above,
                                  EngineLayer& handoff);
int engine_device();  // the single-device engine's CUDA device (-1 without one)
void engine_release_buffers();  // frees the single-device engine's round buffers
void engine_bind_device(int dev);  // (re)binds the single-device engine to CUDA device dev

struct ExpandResult {
    std::vector<State> states;
    bool overflowed = false;
};
ExpandResult device_expand_layer(const Graph& g, int k, const HostSet& forbidden,
                                 const std::vector<State>& input, const DpConfig& cfg,
                                 LayerStats& stats);

// One concurrent batch of Bloom inserts on the device (one key per thread,
// no warp pre-dedup: exercises the striped lock). Filter sized for
// `expected` elements as ConcurrentBloom (bloom.cpp:72-79); returns m.
uint64_t device_bloom_insert(uint64_t expected, int bits_per_element, int hashes,
                             const std::vector<uint64_t>& keys, int words,
                             std::vector<uint8_t>& novel, std::vector<uint32_t>* bits);

// Runtime knobs and counters for the device engine (additive API).
struct DeviceInfo {
    int device = -1;
    int sm_count = 0;
    char name[128] = {0};
};
bool device_available(DeviceInfo* info);

struct KernelTimes {
    // accumulated device milliseconds per kernel class (only when profiling)
    double expand_ms = 0, insert_ms = 0, append_ms = 0, clear_ms = 0, fused_ms = 0;
    uint64_t expand_launches = 0, insert_launches = 0, append_launches = 0, clear_launches = 0,
             fused_launches = 0;
    // algorithmic bytes accumulated by the rounds that ran
    double layer_bytes = 0, dedup_bytes = 0;
    uint64_t kernel_launches = 0;  // all wavefront kernels launched
    double decide_ms = 0;          // device time of decide calls (events)
    uint64_t expanded = 0;
    uint64_t h2d_bytes = 0, d2h_bytes = 0;  // host<->device traffic of the engine
    double exchange_bytes = 0;  // sharded: child records sent to other shards
    uint64_t reruns = 0;        // sharded: rounds re-run after a buffer grew
    // per-kernel-class algorithmic bytes: expand / scatter,
    // insert / partition dedup, append
    double expand_bytes = 0, insert_bytes = 0, append_bytes = 0;
    uint64_t offered = 0, unique = 0;  // children offered to dedup / distinct children
    double records = 0;                // exact rounds: child records written (after the swap pre-dedup)
    // partitioned Bloom rounds: distinct keys probed / rejected by the filter
    uint64_t bloom_probed = 0, bloom_fp = 0;
};
// Brackets a region on the engine's stream with CUDA events; end returns the
// device milliseconds between the two events (synchronizing).
void engine_timer_begin();
double engine_timer_end();
void engine_set_profiling(bool on);
KernelTimes engine_times();
void engine_reset_times();

// Owner-sharded decide over G shards (shard.cu). Active after
// shard_set_virtual(G > 1) — G virtual shards on this process's device, the
// single-GPU test double of the exchange — or shard_init_nccl (one shard per
// process/GPU, NCCL over NVLink). device_decide routes to it while active.
bool shard_active();
DecideResult shard_decide(const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg, int rounds,
                          const LayerObserver* observer);
void shard_set_virtual(int G);
void shard_unique_id(unsigned char* out128);
void shard_init_nccl(const unsigned char* id128, int rank, int world, int device);
void shard_release();
void shard_info(int* world, int* rank, int* virt);
int shard_p2p();  // 1 when the NCCL path pulls records over NVLink (CUDA IPC)
// layers up to `states` run replicated on the single-device engine (0: shard from the root)
void shard_set_handoff(uint64_t states);
// 1: next-layer states stay on their emitting shard (default); 0: on their hash owner
void shard_set_mode(int emitter);
void shard_timer_begin();
double shard_timer_end();
void shard_accumulate(KernelTimes& t);
void shard_reset_times();

// NVTX range for the whole scope (solve, attempt, decide, round chunk,
// sharded round, buffer growth): visible in ncu --nvtx / Nsight timelines.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    template <typename... A>
    NvtxRange(const char* fmt, A... a) {
        char buf[96];
        std::snprintf(buf, sizeof buf, fmt, a...);
        nvtxRangePushA(buf);
    }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace etw
