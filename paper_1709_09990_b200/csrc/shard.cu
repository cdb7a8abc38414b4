// Sharded wavefront across G devices: the multi-GPU
// replacement for the reference's decide / expand_layer (proj/src/dp.cpp:
// 73-194), one shard per B200 (or G virtual shards on one device, the
// single-GPU double of the exchange).
//
// Every child S+v has an owner shard owner(S+v) = mulhi(mix(S+v), G) that
// deduplicates it. A round on every shard:
//
//   k_route     K1 (candidates, graph.hpp:61-78 / dp.cpp:39-69) over the
//               local parents; each child record goes to the outbox bucket
//               (owner, partition) — partition = top bits of an independent
//               hash, sized so one bucket's distinct keys fit shared memory.
//   exchange    owners read their buckets straight from the sources'
//               outboxes: over NVLink through CUDA IPC mappings (a
//               stream-ordered allgather is the barrier), or in place between
//               virtual shards; fallback: NCCL grouped send/recv.
//   emitter-stored layers (default):
//     k_owner_emit   per partition: min emission rank per key (dp.cpp:140-151
//                    semantics, emitters ranked cyclically from the owner so
//                    every shard keeps its share), optional Bloom filter on
//                    the owner's slice (bloom.cpp:86-97); one mark per winner
//                    back to its emitter
//     k_apply_marks  each shard ORs its marks into its parents' winner masks
//     k_emit_append  ordered append of the marked children (rank order)
//   owner-stored layers (ETWG_SHARD_MODE=owner, and the NCCL fallback):
//     k_owner        per partition: min rank + history per key, rank sort,
//                    survivors to staging; k_owner_compact builds the layer
//   allgather   per-shard counters (ncclAllGather / copies) — the per-level
//               count reduction that decides termination (dp.cpp:176-188).
//   k_finish    global stats, the capacity wall applied shard-major
//               (emitted = min(unique, cap), dp.cpp:84-86, 152-155).
//
// Layers of up to 2^19 states are expanded redundantly on every shard by the
// single-device engine first (no communication); the first larger layer is
// split between the shards. Exact-mode per-level sets and counters
// (expanded, emitted, duplicates, mmw_pruned) equal the single-device
// engine's; layer order is deterministic for a given G. The host plans each
// round's bucket geometry from the previous round's growth and re-runs a
// round whose buffers overflowed on any shard.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cub/block/block_scan.cuh>
#include <nccl.h>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <type_traits>
#include <vector>

#include "engine.hpp"
#include "wave_device.cuh"

namespace etw {

namespace {

constexpr int kMaxShards = 8;
#ifndef ETWG_OWNER_TARGET
#define ETWG_OWNER_TARGET 640
#endif
#ifndef ETWG_ROUTE_COMPACT
#define ETWG_ROUTE_COMPACT true  // rank-indexed boundary table for hash-ordered layers
#endif
constexpr int kOwnerThreads = 512;
constexpr int kRouteThreads = 256;
#ifndef ETWG_ROUTE_LANE_EMIT
#define ETWG_ROUTE_LANE_EMIT 1  // k_route: each lane routes its own children (0: flattened over the warp)
#endif
// parents per look-back tile of k_emit_append (its ITEMS x kRouteThreads);
// the host sizes the tile-status array from the same figure
constexpr unsigned long long emit_span(int W) { return static_cast<unsigned long long>(kRouteThreads) * (W == 1 ? 8 : 4); }

template <int W>
constexpr int owner_slots() { return 2048; }
template <int W>
constexpr int owner_target() { return ETWG_OWNER_TARGET; }  // distinct keys aimed for per partition
// Child record: {key words, parent index << 32 | history}. The emission
// rank (source shard, parent index, vertex) is rebuilt by the owner: the
// source is the block it reads, the vertex the history's low byte.
template <int W>
constexpr int srec_words() { return W + 1; }
template <int W>
constexpr int owner_smem_bytes() {
    return owner_slots<W>() * (8 * W + 16 + 8);  // keys, {min rank, history}, sort keys
}

__device__ __forceinline__ u64 owner_rank(int src, u64 packed) {
    return (static_cast<u64>(src) << 40) | ((packed >> 32) << 7) | (packed & 0x7F);
}

enum ShardAbort : unsigned { kAbortLayer = 1, kAbortRecs = 2, kAbortParts = 4, kAbortMarks = 8 };

struct ShardStat {
    u64 expanded, offered, pruned, routed, unique;
    u64 need_layer, need_recs, need_parts, need_marks;
    unsigned abort, pad;
};

struct ShardRound {
    u64 expanded, offered, unique, emitted, pruned, routed;
    unsigned overflowed, valid;
};

struct ShardCtl {
    u64 count[2];  // local layer sizes, ping-pong by round parity
    unsigned round, stop, epoch, pad;
    u64 ticket;   // owner-pass partition ticket
    u64 ticket2;  // compaction tile ticket
    ShardStat mine;
    ShardStat all[kMaxShards];
    ShardRound rs[kMaxRounds];
};

// Round geometry, identical on every shard (host-planned).
struct Plan {
    u64 np;       // partitions per owner (power of two)
    u64 cap;      // records per (owner, partition) bucket of one source
    u64 bloom_m;  // bits of the owner's Bloom slice (0: exact mode)
    u64 layer_est;  // host sizing hint: next-layer states per owner
    int lg, G, me, rounds;
    int shared_r;   // k_route keeps K1's boundary tables in (dynamic) shared memory
    int emit;       // emitter-stored layers: records carry (index << 7 | vertex), no history
    int direct;     // emitter-stored: owners OR each winner straight into the emitter's mask
};

struct ShardBufs {
    u64* keys[2];
    unsigned* hist[2];
    u64 layer_cap;
    u64* out;            // outbox: [owner][partition][cap] records
    unsigned* out_cnt;   // [owner][partition]
    u64* in;             // inbox: [source][partition][cap] records
    unsigned* in_cnt;    // [source][partition]
    u64 box_cap;         // records per box
    u64 cnt_cap;         // counters per box
    // where the owner reads source s's records for it: the inbox block the
    // exchange filled (NCCL), or source s's own outbox block (virtual shards
    // of one device, and a shard's records for itself — no copy)
    const u64* src_recs[kMaxShards];
    const unsigned* src_cnt[kMaxShards];
    u64* tiles;          // look-back status per compaction tile (256 partitions)
    u64 tile_cap;
    u64* stage;          // owner output staging: [partition][owner_slots] keys
    unsigned* stage_hist;
    unsigned* pcount;    // survivors per partition
    u64 stage_cap;       // partitions the staging holds
    unsigned* bloom;     // the owner's Bloom slice (32-bit words)
    u64 bloom_cap;       // words
    // emitter-stored layers (ETWG_SHARD_MODE=emitter): winner marks the
    // owner returns to each emitting shard, [emitter][mark_cap] of
    // (parent index << 7 | vertex), and the emitter's parent winner masks
    u64* marks;
    unsigned* mark_cnt;  // [emitter]
    u64 mark_cap;        // marks per emitter
    const u64* src_marks[kMaxShards];       // owner o's marks for this shard
    const unsigned* src_mark_cnt[kMaxShards];
    u64* cmask;          // u64[W] per local parent
    // direct marks: every emitter's winner masks (virtual shards: the other
    // shard's buffer; NVLink: the peer's mask mapped over CUDA IPC)
    u64* dst_cmask[kMaxShards];
};

template <int W>
__device__ __forceinline__ unsigned owner_of(const Set<W>& key, int G) {
    u64 h = fmix64(key.w[0] ^ 0xD6E8FEB86659FD93ULL);
    if constexpr (W == 2) h = fmix64(h ^ key.w[1]);
    return static_cast<unsigned>(__umul64hi(h, static_cast<u64>(G)));
}

// partition of a key inside its owner: top bits of the slot hash (the
// shared-memory table of k_owner indexes with the low bits)
template <int W>
__device__ __forceinline__ u64 part_hash_bits(const Set<W>& key, int lg) {
    return lg ? slot_hash<W>(key) >> (64 - lg) : 0;
}

// ----------------------------------------------------------------------
// k_route: candidates of the local parents, children to owner buckets

template <int W>
constexpr int route_tile_slots() { return W == 1 ? 4096 : 2048; }
template <int W>
constexpr int route_smem_bytes() { return static_cast<int>(sizeof(TileSet<W, route_tile_slots<W>()>)); }

// TILE: identical children of one tile of 256 consecutive parents are
// resolved in shared memory first (tile_dedup keeps the minimum emission
// rank, so the owner's min-rank choice is unchanged) — fewer records cross
// NVLink at the cost of two shared-memory passes per child.
template <int W, bool MMW, bool TILE>
__global__ void __launch_bounds__(kRouteThreads) k_route(const Params* __restrict__ P, ShardCtl* C,
                                                         ShardBufs B, Plan pl) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto& ts = *reinterpret_cast<TileSet<W, route_tile_slots<W>()>*>(smem_raw);
    __shared__ Set<W> adj[64 * W];
    __shared__ unsigned win[kRouteThreads][2 * W];
    __shared__ unsigned mmw_keep[MMW ? kRouteThreads : 1][2 * W];
    if (C->stop) return;
    const unsigned r = C->round;
    const u64 E = C->count[r & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) C->mine.expanded = E;
    load_adjacency<W>(P, adj);
    const int lane = threadIdx.x & 31;
    const Set<W> forbidden = param_set<W>(P->forbidden);
    const u64* in = B.keys[r & 1];
    const unsigned* hin = B.hist[r & 1];
    const u64 ntiles = (E + kRouteThreads - 1) / kRouteThreads;
    u64 offered = 0, pruned = 0, routed = 0;
    bool full = false;
    __syncthreads();
    for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const u64 idx = tile * kRouteThreads + threadIdx.x;
        const bool valid = idx < E;
        const Set<W> S = valid ? load_set<W>(in, idx) : Set<W>::zero();
        const unsigned H = valid ? hin[idx] : 0u;
        Set<W> M = warp_candidates<W, MMW, ETWG_ROUTE_COMPACT>(
            adj, P->n, P->k, S, valid, forbidden, pruned, mmw_keep,
            (!TILE && !MMW && W == 1 && pl.shared_r) ? reinterpret_cast<Set<W>*>(smem_raw) : nullptr);
        offered += M.count();
        if constexpr (ETWG_SWAP_DEDUP && W == 1 && !MMW && !TILE) {
            // sibling swap pre-dedup (as in k_exact_scatter): of two parents
            // of this warp whose sets differ by one swap, the higher-rank one
            // does not route the child they share — fewer records cross NVLink
            const u64 Sm = S.w[0], M0 = M.w[0];
            u64 drop = 0;
#pragma unroll 4
            for (int d = 1; d < 32; ++d) {
                const u64 So = __shfl_up_sync(kFull, Sm, d);
                const u64 Mo = __shfl_up_sync(kFull, M0, d);
                const u64 x = So ^ Sm;
                if (lane >= d && __popcll(x) == 2 && (Mo & x & Sm) != 0) drop |= x & So;
            }
            M.w[0] = M0 & ~drop;
        }
        if (pl.emit && valid) store_set<W>(B.cmask, idx, Set<W>::zero());
        if constexpr (TILE) {
            tile_set_clear<W, route_tile_slots<W>()>(ts);
            __syncthreads();
            tile_dedup<W, route_tile_slots<W>()>(ts, win, S, M);
        }
        routed += M.count();
#if ETWG_ROUTE_LANE_EMIT
        // each lane routes its own parent's children (no flattening
        // shuffles; the trip count is the warp's largest child count)
        {
            Set<W> rest = M;
            while (rest.any()) {
                const int v = pop_any(rest);
                Set<W> key = S;
                key.add(v);
                const u64 bucket = static_cast<u64>(owner_of<W>(key, pl.G)) * pl.np + part_hash_bits<W>(key, pl.lg);
                const unsigned slot = atomicAdd(B.out_cnt + bucket, 1u);
                if (slot < pl.cap) {
                    u64* rec = B.out + (bucket * pl.cap + slot) * srec_words<W>();
                    const u64 packed = pl.emit ? ((idx << 7) | static_cast<u64>(v))
                                               : ((idx << 32) | ((H << 8) | static_cast<unsigned>(v)));  // push_history
                    if constexpr (W == 1) {
                        *reinterpret_cast<ulonglong2*>(rec) = make_ulonglong2(key.w[0], packed);
                    } else {
                        rec[0] = key.w[0];
                        rec[1] = key.w[1];
                        rec[2] = packed;
                    }
                } else {
                    full = true;
                }
            }
        }
        if (false)
#endif
        {
        WarpFlat f;
        f.scan(M.count());
        const u64 warp_base = tile * kRouteThreads + (threadIdx.x & ~31);
        for (int t = 0; t < f.total; t += 32) {
            const int j = t + lane;
            const int src = f.source(j);
            const int excl = __shfl_sync(kFull, f.incl, src) - __shfl_sync(kFull, f.cnt, src);
            const Set<W> Ms = shfl_set<W>(M, src);
            const Set<W> Ss = shfl_set<W>(S, src);
            const unsigned Hs = __shfl_sync(kFull, H, src);
            if (j < f.total) {
                const int v = nth_member<W>(Ms, j - excl);
                Set<W> key = Ss;
                key.add(v);
                const u64 bucket = static_cast<u64>(owner_of<W>(key, pl.G)) * pl.np + part_hash_bits<W>(key, pl.lg);
                const unsigned slot = atomicAdd(B.out_cnt + bucket, 1u);
                if (slot < pl.cap) {
                    u64* rec = B.out + (bucket * pl.cap + slot) * srec_words<W>();
                    const u64 packed = pl.emit ? (((warp_base + src) << 7) | static_cast<u64>(v))
                                               : (((warp_base + src) << 32) | ((Hs << 8) | static_cast<unsigned>(v)));  // push_history
                    if constexpr (W == 1) {
                        *reinterpret_cast<ulonglong2*>(rec) = make_ulonglong2(key.w[0], packed);
                    } else {
                        rec[0] = key.w[0];
                        rec[1] = key.w[1];
                        rec[2] = packed;
                    }
                } else {
                    full = true;
                }
            }
        }
        }
        if constexpr (TILE) __syncthreads();  // the next tile clears the tile set
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        offered += __shfl_xor_sync(kFull, offered, o);
        pruned += __shfl_xor_sync(kFull, pruned, o);
        routed += __shfl_xor_sync(kFull, routed, o);
    }
    full = __any_sync(kFull, full);
    if (lane == 0) {
        if (offered) atomicAdd(&C->mine.offered, offered);
        if (routed) atomicAdd(&C->mine.routed, routed);
        if (pruned) atomicAdd(&C->mine.pruned, pruned);
        if (full) {
            atomicOr(&C->mine.abort, static_cast<unsigned>(kAbortRecs));
            atomicMax(&C->mine.need_recs, 2 * pl.cap);
        }
    }
}

// ----------------------------------------------------------------------
// k_owner: per partition exact dedup (+ Bloom), rank sort, ordered append

template <int W>
__device__ __forceinline__ void load_srec(const u64* rec, Set<W>& key, u64& packed) {
    if constexpr (W == 1) {
        const ulonglong2 r = __ldcs(reinterpret_cast<const ulonglong2*>(rec));
        key.w[0] = r.x;
        packed = r.y;
    } else {
        key.w[0] = __ldcs(rec);
        key.w[1] = __ldcs(rec + 1);
        packed = __ldcs(rec + 2);
    }
}

// {rank, history} of a table slot lowered to (rank, hist) if rank is smaller
// (128-bit CAS in shared memory, so the history always belongs to the rank)
__device__ __forceinline__ void smem_min_pair(ulonglong2* slot, u64 rank, u64 hist) {
    u64 er = slot->x, eh = slot->y;
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(slot));
    while (rank < er) {
        u64 orr, oh;
        asm volatile(
            "{\n\t.reg .b128 c, s, d;\n\t"
            "mov.b128 c, {%2, %3};\n\t"
            "mov.b128 s, {%4, %5};\n\t"
            "atom.shared.cas.b128 d, [%6], c, s;\n\t"
            "mov.b128 {%0, %1}, d;\n\t}"
            : "=l"(orr), "=l"(oh)
            : "l"(er), "l"(eh), "l"(rank), "l"(hist), "r"(sa)
            : "memory");
        if (orr == er && oh == eh) return;
        er = orr;
        eh = oh;
    }
}

template <int W, bool BLOOM>
__global__ void __launch_bounds__(kOwnerThreads) k_owner(const Params* __restrict__ P, ShardCtl* C,
                                                         ShardBufs B, Plan pl) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int SLOTS = owner_slots<W>();
    ulonglong2* vals = reinterpret_cast<ulonglong2*>(smem_raw);  // {min rank, history}
    u64* keys = reinterpret_cast<u64*>(vals + SLOTS);
    u64* sortk = keys + SLOTS * W;
    __shared__ unsigned s_full, s_cnt;
    __shared__ u64 s_part;
    if (C->stop) return;
    for (;;) {
        if (threadIdx.x == 0) s_part = atomicAdd(&C->ticket, 1ull);
        __syncthreads();
        const u64 part = s_part;
        if (part >= pl.np) break;
        for (int i = threadIdx.x; i < SLOTS * W; i += blockDim.x) keys[i] = 0;
        for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) vals[i] = make_ulonglong2(~u64{0}, 0);
        if (threadIdx.x == 0) {
            s_full = 0;
            s_cnt = 0;
        }
        __syncthreads();
        // every source's records of this partition -> min emission rank per
        // key, with that emission's history (dp.cpp:140-151)
        for (int s = 0; s < pl.G; ++s) {
            const unsigned cnt = min(B.src_cnt[s][part], static_cast<unsigned>(pl.cap));
            const u64* recs = B.src_recs[s] + part * pl.cap * srec_words<W>();
            for (unsigned i = threadIdx.x; i < cnt; i += blockDim.x) {
                Set<W> key;
                u64 packed;
                load_srec<W>(recs + static_cast<u64>(i) * srec_words<W>(), key, packed);
                unsigned h = static_cast<unsigned>(slot_hash<W>(key)) & (SLOTS - 1);
                bool placed = false;
                for (int probe = 0; probe < SLOTS && !placed; ++probe) {
                    placed = smem_claim<W>(keys, h, key);
                    if (!placed) h = (h + 1) & (SLOTS - 1);
                }
                if (placed)
                    smem_min_pair(vals + h, owner_rank(s, packed), packed & 0xFFFFFFFFull);
                else
                    s_full = 1;
            }
        }
        __syncthreads();
        const bool full = s_full != 0;
        if (!full) {
            // compact the distinct keys (Bloom mode: only those the filter calls novel)
            for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
                const u64 rank = vals[i].x;
                if (rank == ~u64{0}) continue;
                bool keep = true;
                if constexpr (BLOOM) {
                    Set<W> key;
#pragma unroll
                    for (int w = 0; w < W; ++w) key.w[w] = keys[W * i + w];
                    const unsigned h1 = murmur_key<W>(key, kSeed1);
                    const unsigned h2 = murmur_key<W>(key, kSeed2);
                    u64 pos, step;
                    probe_start(h1, h2, pl.bloom_m, pos, step);
                    // distinct keys of one round meet the filter exactly once, so the
                    // reference's "any probed bit was clear" is the novelty test
                    keep = bloom_or_probes(B.bloom, pl.bloom_m, pos, step, P->hashes);
                }
                if (keep) sortk[atomicAdd(&s_cnt, 1u)] = (rank << 12) | static_cast<u64>(i);
            }
        }
        __syncthreads();
        const unsigned cnt = full ? 0u : s_cnt;
        // bitonic sort of the partition's survivors by emission rank
        unsigned m = 1;
        while (m < cnt) m <<= 1;
        for (unsigned i = cnt + threadIdx.x; i < m; i += blockDim.x) sortk[i] = ~u64{0};
        __syncthreads();
        for (unsigned size = 2; size <= m; size <<= 1) {
            for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
                for (unsigned i = threadIdx.x; i < m; i += blockDim.x) {
                    const unsigned j = i ^ stride;
                    if (j > i) {
                        const u64 a = sortk[i], b = sortk[j];
                        const bool up = (i & size) == 0;
                        if ((a > b) == up) {
                            sortk[i] = b;
                            sortk[j] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // sorted survivors to the partition's staging slot; k_owner_compact
        // places them (no look-back chain between partitions here)
        u64* stage = B.stage + part * SLOTS * W;
        unsigned* shist = B.stage_hist + part * SLOTS;
        for (unsigned i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int slot = static_cast<int>(sortk[i] & 0xFFF);
#pragma unroll
            for (int w = 0; w < W; ++w) stage[W * i + w] = keys[W * slot + w];
            shist[i] = static_cast<unsigned>(vals[slot].y);
        }
        if (threadIdx.x == 0) {
            B.pcount[part] = cnt;
            if (full) {
                atomicOr(&C->mine.abort, static_cast<unsigned>(kAbortParts));
                atomicMax(&C->mine.need_parts, 2 * pl.np);
            }
        }
        __syncthreads();
    }
}

// Partition survivors -> the contiguous next layer: tiles of 256
// partitions, block scan of their counts, one decoupled look-back per tile,
// then each warp copies its partitions' staged states (coalesced).
template <int W>
__global__ void __launch_bounds__(kRouteThreads) k_owner_compact(ShardCtl* C, ShardBufs B, Plan pl) {
    using BlockScan = cub::BlockScan<unsigned, kRouteThreads>;
    constexpr int SLOTS = owner_slots<W>();
    __shared__ typename BlockScan::TempStorage scan_tmp;
    __shared__ unsigned s_excl[kRouteThreads], s_cnt[kRouteThreads];
    __shared__ u64 s_prefix, s_tile;
    if (C->stop) return;
    const unsigned r = C->round;
    const unsigned epoch = C->epoch;
    u64* out = B.keys[(r + 1) & 1];
    unsigned* hout = B.hist[(r + 1) & 1];
    const u64 ntiles = (pl.np + kRouteThreads - 1) / kRouteThreads;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&C->ticket2, 1ull);
        __syncthreads();
        const u64 tile = s_tile;
        if (tile >= ntiles) break;
        const u64 part = tile * kRouteThreads + threadIdx.x;
        const unsigned cnt = part < pl.np ? B.pcount[part] : 0u;
        unsigned excl, total;
        BlockScan(scan_tmp).ExclusiveSum(cnt, excl, total);
        s_excl[threadIdx.x] = excl;
        s_cnt[threadIdx.x] = cnt;
        if (threadIdx.x == 0) s_prefix = look_back(B.tiles, tile, total, epoch);
        __syncthreads();
        const u64 prefix = s_prefix;
        for (int j = warp; j < kRouteThreads; j += kRouteThreads / 32) {
            const u64 p = tile * kRouteThreads + j;
            if (p >= pl.np) break;
            const unsigned c = s_cnt[j];
            const u64 base = prefix + s_excl[j];
            const u64* stage = B.stage + p * SLOTS * W;
            const unsigned* shist = B.stage_hist + p * SLOTS;
            for (unsigned i = lane; i < c; i += 32) {
                const u64 pos = base + i;
                if (pos >= B.layer_cap) break;
                Set<W> key;
#pragma unroll
                for (int w = 0; w < W; ++w) key.w[w] = stage[W * i + w];
                store_set<W>(out, pos, key);
                hout[pos] = shist[i];
            }
        }
        if (threadIdx.x == 0 && tile == ntiles - 1) {
            const u64 unique = prefix + total;
            C->mine.unique = unique;
            if (unique > B.layer_cap) {
                atomicOr(&C->mine.abort, static_cast<unsigned>(kAbortLayer));
                atomicMax(&C->mine.need_layer, unique);
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------------
// Emitter-stored layers. The owner of a key only deduplicates it: of all
// emissions it keeps one winner — the emitting shard closest after the owner
// in cyclic order (so every shard stores about its share), then the smallest
// (parent index, vertex) there — and returns a mark to that emitter, which
// keeps the state in its own next layer. Layers stay in rank order on every
// shard, histories are computed where the parent lives, and the owner
// neither sorts nor stages.

template <int W, bool BLOOM>
__global__ void __launch_bounds__(kOwnerThreads) k_owner_emit(const Params* __restrict__ P, ShardCtl* C,
                                                              ShardBufs B, Plan pl) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int SLOTS = owner_slots<W>();
    u64* ranks = reinterpret_cast<u64*>(smem_raw);
    u64* keys = ranks + SLOTS;
    __shared__ unsigned s_full, s_cnt[kMaxShards], s_pos[kMaxShards];
    __shared__ u64 s_part, s_base[kMaxShards];
    if (C->stop) return;
    for (;;) {
        if (threadIdx.x == 0) s_part = atomicAdd(&C->ticket, 1ull);
        __syncthreads();
        const u64 part = s_part;
        if (part >= pl.np) break;
        for (int i = threadIdx.x; i < SLOTS * W; i += blockDim.x) keys[i] = 0;
        for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) ranks[i] = ~u64{0};
        if (threadIdx.x < kMaxShards) {
            s_cnt[threadIdx.x] = 0;
            s_pos[threadIdx.x] = 0;
        }
        if (threadIdx.x == 0) s_full = 0;
        __syncthreads();
        for (int s = 0; s < pl.G; ++s) {
            const u64 pri = static_cast<u64>((s - pl.me + pl.G) % pl.G) << 40;
            const unsigned cnt = min(B.src_cnt[s][part], static_cast<unsigned>(pl.cap));
            const u64* recs = B.src_recs[s] + part * pl.cap * srec_words<W>();
            for (unsigned i = threadIdx.x; i < cnt; i += blockDim.x) {
                Set<W> key;
                u64 packed;
                load_srec<W>(recs + static_cast<u64>(i) * srec_words<W>(), key, packed);
                unsigned h = static_cast<unsigned>(slot_hash<W>(key)) & (SLOTS - 1);
                bool placed = false;
                for (int probe = 0; probe < SLOTS && !placed; ++probe) {
                    placed = smem_claim<W>(keys, h, key);
                    if (!placed) h = (h + 1) & (SLOTS - 1);
                }
                if (placed) {
                    const u64 mine = pri | packed;  // ranks only decrease: skip the atomic when already beaten
                    if (!ETWG_CLAIM_PEEK || mine < *reinterpret_cast<volatile u64*>(ranks + h))
                        atomicMin(reinterpret_cast<unsigned long long*>(ranks + h), mine);
                }
                else
                    s_full = 1;
            }
        }
        __syncthreads();
        if (s_full) {
            if (threadIdx.x == 0) {
                atomicOr(&C->mine.abort, static_cast<unsigned>(kAbortParts));
                atomicMax(&C->mine.need_parts, 2 * pl.np);
            }
            __syncthreads();
            continue;
        }
        if (pl.direct) {
            // winners (Bloom: those the owner's filter calls novel) set their
            // bit in the emitting shard's winner mask directly — a local or
            // NVLink peer atomic — instead of a mark list the emitter applies
            for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
                const u64 rank = ranks[i];
                if (rank == ~u64{0}) continue;
                if constexpr (BLOOM) {
                    Set<W> key;
#pragma unroll
                    for (int w = 0; w < W; ++w) key.w[w] = keys[W * i + w];
                    const unsigned h1 = murmur_key<W>(key, kSeed1);
                    const unsigned h2 = murmur_key<W>(key, kSeed2);
                    u64 pos, step;
                    probe_start(h1, h2, pl.bloom_m, pos, step);
                    if (!bloom_or_probes(B.bloom, pl.bloom_m, pos, step, P->hashes)) continue;
                }
                const int emitter = static_cast<int>(((rank >> 40) + pl.me) % pl.G);
                const u64 m = rank & ((u64{1} << 40) - 1);
                const int v = static_cast<int>(m & 127);
                atomicOr(reinterpret_cast<unsigned long long*>(B.dst_cmask[emitter]) + (m >> 7) * W + (v >> 6),
                         u64{1} << (v & 63));
            }
            __syncthreads();
            continue;
        }
        // winners (Bloom: those the owner's filter calls novel) -> marks
        for (int pass = 0; pass < 2; ++pass) {
            for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
                const u64 rank = ranks[i];
                if (rank == ~u64{0}) continue;
                if constexpr (BLOOM) {
                    if (pass == 0) {
                        Set<W> key;
#pragma unroll
                        for (int w = 0; w < W; ++w) key.w[w] = keys[W * i + w];
                        const unsigned h1 = murmur_key<W>(key, kSeed1);
                        const unsigned h2 = murmur_key<W>(key, kSeed2);
                        u64 pos, step;
                        probe_start(h1, h2, pl.bloom_m, pos, step);
                        if (!bloom_or_probes(B.bloom, pl.bloom_m, pos, step, P->hashes)) {
                            ranks[i] = ~u64{0};  // a false positive: dropped as the reference drops it
                            continue;
                        }
                    }
                }
                const int emitter = static_cast<int>(((rank >> 40) + pl.me) % pl.G);
                if (pass == 0) {
                    atomicAdd(&s_cnt[emitter], 1u);
                } else {
                    const u64 slot = s_base[emitter] + atomicAdd(&s_pos[emitter], 1u);
                    if (slot < B.mark_cap) B.marks[emitter * B.mark_cap + slot] = rank & ((u64{1} << 40) - 1);
                }
            }
            __syncthreads();
            if (pass == 0 && threadIdx.x < pl.G) {
                const unsigned c = s_cnt[threadIdx.x];
                s_base[threadIdx.x] = c ? atomicAdd(B.mark_cnt + threadIdx.x, c) : 0;
                if (c && s_base[threadIdx.x] + c > B.mark_cap) {
                    atomicOr(&C->mine.abort, static_cast<unsigned>(kAbortMarks));
                    atomicMax(&C->mine.need_marks, 2 * B.mark_cap);
                }
            }
            __syncthreads();
        }
    }
}

// marks from every owner -> this shard's parents' winner masks
template <int W>
__global__ void k_apply_marks(ShardCtl* C, ShardBufs B, Plan pl) {
    if (C->stop) return;
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (int o = 0; o < pl.G; ++o) {
        const u64 cnt = min(static_cast<u64>(B.src_mark_cnt[o][pl.me]), B.mark_cap);
        const u64* marks = B.src_marks[o] + static_cast<u64>(pl.me) * B.mark_cap;
        for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < cnt; i += stride) {
            const u64 m = __ldcs(marks + i);
            const u64 idx = m >> 7;
            const int v = static_cast<int>(m & 127);
            atomicOr(reinterpret_cast<unsigned long long*>(B.cmask) + idx * W + (v >> 6), u64{1} << (v & 63));
        }
    }
}

// marked children -> this shard's next layer in rank order (tiles of 2048
// parents, one decoupled look-back per tile; histories pushed here)
template <int W>
__global__ void __launch_bounds__(kRouteThreads) k_emit_append(ShardCtl* C, ShardBufs B, Plan pl) {
    using BlockScan = cub::BlockScan<unsigned, kRouteThreads>;
    constexpr int ITEMS = W == 1 ? 8 : 4;
    constexpr u64 kSpan = static_cast<u64>(kRouteThreads) * ITEMS;
    static_assert(kSpan == emit_span(W), "host tile sizing");
    __shared__ typename BlockScan::TempStorage scan_tmp;
    __shared__ u64 s_prefix, s_tile;
    if (C->stop) return;
    const unsigned r = C->round;
    const unsigned epoch = C->epoch;
    const u64 E = C->count[r & 1];
    const u64 ntiles = (E + kSpan - 1) / kSpan;
    const u64* in = B.keys[r & 1];
    const unsigned* hin = B.hist[r & 1];
    u64* out = B.keys[(r + 1) & 1];
    unsigned* hout = B.hist[(r + 1) & 1];
    const int lane = threadIdx.x & 31;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&C->ticket2, 1ull);
        __syncthreads();
        const u64 tile = s_tile;
        if (tile >= ntiles) break;
        Set<W> S[ITEMS], M[ITEMS];
        unsigned H[ITEMS], excl[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const u64 idx = tile * kSpan + static_cast<u64>(i) * kRouteThreads + threadIdx.x;
            const bool valid = idx < E;
            S[i] = valid ? load_set<W>(in, idx) : Set<W>::zero();
            H[i] = valid ? hin[idx] : 0u;
            M[i] = valid ? load_set<W>(B.cmask, idx) : Set<W>::zero();
        }
        unsigned total = 0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            unsigned slice_total;
            BlockScan(scan_tmp).ExclusiveSum(static_cast<unsigned>(M[i].count()), excl[i], slice_total);
            excl[i] += total;
            total += slice_total;
            __syncthreads();
        }
        if (threadIdx.x == 0) s_prefix = look_back(B.tiles, tile, total, epoch);
        __syncthreads();
        const u64 prefix = s_prefix;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const Set<W> Mi = M[i];
            WarpFlat f;
            f.scan(Mi.count());
            const u64 warp_start = prefix + __shfl_sync(kFull, excl[i], 0);
            for (int t = 0; t < f.total; t += 32) {
                const int j = t + lane;
                const int src = f.source(j);
                const int ex = __shfl_sync(kFull, f.incl, src) - __shfl_sync(kFull, f.cnt, src);
                const Set<W> Ms = shfl_set<W>(Mi, src);
                const Set<W> Ss = shfl_set<W>(S[i], src);
                const unsigned Hs = __shfl_sync(kFull, H[i], src);
                const u64 pos = warp_start + j;
                if (j < f.total && pos < B.layer_cap) {
                    const int v = nth_member<W>(Ms, j - ex);
                    Set<W> key = Ss;
                    key.add(v);
                    store_set<W>(out, pos, key);
                    hout[pos] = (Hs << 8) | static_cast<unsigned>(v & 0xFF);  // push_history
                }
            }
        }
        if (threadIdx.x == 0 && tile == ntiles - 1) {
            const u64 unique = prefix + total;
            C->mine.unique = unique;
            if (unique > B.layer_cap) {
                atomicOr(&C->mine.abort, static_cast<unsigned>(kAbortLayer));
                atomicMax(&C->mine.need_layer, unique);
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------------
// Handoff from the replicated prefix: every rank holds the whole layer (in
// rank order); each keeps the states it owns, in the same order.

template <int W>
__global__ void k_owner_histogram(const u64* __restrict__ keys, u64 E, int G, unsigned long long* counts) {
    __shared__ unsigned local[kMaxShards];
    if (threadIdx.x < kMaxShards) local[threadIdx.x] = 0;
    __syncthreads();
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < E; i += stride)
        atomicAdd(&local[owner_of<W>(load_set<W>(keys, i), G)], 1u);
    __syncthreads();
    if (threadIdx.x < G && local[threadIdx.x]) atomicAdd(counts + threadIdx.x, static_cast<unsigned long long>(local[threadIdx.x]));
}

// tiles of 2048 states by ticket: block scan of the owned flags, decoupled
// look-back over tiles, ordered stores
template <int W>
__global__ void __launch_bounds__(kRouteThreads) k_take_owned(const u64* __restrict__ keys,
                                                              const unsigned* __restrict__ hist, u64 E, int G,
                                                              int me, u64* out, unsigned* hout, u64* tiles,
                                                              unsigned epoch, unsigned long long* ticket) {
    using BlockScan = cub::BlockScan<unsigned, kRouteThreads>;
    constexpr int ITEMS = 8;
    constexpr u64 kSpan = static_cast<u64>(kRouteThreads) * ITEMS;
    __shared__ typename BlockScan::TempStorage scan_tmp;
    __shared__ u64 s_prefix, s_tile;
    const u64 ntiles = (E + kSpan - 1) / kSpan;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1ull);
        __syncthreads();
        const u64 tile = s_tile;
        if (tile >= ntiles) break;
        // thread t holds states tile*span + t*ITEMS + i: its run is contiguous
        Set<W> S[ITEMS];
        unsigned H[ITEMS], mine = 0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const u64 idx = tile * kSpan + static_cast<u64>(threadIdx.x) * ITEMS + i;
            const bool valid = idx < E;
            S[i] = valid ? load_set<W>(keys, idx) : Set<W>::zero();
            H[i] = valid ? hist[idx] : 0u;
            if (valid && static_cast<int>(owner_of<W>(S[i], G)) == me) mine |= 1u << i;
        }
        unsigned excl, total;
        BlockScan(scan_tmp).ExclusiveSum(static_cast<unsigned>(__popc(mine)), excl, total);
        if (threadIdx.x == 0) s_prefix = look_back(tiles, tile, total, epoch);
        __syncthreads();
        u64 pos = s_prefix + excl;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (!(mine >> i & 1u)) continue;
            store_set<W>(out, pos, S[i]);
            hout[pos] = H[i];
            ++pos;
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------------
// k_finish: global counters (all[] holds every shard's ShardStat)

__global__ void k_shard_finish(const Params* __restrict__ P, ShardCtl* C, Plan pl) {
    if (threadIdx.x != 0 || C->stop) return;
    unsigned abort = 0;
    u64 E = 0, offered = 0, pruned = 0, unique = 0, routed = 0, before = 0;
    for (int s = 0; s < pl.G; ++s) {
        const ShardStat& st = C->all[s];
        abort |= st.abort;
        E += st.expanded;
        offered += st.offered;
        pruned += st.pruned;
        unique += st.unique;
        routed += st.routed;
        if (s < pl.me) before += st.unique;
    }
    if (abort) return;  // the host grows what the round asked for and re-runs it
    const unsigned r = C->round;
    const u64 cap = round_cap(*P, E);
    const u64 emitted = unique < cap ? unique : cap;
    const u64 mine = C->all[pl.me].unique;
    const u64 room = cap > before ? cap - before : 0;  // shard-major capacity wall
    ShardRound& rs = C->rs[r];
    rs.expanded = E;
    rs.offered = offered;
    rs.unique = unique;
    rs.emitted = emitted;
    rs.pruned = pruned;
    rs.routed = routed;
    rs.overflowed = unique > cap ? 1u : 0u;
    rs.valid = 1;
    C->count[(r + 1) & 1] = mine < room ? mine : room;
    C->round = r + 1;
    C->epoch = (C->epoch & kEpochMask) == kEpochMask ? 1 : C->epoch + 1;
    C->ticket = 0;
    C->ticket2 = 0;
    C->mine = ShardStat{};
    if (emitted == 0 || static_cast<int>(r) + 1 >= pl.rounds) C->stop = 1;
}

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw DeviceError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// ----------------------------------------------------------------------
// NCCL, loaded on first use (the product links no NCCL unless sharded)

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    static Nccl& get() {
        static Nccl n;
        static std::once_flag once;
        std::call_once(once, [] { n.load(); });
        if (!n.GetUniqueId) throw DeviceError("NCCL (libnccl.so.2) could not be loaded");
        return n;
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess)
            throw DeviceError(std::string("NCCL error in ") + what + ": " +
                              (GetErrorString ? GetErrorString(r) : "?"));
    }

private:
    void load() {
        const char* names[] = {std::getenv("ETWG_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        void* h = nullptr;
        for (const char* nm : names)
            if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) return;
        auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(h, name)); };
        sym(CommInitRank, "ncclCommInitRank");
        sym(CommDestroy, "ncclCommDestroy");
        sym(AllGather, "ncclAllGather");
        sym(Broadcast, "ncclBroadcast");
        sym(Send, "ncclSend");
        sym(Recv, "ncclRecv");
        sym(GroupStart, "ncclGroupStart");
        sym(GroupEnd, "ncclGroupEnd");
        sym(GetErrorString, "ncclGetErrorString");
        sym(GetUniqueId, "ncclGetUniqueId");
    }
};

// ----------------------------------------------------------------------
// host side

struct Shard {
    int me = 0;
    Params* d_params = nullptr;
    Params* h_params = nullptr;
    ShardCtl* d_ctl = nullptr;
    ShardCtl* h_ctl = nullptr;
    ShardBufs b{};
    u64 bloom_dirty = 0;  // words of the Bloom slice that may hold bits
    int box_words = 0;    // W the boxes were sized for
    int stage_words = 0;  // W the owner staging was sized for
    u64 mark_alloc = 0;   // emitter mode: marks allocated
    u64 cmask_cap = 0;    // emitter mode: parents the winner masks cover
};

class ShardSet {
public:
    static ShardSet& instance() {
        static ShardSet* s = new ShardSet();
        return *s;
    }
    std::mutex mu;

    // a one-rank NCCL communicator is active too: it runs the whole NCCL
    // host flow (allgather, witness broadcast) on a single GPU
    bool active() const { return G_ > 1 || comm_ != nullptr; }

    void set_virtual(int G) {
        if (G < 1 || G > kMaxShards) throw std::invalid_argument("virtual shard count must be 1..8");
        if (comm_) throw std::invalid_argument("sharding already initialised over NCCL");
        release();
        if (G == 1) return;
        int dev = 0;
        if (const char* e = std::getenv("ETWG_DEVICE")) dev = std::atoi(e);
        engine_release_buffers();  // the shards take over the device's HBM
        init_device(dev);
        G_ = G;
        local_.resize(G);
        for (int s = 0; s < G; ++s) create_shard(local_[s], s);
    }

    void init_nccl(const unsigned char* id, int rank, int world, int device) {
        if (world < 1 || world > kMaxShards) throw std::invalid_argument("world size must be 1..8");
        if (rank < 0 || rank >= world) throw std::invalid_argument("rank out of range");
        release();
        Nccl& nc = Nccl::get();
        engine_release_buffers();
        engine_bind_device(device);  // the replicated prefix runs on the shard's GPU too
        init_device(device);
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        nc.check(nc.CommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
        G_ = world;
        rank_ = rank;
        local_.resize(1);
        create_shard(local_[0], rank);
        // owners pull their buckets from the peers' outboxes over NVLink
        // (CUDA IPC) unless ETWG_EXCHANGE=nccl or a peer mapping fails
        const char* ex = std::getenv("ETWG_EXCHANGE");
        p2p_ = world > 1 && !(ex && std::strcmp(ex, "nccl") == 0);
        handles_dirty_ = true;
    }

    void release() {
        close_peers();
        for (Shard& s : local_) destroy_shard(s);
        local_.clear();
        if (comm_) {
            Nccl::get().CommDestroy(comm_);
            comm_ = nullptr;
        }
        G_ = 1;
        rank_ = 0;
    }

    void set_handoff(u64 states) { handoff_ = states; }
    void set_mode(int emitter) { emit_request_ = emitter != 0; }
    int mode() const { return emit_request_ ? 1 : 0; }
    u64 handoff() const { return handoff_; }

    // exchange mode of the NCCL path: 1 = owners read peers' outboxes over
    // NVLink (CUDA IPC), 0 = NCCL grouped send/recv of the outbox blocks
    int p2p() const { return p2p_ ? 1 : 0; }

    void info(int* world, int* rank, int* virt) const {
        if (world) *world = G_;
        if (rank) *rank = rank_;
        if (virt) *virt = (G_ > 1 && !comm_) ? 1 : 0;
    }

    void timer_begin() { check(cudaEventRecord(tev_[0], stream_), "timer"); }
    double timer_end() {
        check(cudaEventRecord(tev_[1], stream_), "timer");
        check(cudaEventSynchronize(tev_[1]), "timer sync");
        float t = 0;
        check(cudaEventElapsedTime(&t, tev_[0], tev_[1]), "timer elapsed");
        return t;
    }
    // adds this engine's counters to t (engine_times) / clears them
    void accumulate(KernelTimes& t) const {
        t.decide_ms += decide_ms_;
        t.kernel_launches += launches_;
        t.layer_bytes += layer_bytes_;
        t.dedup_bytes += dedup_bytes_;
        t.expanded += expanded_;
        t.h2d_bytes += h2d_;
        t.d2h_bytes += d2h_;
        t.exchange_bytes += exchange_bytes_;
        t.reruns += reruns_;
        t.offered += offered_;
        t.unique += unique_;
    }
    void reset_counters() {
        decide_ms_ = layer_bytes_ = dedup_bytes_ = exchange_bytes_ = 0;
        launches_ = expanded_ = h2d_ = d2h_ = reruns_ = offered_ = unique_ = 0;
    }

    DecideResult decide(const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg, int rounds,
                        const LayerObserver* observer) {
        NvtxRange nvtx("shard decide k=%d G=%d", k, G_);
        check(cudaSetDevice(device_), "cudaSetDevice");
        const int n = g.vertex_count();
        const int W = n > 64 ? 2 : 1;
        if (rounds < 0) rounds = std::max(0, n - k - 1);
        if (rounds > kMaxRounds - 1) throw std::invalid_argument("too many rounds");
        DecideResult res;
        if (rounds == 0) {
            res.outcome = Outcome::feasible;
            return res;
        }
        check(cudaEventRecord(ev_[0], stream_), "event");
        np_floor_ = 1;
        cap_floor_ = 0;
        mark_floor_ = 0;
        emit_ = emit_request_ && (!comm_ || p2p_);
        const bool bloom = cfg.dedup == DedupMode::bloom;
        // host mirror of the global round state
        std::vector<u64> count(G_, 0);
        ShardRound prev{};
        int r = 0;
        if (handoff_ > 0) {
            // replicated prefix: small layers run on the single-device engine on
            // every rank (identical results, no communication)
            if (engine_device() != device_)
                throw DeviceError("the single-device engine and the shard run on different devices "
                                  "(set ETWG_DEVICE to the shard's device before the first call)");
            EngineLayer lay;
            DecideResult pre = device_decide_prefix(g, k, forbidden, cfg, rounds, observer, handoff_, lay);
            if (!lay.handed) {
                check(cudaEventRecord(ev_[1], stream_), "event");
                check(cudaEventSynchronize(ev_[1]), "event sync");
                float ms = 0;
                cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
                decide_ms_ += ms;
                return pre;
            }
            r = lay.rounds_done;
            res.rounds = pre.rounds;
            const LayerStats& last = pre.rounds.back();
            prev.expanded = last.expanded;
            prev.unique = last.emitted;
            prev.routed = last.emitted + last.duplicates;
            prev.emitted = last.emitted;
            if (emit_) {  // any split works: contiguous slices keep rank order
                for (int q = 0; q < G_; ++q) count[q] = lay.count * (q + 1) / G_ - lay.count * q / G_;
            } else {
                count = owner_counts(lay);
            }
            for (Shard& s : local_) setup(s, g, k, forbidden, cfg, rounds, r, &lay, count[s.me]);
        } else {
            for (Shard& s : local_) setup(s, g, k, forbidden, cfg, rounds);
            count[0] = 1;  // the root (empty set, history 0xFFFFFFFF) starts on shard 0
        }
        const int r_first = r;
        bool stopped = false;
        while (r < rounds && !stopped) {
            NvtxRange round_range("shard round %d", r);
            Plan pl = plan(r, count, prev, cfg, W);
            pl_round_parity_ = r & 1;
            if (trace_)
                std::fprintf(stderr, "[shard] k=%d r=%d E=%llu np=%llu cap=%llu recs/shard=%llu prev(exp=%llu routed=%llu uniq=%llu)\n",
                             k, r, static_cast<unsigned long long>(std::accumulate(count.begin(), count.end(), u64{0})),
                             static_cast<unsigned long long>(pl.np), static_cast<unsigned long long>(pl.cap),
                             static_cast<unsigned long long>(G_ * pl.np * pl.cap),
                             static_cast<unsigned long long>(prev.expanded), static_cast<unsigned long long>(prev.routed),
                             static_cast<unsigned long long>(prev.unique));
            for (u64 c : count)
                if (c >> 32) throw DeviceError("sharded layer slice exceeds 2^32 states");
            for (Shard& s : local_) prepare_round(s, pl, W, bloom, count);
            if (comm_ && p2p_ && handles_dirty_) {
                share_outboxes(local_[0]);
                if (!p2p_) {  // a peer mapping failed on some rank: NCCL exchange, owner-stored layers
                    pl = plan(r, count, prev, cfg, W);
                    for (Shard& s : local_) prepare_round(s, pl, W, bloom, count);
                }
            }
            for (Shard& s : local_) launch_route(s, pl, W, cfg.use_mmw);
            exchange(pl, W);
            if (emit_) {
                for (Shard& s : local_) launch_owner_emit(s, pl, W, bloom);
                if (comm_) route_barrier();  // every owner's marks are complete
                for (Shard& s : local_) launch_emit_append(s, pl, W);
            } else {
                for (Shard& s : local_) launch_owner(s, pl, W, bloom);
                for (Shard& s : local_) launch_compact(s, pl, W);
            }
            allgather_stats();
            for (Shard& s : local_) {
                Plan p = pl;
                p.me = s.me;
                k_shard_finish<<<1, 32, 0, stream_>>>(s.d_params, s.d_ctl, p);
                check(cudaGetLastError(), "finish launch");
                ++launches_;
            }
            for (Shard& s : local_) {
                check(cudaMemcpyAsync(s.h_ctl, s.d_ctl, sizeof(ShardCtl), cudaMemcpyDeviceToHost, stream_),
                      "control d2h");
                d2h_ += sizeof(ShardCtl);
            }
            check(cudaStreamSynchronize(stream_), "round sync");
            const ShardCtl& c0 = *local_[0].h_ctl;
            unsigned abort = 0;
            u64 need_layer = 0, need_recs = 0, need_parts = 0;
            for (int s = 0; s < G_; ++s) {
                abort |= c0.all[s].abort;
                need_layer = std::max(need_layer, c0.all[s].need_layer);
                need_recs = std::max(need_recs, c0.all[s].need_recs);
                need_parts = std::max(need_parts, c0.all[s].need_parts);
            }
            if (abort) {
                if (abort & kAbortRecs) cap_floor_ = std::max(cap_floor_, need_recs);
                if (abort & kAbortMarks) {
                    u64 need_marks = 0;
                    for (int q = 0; q < G_; ++q) need_marks = std::max(need_marks, c0.all[q].need_marks);
                    mark_floor_ = std::max(mark_floor_, need_marks);
                }
                if (abort & kAbortParts) np_floor_ = std::max(np_floor_, need_parts);
                for (Shard& s : local_) {
                    if (abort & kAbortLayer) grow_layers(s, need_layer + need_layer / 2, r & 1, count[s.me]);
                    rearm(s);
                }
                ++reruns_;
                continue;
            }
            prev = c0.rs[r];
            np_floor_ = 1;  // floors only widen the round that overflowed
            cap_floor_ = 0;
            mark_floor_ = 0;
            // every shard's kept count, shard-major (as k_shard_finish computed it)
            const u64 cap = host_round_cap(prev.expanded);
            u64 before = 0;
            for (int s = 0; s < G_; ++s) {
                const u64 u = c0.all[s].unique;
                const u64 room = cap > before ? cap - before : 0;
                count[s] = std::min(u, room);
                before += u;
            }
            if (observer) {
                std::vector<State> layer;
                for (Shard& s : local_) {
                    std::vector<State> part = fetch_layer(s, (r + 1) & 1, count[s.me], W);
                    layer.insert(layer.end(), part.begin(), part.end());
                }
                (*observer)(k, r, layer);
            }
            stopped = c0.stop != 0;
            ++r;
        }
        const ShardCtl& c0 = *local_[0].h_ctl;
        bool any_ovf = false;
        for (const LayerStats& ls : res.rounds) any_ovf = any_ovf || ls.overflowed;
        for (int i = r_first; i < rounds; ++i) {
            const ShardRound& s = c0.rs[i];
            if (!s.valid) break;
            LayerStats ls;
            ls.k = k;
            ls.round = i;
            ls.expanded = s.expanded;
            ls.emitted = s.emitted;
            ls.duplicates = s.offered - s.unique;
            ls.mmw_pruned = s.pruned;
            ls.overflowed = s.overflowed != 0;
            any_ovf = any_ovf || ls.overflowed;
            res.rounds.push_back(ls);
            if (s.emitted == 0) break;
        }
        res.overflowed = any_ovf;
        // SURVEY §8d algorithmic bytes (same model as the single-device engine)
        // plus the records that crossed to other shards
        const double wb = 8.0 * W + 4.0, db = cfg.dedup == DedupMode::bloom ? 4.0 * cfg.bloom_hashes : 8.0 * W + 8.0;
        for (int i = r_first; i < rounds && c0.rs[i].valid; ++i) {
            const ShardRound& s = c0.rs[i];
            layer_bytes_ += wb * static_cast<double>(s.expanded + s.emitted);
            dedup_bytes_ += db * static_cast<double>(s.offered);
            expanded_ += s.expanded;
            offered_ += s.offered;
            unique_ += s.emitted;
            exchange_bytes_ += 8.0 * (W + 1) * static_cast<double>(s.routed) * (G_ - 1) / G_;
        }
        check(cudaEventRecord(ev_[1], stream_), "event");
        check(cudaEventSynchronize(ev_[1]), "event sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
        decide_ms_ += ms;
        const bool empty = !res.rounds.empty() && res.rounds.back().emitted == 0;
        if (empty) {
            res.outcome = any_ovf ? Outcome::indeterminate : Outcome::infeasible;
            return res;
        }
        if (static_cast<int>(res.rounds.size()) != rounds)
            throw DeviceError("sharded decide stopped early without an empty layer");
        res.outcome = Outcome::feasible;
        // witness = front of the final layer on the lowest shard holding states
        int root = 0;
        while (root < G_ && count[root] == 0) ++root;
        res.witness = witness(root, rounds & 1, W);
        return res;
    }

private:
    int G_ = 1, rank_ = 0, device_ = -1;
    ncclComm_t comm_ = nullptr;
    cudaStream_t stream_ = nullptr;
    cudaEvent_t ev_[2] = {nullptr, nullptr};
    std::vector<Shard> local_;
    u64 np_floor_ = 1, cap_floor_ = 0;
    u64 free_count_ = 0, max_states_ = 0;
    double decide_ms_ = 0, layer_bytes_ = 0, dedup_bytes_ = 0, exchange_bytes_ = 0;
    uint64_t launches_ = 0, reruns_ = 0, expanded_ = 0, h2d_ = 0, d2h_ = 0, offered_ = 0, unique_ = 0;
    cudaEvent_t tev_[2] = {nullptr, nullptr};
    int grid_route_[2] = {0, 0}, grid_owner_[2] = {0, 0};
    int grid_route_sh_ = 0;  // grid of the shared-boundary-table route variant
    bool shared_r_ = true;
    bool tile_dedup_ = false;
    bool trace_ = std::getenv("ETWG_SHARD_TRACE") != nullptr;
    u64* d_wit_ = nullptr;
    int pl_round_parity_ = 0;  // buffer holding the current round's input layer
    u64* d_scratch_ = nullptr;  // histogram counters + handoff ticket
    bool tight_ = std::getenv("ETWG_SHARD_TIGHT") != nullptr;  // tests: force aborts / re-runs
    // Emitter-stored layers (default; ETWG_SHARD_MODE=owner or
    // etwg_set_shard_mode(0) selects owner-stored): next-layer states stay
    // on the shard that emitted them, owners only deduplicate and return
    // marks. Virtual shards and the NVLink pull; the NCCL send/recv exchange
    // keeps owner-stored layers.
    bool emit_request_ = [] {
        const char* e = std::getenv("ETWG_SHARD_MODE");
        return !(e && std::strcmp(e, "owner") == 0);
    }();
    bool emit_ = false;
    u64 mark_cap_plan_ = 0, mark_floor_ = 0;
    // layers up to this many states are expanded redundantly by every shard
    // on the single-device engine (no routing); the first larger layer is
    // split by owner. ETWG_HANDOFF=0 shards from the root.
    u64 handoff_ = [] {
        const char* e = std::getenv("ETWG_HANDOFF");
        return e ? std::strtoull(e, nullptr, 10) : (u64{1} << 19);
    }();
    bool p2p_ = false;          // NCCL mode: pull records over NVLink instead of send/recv
    bool handles_dirty_ = false;  // outboxes (re)allocated since the last handle exchange
    const u64* peer_out_[kMaxShards] = {};
    const unsigned* peer_cnt_[kMaxShards] = {};
    const u64* peer_marks_[kMaxShards] = {};
    u64* peer_cmask_[kMaxShards] = {};
    bool direct_request_ = [] {  // ETWG_DIRECT_MARKS=0: owners return mark lists instead
        const char* e = std::getenv("ETWG_DIRECT_MARKS");
        return !(e && e[0] == '0');
    }();
    const unsigned* peer_mark_cnt_[kMaxShards] = {};
    unsigned char* d_handles_ = nullptr;

    void init_device(int dev) {
        if (device_ == dev && stream_) return;
        check(cudaSetDevice(dev), "cudaSetDevice");
        device_ = dev;
        cudaDeviceProp prop;
        check(cudaGetDeviceProperties(&prop, dev), "device properties");
        check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
        check(cudaEventCreate(&ev_[0]), "event");
        check(cudaEventCreate(&ev_[1]), "event");
        check(cudaEventCreate(&tev_[0]), "event");
        check(cudaEventCreate(&tev_[1]), "event");
        check(cudaMalloc(&d_wit_, 32), "witness");
        auto allow = [&](auto kernel, int bytes, int& grid) {
            check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "smem");
            int blocks = 0;
            check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, kOwnerThreads, bytes), "occupancy");
            grid = prop.multiProcessorCount * std::max(1, blocks);
        };
        allow(k_owner<1, false>, owner_smem_bytes<1>(), grid_owner_[0]);
        allow(k_owner<1, true>, owner_smem_bytes<1>(), grid_owner_[0]);
        allow(k_owner<2, false>, owner_smem_bytes<2>(), grid_owner_[1]);
        allow(k_owner<2, true>, owner_smem_bytes<2>(), grid_owner_[1]);
        {
            int g;
            allow(k_owner_emit<1, false>, owner_smem_bytes<1>(), g);
            allow(k_owner_emit<1, true>, owner_smem_bytes<1>(), g);
            allow(k_owner_emit<2, false>, owner_smem_bytes<2>(), g);
            allow(k_owner_emit<2, true>, owner_smem_bytes<2>(), g);
        }
        auto allow_route = [&](auto kernel, int bytes, int& grid) {
            check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "smem");
            int blocks = 0;
            check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, kRouteThreads, bytes), "occupancy");
            grid = prop.multiProcessorCount * std::max(1, blocks);
        };
        // ETWG_ROUTE_DEDUP=1 pre-dedups each tile of parents before routing.
        // Off by default: a shard's layer is in (partition, rank) order, so
        // consecutive parents are rarely siblings and the tile finds almost
        // no duplicates (measured: 0.01 % of the routed records on G(48,0.2)).
        const char* td = std::getenv("ETWG_ROUTE_DEDUP");
        tile_dedup_ = td && td[0] == '1';
        // grid = resident CTAs of the variant that will run (the MMW one bounds it)
        int g_mmw[2];
        if (tile_dedup_) {
            allow_route(k_route<1, false, true>, route_smem_bytes<1>(), grid_route_[0]);
            allow_route(k_route<1, true, true>, route_smem_bytes<1>(), g_mmw[0]);
            allow_route(k_route<2, false, true>, route_smem_bytes<2>(), grid_route_[1]);
            allow_route(k_route<2, true, true>, route_smem_bytes<2>(), g_mmw[1]);
        } else {
            allow_route(k_route<1, false, false>, 0, grid_route_[0]);
            allow_route(k_route<1, true, false>, 0, g_mmw[0]);
            allow_route(k_route<2, false, false>, 0, grid_route_[1]);
            allow_route(k_route<2, true, false>, 0, g_mmw[1]);
        }
        grid_route_[0] = std::min(grid_route_[0], g_mmw[0]);
        grid_route_[1] = std::min(grid_route_[1], g_mmw[1]);
        {
            const char* e = std::getenv("ETWG_ROUTE_SHARED_R");
            shared_r_ = !(e && e[0] == '0');
            allow_route(k_route<1, false, false>, kShSlots * 8 * kRouteThreads, grid_route_sh_);
        }
        if (const char* c = std::getenv("ETWG_ROUTE_CTAS")) {  // CTAs per SM (tuning sweeps)
            const int per = std::atoi(c);
            for (int w = 0; w < 2; ++w) grid_route_[w] = std::min(grid_route_[w], prop.multiProcessorCount * per);
        }
    }

    void create_shard(Shard& s, int me) {
        s = Shard{};
        s.me = me;
        check(cudaMalloc(&s.d_params, sizeof(Params)), "params");
        check(cudaMallocHost(&s.h_params, sizeof(Params)), "params");
        check(cudaMalloc(&s.d_ctl, sizeof(ShardCtl)), "control");
        check(cudaMallocHost(&s.h_ctl, sizeof(ShardCtl)), "control");
        std::memset(s.h_ctl, 0, sizeof(ShardCtl));
    }

    static void destroy_shard(Shard& s) {
        cudaFree(s.d_params);
        cudaFreeHost(s.h_params);
        cudaFree(s.d_ctl);
        cudaFreeHost(s.h_ctl);
        for (int i = 0; i < 2; ++i) {
            cudaFree(s.b.keys[i]);
            cudaFree(s.b.hist[i]);
        }
        cudaFree(s.b.out);
        cudaFree(s.b.out_cnt);
        cudaFree(s.b.in);
        cudaFree(s.b.in_cnt);
        cudaFree(s.b.tiles);
        cudaFree(s.b.bloom);
        cudaFree(s.b.stage);
        cudaFree(s.b.stage_hist);
        cudaFree(s.b.pcount);
        cudaFree(s.b.marks);
        cudaFree(s.b.mark_cnt);
        cudaFree(s.b.cmask);
        s = Shard{};
    }

    // Params + control of shard s for a decide starting at round r0: the
    // root on shard 0 (r0 = 0), or this shard's owned part of the engine's
    // replicated layer (handoff).
    void setup(Shard& s, const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg, int rounds,
               int r0 = 0, const EngineLayer* from = nullptr, u64 owned = 0) {
        Params& p = *s.h_params;
        std::memset(&p, 0, sizeof p);
        p.n = g.vertex_count();
        p.k = k;
        p.rounds = rounds;
        p.free_count = std::max(0, g.vertex_count() - forbidden.count());
        p.hashes = cfg.bloom_hashes;
        p.bpe = cfg.bloom_bits_per_element;
        p.max_states = cfg.max_layer_states;
        p.forbidden[0] = forbidden.w[0];
        p.forbidden[1] = forbidden.w[1];
        for (int v = 0; v < g.vertex_count(); ++v) {
            p.rows[v][0] = g.neighbors(v).w[0];
            p.rows[v][1] = g.neighbors(v).w[1];
        }
        free_count_ = static_cast<u64>(p.free_count);
        max_states_ = p.max_states;
        check(cudaMemcpyAsync(s.d_params, s.h_params, sizeof(Params), cudaMemcpyHostToDevice, stream_), "params");
        h2d_ += sizeof(Params) + sizeof(ShardCtl);
        ShardCtl& c = *s.h_ctl;
        const unsigned epoch = c.epoch;
        std::memset(&c, 0, sizeof c);
        c.epoch = next_epoch(s, epoch);
        if (from) {
            c.round = static_cast<unsigned>(r0);
            c.count[r0 & 1] = owned;
            grow_layers(s, owned + owned / 4 + 1024, 0, 0);
            if (emit_) {
                const u64 first = from->count * static_cast<u64>(s.me) / G_;
                const int W = from->W;
                check(cudaMemcpyAsync(s.b.keys[r0 & 1], static_cast<const u64*>(from->keys) + first * W, owned * 8 * W,
                                      cudaMemcpyDeviceToDevice, stream_), "handoff slice");
                check(cudaMemcpyAsync(s.b.hist[r0 & 1], from->hist + first, owned * 4, cudaMemcpyDeviceToDevice, stream_),
                      "handoff slice");
            } else {
                take_owned(s, *from, r0 & 1);
            }
            check(cudaMemcpyAsync(s.d_ctl, s.h_ctl, sizeof(ShardCtl), cudaMemcpyHostToDevice, stream_), "control");
            return;
        }
        c.count[0] = s.me == 0 ? 1 : 0;
        check(cudaMemcpyAsync(s.d_ctl, s.h_ctl, sizeof(ShardCtl), cudaMemcpyHostToDevice, stream_), "control");
        grow_layers(s, 1 << 16, 0, 0);
        if (s.me == 0) {
            const u64 zero2[2] = {0, 0};
            const unsigned root_hist = 0xFFFFFFFFu;
            check(cudaMemcpyAsync(s.b.keys[0], zero2, 16, cudaMemcpyHostToDevice, stream_), "root");
            check(cudaMemcpyAsync(s.b.hist[0], &root_hist, 4, cudaMemcpyHostToDevice, stream_), "root");
            check(cudaStreamSynchronize(stream_), "root");
        }
    }

    // per-owner state counts of the engine's layer (identical on every rank)
    std::vector<u64> owner_counts(const EngineLayer& L) {
        if (!d_scratch_) check(cudaMalloc(&d_scratch_, 256), "scratch");
        check(cudaMemsetAsync(d_scratch_, 0, 8 * kMaxShards, stream_), "scratch");
        const int grid = static_cast<int>(std::min<u64>((L.count + 255) / 256, 4096));
        if (L.W == 1)
            k_owner_histogram<1><<<std::max(grid, 1), 256, 0, stream_>>>(static_cast<const u64*>(L.keys), L.count, G_,
                                                                         reinterpret_cast<unsigned long long*>(d_scratch_));
        else
            k_owner_histogram<2><<<std::max(grid, 1), 256, 0, stream_>>>(static_cast<const u64*>(L.keys), L.count, G_,
                                                                         reinterpret_cast<unsigned long long*>(d_scratch_));
        check(cudaGetLastError(), "owner histogram");
        ++launches_;
        std::vector<u64> c(G_);
        check(cudaMemcpyAsync(c.data(), d_scratch_, 8 * G_, cudaMemcpyDeviceToHost, stream_), "owner counts");
        check(cudaStreamSynchronize(stream_), "owner counts");
        return c;
    }

    // the engine's layer -> this shard's layer buffer `buf`, owned states only, in order
    void take_owned(Shard& s, const EngineLayer& L, int buf) {
        const u64 tiles_needed = (L.count + 2047) / 2048 + 1;
        if (tiles_needed > s.b.tile_cap || !s.b.tiles) {
            const u64 cap = std::max<u64>(tiles_needed * 2, u64{1} << 12);
            cudaFree(s.b.tiles);
            check(cudaMalloc(&s.b.tiles, cap * 8), "tiles");
            check(cudaMemsetAsync(s.b.tiles, 0, cap * 8, stream_), "tiles");
            s.b.tile_cap = cap;
        }
        s.h_ctl->epoch = next_epoch(s, s.h_ctl->epoch);
        const unsigned epoch = s.h_ctl->epoch;
        s.h_ctl->epoch = next_epoch(s, epoch);  // the first sharded round gets a fresh epoch
        if (!d_scratch_) check(cudaMalloc(&d_scratch_, 256), "scratch");
        unsigned long long* ticket = reinterpret_cast<unsigned long long*>(d_scratch_) + kMaxShards;
        check(cudaMemsetAsync(ticket, 0, 8, stream_), "ticket");
        const int grid = std::max(1, std::min(grid_route_[0], static_cast<int>((L.count + 2047) / 2048)));
        if (L.W == 1)
            k_take_owned<1><<<grid, kRouteThreads, 0, stream_>>>(static_cast<const u64*>(L.keys), L.hist, L.count, G_,
                                                                 s.me, s.b.keys[buf], s.b.hist[buf], s.b.tiles, epoch, ticket);
        else
            k_take_owned<2><<<grid, kRouteThreads, 0, stream_>>>(static_cast<const u64*>(L.keys), L.hist, L.count, G_,
                                                                 s.me, s.b.keys[buf], s.b.hist[buf], s.b.tiles, epoch, ticket);
        check(cudaGetLastError(), "take owned");
        ++launches_;
    }

    unsigned next_epoch(Shard& s, unsigned e) {
        e = (e + 1) & kEpochMask;
        if (e == 0) {
            e = 1;
            if (s.b.tiles) check(cudaMemsetAsync(s.b.tiles, 0, s.b.tile_cap * 8, stream_), "tiles clear");
        }
        return e;
    }

    u64 host_round_cap(u64 e_in) const {
        u64 upper = e_in * free_count_;
        if (upper < 1) upper = 1;
        return std::min<u64>(max_states_, upper);
    }

    static u64 pow2_at_least(u64 x) {
        u64 s = 1;
        while (s < x) s <<= 1;
        return s;
    }

    Plan plan(int r, const std::vector<u64>& count, const ShardRound& prev, const DpConfig& cfg, int W) {
        u64 E = 0, Emax = 0;
        for (u64 c : count) {
            E += c;
            Emax = std::max(Emax, c);
        }
        const u64 fc = std::max<u64>(free_count_, 1);
        u64 distinct = std::max<u64>(E * fc, 1), routed_max = std::max<u64>(Emax * fc, 1);
        if (r > 0 && prev.expanded) {
            const double grow_u = static_cast<double>(prev.unique) / static_cast<double>(prev.expanded);
            const double grow_r = static_cast<double>(prev.routed) / static_cast<double>(prev.expanded);
            distinct = std::min<u64>(distinct, static_cast<u64>(static_cast<double>(E) * grow_u * 1.25) + 64);
            routed_max = std::min<u64>(routed_max, static_cast<u64>(static_cast<double>(Emax) * grow_r * 1.25) + 64);
        }
        Plan pl{};
        pl.G = G_;
        pl.rounds = local_[0].h_params->rounds;
        const u64 per_owner = (distinct + G_ - 1) / G_;
        pl.np = std::max<u64>(pow2_at_least((per_owner + owner_target<1>() - 1) / owner_target<1>()), np_floor_);
        pl.lg = 0;
        while ((u64{1} << pl.lg) < pl.np) ++pl.lg;
        const u64 per = (routed_max + G_ * pl.np - 1) / (G_ * pl.np);
        pl.cap = std::max<u64>(per + per / 4 + 64, cap_floor_);
        pl.layer_est = per_owner + per_owner / 4 + 1024;
        pl.emit = emit_ ? 1 : 0;
        pl.direct = 0;  // decided per launch (launch_owner_emit): needs every emitter's mask mapped
        mark_cap_plan_ = std::max<u64>(per_owner + per_owner / 2 + 4096, mark_floor_);
        if (tight_) {  // tests: undersized plans, so rounds abort, grow and re-run
            pl.np = std::max<u64>(std::max<u64>(pl.np / 16, 1), np_floor_);
            pl.lg = 0;
            while ((u64{1} << pl.lg) < pl.np) ++pl.lg;
            const u64 per2 = (routed_max + G_ * pl.np - 1) / (G_ * pl.np);
            pl.cap = std::max<u64>(per2 / 4 + 1, cap_floor_);
            pl.layer_est = 0;
            mark_cap_plan_ = std::max<u64>(per_owner / 8 + 1, mark_floor_);
        }
        pl.bloom_m = 0;
        if (cfg.dedup == DedupMode::bloom) {
            const u64 cap = host_round_cap(E);
            pl.bloom_m = bloom_bits_for((cap + G_ - 1) / G_, cfg.bloom_bits_per_element);
        }
        (void)W;
        return pl;
    }

    void grow_layers(Shard& s, u64 states, int keep_buf, u64 keep_count) {
        if (states <= s.b.layer_cap && s.b.keys[0]) return;
        const u64 cap = std::max<u64>(states, std::max<u64>(s.b.layer_cap * 2, u64{1} << 16));
        u64* keys[2];
        unsigned* hist[2];
        for (int i = 0; i < 2; ++i) {
            check(cudaMalloc(&keys[i], cap * 16), "layer keys");
            check(cudaMalloc(&hist[i], cap * 4), "layer hist");
        }
        if (s.b.keys[0] && keep_count) {
            check(cudaMemcpyAsync(keys[keep_buf], s.b.keys[keep_buf], keep_count * 16, cudaMemcpyDeviceToDevice, stream_),
                  "keep layer");
            check(cudaMemcpyAsync(hist[keep_buf], s.b.hist[keep_buf], keep_count * 4, cudaMemcpyDeviceToDevice, stream_),
                  "keep layer");
        }
        check(cudaStreamSynchronize(stream_), "sync");
        for (int i = 0; i < 2; ++i) {
            cudaFree(s.b.keys[i]);
            cudaFree(s.b.hist[i]);
            s.b.keys[i] = keys[i];
            s.b.hist[i] = hist[i];
        }
        s.b.layer_cap = cap;
    }

    void prepare_round(Shard& s, const Plan& pl, int W, bool bloom, const std::vector<u64>& count) {
        const u64 recs = static_cast<u64>(G_) * pl.np * pl.cap;
        const u64 cnts = static_cast<u64>(G_) * pl.np;
        if (W != s.box_words) {  // record size changed: reallocate at the new width
            s.b.box_cap = 0;
            s.box_words = W;
        }
        if (recs > s.b.box_cap || !s.b.out) {
            const u64 cap = std::max<u64>(recs + recs / 16, u64{1} << 16);
            cudaFree(s.b.out);
            cudaFree(s.b.in);
            s.b.in = nullptr;
            check(cudaMalloc(&s.b.out, cap * 8 * (W + 1)), "outbox");
            if (comm_ && !p2p_) check(cudaMalloc(&s.b.in, cap * 8 * (W + 1)), "inbox");
            s.b.box_cap = cap;
            handles_dirty_ = true;
        }
        if (cnts > s.b.cnt_cap || !s.b.out_cnt) {
            const u64 cap = std::max<u64>(cnts * 2, u64{1} << 12);
            cudaFree(s.b.out_cnt);
            cudaFree(s.b.in_cnt);
            s.b.in_cnt = nullptr;
            check(cudaMalloc(&s.b.out_cnt, cap * 4), "outbox counts");
            if (comm_ && !p2p_) check(cudaMalloc(&s.b.in_cnt, cap * 4), "inbox counts");
            s.b.cnt_cap = cap;
            handles_dirty_ = true;
        }
        if (pl.np > s.b.stage_cap || !s.b.stage) {
            const u64 cap = std::max<u64>(pl.np + pl.np / 4, 64);
            cudaFree(s.b.stage);
            cudaFree(s.b.stage_hist);
            cudaFree(s.b.pcount);
            check(cudaMalloc(&s.b.stage, cap * owner_slots<1>() * 8 * W), "owner staging");
            check(cudaMalloc(&s.b.stage_hist, cap * owner_slots<1>() * 4), "owner staging");
            check(cudaMalloc(&s.b.pcount, cap * 4), "partition counts");
            s.b.stage_cap = cap;
            s.stage_words = W;
        }
        if (W != s.stage_words) {  // staging sized for one-word keys: regrow at the new width
            cudaFree(s.b.stage);
            check(cudaMalloc(&s.b.stage, s.b.stage_cap * owner_slots<1>() * 8 * W), "owner staging");
            s.stage_words = W;
        }
        if (emit_) {
            const u64 need = static_cast<u64>(G_) * mark_cap_plan_;
            if (need > s.mark_alloc || !s.b.marks) {
                const u64 cap = need + need / 4;
                cudaFree(s.b.marks);
                check(cudaMalloc(&s.b.marks, cap * 8), "marks");
                s.mark_alloc = cap;
                handles_dirty_ = true;
            }
            if (!s.b.mark_cnt) {
                check(cudaMalloc(&s.b.mark_cnt, kMaxShards * 4), "mark counts");
                handles_dirty_ = true;
            }
            s.b.mark_cap = mark_cap_plan_;
            check(cudaMemsetAsync(s.b.mark_cnt, 0, kMaxShards * 4, stream_), "mark counts");
            if (s.cmask_cap < s.b.layer_cap || !s.b.cmask) {
                cudaFree(s.b.cmask);
                check(cudaMalloc(&s.b.cmask, s.b.layer_cap * 16), "winner masks");
                s.cmask_cap = s.b.layer_cap;
                handles_dirty_ = true;  // peers map the masks for direct marks
            }
            const u64 tiles_needed = (count[s.me] + emit_span(W) - 1) / emit_span(W) + 2;
            if (tiles_needed > s.b.tile_cap) {
                const u64 cap = std::max<u64>(tiles_needed * 2, u64{1} << 12);
                cudaFree(s.b.tiles);
                check(cudaMalloc(&s.b.tiles, cap * 8), "tiles");
                check(cudaMemsetAsync(s.b.tiles, 0, cap * 8, stream_), "tiles");
                s.b.tile_cap = cap;
            }
        }
        if (pl.np + 1 > s.b.tile_cap || !s.b.tiles) {
            const u64 cap = std::max<u64>((pl.np + 1) * 2, u64{1} << 12);
            cudaFree(s.b.tiles);
            check(cudaMalloc(&s.b.tiles, cap * 8), "tiles");
            check(cudaMemsetAsync(s.b.tiles, 0, cap * 8, stream_), "tiles");
            s.b.tile_cap = cap;
        }
        // the next layer holds about this shard's share of the distinct keys
        grow_layers(s, pl.layer_est, pl_round_parity_, count[s.me]);
        check(cudaMemsetAsync(s.b.out_cnt, 0, cnts * 4, stream_), "outbox counts");
        if (bloom) {
            const u64 words = (pl.bloom_m + 31) / 32;
            if (words > s.b.bloom_cap || !s.b.bloom) {
                const u64 cap = std::max<u64>(words + words / 4, u64{1} << 20);
                cudaFree(s.b.bloom);
                check(cudaMalloc(&s.b.bloom, cap * 4), "bloom slice");
                s.b.bloom_cap = cap;
                s.bloom_dirty = cap;
            }
            // a fresh filter every round (dp.cpp:93-94)
            const u64 clear = std::min(std::max(s.bloom_dirty, words), s.b.bloom_cap);
            check(cudaMemsetAsync(s.b.bloom, 0, clear * 4, stream_), "bloom clear");
            s.bloom_dirty = words;
        }
    }

    template <int W, bool MMW>
    void route_kernel(Shard& s, const Plan& p) {
        if (tile_dedup_)
            k_route<W, MMW, true><<<grid_route_[W - 1], kRouteThreads, route_smem_bytes<W>(), stream_>>>(
                s.d_params, s.d_ctl, s.b, p);
        else if (W == 1 && !MMW && shared_r_)
            k_route<W, MMW, false><<<grid_route_sh_, kRouteThreads, kShSlots * 8 * kRouteThreads, stream_>>>(
                s.d_params, s.d_ctl, s.b, p);
        else
            k_route<W, MMW, false><<<grid_route_[W - 1], kRouteThreads, 0, stream_>>>(s.d_params, s.d_ctl, s.b, p);
    }

    void launch_route(Shard& s, const Plan& pl, int W, bool mmw) {
        Plan p = pl;
        p.me = s.me;
        p.shared_r = shared_r_ ? 1 : 0;
        if (W == 1) {
            if (mmw) route_kernel<1, true>(s, p);
            else route_kernel<1, false>(s, p);
        } else {
            if (mmw) route_kernel<2, true>(s, p);
            else route_kernel<2, false>(s, p);
        }
        check(cudaGetLastError(), "route launch");
        ++launches_;
    }

    void launch_owner(Shard& s, const Plan& pl, int W, bool bloom) {
        Plan p = pl;
        p.me = s.me;
        const u64 block = pl.np * pl.cap * (W + 1);
        for (int src = 0; src < G_; ++src) {
            if (!comm_) {  // virtual shards: read the source's outbox in place
                const Shard& from = local_[src];
                s.b.src_recs[src] = from.b.out + s.me * block;
                s.b.src_cnt[src] = from.b.out_cnt + s.me * pl.np;
            } else if (src == s.me) {
                s.b.src_recs[src] = s.b.out + s.me * block;
                s.b.src_cnt[src] = s.b.out_cnt + s.me * pl.np;
            } else if (p2p_) {  // the peer's outbox, read over NVLink
                s.b.src_recs[src] = peer_out_[src] + s.me * block;
                s.b.src_cnt[src] = peer_cnt_[src] + s.me * pl.np;
            } else {
                s.b.src_recs[src] = s.b.in + src * block;
                s.b.src_cnt[src] = s.b.in_cnt + src * pl.np;
            }
        }
        if (W == 1) {
            if (bloom) k_owner<1, true><<<grid_owner_[0], kOwnerThreads, owner_smem_bytes<1>(), stream_>>>(s.d_params, s.d_ctl, s.b, p);
            else k_owner<1, false><<<grid_owner_[0], kOwnerThreads, owner_smem_bytes<1>(), stream_>>>(s.d_params, s.d_ctl, s.b, p);
        } else {
            if (bloom) k_owner<2, true><<<grid_owner_[1], kOwnerThreads, owner_smem_bytes<2>(), stream_>>>(s.d_params, s.d_ctl, s.b, p);
            else k_owner<2, false><<<grid_owner_[1], kOwnerThreads, owner_smem_bytes<2>(), stream_>>>(s.d_params, s.d_ctl, s.b, p);
        }
        check(cudaGetLastError(), "owner launch");
        ++launches_;
    }

    void set_sources(Shard& s, const Plan& pl, int W) {
        const u64 block = pl.np * pl.cap * (W + 1);
        for (int src = 0; src < G_; ++src) {
            if (!comm_) {
                const Shard& from = local_[src];
                s.b.src_recs[src] = from.b.out + s.me * block;
                s.b.src_cnt[src] = from.b.out_cnt + s.me * pl.np;
            } else if (src == s.me) {
                s.b.src_recs[src] = s.b.out + s.me * block;
                s.b.src_cnt[src] = s.b.out_cnt + s.me * pl.np;
            } else if (p2p_) {
                s.b.src_recs[src] = peer_out_[src] + s.me * block;
                s.b.src_cnt[src] = peer_cnt_[src] + s.me * pl.np;
            } else {
                s.b.src_recs[src] = s.b.in + src * block;
                s.b.src_cnt[src] = s.b.in_cnt + src * pl.np;
            }
        }
    }

    // direct marks: every emitter's winner mask reachable from this shard
    bool direct_marks(Shard& s) {
        if (!direct_request_) return false;
        for (int e = 0; e < G_; ++e) {
            u64* m = !comm_ ? local_[e].b.cmask : (e == s.me ? s.b.cmask : (p2p_ ? peer_cmask_[e] : nullptr));
            if (!m) return false;
            s.b.dst_cmask[e] = m;
        }
        return true;
    }

    void launch_owner_emit(Shard& s, const Plan& pl, int W, bool bloom) {
        Plan p = pl;
        p.me = s.me;
        p.direct = direct_marks(s) ? 1 : 0;
        set_sources(s, pl, W);
        if (W == 1) {
            if (bloom) k_owner_emit<1, true><<<grid_owner_[0], kOwnerThreads, owner_smem_bytes<1>(), stream_>>>(s.d_params, s.d_ctl, s.b, p);
            else k_owner_emit<1, false><<<grid_owner_[0], kOwnerThreads, owner_smem_bytes<1>(), stream_>>>(s.d_params, s.d_ctl, s.b, p);
        } else {
            if (bloom) k_owner_emit<2, true><<<grid_owner_[1], kOwnerThreads, owner_smem_bytes<2>(), stream_>>>(s.d_params, s.d_ctl, s.b, p);
            else k_owner_emit<2, false><<<grid_owner_[1], kOwnerThreads, owner_smem_bytes<2>(), stream_>>>(s.d_params, s.d_ctl, s.b, p);
        }
        check(cudaGetLastError(), "owner launch");
        ++launches_;
    }

    // marks from every owner into this shard's winner masks, then its next layer
    void launch_emit_append(Shard& s, const Plan& pl, int W) {
        Plan p = pl;
        p.me = s.me;
        for (int o = 0; o < G_; ++o) {
            if (!comm_) {  // virtual shards: the other shard's marks in place
                s.b.src_marks[o] = local_[o].b.marks;
                s.b.src_mark_cnt[o] = local_[o].b.mark_cnt;
            } else if (o == s.me) {
                s.b.src_marks[o] = s.b.marks;
                s.b.src_mark_cnt[o] = s.b.mark_cnt;
            } else {  // the owner's marks, read over NVLink
                s.b.src_marks[o] = peer_marks_[o];
                s.b.src_mark_cnt[o] = peer_mark_cnt_[o];
            }
        }
        const int grid = grid_route_[0];
        const bool direct = direct_marks(s);  // the owners already set the winner bits
        if (W == 1) {
            if (!direct) k_apply_marks<1><<<grid, kRouteThreads, 0, stream_>>>(s.d_ctl, s.b, p);
            k_emit_append<1><<<grid, kRouteThreads, 0, stream_>>>(s.d_ctl, s.b, p);
        } else {
            if (!direct) k_apply_marks<2><<<grid, kRouteThreads, 0, stream_>>>(s.d_ctl, s.b, p);
            k_emit_append<2><<<grid, kRouteThreads, 0, stream_>>>(s.d_ctl, s.b, p);
        }
        check(cudaGetLastError(), "emit append launch");
        launches_ += 2;
    }

    void route_barrier() {
        Nccl& nc = Nccl::get();
        Shard& s = local_[0];
        nc.check(nc.AllGather(&s.d_ctl->mine, &s.d_ctl->all[0], sizeof(ShardStat), ncclUint8, comm_, stream_),
                 "marks barrier");
    }

    void launch_compact(Shard& s, const Plan& pl, int W) {
        Plan p = pl;
        p.me = s.me;
        const int grid = std::max(1, std::min<int>(static_cast<int>((pl.np + kRouteThreads - 1) / kRouteThreads),
                                                   grid_route_[0]));
        if (W == 1)
            k_owner_compact<1><<<grid, kRouteThreads, 0, stream_>>>(s.d_ctl, s.b, p);
        else
            k_owner_compact<2><<<grid, kRouteThreads, 0, stream_>>>(s.d_ctl, s.b, p);
        check(cudaGetLastError(), "compact launch");
        ++launches_;
    }

    // outbox block d of shard s -> inbox slot s of shard d (NCCL); virtual
    // shards and a shard's own block are read in place by k_owner
    void exchange(const Plan& pl, int W) {
        if (!comm_) return;
        if (p2p_) {
            // every route must be complete before any owner reads a peer's
            // outbox: a stream-ordered allgather of the route counters is the
            // barrier (the post-owner allgather refreshes all[] anyway)
            Nccl& nc = Nccl::get();
            Shard& s = local_[0];
            nc.check(nc.AllGather(&s.d_ctl->mine, &s.d_ctl->all[0], sizeof(ShardStat), ncclUint8, comm_, stream_),
                     "route barrier");
            return;
        }
        const u64 block = pl.np * pl.cap * (W + 1);
        const u64 bytes = block * 8, cnt_bytes = pl.np * 4;
        Nccl& nc = Nccl::get();
        Shard& s = local_[0];
        nc.check(nc.GroupStart(), "group start");
        for (int d = 0; d < G_; ++d) {
            if (d == s.me) continue;
            nc.check(nc.Send(s.b.out + d * block, bytes, ncclUint8, d, comm_, stream_), "send");
            nc.check(nc.Recv(s.b.in + d * block, bytes, ncclUint8, d, comm_, stream_), "recv");
            nc.check(nc.Send(s.b.out_cnt + d * pl.np, cnt_bytes, ncclUint8, d, comm_, stream_), "send counts");
            nc.check(nc.Recv(s.b.in_cnt + d * pl.np, cnt_bytes, ncclUint8, d, comm_, stream_), "recv counts");
        }
        nc.check(nc.GroupEnd(), "group end");
    }

    void allgather_stats() {
        if (!comm_) {
            for (Shard& src : local_)
                for (Shard& dst : local_)
                    check(cudaMemcpyAsync(&dst.d_ctl->all[src.me], &src.d_ctl->mine, sizeof(ShardStat),
                                          cudaMemcpyDeviceToDevice, stream_), "stat gather");
            return;
        }
        Nccl& nc = Nccl::get();
        Shard& s = local_[0];
        nc.check(nc.AllGather(&s.d_ctl->mine, &s.d_ctl->all[0], sizeof(ShardStat), ncclUint8, comm_, stream_),
                 "allgather stats");
    }

    // Collective: every rank publishes CUDA IPC handles of its outbox and
    // bucket counts and maps its peers'. If any rank fails to map, all fall
    // back to the NCCL send/recv exchange.
    struct IpcRecord {
        cudaIpcMemHandle_t out, cnt, marks, mark_cnt, cmask;
        int ok, has_marks, has_cmask, pad;
    };

    void share_outboxes(Shard& s) {
        close_peers();
        Nccl& nc = Nccl::get();
        const size_t rec = sizeof(IpcRecord);
        if (!d_handles_) check(cudaMalloc(&d_handles_, rec * kMaxShards + 64), "ipc handles");
        std::vector<IpcRecord> h(G_);
        IpcRecord mine{};
        cudaError_t why = cudaSuccess;
        auto ok_or = [&](cudaError_t e) {
            if (e != cudaSuccess && why == cudaSuccess) why = e;
            return e == cudaSuccess;
        };
        mine.ok = ok_or(cudaIpcGetMemHandle(&mine.out, s.b.out)) && ok_or(cudaIpcGetMemHandle(&mine.cnt, s.b.out_cnt));
        mine.has_marks = emit_ && s.b.marks && s.b.mark_cnt;
        if (mine.has_marks)
            mine.ok = mine.ok && ok_or(cudaIpcGetMemHandle(&mine.marks, s.b.marks)) &&
                      ok_or(cudaIpcGetMemHandle(&mine.mark_cnt, s.b.mark_cnt));
        mine.has_cmask = emit_ && s.b.cmask;
        if (mine.has_cmask) mine.ok = mine.ok && ok_or(cudaIpcGetMemHandle(&mine.cmask, s.b.cmask));
        cudaGetLastError();
        check(cudaMemcpyAsync(d_handles_ + rec * s.me, &mine, rec, cudaMemcpyHostToDevice, stream_), "ipc h2d");
        nc.check(nc.AllGather(d_handles_ + rec * s.me, d_handles_, rec, ncclUint8, comm_, stream_), "ipc allgather");
        check(cudaMemcpyAsync(h.data(), d_handles_, rec * G_, cudaMemcpyDeviceToHost, stream_), "ipc d2h");
        check(cudaStreamSynchronize(stream_), "ipc sync");
        int ok = 1;
        for (int p = 0; p < G_; ++p) ok &= h[p].ok;
        if (trace_)
            for (int p = 0; p < G_; ++p)
                std::fprintf(stderr, "[shard %d] ipc record of %d: ok=%d marks=%d (mine ok=%d, %s)\n", s.me, p, h[p].ok,
                             h[p].has_marks, mine.ok, cudaGetErrorString(why));
        for (int p = 0; ok && p < G_; ++p) {
            if (p == s.me) continue;
            void* a = nullptr;
            void* b = nullptr;
            if (trace_) std::fprintf(stderr, "[shard %d] opening peer %d handles\n", s.me, p);
            if (!ok_or(cudaIpcOpenMemHandle(&a, h[p].out, cudaIpcMemLazyEnablePeerAccess)) ||
                !ok_or(cudaIpcOpenMemHandle(&b, h[p].cnt, cudaIpcMemLazyEnablePeerAccess))) {
                cudaGetLastError();
                if (a) cudaIpcCloseMemHandle(a);
                ok = 0;
                break;
            }
            peer_out_[p] = static_cast<const u64*>(a);
            peer_cnt_[p] = static_cast<const unsigned*>(b);
            if (h[p].has_marks) {
                void* c = nullptr;
                void* d = nullptr;
                if (!ok_or(cudaIpcOpenMemHandle(&c, h[p].marks, cudaIpcMemLazyEnablePeerAccess)) ||
                    !ok_or(cudaIpcOpenMemHandle(&d, h[p].mark_cnt, cudaIpcMemLazyEnablePeerAccess))) {
                    cudaGetLastError();
                    if (c) cudaIpcCloseMemHandle(c);
                    ok = 0;
                    break;
                }
                peer_marks_[p] = static_cast<const u64*>(c);
                peer_mark_cnt_[p] = static_cast<const unsigned*>(d);
            }
            if (h[p].has_cmask) {
                void* e = nullptr;
                if (!ok_or(cudaIpcOpenMemHandle(&e, h[p].cmask, cudaIpcMemLazyEnablePeerAccess))) {
                    cudaGetLastError();
                    ok = 0;
                    break;
                }
                peer_cmask_[p] = static_cast<u64*>(e);
            }
        }
        if (trace_) std::fprintf(stderr, "[shard %d] opened: ok=%d (%s)\n", s.me, ok, cudaGetErrorString(why));
        // agree: p2p only if every rank mapped every peer
        int* flags = reinterpret_cast<int*>(d_handles_);
        check(cudaMemcpyAsync(flags + s.me, &ok, sizeof(int), cudaMemcpyHostToDevice, stream_), "ipc flag");
        nc.check(nc.AllGather(flags + s.me, flags, sizeof(int), ncclUint8, comm_, stream_), "ipc flag allgather");
        std::vector<int> all(G_);
        check(cudaMemcpyAsync(all.data(), flags, sizeof(int) * G_, cudaMemcpyDeviceToHost, stream_), "ipc flag d2h");
        check(cudaStreamSynchronize(stream_), "ipc sync");
        for (int v : all) ok &= v;
        if (trace_) std::fprintf(stderr, "[shard %d] flags %d %d -> ok=%d\n", s.me, all[0], G_ > 1 ? all[1] : -1, ok);
        handles_dirty_ = false;
        if (!ok) {
            close_peers();
            p2p_ = false;
            emit_ = false;  // emitter-stored layers need the NVLink pull
            s.b.box_cap = 0;  // reallocate with inboxes for the NCCL exchange
            s.b.cnt_cap = 0;
            std::fprintf(stderr, "[elimtw] CUDA IPC peer mapping unavailable (%s): NCCL send/recv exchange\n",
                         why == cudaSuccess ? "a peer failed" : cudaGetErrorString(why));
        }
    }

    void close_peers() {
        for (int p = 0; p < kMaxShards; ++p) {
            if (peer_out_[p]) cudaIpcCloseMemHandle(const_cast<u64*>(peer_out_[p]));
            if (peer_cnt_[p]) cudaIpcCloseMemHandle(const_cast<unsigned*>(peer_cnt_[p]));
            if (peer_marks_[p]) cudaIpcCloseMemHandle(const_cast<u64*>(peer_marks_[p]));
            if (peer_cmask_[p]) cudaIpcCloseMemHandle(peer_cmask_[p]);
            peer_cmask_[p] = nullptr;
            if (peer_mark_cnt_[p]) cudaIpcCloseMemHandle(const_cast<unsigned*>(peer_mark_cnt_[p]));
            peer_out_[p] = nullptr;
            peer_cnt_[p] = nullptr;
            peer_marks_[p] = nullptr;
            peer_mark_cnt_[p] = nullptr;
        }
    }

    // re-arm an aborted round: counters cleared, new look-back epoch
    void rearm(Shard& s) {
        ShardCtl& c = *s.h_ctl;
        c.ticket = 0;
        c.ticket2 = 0;
        c.mine = ShardStat{};
        c.epoch = next_epoch(s, c.epoch);
        check(cudaMemcpyAsync(s.d_ctl, s.h_ctl, offsetof(ShardCtl, all), cudaMemcpyHostToDevice, stream_), "re-arm");
    }

    std::vector<State> fetch_layer(Shard& s, int buf, u64 count, int W) {
        std::vector<u64> keys(static_cast<size_t>(W) * count);
        std::vector<unsigned> hist(count);
        if (count) {
            check(cudaMemcpyAsync(keys.data(), s.b.keys[buf], keys.size() * 8, cudaMemcpyDeviceToHost, stream_), "layer");
            check(cudaMemcpyAsync(hist.data(), s.b.hist[buf], count * 4, cudaMemcpyDeviceToHost, stream_), "layer");
            check(cudaStreamSynchronize(stream_), "sync");
        }
        std::vector<State> out(count);
        for (u64 i = 0; i < count; ++i) {
            out[i].set.w[0] = keys[W * i];
            out[i].set.w[1] = W == 2 ? keys[W * i + 1] : 0;
            out[i].history = hist[i];
        }
        return out;
    }

    State witness(int root, int buf, int W) {
        u64 h[4] = {0, 0, 0, 0};
        if (!comm_) {
            Shard& s = local_[root];
            check(cudaMemcpyAsync(h, s.b.keys[buf], 8 * W, cudaMemcpyDeviceToHost, stream_), "witness");
            check(cudaMemcpyAsync(&h[2], s.b.hist[buf], 4, cudaMemcpyDeviceToHost, stream_), "witness");
        } else {
            Shard& s = local_[0];
            if (s.me == root) {
                check(cudaMemcpyAsync(d_wit_, s.b.keys[buf], 8 * W, cudaMemcpyDeviceToDevice, stream_), "witness");
                check(cudaMemcpyAsync(d_wit_ + 2, s.b.hist[buf], 4, cudaMemcpyDeviceToDevice, stream_), "witness");
            }
            Nccl& nc = Nccl::get();
            nc.check(nc.Broadcast(d_wit_, d_wit_, 24, ncclUint8, root, comm_, stream_), "broadcast witness");
            check(cudaMemcpyAsync(h, d_wit_, 24, cudaMemcpyDeviceToHost, stream_), "witness");
        }
        check(cudaStreamSynchronize(stream_), "sync");
        State st;
        st.set.w[0] = h[0];
        st.set.w[1] = W == 2 ? h[1] : 0;
        st.history = static_cast<uint32_t>(h[2]);
        return st;
    }
};

}  // namespace

bool shard_active() {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    return s.active();
}

DecideResult shard_decide(const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg, int rounds,
                          const LayerObserver* observer) {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    return s.decide(g, k, forbidden, cfg, rounds, observer);
}

void shard_set_virtual(int G) {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    s.set_virtual(G);
}

void shard_unique_id(unsigned char* out128) {
    Nccl& nc = Nccl::get();
    ncclUniqueId id;
    nc.check(nc.GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof id);
}

void shard_init_nccl(const unsigned char* id128, int rank, int world, int device) {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    s.init_nccl(id128, rank, world, device);
}

void shard_release() {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    s.release();
}

void shard_info(int* world, int* rank, int* virt) {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    s.info(world, rank, virt);
}

void shard_set_mode(int emitter) {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    s.set_mode(emitter);
}

void shard_set_handoff(uint64_t states) {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    s.set_handoff(states);
}

int shard_p2p() {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    return s.p2p();
}

void shard_timer_begin() {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    s.timer_begin();
}

double shard_timer_end() {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    return s.timer_end();
}

void shard_accumulate(KernelTimes& t) {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    s.accumulate(t);
}

void shard_reset_times() {
    ShardSet& s = ShardSet::instance();
    std::lock_guard<std::mutex> lock(s.mu);
    s.reset_counters();
}

}  // namespace etw
