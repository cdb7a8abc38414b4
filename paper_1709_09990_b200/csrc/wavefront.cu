// B200 (sm_100a) wavefront engine: the device replacement for the reference's
// decide / expand_layer / expand_range / q_set / ConcurrentBloom / MMW hot
// path (proj/src/dp.cpp:23-194, graph.hpp:61-78, bloom.cpp:27-125,
// mmw.cpp:20-146) on one GPU. (shard.cu runs the same rounds owner-sharded
// over several GPUs.)
//
// Per round (one BFS layer of the Held-Karp prefix DP) the device runs:
//   exact                  : k_exact_scatter -> k_exact_part -> k_append
//   bloom, filter > 2^28 b : k_exact_scatter<BLOOM> -> k_exact_part<BLOOM> -> k_append
//   bloom, smaller filters : k_bloom_dedup -> k_append
//
//   candidates       (K1, wave_device.cuh) one thread per parent S — one warp
//                    per parent on small layers. The components of G[S] are
//                    flood-filled once with bitmask ops; Q(S,v) for every
//                    candidate is the union of v's outside neighbours and the
//                    outside boundary of every component v touches; with MMW
//                    the surviving children's minor-min-width bounds are
//                    spread over the warp.
//   k_exact_scatter  K1 + every child {key, rank} appended to the bucket of
//                    its key hash (buckets sized so one bucket's distinct
//                    keys fit a shared-memory table).
//   k_exact_part     one CTA per bucket: min emission rank per key in shared
//                    memory (CAS claim + atomicMin), one atomicOr per distinct
//                    key marks its min-rank child in the parent's mask (BLOOM:
//                    the key must first pass the reference's filter).
//   k_bloom_dedup    K1 + the reference's Bloom filter on every child
//                    (32-bit atomicOr on its bit positions, exactly-once
//                    novelty through an epoch-tagged claim table).
//   k_append         single-pass decoupled look-back scan over tiles of 2048
//                    parents; marked children are written in rank order
//                    (parent index major, vertex minor) so exact mode
//                    reproduces the reference's sorted-by-first-emission layer
//                    byte for byte (dp.cpp:140-157), including truncation at
//                    the capacity wall.
//
// All per-round sizes live in device memory (Control), so the host enqueues
// rounds without synchronising; it checks the control block once per chunk.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cub/block/block_scan.cuh>
#include <mutex>
#include <string>

#include "engine.hpp"
#include "wave_device.cuh"

namespace etw {

namespace {

struct RoundStats {
    u64 expanded, offered, unique, emitted, mmw_pruned;
    u64 ticket;  // tile ticket of the round's scan pass
    u64 winners;  // exact mode: children left after the tile pre-dedup
    u64 np;       // exact mode: partitions of the round (power of two)
    u64 pcap;     // exact mode: record capacity per partition
    u64 probed;   // partitioned Bloom: distinct keys sent through the filter
    u64 fp;       // partitioned Bloom: of those, rejected by the filter (false positives)
    unsigned overflowed, valid;
    unsigned compact, nb;  // exact mode: 8-byte records this round (PartPlan)
    unsigned gtab, pad4;   // exact mode: global-table round (PartPlan::gtab; pcap = table slots)
};

enum AbortCode : unsigned {
    kOk = 0,
    kGrowLayer = 1,    // next layer does not fit the layer buffers
    kGrowBloom = 3,    // Bloom filter words
    kGrowClaims = 4,   // Bloom claim table slots
    kGrowParts = 5,    // a partition's distinct keys overflowed its shared table
    kGrowRecs = 6,     // a partition's records overflowed its capacity
    kGrowPartBuf = 7,  // record buffer / cursor array too small for the plan
    kGrowTable = 8,    // a global-table probe chain ran out (raise tab_floor)
};

struct Control {
    u64 count[2];       // layer sizes, ping-pong by round parity
    u64 need;           // size requested by an abort
    unsigned round;     // next round to run
    unsigned stop;      // 1 once a layer came out empty or all rounds ran
    unsigned abort;     // AbortCode
    unsigned epoch;     // look-back tag of the current round attempt (never 0)
    unsigned exits;     // CTAs that finished the round's last pass
    unsigned pad;
    u64 handoff_above;  // >0: stop (handed = 1) once a layer exceeds this many states
    unsigned handed, pad2;
    u64 part_floor;     // exact mode: minimum partitions after a grow (per decide)
    u64 rec_floor;      // exact mode: minimum records per partition after a grow
    u64 tab_floor;      // exact mode: minimum global-table slots after a probe overflow
    unsigned passes;    // exact mode: hash-range passes per round (host-set, >= 1)
    unsigned pass;      // current pass of the round (k_pass_advance; reset by the append)
    unsigned fp_log_n;  // ETWG_DEBUG 2048: first false positives logged (key, h1, h2, m)
    unsigned pad3;
    u64 fp_log[16][4];
    RoundStats rs[kMaxRounds];
};

struct Bufs {
    u64* keys[2];
    unsigned* hist[2];
    u64* cmask;
    u64* recs;          // exact mode: partitioned child records {key.., rank}
    unsigned* cursors;  // exact mode: per-partition record counts (zero between rounds)
    unsigned* bloom[2];  // two filters, alternating by round parity
    unsigned* locks;
    u64* tiles;
    u64 layer_cap;   // states per layer buffer
    u64 rec_cap;     // records
    u64 cursor_cap;  // partitions
    u64 bloom_cap;   // 32-bit words
    u64* claims;     // Bloom-mode claim table, 16-byte {key, epoch} slots
    u64 claim_cap;   // slots
    u64* tab;        // exact mode: global {key, ~min rank} table (empty between rounds)
    u64 tab_cap;     // slots
};

// Bucket cursors sit kCursorStride words apart: the L2's atomic unit
// serialises atomics to one cache line, and ~200 K cursors packed 32 per
// 128-byte line put ten-odd thousand emissions per round behind each line.
#ifndef ETWG_CURSOR_STRIDE
#define ETWG_CURSOR_STRIDE 1
#endif
constexpr u64 kCursorStride = ETWG_CURSOR_STRIDE;
__device__ __forceinline__ unsigned* cursor_at(const Bufs& B, u64 part) { return B.cursors + part * kCursorStride; }

__device__ __forceinline__ bool halted(const Control* C) {
    return (*reinterpret_cast<const volatile unsigned*>(&C->stop) |
            *reinterpret_cast<const volatile unsigned*>(&C->abort)) != 0;
}

// ----------------------------------------------------------------------
// Exact dedup, partitioned (replaces the sort / unique / rank sort of the
// exact branch, dp.cpp:118-157). A round touches each child key through a
// global hash table only at random addresses — on a 10^9-child round that is
// ~150 B of DRAM traffic per child. Instead the children are hash-partitioned
// into record buckets small enough that each bucket's distinct keys fit a
// shared-memory table:
//   k_exact_scatter  K1 per tile of parents + tile pre-dedup; every tile
//                    winner appends {key, rank} to bucket hash(key) >> (64-lg)
//                    and the parent's winner mask is cleared;
//   k_exact_part     one CTA per bucket: min emission rank per key in shared
//                    memory, then one atomicOr per distinct key marks its
//                    min-rank child in the parent's winner mask;
//   k_append<W>      writes the marked children in rank order.
// Bucket count and capacity are planned on the device from the previous
// round's growth; an overflow aborts the round and raises the floor.

#ifndef ETWG_SCATTER_COMPACT
#define ETWG_SCATTER_COMPACT false  // vertex-indexed boundary table (rank order keeps it L1-friendly)
#endif
#ifndef ETWG_APPEND_MINB
#define ETWG_APPEND_MINB 4  // k_append: >= 4 resident CTAs per SM (registers <= 64)
#endif
#ifndef ETWG_EMIT_FLAT
#define ETWG_EMIT_FLAT 0  // 1: children flattened over the warp's lanes; 0: each lane emits its own (-0.8 %)
#endif
#ifndef ETWG_PART_TMA
#define ETWG_PART_TMA 1  // 1: k_exact_part_tma (cp.async.bulk staging) for exact rounds of one-word keys
#endif
#ifndef ETWG_LANE_UNROLL
#define ETWG_LANE_UNROLL 2  // children per lane whose bucket-cursor atomics are in flight together
#endif
#ifndef ETWG_COMPACT
#define ETWG_COMPACT 0  // 1: 8-byte records on every eligible round (see PartPlan)
#endif
#ifndef ETWG_EMIT_UNROLL
#define ETWG_EMIT_UNROLL 2  // children emitted per lane per step in k_exact_scatter
#endif
#ifndef ETWG_PART_BATCH
#define ETWG_PART_BATCH 4  // records loaded per thread before probing (k_exact_part)
#endif
#ifndef ETWG_PART_DIV
#define ETWG_PART_DIV 4  // table slots per targeted distinct key (3: +0.6 %, 5: +1.3 % per solve)
#endif

template <int W>
constexpr int part_slots() { return W == 1 ? 4096 : 2048; }
template <int W>
constexpr int part_target() { return part_slots<W>() / ETWG_PART_DIV; }  // distinct keys aimed for per bucket
template <int W>
constexpr int rec_words() { return W == 1 ? 2 : 4; }  // {key, rank} / {lo, hi, rank, pad}
template <int W>
constexpr int part_smem_bytes() { return part_slots<W>() * (8 * W + 8); }

__device__ __forceinline__ u64 ceil_pow2(u64 x) {
    u64 s = 1;
    while (s < x) s <<= 1;
    return s;
}

// Compact 8-byte records (n <= 64, one-word keys). The key is replaced by an
// n-bit bijective mix m = mixn(key); the bucket is the top lg bits of m, so a
// record only carries the low nb = n - lg bits of m plus the 32-bit parent
// index: {low << 32 | parent}. Among emissions of one key the minimum
// emission rank idx*64+v (dp.cpp:66) is the minimum parent index (one key
// comes at most once from each parent), so the parent index is the rank; v
// is recovered as the one bit of key \ S[parent] when the winner is marked.
// Needs nb <= 31 (the 32-bit table key 0xFFFFFFFF means empty) and layers
// below 2^32 states; other rounds keep the 16-byte {key, rank} records.
constexpr u64 kMixC1 = 0xff51afd7ed558ccdULL;
constexpr u64 kMixC2 = 0xc4ceb9fe1a85ec53ULL;
__host__ __device__ constexpr u64 inv_odd(u64 c) {
    u64 x = c;  // Newton: x <- x (2 - c x) doubles the correct low bits
    for (int i = 0; i < 6; ++i) x *= 2 - c * x;
    return x;
}
constexpr u64 kMixC1inv = inv_odd(kMixC1);
constexpr u64 kMixC2inv = inv_odd(kMixC2);
static_assert(kMixC1 * kMixC1inv == 1 && kMixC2 * kMixC2inv == 1, "modular inverses");

__device__ __forceinline__ u64 nmask(int n) { return n >= 64 ? ~u64{0} : (u64{1} << n) - 1; }

// x ^= x >> s with 2s >= n is an involution on n-bit values
__device__ __forceinline__ u64 mixn(u64 x, int n) {
    const int s = (n + 1) >> 1;
    const u64 m = nmask(n);
    x ^= x >> s;
    x = (x * kMixC1) & m;
    x ^= x >> s;
    x = (x * kMixC2) & m;
    x ^= x >> s;
    return x;
}

__device__ __forceinline__ u64 unmixn(u64 x, int n) {
    const int s = (n + 1) >> 1;
    const u64 m = nmask(n);
    x ^= x >> s;
    x = (x * kMixC2inv) & m;
    x ^= x >> s;
    x = (x * kMixC1inv) & m;
    x ^= x >> s;
    return x;
}

constexpr int kCompactSlots = 4096;  // 32-bit key + 32-bit parent per slot: 32 KB
constexpr int compact_smem_bytes() { return kCompactSlots * 8; }

struct PartPlan {
    u64 np, cap;
    int lg;
    int compact;  // 8-byte records this round
    int nb;       // bits of the mixed key a compact record carries (n - lg)
    // Hash-range passes (records beyond HBM): pass p of `passes` handles the
    // buckets with part % passes == p; K1 reruns per pass, records of one
    // pass only are held, so the record buffer is np/passes * cap.
    unsigned passes, pass;
    int lgp;  // log2(passes)
    // Global-table rounds (exact, one-word keys, the round's table fits
    // 2^P->gtab slots, i.e. stays L2-resident): no buckets; every child goes
    // straight into an open-addressing {key, ~min rank} table of `cap` slots
    // (a power of two) in B.tab; np = passes, so `part` is only the pass
    // selector. Larger rounds keep the bucket records: random 16-byte probes
    // into a multi-GB table measured 1.59 s vs 1.03 s per G(48,0.2) solve.
    int gtab;
    __device__ __forceinline__ bool mine(u64 part) const { return (part & (passes - 1)) == pass; }
    __device__ __forceinline__ u64 local(u64 part) const { return part >> lgp; }
};

template <int W>
__device__ __forceinline__ PartPlan part_plan(const Params* P, const Control* C, unsigned r, u64 E, u64 B_tab_cap) {
    const u64 upper = E * static_cast<u64>(P->free_count > 0 ? P->free_count : 1);
    u64 distinct = upper, winners = upper;
    if (r > 0 && C->rs[r - 1].expanded) {
        const double e = static_cast<double>(E) / static_cast<double>(C->rs[r - 1].expanded);
        const u64 d = static_cast<u64>(e * static_cast<double>(C->rs[r - 1].unique) * 1.25) + 64;
        const u64 w = static_cast<u64>(e * static_cast<double>(C->rs[r - 1].winners) * 1.25) + 64;
        distinct = d < upper ? d : upper;
        winners = w < upper ? w : upper;
    }
    const bool tight = (P->flags & 1024) != 0;  // tests: undersized plans force aborts / re-runs
    PartPlan pl;
    pl.np = ceil_pow2((distinct + part_target<W>() - 1) / part_target<W>());
    if (tight) pl.np = pl.np > 16 ? pl.np / 16 : 1;
    if (pl.np < C->part_floor) pl.np = C->part_floor;
    pl.lg = 0;
    while ((u64{1} << pl.lg) < pl.np) ++pl.lg;
    pl.compact = 0;
    pl.nb = 0;
    // compact records: ETWG_COMPACT=1 at build time or ETWG_DEBUG 8192; off by
    // default (measured on G(48,0.2): 1.054 s vs 1.033 s with 16-byte records —
    // the per-distinct-key read of the parent set costs more than the halved
    // record traffic saves)
    if (W == 1 && (ETWG_COMPACT || (P->flags & 8192)) && E <= 0xFFFFFFFFull) {
        // up to 4x the planned buckets to bring the record's key bits to 31
        const int need = P->n - 31 > pl.lg ? P->n - 31 : pl.lg;
        if (need - pl.lg <= 2) {
            pl.np <<= need - pl.lg;
            pl.lg = need;
            pl.compact = 1;
            pl.nb = P->n - pl.lg;
        }
    }
    pl.passes = C->passes ? C->passes : 1;
    pl.pass = C->pass;
    if (pl.np < pl.passes) {
        pl.lg += __ffs(static_cast<int>(pl.passes)) - 1 - (__ffsll(static_cast<long long>(pl.np)) - 1);
        pl.np = pl.passes;
        if (pl.compact) pl.nb = P->n - pl.lg;
    }
    pl.lgp = __ffs(static_cast<int>(pl.passes)) - 1;
    pl.gtab = 0;
    if (W == 1 && P->gtab) {
        // load factor <= 1/2 on the planned distinct keys of this pass; a
        // probe chain past kTabProbes aborts the round and raises tab_floor
        const u64 per_pass = (distinct + pl.passes - 1) / pl.passes;
        u64 t = ceil_pow2(2 * per_pass);
        if (tight) t = t > 256 ? t / 16 : 16;
        if (t < 16) t = 16;
        while (t < C->tab_floor) t <<= 1;
        if (t <= (u64{1} << P->gtab) && t <= B_tab_cap) {
            pl.gtab = 1;
            pl.compact = 0;
            pl.nb = 0;
            pl.np = pl.passes;
            pl.lg = pl.lgp;
            pl.cap = t;
            return pl;
        }
    }
    const u64 per = (winners + pl.np - 1) / pl.np;
    pl.cap = tight ? per / 4 + 1 : per + per / 4 + 64;
    if (pl.cap < C->rec_floor) pl.cap = C->rec_floor;
    return pl;
}

template <int W>
__device__ __forceinline__ u64 part_of(const Set<W>& key, int lg) {
    return lg ? slot_hash<W>(key) >> (64 - lg) : 0;
}

// Bucket of a child, and (compact rounds) the record's mixed-key low bits.
template <int W>
__device__ __forceinline__ u64 record_part(const Set<W>& key, const PartPlan& pl, int n, u64& low) {
    if (W == 1 && pl.compact) {
        const u64 m = mixn(key.w[0], n);
        low = m & nmask(pl.nb);
        return pl.nb >= 64 ? 0 : m >> pl.nb;
    }
    low = 0;
    return part_of<W>(key, pl.lg);
}

template <int W>
__device__ __forceinline__ void record_store(const Bufs& B, const PartPlan& pl, u64 part, unsigned slot,
                                             const Set<W>& key, u64 low, u64 parent, int v) {
    const u64 lp = pl.local(part);
    if (W == 1 && pl.compact) {
        B.recs[lp * pl.cap + slot] = (low << 32) | parent;
        return;
    }
    u64* rec = B.recs + (lp * pl.cap + slot) * rec_words<W>();
    if constexpr (W == 1) {
        *reinterpret_cast<ulonglong2*>(rec) = make_ulonglong2(key.w[0], child_rank<W>(parent, v));
    } else {
        *reinterpret_cast<ulonglong4*>(rec) = make_ulonglong4(key.w[0], key.w[1], child_rank<W>(parent, v), 0);
    }
}


// Emission of one parent's children by its own lane (the default scatter
// emission): two bucket-cursor atomics in flight per lane, one 16-byte record
// per child, `full` set when a bucket is out of room.
template <int W>
__device__ __forceinline__ void emit_lane(const Bufs& B, const PartPlan& pl, int n, const Set<W>& S,
                                          const Set<W>& M, u64 idx, bool& full, int diag = 0) {
    Set<W> rest = M;
    if (diag == 1 || diag == 2) {
        // diagnostics (ETWG_DEBUG 32768 / 65536, last round of a decide,
        // results invalid): the same records without the cursor atomic's
        // return — 1: slot from a per-lane sequence, no atomic; 2: the
        // cursor bumped by a fire-and-forget RED, slot from the sequence
        unsigned seq = static_cast<unsigned>(idx * 0x9E3779B1u);
        while (rest.any()) {
            const int v = pop_any(rest);
            Set<W> key = S;
            key.add(v);
            u64 low;
            const u64 part = record_part<W>(key, pl, n, low);
            if (!pl.mine(part)) continue;
            if (diag == 2) atomicAdd(cursor_at(B, part), 1u);  // result unused: RED
            const unsigned slot = (seq += 0x61C88647u) % static_cast<unsigned>(pl.cap);
            record_store<W>(B, pl, part, slot, key, low, idx, v);
        }
        return;
    }
    constexpr int LU = ETWG_LANE_UNROLL;
    while (rest.any()) {
        Set<W> key[LU];
        u64 part[LU], low[LU];
        int vv[LU];
        unsigned slot[LU];
#pragma unroll
        for (int u = 0; u < LU; ++u) slot[u] = ~0u;
#pragma unroll
        for (int u = 0; u < LU; ++u) {
            if (!rest.any()) break;
            vv[u] = pop_any(rest);
            key[u] = S;
            key[u].add(vv[u]);
            part[u] = record_part<W>(key[u], pl, n, low[u]);
            if (pl.mine(part[u])) slot[u] = atomicAdd(cursor_at(B, part[u]), 1u);
        }
        if (diag == 3) {  // diagnostics: a second returning atomic per record (to another cursor)
#pragma unroll
            for (int u = 0; u < LU; ++u)
                if (slot[u] != ~0u &&
                    atomicAdd(cursor_at(B, (part[u] + (pl.np >> 1) + 17) & (pl.np - 1)), 0u) == 0xFFFFFFFFu)
                    full = true;  // (a cursor in another line)
        }
#pragma unroll
        for (int u = 0; u < LU; ++u) {
            if (slot[u] == ~0u) continue;
            if (slot[u] < pl.cap)
                record_store<W>(B, pl, part[u], slot[u], key[u], low[u], idx, vv[u]);
            else
                full = true;
        }
    }
}

// Global-table emission (PartPlan::gtab): slot = {key, ~rank}, key 0 =
// empty (a child is never the empty set), the inverted rank so that an
// all-zero slot is "no rank yet" and the minimum rank is an atomicMax.
// Linear probing from slot_hash & (cap-1); a 32-byte sector holds two slots.
// The first slot of each of ETWG_TAB_UNROLL children is loaded (L2 only)
// before any is resolved, so the lane has that many random reads in flight;
// a slot that already holds the key with a lower rank costs no atomic.
#ifndef ETWG_TAB_UNROLL
#define ETWG_TAB_UNROLL 2  // 4: 127 registers (80 at 2), slower
#endif
#ifndef ETWG_GTAB_LG
#define ETWG_GTAB_LG 22  // global table up to 2^22 slots = 64 MB (L2 is 126 MB)
#endif
constexpr int kGtabLg = ETWG_GTAB_LG;
constexpr int kTabProbes = 64;

__device__ __forceinline__ void tab_settle(ulonglong2* tab, u64 mask, u64 key, u64 inv, u64 s, ulonglong2 cur,
                                           bool& full) {
    for (int p = 0;;) {
        u64 k = cur.x;
        if (k == 0) {
            k = atomicCAS(reinterpret_cast<unsigned long long*>(&tab[s].x), 0ull, key);
            if (k == 0) k = key;
        }
        if (k == key) {
            if (cur.y < inv) atomicMax(reinterpret_cast<unsigned long long*>(&tab[s].y), inv);
            return;
        }
        if (++p == kTabProbes) {
            full = true;
            return;
        }
        s = (s + 1) & mask;
        cur = __ldcg(tab + s);
    }
}

__device__ __forceinline__ void emit_lane_tab(const Bufs& B, const PartPlan& pl, u64 S, u64 M, u64 idx,
                                              bool& full) {
    ulonglong2* tab = reinterpret_cast<ulonglong2*>(B.tab);
    const u64 mask = pl.cap - 1;
    constexpr int LU = ETWG_TAB_UNROLL;
    while (M) {
        u64 key[LU], inv[LU], s[LU];
        ulonglong2 cur[LU];
        bool act[LU];
#pragma unroll
        for (int u = 0; u < LU; ++u) {
            act[u] = false;
            if (!M) continue;
            const int v = __ffsll(static_cast<long long>(M)) - 1;
            M &= M - 1;
            key[u] = S | (u64{1} << v);
            const u64 h = fmix64(key[u]);  // slot_hash<1>
            if (!pl.mine(pl.lg ? h >> (64 - pl.lg) : 0)) continue;
            act[u] = true;
            inv[u] = ~child_rank<1>(idx, v);
            s[u] = h & mask;
            cur[u] = __ldcg(tab + s[u]);
        }
#pragma unroll
        for (int u = 0; u < LU; ++u)
            if (act[u]) tab_settle(tab, mask, key[u], inv[u], s[u], cur[u], full);
    }
}

// mbarrier helpers (shared::cta) for the warp-specialised scatter
__device__ __forceinline__ void mbar_init(u64* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
                 "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, unsigned parity) {
    // (a try_wait suspend-time hint, CUTLASS-style, measured no change: 0.995 vs 0.995 s)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WSWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WSWAIT_%=;\n\t}" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
        "r"(parity)
        : "memory");
}

#ifndef ETWG_WS
#define ETWG_WS 1  // warp-specialised scatter: K1 warps feed emission warps through shared memory
#endif
#ifndef ETWG_SWAP_PAIR
#define ETWG_SWAP_PAIR 1  // producer iterations take adjacent tile pairs: 64-parent swap window (0: one tile)
#endif
#ifndef ETWG_SWAP_CTA
#define ETWG_SWAP_CTA 0  // 1: the swap test spans the CTA's kWsProd producer tiles (128 parents)
#endif
#ifndef ETWG_WS_PROD
#define ETWG_WS_PROD 4  // producer warps per CTA; the other warps consume, kWsCpp per producer
#endif
constexpr int kWsProd = ETWG_WS_PROD;
constexpr int kWsCpp = (kThreads / 32 - kWsProd) / kWsProd;  // consumer warps per producer
constexpr int kWsRing = 2 * kWsCpp;                           // shared slots per producer
static_assert(kWsProd * (1 + kWsCpp) == kThreads / 32, "warp roles must fill the CTA");

#ifndef ETWG_SCATTER_MINB
#define ETWG_SCATTER_MINB 0  // >0: resident CTAs per SM asked of ptxas for the scatter instantiations other than the bucket-only exact one
#endif

// GT: 0 = this instantiation runs every round (both emission paths
// compiled in); 1 = bucket rounds only, 2 = global-table rounds only (the
// exact one-word instantiations: the host launches both, the plan picks,
// the other returns at once — with both emission paths in one kernel ptxas
// allocated 80 registers instead of 64, one resident CTA per SM less).
// The bucket-only exact instantiation is held to 64 registers (4 CTAs per
// SM): with the tile-pair swap window ptxas otherwise takes 79 (measured
// 0.911 vs 0.921 s per G48 solve with the cap).
template <int W, bool MMW, bool BLOOM, int GT = 0>
__global__ void __launch_bounds__(kThreads, (W == 1 && !MMW && !BLOOM && GT != 0) ? 4 : (ETWG_SCATTER_MINB > 0 ? ETWG_SCATTER_MINB : 2))
k_exact_scatter(const Params* __restrict__ P, Control* C,
                                                            Bufs B) {
    __shared__ Set<W> adj[64 * W];
    __shared__ unsigned mmw_keep[MMW ? kThreads : 1][2 * W];

    __shared__ Set<W> warp_tables[kThreads / 32][MMW ? 2 : 1][64 * W];  // small-layer mode
    if (halted(C)) return;
    const unsigned r = C->round;
    const u64 E = C->count[r & 1];
    const PartPlan pl = part_plan<W>(P, C, r, E, B.tab_cap);
    if ((GT == 1 && pl.gtab) || (GT == 2 && !pl.gtab)) return;
    const bool gt = GT == 2 ? true : GT == 1 ? false : pl.gtab != 0;  // compile-time where GT fixes it
    const u64 rec_need = pl.gtab ? 0 : (pl.np >> pl.lgp) * pl.cap * (W == 1 && pl.compact ? 1 : rec_words<W>());  // u64 words
    if (pl.np > B.cursor_cap || rec_need > B.rec_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            C->need = rec_need;
            C->abort = kGrowPartBuf;
        }
        return;
    }
    if constexpr (BLOOM) {
        // partitioned Bloom round: a fresh filter of the reference's size per
        // round (dp.cpp:93-94), ping-pong by parity; the filter of round r-1
        // is cleared here for round r+1
        const u64 m = bloom_bits_for(round_cap(*P, E), P->bpe);
        if (m / 32 + 1 > B.bloom_cap) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                C->need = m / 32 + 1;
                C->abort = kGrowBloom;
            }
            return;
        }
        if (r > 0 && pl.pass == 0) {
            const u64 gtid = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
            const u64 gstride = static_cast<u64>(gridDim.x) * blockDim.x;
            const u64 prev_words = bloom_bits_for(round_cap(*P, C->rs[r - 1].expanded), P->bpe) / 32 + 1;
            uint4* w4 = reinterpret_cast<uint4*>(B.bloom[(r + 1) & 1]);
            const u64 n4 = prev_words / 4;
            for (u64 i = gtid; i < n4; i += gstride) w4[i] = make_uint4(0, 0, 0, 0);
            for (u64 i = n4 * 4 + gtid; i < prev_words; i += gstride) B.bloom[(r + 1) & 1][i] = 0;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        C->rs[r].np = pl.np;
        C->rs[r].pcap = pl.cap;
        C->rs[r].compact = pl.compact;
        C->rs[r].nb = pl.nb;
        C->rs[r].gtab = pl.gtab;
    }
    const int n = P->n;
    const int lane = threadIdx.x & 31;
    const Set<W> forbidden = param_set<W>(P->forbidden);
    const u64* in = B.keys[r & 1];
    load_adjacency<W>(P, adj);
    __syncthreads();
    // warp-granular: no block barrier inside the loop, so a warp whose
    // parents are cheap never waits for the CTA's slowest warp
    const u64 nwarps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    u64 offered = 0, pruned = 0, winners = 0;
    // Small layer (fewer than 1/8 of the resident threads): one warp per
    // parent, candidates and MMW bounds spread over the lanes.
    const bool small = (P->flags & 256) || (!(P->flags & 128) && E * 8 <= static_cast<u64>(gridDim.x) * blockDim.x);
    if (ETWG_WS && W == 1 && !MMW && !small) {
        // Warp specialisation (measured: K1 alone is ~46 % of this kernel,
        // the bucket scatter the rest, and in one warp they serialise). A
        // producer warp runs K1 for 32 consecutive parents and puts
        // (S, child mask) into the next slot of its ring; its consumer warps
        // take slots in turn, release them and emit the children (atomics +
        // stores) while the producer already evaluates the next 32 parents.
        // full/empty handshakes on mbarriers.
        __shared__ u64 ws_S[kWsProd][kWsRing][32], ws_M[kWsProd][kWsRing][32], ws_base[kWsProd][kWsRing];
        __shared__ __align__(8) u64 ws_bar[kWsProd][kWsRing][2];  // [producer][slot][full, empty]
        const int warp = threadIdx.x >> 5;
        // producer p = warp < kWsProd; consumer warp kWsProd + p*kWsCpp + c
        // takes producer p's tiles t with t % kWsCpp == c (slot t % kWsRing)
        const int pair = warp < kWsProd ? warp : (warp - kWsProd) / kWsCpp;
        const int role = warp < kWsProd ? 0 : (warp - kWsProd) % kWsCpp;
        for (int i = threadIdx.x; i < kWsProd * kWsRing * 2; i += blockDim.x) mbar_init(&ws_bar[0][0][0] + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncthreads();
        const u64 producers = static_cast<u64>(gridDim.x) * kWsProd;
        const u64 me = static_cast<u64>(blockIdx.x) * kWsProd + pair;
        if (warp < kWsProd) {
            // slot of tile t is free once the consumer of tile t - kWsRing released it
            auto acquire = [&](unsigned t) {
                if (t >= static_cast<unsigned>(kWsRing))
                    mbar_wait(&ws_bar[pair][t % kWsRing][1], ((t / kWsRing) - 1) & 1u);
            };
            // ETWG_SWAP_CTA: the CTA's producers hold kWsProd consecutive tiles
            // per iteration (tiles blockIdx*kWsProd + p + it*producers); they
            // share (S, M) through shared memory on a producer-only named
            // barrier, so the swap test spans 32*kWsProd consecutive parents.
            // Their stop decision must then be uniform: the group's first tile
            // and an abort flag sampled by producer 0 before the barrier.
            __shared__ u64 sw_S[ETWG_SWAP_CTA ? 2 : 1][kWsProd][32], sw_M[ETWG_SWAP_CTA ? 2 : 1][kWsProd][32];
            __shared__ unsigned sw_stop[2];
            if (ETWG_SWAP_CTA && threadIdx.x < 2) sw_stop[threadIdx.x] = 0;
            if (ETWG_SWAP_CTA) asm volatile("bar.sync 1, %0;" ::"n"(kWsProd * 32) : "memory");
            // ETWG_SWAP_PAIR: iterations 2q, 2q+1 take two adjacent tiles, so
            // the odd one also tests against the even one's 32 parents
            u64 prevS = 0, prevM = 0;
            for (unsigned it = 0;; ++it) {
                const int b = it % kWsRing;
                acquire(it);
                const u64 base = ETWG_SWAP_PAIR ? ((me + (it >> 1) * producers) * 2 + (it & 1)) * 32
                                                : (me + it * producers) * 32;
                const bool done =
                    ETWG_SWAP_CTA
                        ? (static_cast<u64>(blockIdx.x) * kWsProd + it * producers) * 32 >= E ||
                              *reinterpret_cast<volatile unsigned*>(&sw_stop[it & 1]) != 0
                        : base >= E || *reinterpret_cast<volatile unsigned*>(&C->abort) != 0;
                if (done) {  // one end marker per consumer: tiles it .. it + kWsCpp - 1
                    for (unsigned u = it; u < it + kWsCpp; ++u) {
                        if (u != it) acquire(u);
                        if (lane == 0) {
                            ws_base[pair][u % kWsRing] = ~u64{0};
                            mbar_arrive(&ws_bar[pair][u % kWsRing][0]);
                        }
                    }
                    break;
                }
                const u64 idx = base + lane;
                const bool valid = idx < E;
                const Set<W> S = valid ? load_set<W>(in, idx) : Set<W>::zero();
                Set<W> M;
                if ((P->flags & 131072) && static_cast<int>(r) + 1 == P->rounds) {
                    // diagnostics (results invalid): no K1 — about half of the
                    // open vertices as pseudo-random children, ~ the real
                    // child count, to time the emission alone
                    M = Set<W>::zero();
                    if (valid) M.w[0] = nmask(P->n) & ~S.w[0] & fmix64(S.w[0] ^ 0x5bd1e995u);
                } else {
                    M = warp_candidates<W, MMW, ETWG_SCATTER_COMPACT>(adj, P->n, P->k, S, valid, forbidden, pruned,
                                                                      mmw_keep);
                }
                const int offered_here = M.count();
                if (ETWG_SWAP_DEDUP) {
                    // Sibling swap pre-dedup: parents i < j of this tile with
                    // S_i ^ S_j = {v, w} (v in S_j, w in S_i) share the child
                    // S_i | S_j, offered by i through v and by j through w. When
                    // both offer it, j's copy can never be the min-rank
                    // emission (rank = idx*64 + vertex, idx_i < idx_j), so j
                    // drops it before it becomes a record; the min-rank copy
                    // of every key survives (the lowest lane never drops it).
                    // Consecutive parents are often siblings (the layer is in
                    // rank order), so this removes records at shuffle cost.
                    const u64 Sm = S.w[0], M0 = M.w[0];
                    u64 drop = 0;
                    if (ETWG_SWAP_CTA) {
                        sw_S[it & 1][pair][lane] = Sm;
                        sw_M[it & 1][pair][lane] = M0;
                        if (pair == 0 && lane == 0)
                            sw_stop[(it + 1) & 1] = *reinterpret_cast<volatile unsigned*>(&C->abort) != 0;
                        asm volatile("bar.sync 1, %0;" ::"n"(kWsProd * 32) : "memory");
                        for (int q = 0; q < pair; ++q) {  // lower producers' tiles: all 32 parents rank lower
#pragma unroll 4
                            for (int d = 0; d < 32; ++d) {
                                const u64 So = sw_S[it & 1][q][d];
                                const u64 Mo = sw_M[it & 1][q][d];
                                const u64 x = So ^ Sm;
                                if (__popcll(x) == 2 && (Mo & x & Sm) != 0) drop |= x & So;
                            }
                        }
                    }
#pragma unroll 4
                    for (int d = 1; d < 32; ++d) {
                        const u64 So = __shfl_up_sync(kFull, Sm, d);
                        const u64 Mo = __shfl_up_sync(kFull, M0, d);
                        const u64 x = So ^ Sm;
                        if (lane >= d && __popcll(x) == 2 && (Mo & x & Sm) != 0) drop |= x & So;
                    }
                    if (ETWG_SWAP_PAIR) {
                        if (it & 1) {  // the even tile's 32 parents all rank lower
#pragma unroll 4
                            for (int d = 0; d < 32; ++d) {
                                const u64 So = __shfl_sync(kFull, prevS, d);
                                const u64 Mo = __shfl_sync(kFull, prevM, d);
                                const u64 x = So ^ Sm;
                                if (__popcll(x) == 2 && (Mo & x & Sm) != 0) drop |= x & So;
                            }
                        } else {
                            prevS = Sm;
                            prevM = M0;
                        }
                    }
                    M.w[0] = M0 & ~drop;
                }
                if (pl.pass == 0) {
                    offered += offered_here;
                    winners += M.count();
                    if (valid) store_set<W>(B.cmask, idx, Set<W>::zero());
                }
                ws_S[pair][b][lane] = S.w[0];
                ws_M[pair][b][lane] = M.w[0];
                if (lane == 0) ws_base[pair][b] = base;
                __syncwarp();
                if (lane == 0) mbar_arrive(&ws_bar[pair][b][0]);
            }
        } else {
            const bool k1_only = (P->flags & 16384) && static_cast<int>(r) + 1 == P->rounds;  // diagnostics
            for (unsigned it = role;; it += kWsCpp) {
                const int b = it % kWsRing;
                mbar_wait(&ws_bar[pair][b][0], (it / kWsRing) & 1u);
                const u64 base = ws_base[pair][b];
                if (base == ~u64{0}) break;
                Set<W> S, M;
                S.w[0] = ws_S[pair][b][lane];
                M.w[0] = ws_M[pair][b][lane];
                __syncwarp();
                if (lane == 0) mbar_arrive(&ws_bar[pair][b][1]);
                bool full = false;
                if (k1_only) {
                } else if (gt) {
                    emit_lane_tab(B, pl, S.w[0], M.w[0], base + lane, full);
                } else {
                    const int diag = static_cast<int>(r) + 1 == P->rounds
                                         ? ((P->flags & 32768) ? 1 : (P->flags & 65536) ? 2 : (P->flags & 262144) ? 3 : 0) : 0;
                    emit_lane<W>(B, pl, n, S, M, base + lane, full, diag);
                }
                if (__any_sync(kFull, full) && lane == 0) {
                    C->need = 2 * pl.cap;
                    C->abort = gt ? kGrowTable : kGrowRecs;
                }
            }
        }
    } else
    if (small) {  // ETWG_DEBUG 128 / 256 force the thread / warp mode (tests)
        Set<W>* R = warp_tables[threadIdx.x >> 5][0];
        Set<W>* rows = warp_tables[threadIdx.x >> 5][MMW ? 1 : 0];
        bool full = false;
        for (u64 p = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 5; p < E; p += nwarps) {
            if (*reinterpret_cast<volatile unsigned*>(&C->abort)) break;
            const Set<W> S = load_set<W>(in, p);
            const Set<W> M = warp_parent_candidates<W, MMW>(adj, P->n, P->k, S, forbidden, pruned, R, rows);
            const int cnt = M.count();
            if (lane == 0 && pl.pass == 0) {  // counters and mask clear once per round, not per pass
                offered += cnt;
                winners += cnt;
                store_set<W>(B.cmask, p, Set<W>::zero());
            }
            for (int i = lane; i < cnt; i += 32) {
                const int v = nth_member<W>(M, i);
                Set<W> key = S;
                key.add(v);
                u64 low;
                if (W == 1 && gt) {
                    emit_lane_tab(B, pl, S.w[0], key.w[0] ^ S.w[0], p, full);
                    continue;
                }
                const u64 part = record_part<W>(key, pl, n, low);
                if (!pl.mine(part)) continue;
                const unsigned slot = atomicAdd(cursor_at(B, part), 1u);
                if (slot < pl.cap)
                    record_store<W>(B, pl, part, slot, key, low, p, v);
                else
                    full = true;
            }
        }
        if (__any_sync(kFull, full) && lane == 0) {
            C->need = 2 * pl.cap;
            C->abort = gt ? kGrowTable : kGrowRecs;
        }
    } else if constexpr (!(ETWG_WS && W == 1 && !MMW)) {  // (dead for warp-specialised instantiations:
                                                          // compiled out so its registers do not count)
    for (u64 base = ((blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 5) * 32; base < E;
         base += nwarps * 32) {
        if (*reinterpret_cast<volatile unsigned*>(&C->abort)) break;  // warp-uniform read
        const u64 idx = base + lane;
        const bool valid = idx < E;
        const Set<W> S = valid ? load_set<W>(in, idx) : Set<W>::zero();
        const Set<W> M =
            warp_candidates<W, MMW, ETWG_SCATTER_COMPACT>(adj, P->n, P->k, S, valid, forbidden, pruned, mmw_keep);
        Set<W> Me = M;  // the children this lane emits
        if constexpr (ETWG_SWAP_DEDUP && W == 1) {  // sibling swap pre-dedup over the warp's 32 parents
            const u64 Sm = S.w[0], M0 = M.w[0];
            u64 drop = 0;
#pragma unroll 4
            for (int d = 1; d < 32; ++d) {
                const u64 So = __shfl_up_sync(kFull, Sm, d);
                const u64 Mo = __shfl_up_sync(kFull, M0, d);
                const u64 x = So ^ Sm;
                if (lane >= d && __popcll(x) == 2 && (Mo & x & Sm) != 0) drop |= x & So;
            }
            Me.w[0] = M0 & ~drop;
        }
        if (pl.pass == 0) {  // counters and mask clear once per round, not per pass
            offered += M.count();
            winners += Me.count();
            if (valid) store_set<W>(B.cmask, idx, Set<W>::zero());
        }
        bool full = false;
        // ETWG_DEBUG 16384 (diagnostics only, results invalid): the decide's
        // last round evaluates its candidates but emits no records — times K1
        // without the bucket scatter
        if ((P->flags & 16384) && static_cast<int>(r) + 1 == P->rounds) continue;
        if (W == 1 && gt) {
            emit_lane_tab(B, pl, S.w[0], Me.w[0], idx, full);
        } else {
#if ETWG_EMIT_FLAT == 0
        emit_lane<W>(B, pl, n, S, Me, idx, full);
#else
        WarpFlat f;
        f.scan(M.count());
        // ETWG_EMIT_UNROLL children per lane per step: their bucket-cursor
        // atomics are in flight together instead of one round trip each
        constexpr int U = ETWG_EMIT_UNROLL;
        for (int t = 0; t < f.total; t += 32 * U) {
            Set<W> key[U];
            u64 part[U], low[U];
            int vv[U], srcs[U];
            unsigned slot[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = t + 32 * u + lane;
                const int src = f.source(j);
                const int excl = __shfl_sync(kFull, f.incl, src) - __shfl_sync(kFull, f.cnt, src);
                const Set<W> Ms = shfl_set<W>(M, src);
                key[u] = shfl_set<W>(S, src);
                slot[u] = ~0u;
                srcs[u] = src;
                if (j < f.total) {
                    vv[u] = nth_member<W>(Ms, j - excl);
                    key[u].add(vv[u]);
                    part[u] = record_part<W>(key[u], pl, n, low[u]);
                    if (pl.mine(part[u])) slot[u] = atomicAdd(cursor_at(B, part[u]), 1u);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (slot[u] == ~0u) continue;
                if (slot[u] < pl.cap)
                    record_store<W>(B, pl, part[u], slot[u], key[u], low[u], base + srcs[u], vv[u]);
                else
                    full = true;
            }
        }
#endif
        }
        if (__any_sync(kFull, full) && lane == 0) {
            C->need = 2 * pl.cap;
            C->abort = gt ? kGrowTable : kGrowRecs;
        }
    }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        offered += __shfl_xor_sync(kFull, offered, o);
        pruned += __shfl_xor_sync(kFull, pruned, o);
        winners += __shfl_xor_sync(kFull, winners, o);
    }
    if (lane == 0) {
        if (offered) atomicAdd(&C->rs[r].offered, offered);
        if (pruned && pl.pass == 0) atomicAdd(&C->rs[r].mmw_pruned, pruned);
        if (winners) atomicAdd(&C->rs[r].winners, winners);
    }
}

// pass p of a hash-range-partitioned round is done: the next scatter / part
// pair takes pass p+1 (the round's append resets it)
__global__ void k_pass_advance(Control* C) {
    if (!halted(C)) C->pass += 1;
}

constexpr int kPartThreads = 512;

// dynamic shared memory of k_exact_scatter<W, false, *> (none: K1's state lives in registers)
template <int W>
constexpr int scatter_smem() { return 0; }

// BLOOM: the round's distinct keys then meet the reference's Bloom filter
// (bit positions (h1 + i*h2) mod m, bloom.cpp:86-97), each exactly once, so
// "any probed bit was clear" is the novelty test; keys the filter calls
// duplicates (false positives) are dropped as the reference drops them.
// ----------------------------------------------------------------------
// k_exact_part_tma (one-word keys, 16-byte records): the same per-bucket
// min-rank dedup as k_exact_part, with each bucket's contiguous records
// staged into shared memory by the Blackwell bulk-copy engine
// (cp.async.bulk, 1D TMA, completion on an mbarrier): two 24 KB stages in
// flight, the next bucket's first two chunks issued before the current
// bucket's mark pass, so no thread waits on a global load. Two 112 KB CTAs
// per SM.
constexpr int kTmaChunk = 1536;  // records per stage (24 KB)
constexpr int kTmaThreads = 512;
constexpr int tma_part_smem_bytes() { return part_smem_bytes<1>() + 2 * kTmaChunk * 16 + 16; }

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, u64* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void bar_wait(u64* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

template <bool BLOOM>
__global__ void __launch_bounds__(kTmaThreads, 2) k_exact_part_tma(const Params* __restrict__ P, Control* C, Bufs B) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int SLOTS = part_slots<1>();
    u64* keys = reinterpret_cast<u64*>(smem_raw);
    u64* ranks = keys + SLOTS;
    u64* stage = ranks + SLOTS;                      // [2][kTmaChunk * 2] u64
    u64* bars = stage + 2 * kTmaChunk * 2;           // 2 mbarriers
    __shared__ unsigned s_full;
    if (halted(C)) return;
    const unsigned r = C->round;
    if (C->rs[r].compact || C->rs[r].gtab) return;
    const u64 passes = C->passes ? C->passes : 1;
    const u64 pass = C->pass;
    const u64 np = C->rs[r].np / passes;
    const u64 cap = C->rs[r].pcap;
    u64 probed = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bars)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bars + 1)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned phases = 0;  // bit st: parity of stage st's next completion (a register, not an array)
    auto count_of = [&](u64 lp) -> unsigned {
        const unsigned c = *cursor_at(B, lp * passes + pass);
        return c < cap ? c : static_cast<unsigned>(cap);
    };
    // issues chunks [c0, c0+k) of local bucket lp into their stages (thread 0)
    auto issue = [&](u64 lp, unsigned cnt, unsigned c0, unsigned k) {
        const u64* recs = B.recs + lp * cap * 2;
        for (unsigned c = c0; c < c0 + k; ++c) {
            const unsigned first = c * kTmaChunk;
            if (first >= cnt) break;
            const unsigned n = min(cnt - first, static_cast<unsigned>(kTmaChunk));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_load(stage + (c & 1) * kTmaChunk * 2, recs + 2 * static_cast<u64>(first), n * 16, bars + (c & 1));
        }
    };
    u64 lp = blockIdx.x;
    if (lp < np && threadIdx.x == 0) issue(lp, count_of(lp), 0, 2);
    // the table is cleared once; each bucket's mark pass empties the slots it used
    for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
        keys[i] = 0;
        ranks[i] = ~u64{0};
    }
    for (; lp < np; lp += gridDim.x) {
        const u64 part = lp * passes + pass;
        const unsigned cnt = count_of(lp);
        if (threadIdx.x == 0) s_full = 0;
        __syncthreads();
        const unsigned nch = (cnt + kTmaChunk - 1) / kTmaChunk;
        for (unsigned c = 0; c < nch; ++c) {
            const int st = c & 1;
            bar_wait(bars + st, (phases >> st) & 1u);
            phases ^= 1u << st;
            const unsigned n = min(cnt - c * kTmaChunk, static_cast<unsigned>(kTmaChunk));
            const u64* sb = stage + st * kTmaChunk * 2;
            for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
                const ulonglong2 rec = *reinterpret_cast<const ulonglong2*>(sb + 2 * i);
                Set<1> key;
                key.w[0] = rec.x;
                const u64 rank = rec.y;
                unsigned h = static_cast<unsigned>(slot_hash<1>(key)) & (SLOTS - 1);
                bool placed = false;
                for (int probe = 0; probe < 128 && !placed; ++probe) {
                    placed = smem_claim<1>(keys, h, key);
                    if (!placed) h = (h + 1) & (SLOTS - 1);
                }
                if (placed && rank < *reinterpret_cast<volatile u64*>(ranks + h))
                    atomicMin(reinterpret_cast<unsigned long long*>(ranks + h), rank);
                if (!placed) s_full = 1;
            }
            __syncthreads();  // stage st consumed by every thread
            if (threadIdx.x == 0 && c + 2 < nch) issue(lp, cnt, c + 2, 1);
        }
        if (s_full) {  // block-uniform; no load is in flight here
            if (threadIdx.x == 0) {
                C->need = 2 * np * passes;
                C->abort = kGrowParts;
            }
            break;
        }
        // both stages free: start the next bucket's loads under this bucket's mark pass
        const u64 nxt = lp + gridDim.x;
        if (threadIdx.x == 0 && nxt < np) issue(nxt, count_of(nxt), 0, 2);
        for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
            const u64 rank = ranks[i];
            if (rank == ~u64{0}) continue;  // never claimed (a claimed slot always got a rank)
            const u64 kw = keys[i];
            keys[i] = 0;  // empty again for the next bucket
            ranks[i] = ~u64{0};
            if constexpr (BLOOM) {
                Set<1> key;
                key.w[0] = kw;
                const u64 m = bloom_bits_for(round_cap(*P, C->count[r & 1]), P->bpe);
                unsigned* bits = B.bloom[r & 1];
                const unsigned h1 = murmur_key<1>(key, kSeed1);
                const unsigned h2 = murmur_key<1>(key, kSeed2);
                u64 pos, step;
                probe_start(h1, h2, m, pos, step);
                ++probed;
                if (!bloom_or_probes(bits, m, pos, step, P->hashes)) {
                    atomicAdd(&C->rs[r].fp, 1ull);
                    continue;
                }
            }
            const u64 parent = rank / 64;
            const int v = static_cast<int>(rank % 64);
            atomicOr(reinterpret_cast<unsigned long long*>(B.cmask) + parent, u64{1} << v);
        }
        if (threadIdx.x == 0) *cursor_at(B, part) = 0;
        __syncthreads();
    }
    if (BLOOM) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) probed += __shfl_xor_sync(kFull, probed, o);
        if ((threadIdx.x & 31) == 0 && probed) atomicAdd(&C->rs[r].probed, probed);
    }
}

// Global-table rounds: one streaming pass over the pass's table marks each
// key's min-rank child in its parent's winner mask (what k_exact_part does
// per bucket) and leaves every slot empty for the next round / pass.
__global__ void __launch_bounds__(kThreads) k_tab_mark(Control* C, Bufs B) {
    if (halted(C)) return;
    const unsigned r = C->round;
    if (!C->rs[r].gtab) return;  // a bucket round: k_exact_part* runs it
    const u64 slots = C->rs[r].pcap;
    ulonglong2* tab = reinterpret_cast<ulonglong2*>(B.tab);
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < slots; i += stride) {
        const ulonglong2 e = __ldcs(tab + i);
        if (e.x == 0) continue;
        const u64 rank = ~e.y;
        atomicOr(reinterpret_cast<unsigned long long*>(B.cmask) + rank / 64, u64{1} << (rank % 64));
        tab[i] = make_ulonglong2(0, 0);
    }
}

template <int W, bool BLOOM>
__global__ void __launch_bounds__(kPartThreads) k_exact_part(const Params* __restrict__ P, Control* C, Bufs B) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int SLOTS = part_slots<W>();
    u64* keys = reinterpret_cast<u64*>(smem_raw);
    u64* ranks = keys + SLOTS * W;
    __shared__ unsigned s_full;
    if (halted(C)) return;
    const unsigned r = C->round;
    if (W == 1 && (C->rs[r].compact || C->rs[r].gtab)) return;  // k_exact_part_compact's / k_tab_mark's round
    const u64 passes = C->passes ? C->passes : 1;
    const u64 pass = C->pass;
    const u64 np = C->rs[r].np / passes;  // this pass's buckets: part = lp * passes + pass
    const u64 cap = C->rs[r].pcap;
    u64 probed = 0;  // BLOOM: distinct keys sent through the filter (one atomic per thread at exit)
    // the table is cleared once; each bucket's mark pass empties the slots it used
    for (int i = threadIdx.x; i < SLOTS * W; i += blockDim.x) keys[i] = 0;
    for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) ranks[i] = ~u64{0};
    for (u64 lp = blockIdx.x; lp < np; lp += gridDim.x) {
        const u64 part = lp * passes + pass;
        if (threadIdx.x == 0) s_full = 0;
        __syncthreads();
        const unsigned cnt = *cursor_at(B, part);
        const u64* recs = B.recs + lp * cap * rec_words<W>();
        // PART_BATCH records in flight per thread before any probing: one
        // outstanding 16 B load per thread cannot cover HBM latency at the
        // 3 CTAs/SM the 64 KB tables allow
        constexpr int kBatch = ETWG_PART_BATCH;
        for (unsigned base = threadIdx.x; base < cnt; base += kBatch * blockDim.x) {
            Set<W> keyv[kBatch];
            u64 rankv[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const unsigned i = base + j * blockDim.x;
                if (i >= cnt) break;
                if constexpr (W == 1) {
                    const ulonglong2 rec = __ldcs(reinterpret_cast<const ulonglong2*>(recs) + i);
                    keyv[j].w[0] = rec.x;
                    rankv[j] = rec.y;
                } else {
                    const ulonglong2 k2 = __ldcs(reinterpret_cast<const ulonglong2*>(recs) + 2 * i);
                    const ulonglong2 r2 = __ldcs(reinterpret_cast<const ulonglong2*>(recs) + 2 * i + 1);
                    keyv[j].w[0] = k2.x;
                    keyv[j].w[1] = k2.y;
                    rankv[j] = r2.x;
                }
            }
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                if (base + j * blockDim.x >= cnt) break;
                const Set<W>& key = keyv[j];
                const u64 rank = rankv[j];
                unsigned h = static_cast<unsigned>(slot_hash<W>(key)) & (SLOTS - 1);
                bool placed = false;
                for (int probe = 0; probe < 128 && !placed; ++probe) {
                    placed = smem_claim<W>(keys, h, key);
                    if (!placed) h = (h + 1) & (SLOTS - 1);
                }
                // ranks only decrease: a slot already at or below ours needs no atomic
                if (placed && (!ETWG_CLAIM_PEEK || rank < *reinterpret_cast<volatile u64*>(ranks + h)))
                    atomicMin(reinterpret_cast<unsigned long long*>(ranks + h), rank);
                if (!placed) s_full = 1;
            }
        }
        __syncthreads();
        if (s_full) {
            if (threadIdx.x == 0) {
                C->need = 2 * np * passes;
                C->abort = kGrowParts;
            }
            return;  // block-uniform
        }
        // mark each key's min-rank child in its parent's winner mask
        for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
            const u64 rank = ranks[i];
            if (rank == ~u64{0}) continue;  // never claimed
            Set<W> key;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                key.w[w] = keys[W * i + w];
                keys[W * i + w] = 0;  // empty again for the next bucket
            }
            ranks[i] = ~u64{0};
            if constexpr (BLOOM) {
                const u64 m = bloom_bits_for(round_cap(*P, C->count[r & 1]), P->bpe);
                unsigned* bits = B.bloom[r & 1];
                const unsigned h1 = murmur_key<W>(key, kSeed1);
                const unsigned h2 = murmur_key<W>(key, kSeed2);
                u64 pos, step;
                probe_start(h1, h2, m, pos, step);
                ++probed;
                if (!bloom_or_probes(bits, m, pos, step, P->hashes)) {
                    // a distinct key of the round whose probe bits were all set
                    // by other keys: a false positive (the reference drops it too)
                    atomicAdd(&C->rs[r].fp, 1ull);
                    if (P->flags & 2048) {
                        const unsigned at = atomicAdd(&C->fp_log_n, 1u);
                        if (at < 16) {
                            C->fp_log[at][0] = key.w[0];
                            C->fp_log[at][1] = W == 2 ? key.w[W - 1] : 0;
                            C->fp_log[at][2] = (static_cast<u64>(h1) << 32) | h2;
                            C->fp_log[at][3] = m;
                        }
                    }
                    continue;
                }
            }
            const u64 parent = rank / (64 * W);
            const int v = static_cast<int>(rank % (64 * W));
            atomicOr(reinterpret_cast<unsigned long long*>(B.cmask) + parent * W + (v >> 6), u64{1} << (v & 63));
        }
        if (threadIdx.x == 0) *cursor_at(B, part) = 0;  // clean for the next round
        __syncthreads();
    }
    if (BLOOM) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) probed += __shfl_xor_sync(kFull, probed, o);
        if ((threadIdx.x & 31) == 0 && probed) atomicAdd(&C->rs[r].probed, probed);
    }
}

// Compact rounds (8-byte records {low << 32 | parent}, see PartPlan): the
// same per-bucket min-rank dedup as k_exact_part with a 32-bit key (the
// mixed key's low bits; the bucket fixes the rest) and the parent index as
// the rank, in a 32 KB table. The winner's vertex is the one bit of
// key \ S[parent]: one read of the parent's set per distinct key.
template <bool BLOOM>
__global__ void __launch_bounds__(kPartThreads) k_exact_part_compact(const Params* __restrict__ P, Control* C,
                                                                     Bufs B) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int SLOTS = kCompactSlots;
    unsigned* keys = reinterpret_cast<unsigned*>(smem_raw);
    unsigned* ranks = keys + SLOTS;
    __shared__ unsigned s_full;
    if (halted(C)) return;
    const unsigned r = C->round;
    if (!C->rs[r].compact) return;
    const u64 passes = C->passes ? C->passes : 1;
    const u64 pass = C->pass;
    const u64 np = C->rs[r].np / passes;
    const u64 cap = C->rs[r].pcap;
    const int nb = static_cast<int>(C->rs[r].nb);
    u64 probed = 0;
    const int n = P->n;
    const u64* layer = B.keys[r & 1];
    for (u64 lp = blockIdx.x; lp < np; lp += gridDim.x) {
        const u64 part = lp * passes + pass;
        for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
            keys[i] = ~0u;
            ranks[i] = ~0u;
        }
        if (threadIdx.x == 0) s_full = 0;
        __syncthreads();
        const unsigned cnt = *cursor_at(B, part);
        const u64* recs = B.recs + lp * cap;
        constexpr int kBatch = 2 * ETWG_PART_BATCH;  // 8-byte records: twice as many in flight
        for (unsigned base = threadIdx.x; base < cnt; base += kBatch * blockDim.x) {
            u64 rv[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const unsigned i = base + j * blockDim.x;
                rv[j] = i < cnt ? __ldcs(recs + i) : ~u64{0};
            }
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                if (rv[j] == ~u64{0}) break;
                const unsigned low = static_cast<unsigned>(rv[j] >> 32);
                const unsigned parent = static_cast<unsigned>(rv[j]);
                unsigned h = (low * 0x9E3779B1u) >> (32 - 12);
                bool placed = false;
                for (int probe = 0; probe < 128; ++probe) {
                    const unsigned seen = *reinterpret_cast<volatile unsigned*>(keys + h);
                    if (seen == low) {
                        placed = true;
                    } else if (seen == ~0u) {
                        const unsigned prev = atomicCAS(keys + h, ~0u, low);
                        placed = prev == ~0u || prev == low;
                    }
                    if (placed) break;
                    h = (h + 1) & (SLOTS - 1);
                }
                if (placed) {
                    if (parent < *reinterpret_cast<volatile unsigned*>(ranks + h)) atomicMin(ranks + h, parent);
                } else {
                    s_full = 1;
                }
            }
        }
        __syncthreads();
        if (s_full) {
            if (threadIdx.x == 0) {
                C->need = 2 * np * passes;
                C->abort = kGrowParts;
            }
            return;  // block-uniform
        }
        for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
            const unsigned parent = ranks[i];
            if (parent == ~0u) continue;
            const u64 key = unmixn((nb >= 64 ? 0 : (part << nb)) | keys[i], n);
            if constexpr (BLOOM) {
                const Set<1> k1 = {{key}};
                const u64 m = bloom_bits_for(round_cap(*P, C->count[r & 1]), P->bpe);
                const unsigned h1 = murmur_key<1>(k1, kSeed1);
                const unsigned h2 = murmur_key<1>(k1, kSeed2);
                u64 pos, step;
                probe_start(h1, h2, m, pos, step);
                ++probed;
                if (!bloom_or_probes(reinterpret_cast<unsigned*>(B.bloom[r & 1]), m, pos, step, P->hashes)) {
                    atomicAdd(&C->rs[r].fp, 1ull);
                    if (P->flags & 2048) {
                        const unsigned at = atomicAdd(&C->fp_log_n, 1u);
                        if (at < 16) {
                            C->fp_log[at][0] = key;
                            C->fp_log[at][1] = 0;
                            C->fp_log[at][2] = (static_cast<u64>(h1) << 32) | h2;
                            C->fp_log[at][3] = m;
                        }
                    }
                    continue;
                }
            }
            const u64 bit = key & ~__ldg(layer + parent);  // the one vertex the parent lacks
            atomicOr(reinterpret_cast<unsigned long long*>(B.cmask) + parent, bit);
        }
        if (threadIdx.x == 0) *cursor_at(B, part) = 0;  // clean for the next round
        __syncthreads();
    }
    if (BLOOM) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) probed += __shfl_xor_sync(kFull, probed, o);
        if ((threadIdx.x & 31) == 0 && probed) atomicAdd(&C->rs[r].probed, probed);
    }
}

template <int W>
__global__ void k_bloom_batch(const u64* keys, u64 count, unsigned* bits, unsigned* locks, u64 m,
                              int hashes, unsigned char* novel) {
    const u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    const Set<W> key = load_set<W>(keys, i);
    novel[i] = bloom_insert<W>(bits, locks, m, hashes, key) ? 1 : 0;
}

// ----------------------------------------------------------------------
// Bloom round, pass 1 (replaces expand_range + the Bloom branch of
// expand_layer, dp.cpp:39-69 + 93-117), barrier-free: each warp takes 32
// consecutive parents, evaluates their candidates (K1), flattens the
// children over its lanes, drops duplicates among them with a warp-private
// shared-memory key set (siblings of one grandparent sit next to each other
// in the layer, so most duplicates are local), and sends the rest to the
// global Bloom filter. The novel-children mask of every parent goes to HBM;
// pass 2 (k_append<W>) turns masks into the rank-ordered next layer.
//
// Exactly-once novelty without the stripe-lock fences: an insert sets its
// 17 bits with relaxed atomicOr; if any was clear it *claims* the key in an
// epoch-tagged table with one 128-bit CAS — of several concurrent inserters
// of the same key exactly one claim succeeds (the reference's lock-based
// guarantee, bloom.cpp:86-97). W=2 keys (16 bytes + tag) do not fit a
// 16-byte CAS and use the reference's stripe locks, as does any round whose
// claim table would exceed kClaimMax.

template <int W, bool MMW>
__global__ void __launch_bounds__(kThreads, 3) k_bloom_dedup(const Params* __restrict__ P, Control* C,
                                                          Bufs B) {
    extern __shared__ __align__(16) u64 local_slots[];
    __shared__ Set<W> adj[64 * W];
    __shared__ unsigned novel_words[kThreads][2 * W];
    __shared__ unsigned mmw_keep[MMW ? kThreads : 1][2 * W];
    if (halted(C)) return;
    const unsigned r = C->round;
    const unsigned epoch = C->epoch;
    const u64 E = C->count[r & 1];
    const u64 cap = round_cap(*P, E);
    const u64 m = bloom_bits_for(cap, P->bpe);
    const u64 gtid = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
    const u64 gstride = static_cast<u64>(gridDim.x) * blockDim.x;
    // claim table sized for every key the round can offer (E_in * free)
    const u64 claim_slots = table_slots_for(E * static_cast<u64>(P->free_count));
    const bool use_claims = W == 1 && !(P->flags & 2) && P->hashes == 17 &&
                            m <= 0xFFFFFFFFull && claim_slots <= kClaimMax;
    if (m / 32 > B.bloom_cap || (use_claims && claim_slots > B.claim_cap)) {
        if (gtid == 0) {
            const bool bloom_short = m / 32 > B.bloom_cap;
            C->need = bloom_short ? m / 32 : claim_slots;
            C->abort = bloom_short ? kGrowBloom : kGrowClaims;
        }
        return;
    }
    // clear the other filter's region from round r-1 (needed clean at r+1)
    if (r > 0) {
        const u64 prev_words = bloom_bits_for(round_cap(*P, C->rs[r - 1].expanded), P->bpe) / 32;
        uint4* w4 = reinterpret_cast<uint4*>(B.bloom[(r + 1) & 1]);
        const u64 n4 = prev_words / 4;
        for (u64 i = gtid; i < n4; i += gstride) w4[i] = make_uint4(0, 0, 0, 0);
        for (u64 i = n4 * 4 + gtid; i < prev_words; i += gstride) B.bloom[(r + 1) & 1][i] = 0;
    }
    unsigned* bits = B.bloom[r & 1];
    load_adjacency<W>(P, adj);
    __syncthreads();
    constexpr unsigned kWarpSlots = kWarpLocalBytes / (8 * W);
    const int lane = threadIdx.x & 31;
    const int wslot = threadIdx.x & ~31;
    u64* my_slots = local_slots + (threadIdx.x >> 5) * (kWarpSlots * W);
    const Set<W> forbidden = param_set<W>(P->forbidden);
    const bool single_lock = (P->flags & 2) != 0;
    const u64* in = B.keys[r & 1];
    const u64 warp = gtid >> 5;
    const u64 nwarps = gstride >> 5;
    u64 offered = 0, pruned = 0;
    for (u64 base = warp * 32; base < E; base += nwarps * 32) {
        const u64 idx = base + lane;
        const bool valid = idx < E;
        const Set<W> S = valid ? load_set<W>(in, idx) : Set<W>::zero();
        const Set<W> M = warp_candidates<W, MMW, ETWG_SCATTER_COMPACT>(adj, P->n, P->k, S, valid, forbidden, pruned, mmw_keep);
        offered += M.count();
        for (unsigned i = lane; i < kWarpSlots * W; i += 32) my_slots[i] = 0;
#pragma unroll
        for (int i = 0; i < 2 * W; ++i) novel_words[threadIdx.x][i] = 0;
        __syncwarp();
        WarpFlat f;
        f.scan(M.count());
        for (int t = 0; t < f.total; t += 32) {
            const int j = t + lane;
            const int src = f.source(j);
            const int excl = __shfl_sync(kFull, f.incl, src) - __shfl_sync(kFull, f.cnt, src);
            const Set<W> Ms = shfl_set<W>(M, src);
            const Set<W> Ss = shfl_set<W>(S, src);
            if (j < f.total) {
                const int v = nth_member<W>(Ms, j - excl);
                Set<W> key = Ss;
                key.add(v);
                bool novel = false;
                if (local_first<W>(my_slots, kWarpSlots - 1, key)) {
                    if (use_claims) {
                        const unsigned h1 = murmur_key<W>(key, kSeed1);
                        const unsigned h2 = murmur_key<W>(key, kSeed2);
                        u64 first, step;
                        probe_start(h1, h2, m, first, step);
                        novel = bloom_set_bits<17>(bits, m, first, step) &&
                                claim_key(B.claims, claim_slots - 1, key.w[0], epoch);
                    } else {
                        novel = bloom_insert<W>(bits, B.locks, m, P->hashes, key, single_lock);
                    }
                }
                if (novel) atomicOr(&novel_words[wslot + src][v >> 5], 1u << (v & 31));
            }
        }
        __syncwarp();
        if (valid) {
            Set<W> nm;
#pragma unroll
            for (int i = 0; i < W; ++i)
                nm.w[i] = novel_words[threadIdx.x][2 * i] |
                          (static_cast<u64>(novel_words[threadIdx.x][2 * i + 1]) << 32);
            store_set<W>(B.cmask, idx, nm);
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        offered += __shfl_xor_sync(kFull, offered, o);
        pruned += __shfl_xor_sync(kFull, pruned, o);
    }
    if (lane == 0) {
        if (offered) atomicAdd(&C->rs[r].offered, offered);
        if (pruned) atomicAdd(&C->rs[r].mmw_pruned, pruned);
    }
}

// ----------------------------------------------------------------------
// K3: ordered append with a single-pass decoupled look-back scan
// (replaces the cursor append dp.cpp:96-117 and the rank sort + truncation
// dp.cpp:150-157)

// Writes the tile's survivors (mask M over parents S with histories H) in
// rank order: the warp's survivors occupy one contiguous run starting at
// warp_start, so consecutive lanes store consecutive states.
template <int W>
__device__ __forceinline__ void append_survivors(const Set<W>& M, const Set<W>& S, unsigned H,
                                                 u64 warp_start, u64 limit, u64* out,
                                                 unsigned* hout) {
    const int lane = threadIdx.x & 31;
    WarpFlat f;
    f.scan(M.count());
    for (int t = 0; t < f.total; t += 32) {
        const int j = t + lane;
        const int src = f.source(j);
        const int excl = __shfl_sync(kFull, f.incl, src) - __shfl_sync(kFull, f.cnt, src);
        const Set<W> Ms = shfl_set<W>(M, src);
        const Set<W> Ss = shfl_set<W>(S, src);
        const unsigned Hs = __shfl_sync(kFull, H, src);
        const u64 pos = warp_start + j;
        if (j < f.total && pos < limit) {  // capacity wall: drop the newest (dp.cpp:107,152-155)
            const int v = nth_member<W>(Ms, j - excl);
            Set<W> key = Ss;
            key.add(v);
            store_set<W>(out, pos, key);
            hout[pos] = (Hs << 8) | static_cast<unsigned>(v & 0xFF);  // push_history
        }
    }
}

// The last CTA out publishes the round (all CTAs have read the round state
// by then, so advancing it cannot race with a late starter). Called by every
// CTA with all threads after its last tile.
__device__ __forceinline__ void finish_round(const Params* P, Control* C, const Bufs& B, unsigned r,
                                             u64 E, u64 cap) {
    if (threadIdx.x != 0) return;
    __threadfence();
    const unsigned done = atomicAdd(&C->exits, 1u);
    if (done != gridDim.x - 1) return;
    __threadfence();
    C->exits = 0;
    RoundStats& rs = C->rs[r];
    const u64 unique = *reinterpret_cast<volatile u64*>(&rs.unique);
    const u64 emitted = unique < cap ? unique : cap;
    if (emitted > B.layer_cap) {
        C->need = emitted;
        C->abort = kGrowLayer;
        return;
    }
    rs.expanded = E;
    rs.emitted = emitted;
    rs.overflowed = unique > cap ? 1u : 0u;
    rs.valid = 1;
    C->count[(r + 1) & 1] = emitted;
    C->round = r + 1;
    C->pass = 0;
    C->epoch = (C->epoch & kEpochMask) == kEpochMask ? 1 : C->epoch + 1;
    if (emitted == 0 || static_cast<int>(r) + 1 >= P->rounds) {
        C->stop = 1;
    } else if (C->handoff_above && emitted > C->handoff_above) {
        C->stop = 1;  // the owner-sharded engine takes the layer from here
        C->handed = 1;
    }
}

// A tile is ITEMS slices of kThreads consecutive parents (slice i = parents
// tile*span + i*kThreads + t), so one look-back publishes 2048 parents: the
// look-back chain, not bandwidth, bounded the 256-parent version.
template <int W>
constexpr int append_items() { return W == 1 ? 8 : 4; }

template <int W>
__global__ void __launch_bounds__(kThreads, ETWG_APPEND_MINB) k_append(const Params* __restrict__ P, Control* C,
                                                     Bufs B) {
    using BlockScan = cub::BlockScan<unsigned, kThreads>;
    constexpr int ITEMS = append_items<W>();
    constexpr u64 kSpan = static_cast<u64>(kThreads) * ITEMS;
    __shared__ typename BlockScan::TempStorage scan_tmp;
    __shared__ u64 s_prefix;
    __shared__ u64 s_tile;
    if (halted(C)) return;
    const unsigned r = C->round;
    const unsigned epoch = C->epoch;
    const u64 E = C->count[r & 1];
    const u64 ntiles = (E + kSpan - 1) / kSpan;
    const u64 cap = round_cap(*P, E);
    const u64 limit = cap < B.layer_cap ? cap : B.layer_cap;
    const u64* in = B.keys[r & 1];
    const unsigned* hin = B.hist[r & 1];
    u64* out = B.keys[(r + 1) & 1];
    unsigned* hout = B.hist[(r + 1) & 1];

    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&C->rs[r].ticket, 1ull);
        __syncthreads();
        const u64 tile = s_tile;
        if (tile >= ntiles) break;
        Set<W> S[ITEMS], M[ITEMS];
        unsigned H[ITEMS], excl[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const u64 idx = tile * kSpan + static_cast<u64>(i) * kThreads + threadIdx.x;
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
            __syncthreads();  // scan_tmp is reused by the next slice
        }
        if (threadIdx.x == 0) s_prefix = look_back(B.tiles, tile, total, epoch);
        __syncthreads();
        const u64 prefix = s_prefix;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
            append_survivors<W>(M[i], S[i], H[i], prefix + __shfl_sync(kFull, excl[i], 0), limit, out, hout);
        if (threadIdx.x == 0 && tile == ntiles - 1) {
            // the final tile knows the round's survivor total
            C->rs[r].unique = prefix + total;
        }
        __syncthreads();
    }
    finish_round(P, C, B, r, E, cap);
}

// ----------------------------------------------------------------------
// host engine

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw DeviceError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

struct Profile {
    bool on = false;
    KernelTimes t;
};

class Engine {
public:
    static Engine& instance() {
        static Engine* e = new Engine();
        return *e;
    }

    std::mutex mu;
    Profile prof;

    bool ready() {
        if (init_state_ == 0) init();
        return init_state_ == 1;
    }

    const DeviceInfo& info() { return info_; }

    void timer_begin() {
        require_device();
        check(cudaEventRecord(tev_[0], stream_), "timer");
    }
    double timer_end() {
        require_device();
        check(cudaEventRecord(tev_[1], stream_), "timer");
        check(cudaEventSynchronize(tev_[1]), "timer sync");
        float t = 0;
        check(cudaEventElapsedTime(&t, tev_[0], tev_[1]), "timer elapsed");
        return t;
    }

    DecideResult decide(const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg,
                        int rounds, const LayerObserver* observer, u64 handoff_above = 0,
                        EngineLayer* handoff = nullptr) {
        NvtxRange nvtx("etw decide k=%d", k);
        require_device();
        const int n = g.vertex_count();
        const int W = n > 64 ? 2 : 1;
        if (rounds < 0) rounds = std::max(0, n - k - 1);
        if (rounds > kMaxRounds - 1) throw std::invalid_argument("too many rounds");
        DecideResult res;
        if (rounds == 0) {  // dp.cpp:176 loop never runs; witness = the root
            res.outcome = Outcome::feasible;
            return res;
        }
        setup_params(g, k, forbidden, cfg, rounds, /*any_pop=*/0);
        // root layer: {(empty set, 0xFFFFFFFF)}
        ensure_layers(1, 0, 0);
        reset_control(1, handoff_above);
        u64 zero2[2] = {0, 0};
        unsigned root_hist = 0xFFFFFFFFu;
        copy(b_.keys[0], zero2, 16, cudaMemcpyHostToDevice, "root");
        copy(b_.hist[0], &root_hist, 4, cudaMemcpyHostToDevice, "root");

        run_rounds(W, cfg, rounds, k, observer);

        const Control& c = *h_ctl_;
        bool any_ovf = false;
        for (int r = 0; r < rounds; ++r) {
            const RoundStats& s = c.rs[r];
            if (!s.valid) break;
            LayerStats ls;
            ls.k = k;
            ls.round = r;
            ls.expanded = s.expanded;
            ls.emitted = s.emitted;
            ls.duplicates = s.offered - s.unique;
            ls.mmw_pruned = s.mmw_pruned;
            ls.overflowed = s.overflowed != 0;
            any_ovf = any_ovf || ls.overflowed;
            res.rounds.push_back(ls);
            prof.t.bloom_probed += s.probed;
            prof.t.bloom_fp += s.fp;
            if (s.fp && std::getenv("ETWG_TRACE"))
                std::fprintf(stderr, "[engine] k=%d round %d: %llu of %llu distinct keys rejected by the filter\n", k, r,
                             static_cast<unsigned long long>(s.fp), static_cast<unsigned long long>(s.probed));
            if (s.emitted == 0) break;
        }
        if ((h_params_->flags & 2048) && c.fp_log_n) {
            for (unsigned i = 0; i < std::min(c.fp_log_n, 16u); ++i)
                std::fprintf(stderr, "[fp] k=%d key=%016llx:%016llx h1=%08x h2=%08x m=%llu\n", k,
                             static_cast<unsigned long long>(c.fp_log[i][1]), static_cast<unsigned long long>(c.fp_log[i][0]),
                             static_cast<unsigned>(c.fp_log[i][2] >> 32), static_cast<unsigned>(c.fp_log[i][2]),
                             static_cast<unsigned long long>(c.fp_log[i][3]));
        }
        res.overflowed = any_ovf;
        account(res.rounds, W, cfg);
        if (h_ctl_->handed) {
            if (!handoff) throw DeviceError("device decide handed off without a receiver");
            const int done = static_cast<int>(res.rounds.size());
            handoff->keys = b_.keys[done & 1];
            handoff->hist = b_.hist[done & 1];
            handoff->count = h_ctl_->count[done & 1];
            handoff->W = W;
            handoff->rounds_done = done;
            handoff->handed = true;
            return res;
        }
        if (handoff) handoff->handed = false;
        const bool empty = !res.rounds.empty() && res.rounds.back().emitted == 0;
        if (empty) {
            res.outcome = any_ovf ? Outcome::indeterminate : Outcome::infeasible;
            return res;
        }
        if (static_cast<int>(res.rounds.size()) != rounds)
            throw DeviceError("device decide stopped early without an empty layer");
        res.outcome = Outcome::feasible;
        res.witness = fetch_state(rounds & 1, 0, W);
        return res;
    }

    ExpandResult expand_layer(const Graph& g, int k, const HostSet& forbidden,
                              const std::vector<State>& input, const DpConfig& cfg,
                              LayerStats& stats) {
        require_device();
        ExpandResult out;
        stats.expanded = input.size();
        stats.emitted = stats.duplicates = stats.mmw_pruned = 0;
        stats.overflowed = false;
        if (input.empty()) return out;
        const int n = g.vertex_count();
        const int W = n > 64 ? 2 : 1;
        setup_params(g, k, forbidden, cfg, 1, /*any_pop=*/1);
        ensure_layers(input.size(), 0, 0);
        reset_control(input.size());
        std::vector<u64> keys(static_cast<size_t>(W) * input.size());
        std::vector<unsigned> hist(input.size());
        for (size_t i = 0; i < input.size(); ++i) {
            for (int w = 0; w < W; ++w) keys[W * i + w] = input[i].set.w[w];
            hist[i] = input[i].history;
        }
        copy(b_.keys[0], keys.data(), keys.size() * 8, cudaMemcpyHostToDevice, "expand input");
        copy(b_.hist[0], hist.data(), hist.size() * 4, cudaMemcpyHostToDevice, "expand input");
        run_rounds(W, cfg, 1, k, nullptr);
        const RoundStats& s = h_ctl_->rs[0];
        stats.emitted = s.emitted;
        stats.duplicates = s.offered - s.unique;
        stats.mmw_pruned = s.mmw_pruned;
        stats.overflowed = s.overflowed != 0;
        out.overflowed = stats.overflowed;
        out.states = fetch_layer(1, s.emitted, W);
        return out;
    }

    // Frees every round buffer (they are re-grown on demand): the sharded
    // engine calls this when it takes over the device, so a process that
    // solved a large instance on one GPU does not keep that HBM.
    void release_buffers() {
        if (init_state_ != 1) return;
        check(cudaStreamSynchronize(stream_), "sync");
        drop_graphs();
        for (int i = 0; i < 2; ++i) {
            cudaFree(b_.keys[i]);
            cudaFree(b_.hist[i]);
            cudaFree(b_.bloom[i]);
            b_.keys[i] = nullptr;
            b_.hist[i] = nullptr;
            b_.bloom[i] = nullptr;
            bloom_dirty_[i] = 0;
        }
        cudaFree(b_.cmask);
        cudaFree(b_.tiles);
        cudaFree(b_.recs);
        cudaFree(b_.cursors);
        cudaFree(b_.claims);
        cudaFree(b_.tab);
        b_.tab = nullptr;
        b_.tab_cap = 0;
        b_.cmask = nullptr;
        b_.tiles = nullptr;
        b_.recs = nullptr;
        b_.cursors = nullptr;
        b_.claims = nullptr;
        b_.layer_cap = b_.rec_cap = b_.cursor_cap = b_.bloom_cap = b_.claim_cap = 0;
    }

    uint64_t bloom_batch(uint64_t expected, int bpe, int hashes, const std::vector<uint64_t>& keys,
                         int words, std::vector<uint8_t>& novel, std::vector<uint32_t>* bits) {
        require_device();
        if (words != 1 && words != 2) throw std::invalid_argument("key words must be 1 or 2");
        const u64 count = keys.size() / words;
        const u64 m = bloom_bits_for(expected, bpe);
        ensure_bloom(m / 32);
        check(cudaMemsetAsync(b_.bloom[0], 0, (m / 32) * 4, stream_), "bloom zero");
        bloom_dirty_[0] = std::max<u64>(bloom_dirty_[0], m / 32);
        u64* d_keys = nullptr;
        unsigned char* d_novel = nullptr;
        check(cudaMalloc(&d_keys, std::max<u64>(8, keys.size() * 8)), "keys");
        check(cudaMalloc(&d_novel, std::max<u64>(1, count)), "novel");
        copy(d_keys, keys.data(), keys.size() * 8, cudaMemcpyHostToDevice, "keys h2d");
        const int blocks = static_cast<int>((count + 255) / 256);
        if (count) {
            if (words == 1)
                k_bloom_batch<1><<<blocks, 256, 0, stream_>>>(d_keys, count, b_.bloom[0], b_.locks, m,
                                                             hashes, d_novel);
            else
                k_bloom_batch<2><<<blocks, 256, 0, stream_>>>(d_keys, count, b_.bloom[0], b_.locks, m,
                                                             hashes, d_novel);
            check(cudaGetLastError(), "bloom batch");
            prof.t.kernel_launches++;
        }
        novel.assign(count, 0);
        if (count)
            copy(novel.data(), d_novel, count, cudaMemcpyDeviceToHost, "novel d2h");
        if (bits) {
            bits->assign(m / 32, 0);
            copy(bits->data(), b_.bloom[0], (m / 32) * 4, cudaMemcpyDeviceToHost, "bits d2h");
        }
        check(cudaStreamSynchronize(stream_), "sync");
        cudaFree(d_keys);
        cudaFree(d_novel);
        return m;
    }

private:
    int init_state_ = 0;  // 0 unknown, 1 ok, 2 no device
    int bound_device_ = -1;  // set by bind_device (shard init); else ETWG_DEVICE or 0
    DeviceInfo info_;
    cudaStream_t stream_ = nullptr;
    Params* d_params_ = nullptr;
    Params* h_params_ = nullptr;
    Control* d_ctl_ = nullptr;
    Control* h_ctl_ = nullptr;
    Bufs b_{};
    u64 bloom_dirty_[2] = {0, 0};  // words of each Bloom filter that may hold bits
    unsigned epoch_ = 1;          // look-back epoch carried across decides
    bool bloom_round_ = false;    // current decide runs the fused Bloom round
    int grid_fused_ = 0;
    int grid_exact_[2] = {0, 0};
    int grid_exact_mmw_[2] = {0, 0};
    int carveout_ = [] {
        const char* e = std::getenv("ETWG_CARVEOUT");
        return e ? std::atoi(e) : -1;  // -1: driver default
    }();
    int grid_part_[2] = {0, 0};
    int grid_compact_ = 0;
    int grid_tma_ = 0;
    bool compact_possible_ = false;  // ETWG_COMPACT build or ETWG_DEBUG 8192 this decide
    unsigned passes_ = 1;            // hash-range passes per round (f4: records beyond HBM)
    bool gtab_ = false;              // this decide's small exact rounds may use the global table (W == 1)
    int grid_bkt_ = 0, grid_tab_ = 0;  // k_exact_scatter<1, false, false, 1 / 2> grids
    bool part_bloom_ = false;  // Bloom rounds of this decide use scatter/part/append

    // Epochs tag look-back statuses (24 bits); on wrap-around the status
    // array is cleared so a status from 2^24 attempts ago cannot match.
    unsigned next_epoch() {
        epoch_ = (epoch_ + 1) & kEpochMask;
        if (epoch_ == 0) {
            epoch_ = 1;
            clear_tagged();
        }
        return epoch_;
    }
    int grid_ = 0;
    cudaEvent_t ev_[2] = {nullptr, nullptr};
    cudaEvent_t tev_[2] = {nullptr, nullptr};

    // every host<->device copy of the engine goes through here (counted)
    void copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, const char* what) {
        check(cudaMemcpyAsync(dst, src, bytes, kind, stream_), what);
        if (kind == cudaMemcpyHostToDevice) prof.t.h2d_bytes += bytes;
        if (kind == cudaMemcpyDeviceToHost) prof.t.d2h_bytes += bytes;
    }

public:
    // Moves the engine to device `dev` (a shard's device: one process per
    // GPU under torchrun). Before first use it only records the choice;
    // afterwards the engine is torn down and re-initialised there on next use.
    void bind_device(int dev) {
        if (init_state_ == 1 && info_.device == dev) return;
        if (init_state_ == 1) teardown();
        bound_device_ = dev;
        init_state_ = 0;
    }

    void teardown() {
        release_buffers();
        cudaSetDevice(info_.device);
        cudaStreamDestroy(stream_);
        cudaFree(d_params_);
        cudaFreeHost(h_params_);
        cudaFree(d_ctl_);
        cudaFreeHost(h_ctl_);
        cudaFree(b_.locks);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(ev_[i]);
            cudaEventDestroy(tev_[i]);
            ev_[i] = tev_[i] = nullptr;
        }
        stream_ = nullptr;
        d_params_ = h_params_ = nullptr;
        d_ctl_ = h_ctl_ = nullptr;
        b_.locks = nullptr;
        init_state_ = 0;
    }

private:
    void init() {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            init_state_ = 2;
            return;
        }
        int dev = 0;
        if (const char* e = std::getenv("ETWG_DEVICE")) dev = std::atoi(e);
        if (bound_device_ >= 0) dev = bound_device_;
        check(cudaSetDevice(dev), "cudaSetDevice");
        cudaDeviceProp prop;
        check(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
        info_.device = dev;
        info_.sm_count = prop.multiProcessorCount;
        std::snprintf(info_.name, sizeof info_.name, "%s", prop.name);
        grid_ = prop.multiProcessorCount * 4;
        // fused Bloom round: 64 KB of dynamic shared memory per CTA
        auto allow = [&](auto kernel) {
            check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kLocalBytes),
                  "smem attribute");
        };
        allow(k_bloom_dedup<1, false>);
        allow(k_bloom_dedup<1, true>);
        allow(k_bloom_dedup<2, false>);
        allow(k_bloom_dedup<2, true>);
        int per_sm = 0;
        check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bloom_dedup<1, false>, kThreads,
                                                            kLocalBytes),
              "occupancy");
        grid_fused_ = prop.multiProcessorCount * std::max(1, per_sm);
        auto allow_exact = [&](auto kernel, int bytes, int& grid) {
            check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                  "smem attribute");
            // K1's per-thread boundary tables live in local memory: keep the
            // shared carve-out near what the resident CTAs need (ETWG_CARVEOUT %)
            check(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_),
                  "carveout");
            int blocks = 0;
            check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, kThreads, bytes), "occupancy");
            grid = prop.multiProcessorCount * std::max(1, blocks);
        };
        allow_exact(k_exact_scatter<1, false, false>, scatter_smem<1>(), grid_exact_[0]);
        allow_exact(k_exact_scatter<1, false, false, 1>, scatter_smem<1>(), grid_bkt_);
        allow_exact(k_exact_scatter<1, false, false, 2>, scatter_smem<1>(), grid_tab_);
        allow_exact(k_exact_scatter<2, false, false>, 0, grid_exact_[1]);
        if (const char* c = std::getenv("ETWG_SCATTER_CTAS")) {  // CTAs per SM (tuning sweeps)
            const int per = std::atoi(c);
            for (int w = 0; w < 2; ++w) grid_exact_[w] = std::min(grid_exact_[w], prop.multiProcessorCount * per);
            grid_bkt_ = std::min(grid_bkt_, prop.multiProcessorCount * per);
            grid_tab_ = std::min(grid_tab_, prop.multiProcessorCount * per);
        }
        allow_exact(k_exact_scatter<1, true, false>, 0, grid_exact_mmw_[0]);
        allow_exact(k_exact_scatter<2, true, false>, 0, grid_exact_mmw_[1]);
        {
            // the Bloom variants run on the grid of their exact twin, capped by their own residency
            int g;
            allow_exact(k_exact_scatter<1, false, true>, scatter_smem<1>(), g);
            grid_exact_[0] = std::min(grid_exact_[0], g);
            allow_exact(k_exact_scatter<2, false, true>, 0, g);
            grid_exact_[1] = std::min(grid_exact_[1], g);
            allow_exact(k_exact_scatter<1, true, true>, 0, g);
            grid_exact_mmw_[0] = std::min(grid_exact_mmw_[0], g);
            allow_exact(k_exact_scatter<2, true, true>, 0, g);
            grid_exact_mmw_[1] = std::min(grid_exact_mmw_[1], g);
        }
        auto allow_part = [&](auto kernel, int bytes, int& grid) {
            check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                  "smem attribute");
            int blocks = 0;
            check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, kPartThreads, bytes),
                  "occupancy");
            grid = prop.multiProcessorCount * std::max(1, blocks);
        };
        allow_part(k_exact_part<1, false>, part_smem_bytes<1>(), grid_part_[0]);
        allow_part(k_exact_part<2, false>, part_smem_bytes<2>(), grid_part_[1]);
        {
            int g;
            allow_part(k_exact_part<1, true>, part_smem_bytes<1>(), g);
            allow_part(k_exact_part<2, true>, part_smem_bytes<2>(), g);
            allow_part(k_exact_part_compact<false>, compact_smem_bytes(), grid_compact_);
            auto allow_tma = [&](auto kernel, int& grid) {
                check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tma_part_smem_bytes()),
                      "smem attribute");
                int blocks = 0;
                check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, kTmaThreads, tma_part_smem_bytes()),
                      "occupancy");
                grid = prop.multiProcessorCount * std::max(1, blocks);
            };
            allow_tma(k_exact_part_tma<false>, grid_tma_);
            allow_tma(k_exact_part_tma<true>, g);
            grid_tma_ = std::min(grid_tma_, g);
            allow_part(k_exact_part_compact<true>, compact_smem_bytes(), g);
            grid_compact_ = std::min(grid_compact_, g);
        }
        check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
        check(cudaMalloc(&d_params_, sizeof(Params)), "malloc params");
        check(cudaMallocHost(&h_params_, sizeof(Params)), "host params");
        check(cudaMalloc(&d_ctl_, sizeof(Control)), "malloc control");
        check(cudaMallocHost(&h_ctl_, sizeof(Control)), "host control");
        check(cudaMalloc(&b_.locks, kStripes * sizeof(unsigned)), "locks");
        check(cudaMemset(b_.locks, 0, kStripes * sizeof(unsigned)), "locks");
        check(cudaEventCreate(&ev_[0]), "event");
        check(cudaEventCreate(&ev_[1]), "event");
        check(cudaEventCreate(&tev_[0]), "event");
        check(cudaEventCreate(&tev_[1]), "event");
        init_state_ = 1;
    }

    void require_device() {
        if (!ready())
            throw DeviceError(
                "no CUDA device available: the elimtw B200 engine has no CPU fallback");
    }

    void setup_params(const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg,
                      int rounds, int any_pop) {
        Params& p = *h_params_;
        std::memset(&p, 0, sizeof p);
        p.n = g.vertex_count();
        p.k = k;
        p.rounds = rounds;
        p.free_count = std::max(0, g.vertex_count() - forbidden.count());
        p.hashes = cfg.bloom_hashes;
        p.bpe = cfg.bloom_bits_per_element;
        p.any_pop = any_pop;
        if (const char* dbg = std::getenv("ETWG_DEBUG")) p.flags = std::atoi(dbg);
        // exact rounds of one-word keys: global open-addressing table (default)
        // or bucket records + per-bucket shared-memory tables (ETWG_GTAB=0)
        // ETWG_GTAB=0: every round on buckets; ETWG_GTAB=L: tables up to 2^L slots
        const char* gt = std::getenv("ETWG_GTAB");
        const int lg = gt ? std::atoi(gt) : kGtabLg;
        p.gtab = cfg.dedup == DedupMode::exact_set ? std::max(0, std::min(lg, 30)) : 0;
        p.max_states = cfg.max_layer_states;
        p.forbidden[0] = forbidden.w[0];
        p.forbidden[1] = forbidden.w[1];
        for (int v = 0; v < g.vertex_count(); ++v) {
            p.rows[v][0] = g.neighbors(v).w[0];
            p.rows[v][1] = g.neighbors(v).w[1];
        }
        copy(d_params_, h_params_, sizeof(Params), cudaMemcpyHostToDevice, "params");
    }

    void reset_control(u64 first_count, u64 handoff_above = 0) {
        Control& c = *h_ctl_;
        std::memset(&c, 0, sizeof c);
        c.count[0] = first_count;
        c.handoff_above = handoff_above;
        c.epoch = next_epoch();
        // ETWG_PASSES: minimum hash-range passes per round (a power of two;
        // tests / out-of-HBM rehearsal); the engine doubles it when the child
        // records of a round do not fit the device
        passes_ = 1;
        if (const char* e = std::getenv("ETWG_PASSES"))
            while (passes_ < 1024 && passes_ * 2 <= static_cast<unsigned>(std::max(1, std::atoi(e)))) passes_ *= 2;
        c.passes = passes_;
        compact_possible_ = ETWG_COMPACT || (h_params_->flags & 8192);
        copy(d_ctl_, h_ctl_, sizeof(Control), cudaMemcpyHostToDevice, "control");
    }

    // (Re)allocates both layer buffers, the candidate masks and the tile
    // status words for `states` per layer; keeps `keep_count` states of
    // buffer `keep_buf` when growing.
    void ensure_layers(u64 states, int keep_buf, u64 keep_count) {
        if (states <= b_.layer_cap && b_.keys[0]) return;
        u64 cap = std::max<u64>(states, std::max<u64>(b_.layer_cap * 2, u64{1} << 16));
        u64* keys[2];
        unsigned* hist[2];
        for (int i = 0; i < 2; ++i) {
            check(cudaMalloc(&keys[i], cap * 16), "layer keys");
            check(cudaMalloc(&hist[i], cap * 4), "layer hist");
        }
        if (b_.keys[0] && keep_count) {
            check(cudaMemcpyAsync(keys[keep_buf], b_.keys[keep_buf], keep_count * 16,
                                  cudaMemcpyDeviceToDevice, stream_),
                  "keep layer");
            check(cudaMemcpyAsync(hist[keep_buf], b_.hist[keep_buf], keep_count * 4,
                                  cudaMemcpyDeviceToDevice, stream_),
                  "keep layer");
        }
        check(cudaStreamSynchronize(stream_), "sync");
        for (int i = 0; i < 2; ++i) {
            if (b_.keys[i]) cudaFree(b_.keys[i]);
            if (b_.hist[i]) cudaFree(b_.hist[i]);
            b_.keys[i] = keys[i];
            b_.hist[i] = hist[i];
        }
        if (b_.cmask) cudaFree(b_.cmask);
        if (b_.tiles) cudaFree(b_.tiles);
        check(cudaMalloc(&b_.cmask, cap * 16), "cmask");
        check(cudaMalloc(&b_.tiles, ((cap + kThreads - 1) / kThreads + 1) * 8), "tiles");
        check(cudaMemsetAsync(b_.tiles, 0, ((cap + kThreads - 1) / kThreads + 1) * 8, stream_), "tiles");
        b_.layer_cap = cap;
    }

    // Exact-mode record buckets; cursors start (and are left by every
    // completed round) at zero.
    // records: `words` u64 words (2 per 16-byte record, 4 per 32-byte, 1 per
    // compact); false when the device cannot hold them (the caller then
    // splits the round into more hash-range passes)
    bool ensure_parts(u64 words, u64 parts) {
        if (words > b_.rec_cap || !b_.recs) {
            const u64 cap = std::max<u64>(words, u64{1} << 21);
            if (b_.recs) cudaFree(b_.recs);
            b_.recs = nullptr;
            b_.rec_cap = 0;
            const cudaError_t e = cudaMalloc(&b_.recs, cap * 8);
            if (e == cudaErrorMemoryAllocation && words > (u64{1} << 21)) {
                cudaGetLastError();
                return false;
            }
            check(e, "records");
            b_.rec_cap = cap;
        }
        if (parts > b_.cursor_cap || !b_.cursors) {
            const u64 cap = std::max<u64>(parts, u64{1} << 16);
            if (b_.cursors) cudaFree(b_.cursors);
            check(cudaMalloc(&b_.cursors, cap * 4 * kCursorStride), "cursors");
            check(cudaMemsetAsync(b_.cursors, 0, cap * 4 * kCursorStride, stream_), "cursors zero");
            b_.cursor_cap = cap;
        }
        return true;
    }

    void clean_cursors() {
        check(cudaMemsetAsync(b_.cursors, 0, b_.cursor_cap * 4 * kCursorStride, stream_), "cursors clean");
    }

    // Global table: allocated once at its maximum (2^gtab slots, L2-sized),
    // empty between rounds (k_tab_mark clears what it marks); an aborted
    // global-table round leaves `slots` slots to clear.
    void ensure_tab(u64 slots) {
        if (b_.tab && b_.tab_cap >= slots) return;
        if (b_.tab) cudaFree(b_.tab);
        check(cudaMalloc(&b_.tab, slots * 16), "global table");
        check(cudaMemsetAsync(b_.tab, 0, slots * 16, stream_), "global table zero");
        b_.tab_cap = slots;
    }
    void clean_table(u64 slots) {
        if (b_.tab && slots)
            check(cudaMemsetAsync(b_.tab, 0, std::min(slots, b_.tab_cap) * 16, stream_), "table clean");
    }

    void ensure_bloom(u64 words) {
        if (words <= b_.bloom_cap && b_.bloom[0]) return;
        u64 cap = std::max<u64>(words, u64{1} << 22);
        for (int f = 0; f < 2; ++f) {
            if (b_.bloom[f]) cudaFree(b_.bloom[f]);
            check(cudaMalloc(&b_.bloom[f], cap * 4), "bloom");
            check(cudaMemsetAsync(b_.bloom[f], 0, cap * 4, stream_), "bloom zero");
            bloom_dirty_[f] = 0;
        }
        b_.bloom_cap = cap;
    }

    // Bloom filters must be all-zero when a decide starts; the fused round
    // kernel keeps them clean within a decide, this covers what is left.
    void clean_blooms() {
        for (int f = 0; f < 2; ++f) {
            if (!bloom_dirty_[f]) continue;
            const u64 words = std::min(bloom_dirty_[f], b_.bloom_cap);
            check(cudaMemsetAsync(b_.bloom[f], 0, words * 4, stream_), "bloom clean");
            bloom_dirty_[f] = 0;
        }
    }

    // Claim slots are {key, epoch}; fresh memory is zero (epoch 0 is never a
    // live tag), and a look-back epoch wrap clears the table again.
    void ensure_claims(u64 slots) {
        if (slots <= b_.claim_cap && b_.claims) return;
        const u64 cap = std::max<u64>(slots, u64{1} << 20);
        if (b_.claims) cudaFree(b_.claims);
        check(cudaMalloc(&b_.claims, cap * 16), "claims");
        check(cudaMemsetAsync(b_.claims, 0, cap * 16, stream_), "claims zero");
        b_.claim_cap = cap;
    }

    // Epoch-tagged structures (look-back statuses, claim slots) after a wrap.
    void clear_tagged() {
        if (b_.tiles)
            check(cudaMemsetAsync(b_.tiles, 0, ((b_.layer_cap + kThreads - 1) / kThreads + 1) * 8, stream_),
                  "tiles clear");
        if (b_.claims) check(cudaMemsetAsync(b_.claims, 0, b_.claim_cap * 16, stream_), "claims clear");
    }

    u64 host_round_cap(u64 e_in) const {
        u64 upper = e_in * static_cast<u64>(h_params_->free_count);
        if (upper < 1) upper = 1;
        return std::min<u64>(h_params_->max_states, upper);
    }

    template <int W>
    void launch_round(const DpConfig& cfg) {
        const bool exact = cfg.dedup == DedupMode::exact_set;
        const bool timed = prof.on;
        auto timed_launch = [&](auto&& fn, double& ms, uint64_t& launches) {
            if (timed) check(cudaEventRecord(ev_[0], stream_), "event");
            fn();
            check(cudaGetLastError(), "kernel launch");
            prof.t.kernel_launches++;
            launches++;
            if (timed) {
                check(cudaEventRecord(ev_[1], stream_), "event");
                check(cudaEventSynchronize(ev_[1]), "event sync");
                float t = 0;
                cudaEventElapsedTime(&t, ev_[0], ev_[1]);
                ms += t;
            }
        };
        if (!exact && !part_bloom_) {
            if (cfg.use_mmw)
                timed_launch([&] { k_bloom_dedup<W, true><<<grid_fused_, kThreads, kLocalBytes, stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.insert_ms, prof.t.insert_launches);
            else
                timed_launch([&] { k_bloom_dedup<W, false><<<grid_fused_, kThreads, kLocalBytes, stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.insert_ms, prof.t.insert_launches);
            timed_launch([&] { k_append<W><<<grid_, kThreads, 0, stream_>>>(d_params_, d_ctl_, b_); },
                         prof.t.append_ms, prof.t.append_launches);
            return;
        }
        if (exact)
            launch_partitioned<W, false>(cfg, timed_launch);
        else
            launch_partitioned<W, true>(cfg, timed_launch);
    }

    // scatter -> part -> append (exact mode, and Bloom mode with a large filter)
    template <int W, bool BLOOM, typename Launch>
    void launch_partitioned(const DpConfig& cfg, Launch&& timed_launch) {
        const int smem = 0;
        for (unsigned pass = 0; pass < passes_; ++pass) {
            if (cfg.use_mmw)
                timed_launch([&] { k_exact_scatter<W, true, BLOOM><<<grid_exact_mmw_[W - 1], kThreads, smem, stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.expand_ms, prof.t.expand_launches);
            else if (W == 1 && !BLOOM && gtab_) {  // the plan picks one; the other returns at once
                timed_launch([&] { k_exact_scatter<W, false, BLOOM, 1><<<grid_bkt_, kThreads, scatter_smem<W>(), stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.expand_ms, prof.t.expand_launches);
                timed_launch([&] { k_exact_scatter<W, false, BLOOM, 2><<<grid_tab_, kThreads, scatter_smem<W>(), stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.expand_ms, prof.t.expand_launches);
            } else
                timed_launch([&] { k_exact_scatter<W, false, BLOOM><<<grid_exact_[W - 1], kThreads, scatter_smem<W>(), stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.expand_ms, prof.t.expand_launches);
            // the scatter's plan picks the round's dedup; the other kernels return at once
            if (W == 1 && gtab_ && !BLOOM)
                timed_launch([&] { k_tab_mark<<<grid_, kThreads, 0, stream_>>>(d_ctl_, b_); },
                             prof.t.insert_ms, prof.t.insert_launches);
            if (W == 1 && ETWG_PART_TMA && !BLOOM)  // Bloom probes want the 3-CTA kernel's warps
                timed_launch([&] { k_exact_part_tma<BLOOM><<<grid_tma_, kTmaThreads, tma_part_smem_bytes(), stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.insert_ms, prof.t.insert_launches);
            else
                timed_launch([&] { k_exact_part<W, BLOOM><<<grid_part_[W - 1], kPartThreads, part_smem_bytes<W>(), stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.insert_ms, prof.t.insert_launches);
            if (W == 1 && compact_possible_)  // the plan picks one record format; the other kernel returns at once
                timed_launch([&] { k_exact_part_compact<BLOOM><<<grid_compact_, kPartThreads, compact_smem_bytes(), stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.insert_ms, prof.t.insert_launches);
            if (passes_ > 1) {
                k_pass_advance<<<1, 1, 0, stream_>>>(d_ctl_);
                check(cudaGetLastError(), "pass advance");
            }
        }
        timed_launch([&] { k_append<W><<<grid_, kThreads, 0, stream_>>>(d_params_, d_ctl_, b_); },
                     prof.t.append_ms, prof.t.append_launches);
    }

    // ---- CUDA graphs of round chunks ---------------------------------
    // Every round kernel takes its sizes from device memory (Params,
    // Control), so a chunk of `count` rounds is the same launch sequence
    // for every chunk of that length: it is captured once per (W, mode,
    // passes, count, buffer set) and replayed with one cudaGraphLaunch
    // instead of 3-5 launches per round. A buffer reallocation changes the
    // kernels' by-value Bufs, so the cached graph no longer matches and a
    // new one is captured. Profiling runs (per-kernel events) and
    // ETWG_GRAPHS=0 launch kernel by kernel.
    struct RoundGraph {
        int W, mode, count;
        unsigned passes;
        Bufs bufs;
        cudaGraphExec_t exec;
        uint64_t launches[4];  // kernel / expand / insert / append launches per replay
    };
    std::vector<RoundGraph> graphs_;
    int use_graphs_ = -1;

    void drop_graphs() {
        for (RoundGraph& g : graphs_) cudaGraphExecDestroy(g.exec);
        graphs_.clear();
    }

    template <int W>
    void launch_rounds(const DpConfig& cfg, int count) {
        if (use_graphs_ < 0) {
            const char* e = std::getenv("ETWG_GRAPHS");
            use_graphs_ = !(e && std::atoi(e) == 0);
        }
        if (prof.on || !use_graphs_) {
            for (int i = 0; i < count; ++i) launch_round<W>(cfg);
            return;
        }
        const int mode = (cfg.dedup == DedupMode::exact_set ? 1 : 0) | (cfg.use_mmw ? 2 : 0) | (part_bloom_ ? 4 : 0) |
                         (gtab_ ? 8 : 0) | (compact_possible_ ? 16 : 0);
        for (RoundGraph& g : graphs_) {
            if (g.W == W && g.mode == mode && g.count == count && g.passes == passes_ &&
                std::memcmp(&g.bufs, &b_, sizeof(Bufs)) == 0) {
                check(cudaGraphLaunch(g.exec, stream_), "graph launch");
                prof.t.kernel_launches += g.launches[0];
                prof.t.expand_launches += g.launches[1];
                prof.t.insert_launches += g.launches[2];
                prof.t.append_launches += g.launches[3];
                return;
            }
        }
        const uint64_t before[4] = {prof.t.kernel_launches, prof.t.expand_launches, prof.t.insert_launches,
                                    prof.t.append_launches};
        cudaGraph_t graph = nullptr;
        check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "graph capture");
        for (int i = 0; i < count; ++i) launch_round<W>(cfg);
        check(cudaStreamEndCapture(stream_, &graph), "graph capture end");
        RoundGraph g{W, mode, count, passes_, b_, nullptr, {}};
        check(cudaGraphInstantiate(&g.exec, graph, 0), "graph instantiate");
        cudaGraphDestroy(graph);
        g.launches[0] = prof.t.kernel_launches - before[0];
        g.launches[1] = prof.t.expand_launches - before[1];
        g.launches[2] = prof.t.insert_launches - before[2];
        g.launches[3] = prof.t.append_launches - before[3];
        if (graphs_.size() >= 48) {  // stale buffer sets / chunk lengths
            cudaGraphExecDestroy(graphs_.front().exec);
            graphs_.erase(graphs_.begin());
        }
        graphs_.push_back(g);
        check(cudaGraphLaunch(g.exec, stream_), "graph launch");  // (the capture counted this replay's launches)
    }

    void fetch_control() {
        copy(h_ctl_, d_ctl_, sizeof(Control), cudaMemcpyDeviceToHost, "control d2h");
        check(cudaStreamSynchronize(stream_), "sync");
        // the device advanced the look-back epoch once per round; continue
        // from there (a wrap past 2^24 clears the status array)
        if (h_ctl_->epoch < epoch_) {
            epoch_ = h_ctl_->epoch;
            clear_tagged();
        } else {
            epoch_ = h_ctl_->epoch;
        }
    }

    void run_rounds(int W, const DpConfig& cfg, int rounds, int k, const LayerObserver* observer) {
        NvtxRange nvtx("rounds W=%d", W);
        if (!ensure_parts(u64{1} << 21, u64{1} << 22)) throw DeviceError("device engine: no memory for records");
        ensure_bloom(u64{1} << 22);
        ensure_claims(u64{1} << 20);
        bloom_round_ = cfg.dedup == DedupMode::bloom;
        // Bloom filters beyond 2^28 bits (32 MB: random probes stop hitting L2)
        // take the partitioned path: exact per-bucket dedup in shared memory,
        // then the filter on each distinct key once (17 probes per distinct
        // child instead of per offered child)
        // (and MMW decides: their small layers run the warp-per-parent scatter)
        part_bloom_ = bloom_round_ &&
                      (bloom_bits_for(cfg.max_layer_states, cfg.bloom_bits_per_element) > (u64{1} << 28) ||
                       cfg.use_mmw) &&
                      !(h_params_->flags & 64);
        if (bloom_round_) clean_blooms();
        gtab_ = W == 1 && h_params_->gtab > 0;
        if (gtab_) ensure_tab(u64{1} << h_params_->gtab);
        if (!prof.on) check(cudaEventRecord(ev_[0], stream_), "event");
        auto t0 = std::chrono::steady_clock::now();
        const bool sync_each = (h_params_->flags & 8) != 0;
        int chunk = observer || sync_each ? 1 : 4;
        for (;;) {
            const int start = static_cast<int>(h_ctl_->round);
            const int end = std::min(rounds, start + chunk);
            NvtxRange chunk_range("round chunk %d..%d", start, end - 1);
            if (epoch_ + static_cast<unsigned>(end - start) + 1 >= kEpochMask) {
                // the device advances the epoch once per round and would wrap
                // inside this chunk: restart the tags from a cleared state now
                epoch_ = 1;
                clear_tagged();
                h_ctl_->epoch = epoch_;
                copy(&d_ctl_->epoch, &h_ctl_->epoch, sizeof(unsigned), cudaMemcpyHostToDevice, "epoch reset");
            }
            if (W == 1)
                launch_rounds<1>(cfg, end - start);
            else
                launch_rounds<2>(cfg, end - start);
            fetch_control();
            Control& c = *h_ctl_;
            if (c.abort != kOk) {
                grow(c, W);
                continue;
            }
            if (observer) {
                for (int r = start; r < static_cast<int>(c.round); ++r) {
                    // chunk == 1: exactly one round ran
                    std::vector<State> layer = fetch_layer((r + 1) & 1, c.rs[r].emitted, W);
                    (*observer)(k, r, layer);
                }
            }
            if (c.stop || static_cast<int>(c.round) >= rounds) break;
            if (!observer && !sync_each) chunk = std::min(chunk * 2, 32);  // observer: one round per check
        }
        if (bloom_round_) {  // the last round's filter is left dirty
            int last = -1;
            for (int r = 0; r < rounds; ++r)
                if (h_ctl_->rs[r].valid) last = r;
            if (last >= 0)
                bloom_dirty_[last & 1] = std::max<u64>(
                    bloom_dirty_[last & 1],
                    bloom_bits_for(host_round_cap(h_ctl_->rs[last].expanded), h_params_->bpe) / 32);
        }
        if (!prof.on) {
            check(cudaEventRecord(ev_[1], stream_), "event");
            check(cudaEventSynchronize(ev_[1]), "event sync");
            float t = 0;
            cudaEventElapsedTime(&t, ev_[0], ev_[1]);
            prof.t.decide_ms += t;
        } else {
            prof.t.decide_ms +=
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
    }

    // Grows the structure an aborted round asked for and re-arms the round.
    void grow(Control& c, int W) {
        NvtxRange nvtx("grow abort=%u", c.abort);
        const unsigned r = c.round;
        const u64 tab_dirty = gtab_ && c.rs[r].gtab ? c.rs[r].pcap : 0;  // inserts of the aborted round
        if (bloom_round_) {  // the aborted attempt may have set bits in filter r&1
            bloom_dirty_[r & 1] = std::max<u64>(
                bloom_dirty_[r & 1], bloom_bits_for(host_round_cap(c.count[r & 1]), h_params_->bpe) / 32 + 1);
        }
        if (std::getenv("ETWG_TRACE"))
            std::fprintf(stderr, "[engine] round %u abort %u need %llu (E=%llu np=%llu pcap=%llu)\n", r, c.abort,
                         static_cast<unsigned long long>(c.need), static_cast<unsigned long long>(c.count[r & 1]),
                         static_cast<unsigned long long>(c.rs[r].np), static_cast<unsigned long long>(c.rs[r].pcap));
        switch (c.abort) {
            case kGrowLayer:
                ensure_layers(c.need + c.need / 2, static_cast<int>(r & 1), c.count[r & 1]);
                break;
            case kGrowParts: {
                // more partitions: each gets proportionally fewer records, so a
                // record floor raised at the old partition count shrinks with it
                // (a fixed floor times a doubling partition count grew the record
                // buffer without bound under repeated table overflows)
                const u64 np_old = std::max<u64>(c.rs[r].np, 1);
                const u64 np_new = std::max<u64>(c.part_floor, c.need);
                if (np_new > np_old) c.rec_floor = c.rec_floor * np_old / np_new;
                c.part_floor = np_new;
                clean_cursors();
                break;
            }
            case kGrowRecs:
                c.rec_floor = std::max<u64>(c.rec_floor, c.need);
                clean_cursors();
                break;
            case kGrowPartBuf:
                // f4: child records beyond HBM -> twice the hash-range passes
                // per round (K1 reruns per pass; same layers, same counters)
                while (!ensure_parts(c.need + c.need / 4, 0)) {
                    if (passes_ >= 1024) throw DeviceError("device engine: child records exceed device memory");
                    passes_ *= 2;
                    c.passes = passes_;
                    c.need = (c.need + 1) / 2;
                    if (std::getenv("ETWG_TRACE"))
                        std::fprintf(stderr, "[engine] records do not fit: %u hash-range passes per round\n", passes_);
                }
                clean_cursors();
                break;
            case kGrowBloom:
                ensure_bloom(c.need + c.need / 4);
                break;
            case kGrowTable:  // beyond 2^gtab slots the plan falls back to buckets
                c.tab_floor = std::max<u64>(c.tab_floor, c.need);
                break;
            case kGrowClaims:
                ensure_claims(c.need);
                break;
            default:
                throw DeviceError("device engine: unknown abort code");
        }
        if (bloom_round_) clean_blooms();
        clean_table(tab_dirty);
        // re-arm: clear the abort and the partial statistics of round r
        c.abort = kOk;
        c.need = 0;
        c.exits = 0;
        c.pass = 0;
        c.epoch = next_epoch();  // statuses of the aborted attempt must not match
        std::memset(&c.rs[r], 0, sizeof(RoundStats) * (kMaxRounds - r));
        copy(d_ctl_, h_ctl_, sizeof(Control), cudaMemcpyHostToDevice, "control re-arm");
    }

    State fetch_state(int buf, u64 i, int W) {
        u64 k[2] = {0, 0};
        unsigned h = 0;
        copy(k, b_.keys[buf] + W * i, 8 * W, cudaMemcpyDeviceToHost, "witness");
        copy(&h, b_.hist[buf] + i, 4, cudaMemcpyDeviceToHost, "witness");
        check(cudaStreamSynchronize(stream_), "sync");
        State s;
        s.set.w[0] = k[0];
        s.set.w[1] = W == 2 ? k[1] : 0;
        s.history = h;
        return s;
    }

    std::vector<State> fetch_layer(int buf, u64 count, int W) {
        std::vector<u64> keys(static_cast<size_t>(W) * count);
        std::vector<unsigned> hist(count);
        if (count) {
            copy(keys.data(), b_.keys[buf], keys.size() * 8, cudaMemcpyDeviceToHost, "layer d2h");
            copy(hist.data(), b_.hist[buf], count * 4, cudaMemcpyDeviceToHost, "layer d2h");
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

    // SURVEY §8d algorithmic bytes: W*E_in + W*E_out + D*P per round
    void account(const std::vector<LayerStats>& rounds, int W, const DpConfig& cfg) {
        const double wb = 8.0 * W + 4.0, sb = 8.0 * W;
        const bool bloom = cfg.dedup == DedupMode::bloom;
        const double db = bloom ? 4.0 * cfg.bloom_hashes : (W == 1 ? 16.0 : 24.0);
        for (const LayerStats& s : rounds) {
            const double E = static_cast<double>(s.expanded), U = static_cast<double>(s.emitted);
            const double P = static_cast<double>(s.emitted + s.duplicates);
            prof.t.layer_bytes += wb * (E + U);
            prof.t.dedup_bytes += db * P;
            prof.t.expanded += s.expanded;
            prof.t.offered += s.emitted + s.duplicates;
            prof.t.unique += s.emitted;
            if (bloom) {
                // k_bloom_dedup: parent read + novel-mask write + h probe words per child
                prof.t.insert_bytes += 2 * sb * E + db * P;
            } else if (W == 1 && s.round >= 0 && s.round < kMaxRounds && h_ctl_->rs[s.round].gtab) {
                // global table: k_exact_scatter reads the parent, clears its
                // winner mask, reads one 16-byte slot per offered child and
                // writes one per distinct key; k_tab_mark streams the table
                // (pcap slots), clears each used slot, ORs the winner's bit
                const double slots = s.round >= 0 && s.round < kMaxRounds
                                         ? static_cast<double>(h_ctl_->rs[s.round].pcap) : 0.0;
                prof.t.expand_bytes += 2 * sb * E + 16.0 * P + 16.0 * U;
                prof.t.insert_bytes += 16.0 * slots + 16.0 * U + 8.0 * U;
            } else {
                // k_exact_scatter: parent read, winner-mask clear, one record per child;
                // k_exact_part: record read, one winner-mask OR per distinct key
                // (compact rounds: 8-byte records, plus the parent's set read
                // back per distinct key)
                // Records are the children left after the producers' swap
                // pre-dedup (RoundStats::winners), not every offered child.
                const bool in_range = s.round >= 0 && s.round < kMaxRounds;
                const bool compact = in_range && h_ctl_->rs[s.round].compact;
                const double R = in_range && h_ctl_->rs[s.round].winners ? static_cast<double>(h_ctl_->rs[s.round].winners) : P;
                const double rec = compact ? 8.0 : 8.0 * W + 8.0;
                prof.t.expand_bytes += 2 * sb * E + rec * R;
                prof.t.insert_bytes += rec * R + (compact ? 16.0 : 8.0) * U;
                if (!compact) prof.t.records += R;
                if (std::getenv("ETWG_TRACE") && in_range)
                    std::fprintf(stderr, "[engine] round %d expanded %llu offered %llu records %llu distinct %llu\n", s.round,
                                 static_cast<unsigned long long>(s.expanded), static_cast<unsigned long long>(P),
                                 static_cast<unsigned long long>(R), static_cast<unsigned long long>(U));
            }
            // k_append: parent + history + mask read, state + history written
            prof.t.append_bytes += (sb + 4.0 + sb) * E + wb * U;
        }
    }
};

}  // namespace

DecideResult device_decide(const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg,
                           int rounds, const LayerObserver* observer) {
    if (k < 0) throw std::invalid_argument("k must be non-negative");
    if (cfg.max_layer_states == 0) throw std::invalid_argument("layer capacity must be positive");
    if (shard_active()) return shard_decide(g, k, forbidden, cfg, rounds, observer);
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    return e.decide(g, k, forbidden, cfg, rounds, observer);
}

DecideResult device_decide_prefix(const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg,
                                  int rounds, const LayerObserver* observer, uint64_t handoff_above,
                                  EngineLayer& handoff) {
    if (k < 0) throw std::invalid_argument("k must be non-negative");
    if (cfg.max_layer_states == 0) throw std::invalid_argument("layer capacity must be positive");
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    handoff.handed = false;
    return e.decide(g, k, forbidden, cfg, rounds, observer, handoff_above, &handoff);
}

void engine_release_buffers() {
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    e.release_buffers();
}

void engine_bind_device(int dev) {
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    e.bind_device(dev);
}

int engine_device() {
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    return e.ready() ? e.info().device : -1;
}

ExpandResult device_expand_layer(const Graph& g, int k, const HostSet& forbidden,
                                 const std::vector<State>& input, const DpConfig& cfg,
                                 LayerStats& stats) {
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    return e.expand_layer(g, k, forbidden, input, cfg, stats);
}

uint64_t device_bloom_insert(uint64_t expected, int bpe, int hashes,
                             const std::vector<uint64_t>& keys, int words, std::vector<uint8_t>& novel,
                             std::vector<uint32_t>* bits) {
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    return e.bloom_batch(expected, bpe, hashes, keys, words, novel, bits);
}

bool device_available(DeviceInfo* info) {
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    bool ok = e.ready();
    if (ok && info) *info = e.info();
    return ok;
}

void engine_timer_begin() {
    if (shard_active()) return shard_timer_begin();
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    e.timer_begin();
}

double engine_timer_end() {
    if (shard_active()) return shard_timer_end();
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    return e.timer_end();
}

void engine_set_profiling(bool on) {
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    e.prof.on = on;
}

KernelTimes engine_times() {
    KernelTimes t;
    {
        Engine& e = Engine::instance();
        std::lock_guard<std::mutex> lock(e.mu);
        t = e.prof.t;
    }
    shard_accumulate(t);
    return t;
}

void engine_reset_times() {
    {
        Engine& e = Engine::instance();
        std::lock_guard<std::mutex> lock(e.mu);
        e.prof.t = KernelTimes{};
    }
    shard_reset_times();
}

}  // namespace etw
