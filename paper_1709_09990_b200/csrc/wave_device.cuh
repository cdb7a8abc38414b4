// Device building blocks shared by the single-device engine (wavefront.cu)
// and the owner-sharded engine (shard.cu): vertex-set access, the Q(S,v)
// candidate test (graph.hpp:61-78 / dp.cpp:39-69), Murmur3 + Bloom probes
// (bloom.cpp:27-97), the exact open-addressing table (dp.cpp:118-151
// semantics) and the decoupled look-back scan used by every ordered append.
// Everything lives in an anonymous namespace: each .cu is its own device
// translation unit (no -rdc).
#pragma once

#include <cuda_runtime.h>

#include "mmw.hpp"
#include "vset.hpp"

namespace etw {
namespace {
constexpr int kThreads = 256;
constexpr int kMaxRounds = 130;
constexpr unsigned kFull = 0xffffffffu;
// Bloom stripe locks. The reference uses 65,536 mutex stripes keyed by
// h1 (bloom.cpp:18-23); any key -> stripe map keeps inserts of one key
// serialised, and ~10^5 concurrent device threads need more stripes to keep
// unrelated keys from contending.
constexpr int kStripes = 1 << 20;
constexpr unsigned kSeed1 = 0x9747B28Cu;  // bloom.hpp:24
constexpr unsigned kSeed2 = 0x5EEDBA5Eu;  // bloom.hpp:25

using u64 = unsigned long long;

#ifndef ETWG_SWAP_DEDUP
#define ETWG_SWAP_DEDUP 1  // sibling swap pre-dedup of each warp's 32 parents (k_exact_scatter, k_route)
#endif

struct Params {
    int n, k, rounds, free_count;
    int hashes, bpe, any_pop, flags;  // flags: ETWG_DEBUG bits (tests only)
    int gtab, pad_;                   // >0: exact rounds whose table fits 2^gtab slots dedup in a global table
    u64 max_states;
    u64 forbidden[2];
    u64 rows[kMaxVertices][2];
};

// ----------------------------------------------------------------------
// small device helpers

template <int W>
__device__ __forceinline__ Set<W> load_set(const u64* p, u64 i) {
    Set<W> s;
    if constexpr (W == 1) {
        s.w[0] = p[i];
    } else {
        ulonglong2 v = reinterpret_cast<const ulonglong2*>(p)[i];
        s.w[0] = v.x;
        s.w[1] = v.y;
    }
    return s;
}

template <int W>
__device__ __forceinline__ void store_set(u64* p, u64 i, const Set<W>& s) {
    if constexpr (W == 1) {
        p[i] = s.w[0];
    } else {
        reinterpret_cast<ulonglong2*>(p)[i] = make_ulonglong2(s.w[0], s.w[1]);
    }
}

template <int W>
__device__ __forceinline__ Set<W> shfl_set(const Set<W>& s, int src) {
    Set<W> r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.w[i] = __shfl_sync(kFull, s.w[i], src);
    return r;
}

// position of the r-th (0-based) set bit of x; requires popc(x) > r
__device__ __forceinline__ int nth_bit64(u64 x, int r) {
    int pos = 0;
#pragma unroll
    for (int w = 32; w >= 1; w >>= 1) {
        u64 low = x & ((u64{1} << w) - 1);
        int c = __popcll(low);
        if (r >= c) {
            r -= c;
            x >>= w;
            pos += w;
        }
    }
    return pos;
}

template <int W>
__device__ __forceinline__ int nth_member(const Set<W>& s, int r) {
    if constexpr (W == 1) {
        return nth_bit64(s.w[0], r);
    } else {
        int c0 = __popcll(s.w[0]);
        return r < c0 ? nth_bit64(s.w[0], r) : 64 + nth_bit64(s.w[1], r - c0);
    }
}

// Warp-wide flattening of per-lane child masks: after scan(), iteration t
// hands lane l the child number t*32+l in (lane, vertex) order.
struct WarpFlat {
    int cnt, incl, total;
    __device__ __forceinline__ void scan(int c) {
        const int lane = threadIdx.x & 31;
        cnt = c;
        incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        total = __shfl_sync(kFull, incl, 31);
    }
    // lane holding child j (warp-uniform control flow required)
    __device__ __forceinline__ int source(int j) const {
        int src = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            int c = __shfl_sync(kFull, incl, src + step - 1);
            if (c <= j) src += step;
        }
        return src > 31 ? 31 : src;
    }
};

__device__ __forceinline__ u64 fmix64(u64 k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ULL;
    k ^= k >> 33;
    return k;
}

template <int W>
__device__ __forceinline__ u64 slot_hash(const Set<W>& s) {
    u64 h = fmix64(s.w[0]);
    if constexpr (W == 2) h = fmix64(h ^ (s.w[1] + 0x9E3779B97F4A7C15ULL));
    return h;
}

// Murmur3 x86_32 over the little-endian bytes of the key (bloom.cpp:27-64):
// 8 bytes for n <= 64 (the reference key, bloom.cpp:66-70), 16 for n <= 128.
__device__ __forceinline__ unsigned rotl32(unsigned x, int r) { return __funnelshift_l(x, x, r); }

template <int W>
__device__ __forceinline__ unsigned murmur_key(const Set<W>& key, unsigned seed) {
    unsigned h = seed;
#pragma unroll
    for (int i = 0; i < 2 * W; ++i) {
        unsigned k = static_cast<unsigned>(key.w[i >> 1] >> (32 * (i & 1)));
        k *= 0xcc9e2d51u;
        k = rotl32(k, 15);
        k *= 0x1b873593u;
        h ^= k;
        h = rotl32(h, 13);
        h = h * 5 + 0xe6546b64u;
    }
    h ^= 8u * W;
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

__host__ __device__ __forceinline__ u64 bloom_bits_for(u64 expected, int bpe) {
    u64 bits = expected * static_cast<u64>(bpe);
    u64 m = (bits + 63) / 64 * 64;  // bloom.cpp:74-75
    return m < 64 ? 64 : m;
}

__host__ __device__ __forceinline__ u64 round_cap(const Params& p, u64 e_in) {
    u64 upper = e_in * static_cast<u64>(p.free_count);  // dp.cpp:84-86
    if (upper < 1) upper = 1;
    return p.max_states < upper ? p.max_states : upper;
}

__host__ __device__ __forceinline__ u64 table_slots_for(u64 offered) {
    u64 want = 2 * offered + 1024;
    u64 s = 1024;
    while (s < want) s <<= 1;
    return s;
}

template <int W>
__device__ __forceinline__ Set<W> param_set(const u64 (&w)[2]) {
    Set<W> s;
#pragma unroll
    for (int i = 0; i < W; ++i) s.w[i] = w[i];
    return s;
}

// ----------------------------------------------------------------------
// K1: candidate evaluation (replaces expand_range + q_set, dp.cpp:39-69,
// graph.hpp:61-78, and the MMW prune driven at dp.cpp:51-63)

// Slot of member u of S in the per-parent boundary table R. Vertex-indexed
// (COMPACT = false) costs nothing; rank-indexed (COMPACT = true, the rank of
// u among S's members) keeps a warp's touched slots within the first |S|
// entries when the warp's parents are unrelated (a sharded layer is in hash
// order), so its slice of local memory stays L1-resident. Measured: vertex
// indexing is faster on rank-ordered layers (single device), rank indexing
// on hash-ordered ones (shards).
template <int W, bool COMPACT>
__device__ __forceinline__ int reach_slot(const Set<W>& S, int u) {
    if constexpr (!COMPACT) {
        return u;
    } else if constexpr (W == 1) {
        return __popcll(S.w[0] & ((u64{1} << u) - 1));
    } else {
        return u < 64 ? __popcll(S.w[0] & ((u64{1} << u) - 1))
                      : __popcll(S.w[0]) + __popcll(S.w[1] & ((u64{1} << (u - 64)) - 1));
    }
}

// For every u in S: R[slot(u)] = N(K_u) \ S, the outside boundary of u's
// component K_u of G[S] (flood fill over bitmask rows, one pass per
// component). Components without outside neighbours touch no candidate.
template <int W, bool COMPACT>
__device__ __forceinline__ void component_reach(const Set<W>* adj, const Set<W>& S, Set<W>* R) {
    Set<W> rem = S;
    while (rem.any()) {
        Set<W> frontier = rem;
        Set<W> comp = Set<W>::bit(pop_any(frontier));  // any seed
        frontier = comp;
        Set<W> nb = Set<W>::zero();
        while (frontier.any()) {
            const Set<W> a = adj[pop_any(frontier)];
            nb |= a;
            Set<W> fresh = (a & S) - comp;
            comp |= fresh;
            frontier |= fresh;
        }
        rem = rem - comp;
        const Set<W> boundary = nb - S;
        if (boundary.none()) continue;
        for_each_any(comp, [&](int u) { R[reach_slot<W, COMPACT>(S, u)] = boundary; });
    }
}

// Q(S,v) (graph.hpp:61-78): v's own outside neighbours plus the boundary of
// every component of G[S] that v touches, i.e. of K_u for u in N(v) & S.
// Costs |N(v) & S| mask ORs instead of a DFS per (S, v).
template <int W, bool COMPACT>
__device__ __forceinline__ Set<W> reach_from(const Set<W>* adj, const Set<W>& S, const Set<W>* R,
                                             int v) {
    Set<W> q = adj[v] - S;
    for_each_any(adj[v] & S, [&](int u) { q |= R[reach_slot<W, COMPACT>(S, u)]; });
    q.del(v);
    return q;
}

// Minor-min-width on eliminate(G, S + v) (init_view_after, mmw.cpp:20-43,
// then run_mmw / contract_step, mmw.cpp:81-140) with the minor held
// explicitly as bitmask rows: nb[w] starts as Q(S+v, w) — rows[w], plus
// rows[v] when w is in it — and a contraction of (x, u) is one mask union
// plus |N(u)| row edits, instead of the shared contraction loop's DFS
// through eliminated vertices per step. Same choices as the reference:
// min degree, smallest index on ties; its min-degree neighbour, smallest
// index on ties; degree-0 classes dropped; degrees updated by
// deg[x] + deg[u] - c - 2 and -1 for the c common neighbours. Returns
// early once the bound exceeds cap.
template <int W>
__device__ int mmw_child(int n, int cap, const Set<W>& S, int v, const Set<W>* rows) {
    constexpr int N = 64 * W;
    Set<W> nb[N];
    unsigned char deg[N];
    Set<W> alive = Set<W>::prefix(n) - S;
    alive.del(v);
    const Set<W> rv = rows[v];
    for (int w : members(alive)) {
        Set<W> a = rows[w];
        if (rv.has(w)) a |= rv;  // eliminating v joins Q(S,v) into a clique
        a.del(v);
        a.del(w);
        nb[w] = a;
        deg[w] = static_cast<unsigned char>(a.count());
    }
    int bound = 0;
    while (alive.count() >= 2) {
        int d1 = 1 << 30, d2 = 1 << 30, x1 = -1;
        for (int x : members(alive)) {
            const int d = deg[x];
            if (d < d1) {
                d2 = d1;
                d1 = d;
                x1 = x;
            } else if (d < d2) {
                d2 = d;
            }
        }
        if (d2 > bound) bound = d2;
        if (bound > cap) return bound;
        if (d1 == 0) {  // isolated class: drop it
            alive.del(x1);
            continue;
        }
        int u = -1, du = 1 << 30;
        for (int x : members(nb[x1])) {
            if (deg[x] < du) {
                du = deg[x];
                u = x;
            }
        }
        const Set<W> nu = nb[u];
        const Set<W> common = nb[x1] & nu;
        Set<W> merged = nb[x1] | nu;
        merged.del(x1);
        merged.del(u);
        nb[x1] = merged;
        deg[x1] = static_cast<unsigned char>(deg[x1] + deg[u] - common.count() - 2);
        alive.del(u);
        Set<W> moved = nu;
        moved.del(x1);
        for (int x : members(moved)) {
            nb[x].del(u);
            nb[x].add(x1);
        }
        for (int x : members(common)) --deg[x];
    }
    return bound;
}

// Rank-indexed per-thread boundary table in shared memory, strided by the
// block size (slot j of thread t at [j * blockDim.x + t]): for hash-ordered
// (sharded) layers, whose warps touch unrelated slots, the local-memory
// table thrashes L1. Parents with more than kShSlots members use the
// local-memory table.
constexpr int kShSlots = 24;

template <int W>
__device__ __forceinline__ Set<W> candidates_shared(const Set<W>* adj, int k, const Set<W>& S,
                                                    const Set<W>& eligible, Set<W>* Rsh) {
    Set<W>* R = Rsh + threadIdx.x;
    const int stride = blockDim.x;
    Set<W> rem = S;
    while (rem.any()) {
        Set<W> frontier = rem;
        Set<W> comp = Set<W>::bit(pop_any(frontier));
        frontier = comp;
        Set<W> nb = Set<W>::zero();
        while (frontier.any()) {
            const Set<W> a = adj[pop_any(frontier)];
            nb |= a;
            Set<W> fresh = (a & S) - comp;
            comp |= fresh;
            frontier |= fresh;
        }
        rem = rem - comp;
        const Set<W> boundary = nb - S;
        if (boundary.none()) continue;
        for_each_any(comp, [&](int u) { R[reach_slot<W, true>(S, u) * stride] = boundary; });
    }
    Set<W> keep = Set<W>::zero();
    for_each_any(eligible, [&](int v) {
        Set<W> q = adj[v] - S;
        if (q.count() > k) return;  // |Q(S,v)| >= |N(v) \ S|
        for_each_any(adj[v] & S, [&](int u) { q |= R[reach_slot<W, true>(S, u) * stride]; });
        q.del(v);
        if (q.count() <= k) keep.add(v);
    });
    return keep;
}

// K1 with the boundaries in registers (the degree test of expand_range,
// dp.cpp:55-56, on Q(S,v) of graph.hpp:61-78). Q(S,v) = N(v)\S plus the
// outside boundary B_K of every component K of G[S] that v touches, and v
// touches K exactly when v is in B_K. So instead of a per-vertex table
// R[u] = B_{K(u)} (64 entries per thread, local memory, read at a
// different index by every lane of a warp), the components are kept as a
// short list of boundaries:
//   * a component whose boundary misses every eligible vertex is dropped;
//   * one whose boundary has more than k+1 vertices rejects all of them
//     (|Q(S,v)| >= |B_K| - 1 > k), one mask for all such components;
//   * an isolated member u of S (boundary N(u)) goes into a mask and is
//     read back from the shared adjacency rows;
//   * every other component takes a register slot (kSlotRegs of them;
//     further ones go to a local array walked with a loop-uniform index, so
//     those loads stay coalesced). Measured on G(40,0.3) / G(48,0.2) layers:
//     parents have 0-4 multi-vertex components, >4 in ~1 % of them.
// The flood fill is one flat loop of exactly |S| pops (|S| is the round
// number, the same for every lane), and the candidate loop runs over the
// eligible set, whose size n - |S| - |forbidden| is also warp-uniform.
#ifndef ETWG_K1
#define ETWG_K1 4  // 4: half-word register slots (one-word keys); 2: register slots + isolated-member loop; 1: per-vertex table
#endif
#ifndef ETWG_K1_LOOP
#define ETWG_K1_LOOP 2  // 1: two 32-bit half loops with an early |N(v) \ S| > k exit
#endif
#ifndef ETWG_SLOT_REGS
#define ETWG_SLOT_REGS 4
#endif
constexpr int kSlotRegs = ETWG_SLOT_REGS;

template <int W>
__device__ __forceinline__ bool single_member(const Set<W>& s) {
    if constexpr (W == 1) {
        return (s.w[0] & (s.w[0] - 1)) == 0;
    } else {
        return s.count() == 1;
    }
}

template <int W>
struct Comps {
    Set<W> slot[kSlotRegs];  // constant-index access only: stays in registers
    Set<W> sing, reject;
    int ns;
    // multi-vertex components beyond the register slots live in a separate
    // local array (kept out of the struct so the struct stays in registers)
    using Spill = Set<W>[32 * W];

    // The components of G[S] whose boundary meets `targets`; a boundary of
    // more than `reject_above` vertices goes to `reject` instead of a slot.
    __device__ __forceinline__ void build(const Set<W>* adj, const Set<W>& S, const Set<W>& targets,
                                          int reject_above, Spill& spill) {
#pragma unroll
        for (int j = 0; j < kSlotRegs; ++j) slot[j] = Set<W>::zero();
        sing = reject = Set<W>::zero();
        ns = 0;
        Set<W> rem = S, frontier = Set<W>::zero(), comp = Set<W>::zero(), nb = Set<W>::zero();
        const int r = S.count();
        for (int it = 0; it < r; ++it) {
            if (frontier.none()) {  // next component: seed from the unvisited members
                frontier = Set<W>::bit(pop_any(rem));
                comp = frontier;
                nb = Set<W>::zero();
            }
            const Set<W> a = adj[pop_any(frontier)];
            nb |= a;
            const Set<W> fresh = a & rem;
            rem = rem - fresh;
            comp |= fresh;
            frontier |= fresh;
            if (frontier.any()) continue;
            const Set<W> B = nb - S;  // the finished component's outside boundary
            if ((B & targets).none()) continue;
            if (B.count() > reject_above) {
                reject |= B;
            } else if (single_member<W>(comp)) {
                sing |= comp;
            } else {
#pragma unroll
                for (int j = 0; j < kSlotRegs; ++j)
                    if (ns == j) slot[j] = B;
                if (ns >= kSlotRegs) spill[ns - kSlotRegs] = B;
                ++ns;
            }
        }
    }

    // Q(S,v) \ {v} from its first term N(v) \ S = a - S (exact for v in
    // `targets` outside `reject`)
    __device__ __forceinline__ Set<W> q(const Set<W>* adj, const Set<W>& a, Set<W> q0, int v,
                                        const Spill& spill) const {
        Set<W> x = a & sing;
        while (x.any()) q0 |= adj[pop_any(x)];
#pragma unroll
        for (int j = 0; j < kSlotRegs; ++j)
            if (slot[j].has(v)) q0 |= slot[j];
        for (int j = kSlotRegs; j < ns; ++j)
            if (spill[j - kSlotRegs].has(v)) q0 |= spill[j - kSlotRegs];
        q0.del(v);
        return q0;
    }

    __device__ __forceinline__ Set<W> q(const Set<W>* adj, const Set<W>& S, int v, const Spill& spill) const {
        const Set<W> a = adj[v];
        return q(adj, a, a - S, v, spill);
    }
};

template <int W>
__device__ __forceinline__ Set<W> candidates_slots(const Set<W>* adj, int k, const Set<W>& S,
                                                   const Set<W>& eligible) {
    Comps<W> c;
    typename Comps<W>::Spill spill;
    c.build(adj, S, eligible, k + 1, spill);  // |Q(S,v)| >= |B_K| - 1 for v in B_K
    Set<W> keep = Set<W>::zero();
#if ETWG_K1_LOOP == 1
    for_each_any(eligible - c.reject, [&](int v) {
        const Set<W> a = adj[v];
        const Set<W> q0 = a - S;
        if (q0.count() > k) return;  // |Q(S,v)| >= |N(v) \ S|
        if (c.q(adj, a, q0, v, spill).count() <= k) keep.add(v);
    });
#else
    // one loop over the candidates (|eligible| is warp-uniform, so no lane
    // idles), no early exit: the final test implies |N(v) \ S| <= k
    Set<W> cand = eligible - c.reject;
    while (cand.any()) {
        const int v = pop_any(cand);
        const Set<W> a = adj[v];
        if (c.q(adj, a, a - S, v, spill).count() <= k) keep.add(v);
    }
#endif
    return keep;
}

// K1 for one-word keys with every relevant component in a register slot
// (isolated members too: their boundary is their row), held as 32-bit halves.
// The candidate loop runs once over the low and once over the high half of
// the candidate mask, so a candidate's bit lies in a known half: testing
// whether v touches a component is one AND on that half of its boundary,
// and the whole test costs ~3 instructions per slot, no inner loop.
// Components beyond kHalfSlots go to a local array walked with a
// loop-uniform index (rare: stats in DESIGN.md §4).
#ifndef ETWG_HALF_SLOTS
#define ETWG_HALF_SLOTS 8
#endif
constexpr int kHalfSlots = ETWG_HALF_SLOTS;

__device__ __forceinline__ u64 candidates_half(const Set<1>* adj, int k, u64 S, u64 eligible) {
    unsigned slo[kHalfSlots], shi[kHalfSlots];
#pragma unroll
    for (int j = 0; j < kHalfSlots; ++j) slo[j] = shi[j] = 0;
    u64 spill[32];
    int ns = 0;
    u64 reject = 0;
    u64 rem = S, frontier = 0, nb = 0, comp = 0;
    const int r = __popcll(S);
    for (int it = 0; it < r; ++it) {
        if (!frontier) {
            frontier = u64{1} << (63 - __clzll(rem));
            rem ^= frontier;
            comp = frontier;
            nb = 0;
        }
        const int x = 63 - __clzll(frontier);
        frontier ^= u64{1} << x;
        const u64 a = adj[x].w[0];
        nb |= a;
        const u64 fresh = a & rem;
        rem ^= fresh;
        comp |= fresh;
        frontier |= fresh;
        if (frontier) continue;
        const u64 B = nb & ~S;
        if (!(B & eligible)) continue;
        if (__popcll(B) > k + 1) {
            reject |= B;
            continue;
        }
#pragma unroll
        for (int j = 0; j < kHalfSlots; ++j)
            if (ns == j) {
                slo[j] = static_cast<unsigned>(B);
                shi[j] = static_cast<unsigned>(B >> 32);
            }
        if (ns >= kHalfSlots) spill[ns - kHalfSlots] = B;
        ++ns;
    }
    const u64 cand = eligible & ~reject;
    const unsigned Slo = static_cast<unsigned>(S), Shi = static_cast<unsigned>(S >> 32);
    u64 keep = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        unsigned y = static_cast<unsigned>(cand >> (32 * h));
        while (y) {
            const int b = 31 - __clz(y);
            const unsigned bit = 1u << b;
            y ^= bit;
            const int v = 32 * h + b;
            const u64 a = adj[v].w[0];
            unsigned qlo = static_cast<unsigned>(a) & ~Slo, qhi = static_cast<unsigned>(a >> 32) & ~Shi;
#pragma unroll
            for (int j = 0; j < kHalfSlots; ++j) {
                if (((h ? shi[j] : slo[j]) & bit) != 0) {
                    qlo |= slo[j];
                    qhi |= shi[j];
                }
            }
            for (int j = kHalfSlots; j < ns; ++j) {
                const u64 Bj = spill[j - kHalfSlots];
                if ((Bj >> v) & 1) {
                    qlo |= static_cast<unsigned>(Bj);
                    qhi |= static_cast<unsigned>(Bj >> 32);
                }
            }
            if (h) qhi &= ~bit; else qlo &= ~bit;
            if (__popc(qlo) + __popc(qhi) <= k) keep |= u64{1} << v;
        }
    }
    return keep;
}

// Q(S,w) for every open w (the minor-min-width input, dp.cpp:51-53)
template <int W>
__device__ __forceinline__ void q_rows(const Set<W>* adj, const Set<W>& S, const Set<W>& open, Set<W>* rows) {
    Comps<W> c;
    typename Comps<W>::Spill spill;
    c.build(adj, S, open, 1 << 30, spill);
    for_each_any(open, [&](int w) { rows[w] = c.q(adj, S, w, spill); });
}

template <int W, bool MMW, bool COMPACT = false>
__device__ __forceinline__ Set<W> candidates(const Set<W>* adj, int n, int k, const Set<W>& S,
                                             const Set<W>& forbidden, u64& pruned, Set<W>* Rsh = nullptr) {
    constexpr int N = 64 * W;
    const Set<W> open = Set<W>::prefix(n) - S;
    const Set<W> eligible = open - forbidden;
    Set<W> keep = Set<W>::zero();
    if (eligible.none()) return keep;
    if constexpr (!MMW) {
        if constexpr (W == 1 && ETWG_K1 == 4) {
            keep.w[0] = candidates_half(adj, k, S.w[0], eligible.w[0]);
            return keep;
        }
        if (ETWG_K1 >= 2) return candidates_slots<W>(adj, k, S, eligible);
        if (Rsh && S.count() <= kShSlots) return candidates_shared<W>(adj, k, S, eligible, Rsh);
    }
    Set<W> R[N];
    if (ETWG_K1 < 2) component_reach<W, COMPACT>(adj, S, R);
    if constexpr (!MMW) {
        for_each_any(eligible, [&](int v) {
            if ((adj[v] - S).count() > k) return;  // |Q(S,v)| >= |N(v) \ S|
            if (reach_from<W, COMPACT>(adj, S, R, v).count() <= k) keep.add(v);
        });
    } else {
        Set<W> rows[N];  // dp.cpp:51-53: Q(S,w) for every open w
        if (ETWG_K1 >= 2)
            q_rows<W>(adj, S, open, rows);
        else
            for (int w : members(open)) rows[w] = reach_from<W, COMPACT>(adj, S, R, w);
        for (int v : members(eligible)) {
            if (rows[v].count() > k) continue;
            if (mmw_child<W>(n, k, S, v, rows) > k) {
                ++pruned;
                continue;
            }
            keep.add(v);
        }
    }
    return keep;
}

// Warp-collective candidate evaluation (call with all 32 lanes; `valid`
// marks lanes holding a parent). The degree test runs per parent; with MMW
// the surviving children are then flattened across the warp so each lane
// evaluates the minor-min-width bound of one child (dp.cpp:57-63) — a
// parent's children no longer run serially in one thread, which is what
// bounded small MMW layers. `scratch` is a per-thread row of 2W words in
// shared memory.
template <int W, bool MMW, bool COMPACT = false>
__device__ __forceinline__ Set<W> warp_candidates(const Set<W>* adj, int n, int k, const Set<W>& S, bool valid,
                                                  const Set<W>& forbidden, u64& pruned,
                                                  unsigned (*scratch)[2 * W], Set<W>* Rsh = nullptr) {
    u64 unused = 0;
    Set<W> M = valid ? candidates<W, false, COMPACT>(adj, n, k, S, forbidden, unused, Rsh) : Set<W>::zero();
    if constexpr (!MMW) {
        return M;
    } else {
        constexpr int N = 64 * W;
        const int lane = threadIdx.x & 31;
        const int wslot = threadIdx.x & ~31;
#pragma unroll
        for (int i = 0; i < 2 * W; ++i) scratch[threadIdx.x][i] = 0;
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
                Set<W> rows[N];  // dp.cpp:51-53: Q(S,w) for every open w
                if (ETWG_K1 >= 2) {
                    q_rows<W>(adj, Ss, Set<W>::prefix(n) - Ss, rows);
                } else {
                    Set<W> R[N];
                    component_reach<W, COMPACT>(adj, Ss, R);
                    for (int w : members(Set<W>::prefix(n) - Ss)) rows[w] = reach_from<W, COMPACT>(adj, Ss, R, w);
                }
                if (mmw_child<W>(n, k, Ss, v, rows) > k)
                    ++pruned;
                else
                    atomicOr(&scratch[wslot + src][v >> 5], 1u << (v & 31));
            }
        }
        __syncwarp();
        Set<W> keep;
#pragma unroll
        for (int i = 0; i < W; ++i)
            keep.w[i] = scratch[threadIdx.x][2 * i] | (static_cast<u64>(scratch[threadIdx.x][2 * i + 1]) << 32);
        return valid ? keep : Set<W>::zero();
    }
}

// Warp-per-parent candidate evaluation for small layers (call with all 32
// lanes, S warp-uniform). With one thread per parent a round of a few
// thousand states leaves the GPU idle and each thread walks ~n candidates
// (and, with MMW, ~n minor contractions) serially; here lane 0 flood-fills
// G[S] into the warp's shared boundary table R and the candidates (and
// their MMW bounds) are spread over the lanes. R (and `rows`, for MMW) are
// the warp's 64W-entry shared tables. Returns the warp-uniform keep mask;
// `pruned` counts this lane's MMW prunes.
template <int W, bool MMW>
__device__ __forceinline__ Set<W> warp_parent_candidates(const Set<W>* adj, int n, int k, const Set<W>& S,
                                                         const Set<W>& forbidden, u64& pruned, Set<W>* R,
                                                         Set<W>* rows) {
    const int lane = threadIdx.x & 31;
    const Set<W> open = Set<W>::prefix(n) - S;
    const Set<W> eligible = open - forbidden;
    if (eligible.none()) return Set<W>::zero();
#if ETWG_K1 >= 2
    // S is warp-uniform: every lane builds the same component list (no
    // serial lane-0 fill, no shared table)
    Comps<W> c;
    typename Comps<W>::Spill spill;
    c.build(adj, S, MMW ? open : eligible, MMW ? (1 << 30) : k + 1, spill);
#else
    if (lane == 0) component_reach<W, false>(adj, S, R);
    __syncwarp();
#endif
    Set<W> mine = Set<W>::zero();
    if constexpr (!MMW) {
        const int ne = eligible.count();
        for (int i = lane; i < ne; i += 32) {
            const int v = nth_member<W>(eligible, i);
            const Set<W> q0 = adj[v] - S;
            if (q0.count() > k) continue;
#if ETWG_K1 >= 2
            if (!c.reject.has(v) && c.q(adj, adj[v], q0, v, spill).count() <= k) mine.add(v);
#else
            if (reach_from<W, false>(adj, S, R, v).count() <= k) mine.add(v);
#endif
        }
    } else {
        const int no = open.count();
        for (int i = lane; i < no; i += 32) {  // dp.cpp:51-53: Q(S,w) for every open w
            const int w = nth_member<W>(open, i);
#if ETWG_K1 >= 2
            rows[w] = c.q(adj, S, w, spill);
#else
            rows[w] = reach_from<W, false>(adj, S, R, w);
#endif
        }
        __syncwarp();
        const int ne = eligible.count();
        for (int i = lane; i < ne; i += 32) {
            const int v = nth_member<W>(eligible, i);
            if (rows[v].count() > k) continue;
            if (mmw_child<W>(n, k, S, v, rows) > k)
                ++pruned;
            else
                mine.add(v);
        }
    }
    Set<W> keep;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        const unsigned lo = __reduce_or_sync(kFull, static_cast<unsigned>(mine.w[i]));
        const unsigned hi = __reduce_or_sync(kFull, static_cast<unsigned>(mine.w[i] >> 32));
        keep.w[i] = (static_cast<u64>(hi) << 32) | lo;
    }
    __syncwarp();  // R / rows are reused by the warp's next parent
    return keep;
}

template <int W>
__device__ __forceinline__ void load_adjacency(const Params* P, Set<W>* adj) {
    for (int i = threadIdx.x; i < P->n; i += blockDim.x) adj[i] = param_set<W>(P->rows[i]);
}

// ----------------------------------------------------------------------
// 128-bit global compare-and-swap (atom.global.cas.b128, sm_90+)

__device__ __forceinline__ void cas128(u64* addr, u64 exp_lo, u64 exp_hi, u64 new_lo, u64 new_hi,
                                       u64& old_lo, u64& old_hi) {
    asm volatile(
        "{\n\t.reg .b128 c, s, d;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 s, {%4, %5};\n\t"
        "atom.global.cas.b128 d, [%6], c, s;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(old_lo), "=l"(old_hi)
        : "l"(exp_lo), "l"(exp_hi), "l"(new_lo), "l"(new_hi), "l"(addr)
        : "memory");
}

template <int W>
__device__ __forceinline__ u64 child_rank(u64 parent_idx, int v) {
    return parent_idx * (64 * W) + static_cast<u64>(v);  // dp.cpp:66 (idx*64+v)
}

// Shared-memory open-addressing claim: the slot at `keys + W*h` becomes
// `key` if it was empty (0); true when the slot now holds `key`.
#ifndef ETWG_CLAIM_PEEK
#define ETWG_CLAIM_PEEK 1
#endif
template <int W>
__device__ __forceinline__ bool smem_claim(u64* keys, unsigned h, const Set<W>& key) {
#if ETWG_CLAIM_PEEK
    // A slot only ever goes 0 -> key, so a plain read that shows a complete
    // key is final: ours (claimed, no atomic) or another (probe on). Only an
    // empty slot — or, at 128 bits, a read with a zero half, which may be a
    // half-visible CAS (keys with an empty half always take this path) —
    // takes the atomic.
    if constexpr (W == 1) {
        const u64 seen = *reinterpret_cast<volatile u64*>(keys + h);
        if (seen) return seen == key.w[0];
    } else {
        u64 lo, hi;
        asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];"
                     : "=l"(lo), "=l"(hi)
                     : "r"(static_cast<unsigned>(__cvta_generic_to_shared(keys + 2 * h))));
        if (lo && hi) return lo == key.w[0] && hi == key.w[1];
    }
#endif
    if constexpr (W == 1) {
        const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(keys + h), 0ull, key.w[0]);
        return prev == 0 || prev == key.w[0];
    } else {
        u64 lo, hi;
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(keys + 2 * h));
        asm volatile(
            "{\n\t.reg .b128 c, s, d;\n\t"
            "mov.b128 c, {%2, %3};\n\t"
            "mov.b128 s, {%4, %5};\n\t"
            "atom.shared.cas.b128 d, [%6], c, s;\n\t"
            "mov.b128 {%0, %1}, d;\n\t}"
            : "=l"(lo), "=l"(hi)
            : "l"(0ull), "l"(0ull), "l"(key.w[0]), "l"(key.w[1]), "r"(sa)
            : "memory");
        return (lo | hi) == 0 || (lo == key.w[0] && hi == key.w[1]);
    }
}

// ----------------------------------------------------------------------
// CTA-scope duplicate filter. A tile of consecutive parents (siblings of the
// same grandparents sit next to each other in a rank-ordered layer) offers
// many identical children; resolving them in shared memory first means only
// one instance per key and tile goes on to the global table / filter / owner
// (the one with the smallest emission rank, so min-rank semantics survive).
template <int W, int SLOTS>
struct TileSet {
    u64 keys[SLOTS * W];  // 0 = empty (children are never the empty set)
    unsigned rank[SLOTS];
};

template <int W, int SLOTS>
__device__ __forceinline__ void tile_set_clear(TileSet<W, SLOTS>& t) {
    for (int i = threadIdx.x; i < SLOTS * W; i += blockDim.x) t.keys[i] = 0;
    for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) t.rank[i] = 0xffffffffu;
}

constexpr int kTileProbes = 32;

// Inserts (key, rank); a key whose probe window is full stays out of the set
// for good (slots are never freed), so every instance of it reads as a
// winner in tile_set_winner and goes on to the global structure.
template <int W, int SLOTS>
__device__ __forceinline__ void tile_set_insert(TileSet<W, SLOTS>& t, const Set<W>& key, unsigned rank) {
    unsigned h = static_cast<unsigned>(slot_hash<W>(key)) & (SLOTS - 1);
    for (int probe = 0; probe < kTileProbes; ++probe) {
        if constexpr (W == 1) {
            const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(&t.keys[h]), 0ull, key.w[0]);
            if (prev == 0 || prev == key.w[0]) {
                atomicMin(&t.rank[h], rank);
                return;
            }
        } else {
            u64 lo, hi;
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&t.keys[2 * h]));
            asm volatile(
                "{\n\t.reg .b128 c, s, d;\n\t"
                "mov.b128 c, {%2, %3};\n\t"
                "mov.b128 s, {%4, %5};\n\t"
                "atom.shared.cas.b128 d, [%6], c, s;\n\t"
                "mov.b128 {%0, %1}, d;\n\t}"
                : "=l"(lo), "=l"(hi)
                : "l"(0ull), "l"(0ull), "l"(key.w[0]), "l"(key.w[1]), "r"(sa)
                : "memory");
            if ((lo | hi) == 0 || (lo == key.w[0] && hi == key.w[1])) {
                atomicMin(&t.rank[h], rank);
                return;
            }
        }
        h = (h + 1) & (SLOTS - 1);
    }
}

// After every insert of the tile: true iff `rank` is the key's tile minimum
// (or the key never found room).
template <int W, int SLOTS>
__device__ __forceinline__ bool tile_set_winner(const TileSet<W, SLOTS>& t, const Set<W>& key,
                                                unsigned rank) {
    unsigned h = static_cast<unsigned>(slot_hash<W>(key)) & (SLOTS - 1);
    for (int probe = 0; probe < kTileProbes; ++probe) {
        bool hit = t.keys[W * h] == key.w[0];
        if constexpr (W == 2) hit = hit && t.keys[2 * h + 1] == key.w[1];
        if (hit) return t.rank[h] == rank;
        h = (h + 1) & (SLOTS - 1);
    }
    return true;
}

// Replaces each thread's child mask M (children S+v) by the mask of its
// tile winners. Call with all threads of the CTA; t must be clear on entry
// and `win` is a per-thread scratch row of 2W words.
template <int W, int SLOTS>
__device__ __forceinline__ void tile_dedup(TileSet<W, SLOTS>& t, unsigned (*win)[2 * W], const Set<W>& S,
                                           Set<W>& M) {
    const int lane = threadIdx.x & 31;
    const int wslot = threadIdx.x & ~31;
    WarpFlat f;
    f.scan(M.count());
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
#pragma unroll
            for (int i = 0; i < 2 * W; ++i) win[threadIdx.x][i] = 0;
            __syncthreads();  // every insert of the tile is done
        }
        for (int tt = 0; tt < f.total; tt += 32) {
            const int j = tt + lane;
            const int src = f.source(j);
            const int excl = __shfl_sync(kFull, f.incl, src) - __shfl_sync(kFull, f.cnt, src);
            const Set<W> Ms = shfl_set<W>(M, src);
            const Set<W> Ss = shfl_set<W>(S, src);
            if (j < f.total) {
                const int v = nth_member<W>(Ms, j - excl);
                Set<W> key = Ss;
                key.add(v);
                const unsigned rank = static_cast<unsigned>(wslot + src) * (64 * W) + v;
                if (pass == 0)
                    tile_set_insert<W, SLOTS>(t, key, rank);
                else if (tile_set_winner<W, SLOTS>(t, key, rank))
                    atomicOr(&win[wslot + src][v >> 5], 1u << (v & 31));
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < W; ++i)
        M.w[i] = win[threadIdx.x][2 * i] | (static_cast<u64>(win[threadIdx.x][2 * i + 1]) << 32);
}

// ----------------------------------------------------------------------
// K2b: Bloom dedup on the reference's bit positions (bloom.cpp:86-97)

// Stripe lock with acquire / release semantics (no full fences): the 17
// relaxed atomicOr of a locked insert stay between the two.
__device__ __forceinline__ void stripe_lock(unsigned* lock) {
    unsigned old;
    for (;;) {
        asm volatile("atom.acquire.gpu.global.cas.b32 %0, [%1], 0, 1;" : "=r"(old) : "l"(lock) : "memory");
        if (old == 0) return;
        __nanosleep(64);
    }
}

__device__ __forceinline__ void stripe_unlock(unsigned* lock) {
    asm volatile("st.release.gpu.global.b32 [%0], 0;" ::"l"(lock) : "memory");
}

// Probe positions (h1 + i*h2) mod m, i = 1..hashes (bloom.cpp:90-91),
// stepped incrementally: pos_{i+1} = pos_i + (h2 mod m) - [>= m]*m.
__device__ __forceinline__ void probe_start(unsigned h1, unsigned h2, u64 m, u64& first, u64& step) {
    if (m <= 0xFFFFFFFFull) {  // 32-bit division whenever m fits
        const unsigned m32 = static_cast<unsigned>(m);
        const unsigned s = h2 % m32;
        const u64 f = static_cast<u64>(h1 % m32) + s;
        step = s;
        first = f >= m ? f - m : f;
    } else {
        step = static_cast<u64>(h2) % m;
        first = (static_cast<u64>(h1) + static_cast<u64>(h2)) % m;
    }
}

// insert_and_check (bloom.cpp:86-97) on the device. H > 0 fixes the hash
// count at compile time so all probe loads / atomics are issued back to
// back; H == 0 is the generic runtime-count loop.
template <int W, int H>
__device__ __forceinline__ bool bloom_insert_h(unsigned* bits, unsigned* locks, u64 m, int hashes,
                                               const Set<W>& key, bool single_lock) {
    const unsigned h1 = murmur_key<W>(key, kSeed1);
    const unsigned h2 = murmur_key<W>(key, kSeed2);
    u64 first, step;
    probe_start(h1, h2, m, first, step);
    // Fast path without the lock: when every probe bit is already set the
    // key is a duplicate in any serialisation of the concurrent inserts
    // (most children are: duplicates outnumber novel states ~6:1), so only
    // inserts that can still be novel pay for the stripe lock and atomics.
    bool all_set = true;
    if constexpr (H > 0) {  // requires m < 2^32: positions fit 32 bits
        unsigned pos[H];
        unsigned word[H];
        const unsigned m32 = static_cast<unsigned>(m), step32 = static_cast<unsigned>(step);
        pos[0] = static_cast<unsigned>(first);
#pragma unroll
        for (int i = 1; i < H; ++i) {
            const unsigned p = pos[i - 1] + step32;  // < 2m: wraps past 2^32 only if m > 2^31
            pos[i] = (p >= m32 || p < pos[i - 1]) ? p - m32 : p;
        }
#pragma unroll
        for (int i = 0; i < H; ++i) word[i] = __ldcg(bits + (pos[i] >> 5));
#pragma unroll
        for (int i = 0; i < H; ++i) all_set &= ((word[i] >> (pos[i] & 31)) & 1u) != 0;
        if (all_set) return false;
        unsigned* lock = locks + (single_lock ? 0u : h1 % kStripes);
        stripe_lock(lock);
#pragma unroll
        for (int i = 0; i < H; ++i) word[i] = atomicOr(bits + (pos[i] >> 5), 1u << (pos[i] & 31));
        stripe_unlock(lock);
        bool novel = false;
#pragma unroll
        for (int i = 0; i < H; ++i) novel |= ((word[i] >> (pos[i] & 31)) & 1u) == 0;
        return novel;
    } else {
        u64 pos = first;
        for (int i = 1; i <= hashes; ++i) {
            const unsigned word = __ldcg(bits + (pos >> 5));
            all_set &= ((word >> (pos & 31)) & 1u) != 0;
            pos += step;
            if (pos >= m) pos -= m;
        }
        if (all_set) return false;
        pos = first;
        unsigned* lock = locks + (single_lock ? 0u : h1 % kStripes);
        stripe_lock(lock);
        bool novel = false;
        for (int i = 1; i <= hashes; ++i) {
            const unsigned bit = 1u << (pos & 31);
            const unsigned old = atomicOr(bits + (pos >> 5), bit);
            novel |= (old & bit) == 0;
            pos += step;
            if (pos >= m) pos -= m;
        }
        stripe_unlock(lock);
        return novel;
    }
}

template <int W>
__device__ __forceinline__ bool bloom_insert(unsigned* bits, unsigned* locks, u64 m, int hashes,
                                             const Set<W>& key, bool single_lock = false) {
    return hashes == 17 && m <= 0xFFFFFFFFull
               ? bloom_insert_h<W, 17>(bits, locks, m, hashes, key, single_lock)
               : bloom_insert_h<W, 0>(bits, locks, m, hashes, key, single_lock);
}

constexpr int kWarpLocalBytes = 4096;               // per-warp key set
constexpr int kLocalBytes = kWarpLocalBytes * (kThreads / 32);
constexpr u64 kClaimMax = u64{1} << 27;             // slots (16 B each)

// Warp-private open-addressing set (key 0 = empty; children are never the
// empty set). True for the first inserter, and when the probe budget runs
// out (the global filter then decides: costs dedup efficiency, never states).
template <int W>
__device__ __forceinline__ bool local_first(u64* slots, unsigned mask, const Set<W>& key) {
    unsigned h = static_cast<unsigned>(slot_hash<W>(key)) & mask;
    for (int probe = 0; probe < 16; ++probe) {
        if constexpr (W == 1) {
            const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(slots + h), 0ull, key.w[0]);
            if (prev == 0) return true;
            if (prev == key.w[0]) return false;
        } else {
            u64 lo, hi;
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(slots + 2 * h));
            asm volatile(
                "{\n\t.reg .b128 c, s, d;\n\t"
                "mov.b128 c, {%2, %3};\n\t"
                "mov.b128 s, {%4, %5};\n\t"
                "atom.shared.cas.b128 d, [%6], c, s;\n\t"
                "mov.b128 {%0, %1}, d;\n\t}"
                : "=l"(lo), "=l"(hi)
                : "l"(0ull), "l"(0ull), "l"(key.w[0]), "l"(key.w[1]), "r"(sa)
                : "memory");
            if ((lo | hi) == 0) return true;
            if (lo == key.w[0] && hi == key.w[1]) return false;
        }
        h = (h + 1) & mask;
    }
    return true;
}

// Claims a 64-bit key for this round attempt (tag = epoch) in the
// open-addressing claim table; true iff this call is the first claim.
__device__ __forceinline__ bool claim_key(u64* claims, u64 mask, u64 key, u64 tag) {
    u64 i = fmix64(key ^ 0x9E3779B97F4A7C15ULL) & mask;
    for (;;) {
        u64* slot = claims + 2 * i;
        // A plain 16-byte load may tear, so it only seeds the CAS: a stale
        // tag goes straight to the claiming CAS (which fails on any tear and
        // returns the true value); a live tag is re-read untorn first.
        const ulonglong2 seen = __ldcg(reinterpret_cast<const ulonglong2*>(slot));
        u64 lo = seen.x, hi = seen.y;
        if (hi == tag) cas128(slot, ~u64{0}, ~u64{0}, ~u64{0}, ~u64{0}, lo, hi);
        for (;;) {
            if (hi == tag) {
                if (lo == key) return false;
                break;  // another key of this round: probe on
            }
            u64 plo, phi;
            cas128(slot, lo, hi, key, tag, plo, phi);
            if (plo == lo && phi == hi) return true;
            lo = plo;
            hi = phi;
        }
        i = (i + 1) & mask;
    }
}

// Sets the key's probe bits (relaxed atomicOr); true when one was clear.
template <int H>
__device__ __forceinline__ bool bloom_set_bits(unsigned* bits, u64 m, u64 first, u64 step) {
    unsigned pos[H];
    unsigned word[H];
    const unsigned m32 = static_cast<unsigned>(m), step32 = static_cast<unsigned>(step);
    pos[0] = static_cast<unsigned>(first);
#pragma unroll
    for (int i = 1; i < H; ++i) {
        const unsigned p = pos[i - 1] + step32;
        pos[i] = (p >= m32 || p < pos[i - 1]) ? p - m32 : p;
    }
#pragma unroll
    for (int i = 0; i < H; ++i) word[i] = __ldcg(bits + (pos[i] >> 5));
    bool all_set = true;
#pragma unroll
    for (int i = 0; i < H; ++i) all_set &= ((word[i] >> (pos[i] & 31)) & 1u) != 0;
    if (all_set) return false;  // duplicate (or false positive) in any serialisation
#pragma unroll
    for (int i = 0; i < H; ++i) word[i] = atomicOr(bits + (pos[i] >> 5), 1u << (pos[i] & 31));
    bool any_clear = false;
#pragma unroll
    for (int i = 0; i < H; ++i) any_clear |= ((word[i] >> (pos[i] & 31)) & 1u) == 0;
    return any_clear;
}

// Sets the probe bits (h1 + i*h2) mod m, i = 1..hashes, of a key that meets
// the filter once per round (bloom.cpp:86-97 on a distinct key); true when a
// probed bit was clear. Eight atomics are in flight before any result is
// used — consuming each return before the next probe (the plain loop) makes
// every probe a dependent L2/HBM round trip on filters far larger than L2.
__device__ __forceinline__ bool bloom_or_probes(unsigned* bits, u64 m, u64 first, u64 step, int hashes) {
    constexpr int kInFlight = 8;
    u64 pos = first;
    bool clear = false;
    for (int t = 0; t < hashes; t += kInFlight) {
        unsigned word[kInFlight], bit[kInFlight];
#pragma unroll
        for (int j = 0; j < kInFlight; ++j) {
            bit[j] = 0;
            word[j] = 0;
            if (t + j < hashes) {
                bit[j] = 1u << (pos & 31);
                word[j] = atomicOr(bits + (pos >> 5), bit[j]);
                pos += step;
                if (pos >= m) pos -= m;
            }
        }
#pragma unroll
        for (int j = 0; j < kInFlight; ++j) clear |= bit[j] != 0 && (word[j] & bit[j]) == 0;
    }
    return clear;
}

// Tile status word: [epoch:24][flag:2][value:38]. The epoch changes with
// every round attempt, so statuses left by earlier rounds read as "not yet
// published" and the status array never needs clearing between rounds.
constexpr u64 kFlagAgg = u64{1} << 38;
constexpr u64 kFlagPre = u64{2} << 38;
constexpr u64 kValMask = (u64{1} << 38) - 1;
constexpr unsigned kEpochMask = (1u << 24) - 1;

__device__ __forceinline__ u64 look_back(u64* tiles, u64 tile, u64 total, unsigned epoch) {
    volatile u64* vt = tiles;
    const u64 tag = static_cast<u64>(epoch & kEpochMask) << 40;
    if (tile == 0) {
        vt[0] = tag | kFlagPre | total;
        return 0;
    }
    vt[tile] = tag | kFlagAgg | total;
    u64 prefix = 0;
    u64 t = tile - 1;
    for (;;) {
        const u64 s = vt[t];
        if ((s >> 40) != (tag >> 40) || (s & (kFlagAgg | kFlagPre)) == 0) {
            __nanosleep(20);
            continue;
        }
        prefix += s & kValMask;
        if (s & kFlagPre) break;
        --t;
    }
    __threadfence();
    vt[tile] = tag | kFlagPre | (prefix + total);
    return prefix;
}

}  // namespace
}  // namespace etw
