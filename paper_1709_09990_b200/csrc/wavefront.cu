// B200 (sm_100a) wavefront engine: the device replacement for the reference's
// decide / expand_layer / expand_range / q_set / ConcurrentBloom / MMW hot
// path (proj/src/dp.cpp:23-194, graph.hpp:61-78, bloom.cpp:27-125,
// mmw.cpp:20-146).
//
// Per round (one BFS layer of the Held-Karp prefix DP) the device runs:
//   bloom : k_bloom_dedup -> k_append<mask>
//   exact : k_expand -> k_exact_insert -> k_append<probe>
//
//   k_expand       one thread per parent S. The components of G[S] are
//                  flood-filled once with bitmask ops; Q(S,v) for every
//                  candidate is then the union of v's outside neighbours and
//                  the outside boundary of every component v touches. The
//                  candidate mask (children that pass |Q| <= k and, when
//                  enabled, the minor-min-width bound) goes to HBM.
//   k_*_insert     children are flattened across the warp (warp scan +
//                  shuffle binary search), so the atomic-heavy dedup runs one
//                  child per lane. Bloom: 32-bit atomicOr on the reference's
//                  bit positions, striped lock on h1 % 65536 for exactly-once
//                  novelty, warp __match_any pre-dedup. Exact: open-addressing
//                  table, atomicCAS claim + atomicMin on the emission rank.
//   k_append       single-pass decoupled look-back scan over tiles of
//                  parents; survivors are written in rank order (parent index
//                  major, vertex minor) so exact mode reproduces the
//                  reference's sorted-by-first-emission layer byte for byte
//                  (dp.cpp:140-157), including truncation at the capacity wall.
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

struct RoundStats {
    u64 expanded, offered, unique, emitted, mmw_pruned;
    u64 ticket;  // tile ticket of the round's scan pass
    unsigned overflowed, valid;
};

enum AbortCode : unsigned { kOk = 0, kGrowLayer = 1, kGrowTable = 2, kGrowBloom = 3, kGrowClaims = 4 };

struct Control {
    u64 count[2];       // layer sizes, ping-pong by round parity
    u64 need;           // size requested by an abort
    unsigned round;     // next round to run
    unsigned stop;      // 1 once a layer came out empty or all rounds ran
    unsigned abort;     // AbortCode
    unsigned epoch;     // look-back tag of the current round attempt (never 0)
    unsigned exits;     // CTAs that finished the round's last pass
    unsigned pad;
    RoundStats rs[kMaxRounds];
};

struct Params {
    int n, k, rounds, free_count;
    int hashes, bpe, any_pop, flags;  // flags: ETWG_DEBUG bits (tests only)
    u64 max_states;
    u64 forbidden[2];
    u64 rows[kMaxVertices][2];
};

struct Bufs {
    u64* keys[2];
    unsigned* hist[2];
    u64* cmask;
    u64* table;
    unsigned* bloom[2];  // two filters, alternating by round parity
    unsigned* locks;
    u64* tiles;
    u64 layer_cap;   // states per layer buffer
    u64 table_cap;   // slots
    u64 bloom_cap;   // 32-bit words
    u64* claims;     // Bloom-mode claim table, 16-byte {key, epoch} slots
    u64 claim_cap;   // slots
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

// Outside boundaries N(K) \ S of the components K of G[S]; returns count.
template <int W>
__device__ __forceinline__ int component_boundaries(const Set<W>* adj, const Set<W>& S,
                                                    Set<W>* out) {
    int nc = 0;
    Set<W> rem = S;
    while (rem.any()) {
        Set<W> comp = Set<W>::bit(rem.lowest());
        Set<W> frontier = comp;
        Set<W> nb = Set<W>::zero();
        while (frontier.any()) {
            const Set<W> a = adj[frontier.pop()];
            nb |= a;
            Set<W> fresh = (a & S) - comp;
            comp |= fresh;
            frontier |= fresh;
        }
        rem = rem - comp;
        Set<W> boundary = nb - S;
        if (boundary.any()) out[nc++] = boundary;
    }
    return nc;
}

// Q(S,v) from the component boundaries: v's own outside neighbours plus the
// boundary of every component adjacent to v (v lies in that boundary).
template <int W>
__device__ __forceinline__ Set<W> reach_from(const Set<W>* adj, const Set<W>& S, const Set<W>* bnd,
                                             int nc, int v) {
    Set<W> q = adj[v] - S;
    for (int j = 0; j < nc; ++j)
        if (bnd[j].has(v)) q |= bnd[j];
    q.del(v);
    return q;
}

// Minor-min-width on eliminate(G, S + v) (init_view_after, mmw.cpp:20-43,
// then the shared contraction loop of mmw.hpp). rows[w] = Q(S,w) for every
// w outside S. Returns early once the bound exceeds cap.
template <int W>
__device__ int mmw_child(const Set<W>* adj, int n, int cap, const Set<W>& S, int v,
                         const Set<W>* rows) {
    constexpr int N = 64 * W;
    unsigned char parent[N];
    unsigned char degree[N];
    MinorState<W> m{adj, S, Set<W>::zero(), parent, degree};
    m.elim.add(v);
    m.alive = Set<W>::prefix(n) - m.elim;
    for (int x = 0; x < n; ++x) {
        parent[x] = static_cast<unsigned char>(x);
        degree[x] = 0;
    }
    // eliminating v turns Q(S,v) into a clique; everyone else keeps Q(S,w)
    for (int w : members(m.alive)) {
        if (rows[v].has(w)) {
            Set<W> j = rows[w] | rows[v];
            j.del(v);
            j.del(w);
            degree[w] = static_cast<unsigned char>(j.count());
        } else {
            degree[w] = static_cast<unsigned char>(rows[w].count());
        }
    }
    return minor_min_width<W>(m, cap);
}

template <int W, bool MMW>
__device__ __forceinline__ Set<W> candidates(const Set<W>* adj, int n, int k, const Set<W>& S,
                                             const Set<W>& forbidden, u64& pruned) {
    constexpr int N = 64 * W;
    const Set<W> open = Set<W>::prefix(n) - S;
    const Set<W> eligible = open - forbidden;
    Set<W> keep = Set<W>::zero();
    if (eligible.none()) return keep;
    Set<W> bnd[N];
    const int nc = component_boundaries<W>(adj, S, bnd);
    if constexpr (!MMW) {
        for (int v : members(eligible))
            if (reach_from<W>(adj, S, bnd, nc, v).count() <= k) keep.add(v);
    } else {
        Set<W> rows[N];  // dp.cpp:51-53: Q(S,w) for every open w
        for (int w : members(open)) rows[w] = reach_from<W>(adj, S, bnd, nc, w);
        for (int v : members(eligible)) {
            if (rows[v].count() > k) continue;
            if (mmw_child<W>(adj, n, k, S, v, rows) > k) {
                ++pruned;
                continue;
            }
            keep.add(v);
        }
    }
    return keep;
}

template <int W>
__device__ __forceinline__ void load_adjacency(const Params* P, Set<W>* adj) {
    for (int i = threadIdx.x; i < P->n; i += blockDim.x) adj[i] = param_set<W>(P->rows[i]);
}

__device__ __forceinline__ bool halted(const Control* C) {
    return (*reinterpret_cast<const volatile unsigned*>(&C->stop) |
            *reinterpret_cast<const volatile unsigned*>(&C->abort)) != 0;
}

template <int W, bool MMW>
__global__ void __launch_bounds__(kThreads) k_expand(const Params* __restrict__ P, Control* C,
                                                     Bufs B) {
    __shared__ Set<W> adj[64 * W];
    if (halted(C)) return;
    load_adjacency<W>(P, adj);
    __syncthreads();
    const unsigned r = C->round;
    const u64 E = C->count[r & 1];
    const u64 gtid = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
    const u64 gstride = static_cast<u64>(gridDim.x) * blockDim.x;

    const Set<W> forbidden = param_set<W>(P->forbidden);
    const u64* in = B.keys[r & 1];
    u64 offered = 0, pruned = 0;
    for (u64 idx = gtid; idx < E; idx += gstride) {
        const Set<W> S = load_set<W>(in, idx);
        const Set<W> keep = candidates<W, MMW>(adj, P->n, P->k, S, forbidden, pruned);
        store_set<W>(B.cmask, idx, keep);
        offered += keep.count();
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        offered += __shfl_xor_sync(kFull, offered, o);
        pruned += __shfl_xor_sync(kFull, pruned, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (offered) atomicAdd(&C->rs[r].offered, offered);
        if (pruned) atomicAdd(&C->rs[r].mmw_pruned, pruned);
    }
}

// ----------------------------------------------------------------------
// K2a: exact dedup — open addressing, claim by CAS, keep min emission rank
// (replaces the exact branch's sort/unique, dp.cpp:118-151)

// Rank words carry a round tag in bits 48..63 that shrinks as rounds
// advance, so any stale rank left by an earlier round of this decide loses
// every atomicMin; keys of a round all have popcount round+1, so stale keys
// are recognised without clearing the table between rounds.
__device__ __forceinline__ u64 rank_tag(unsigned r) { return static_cast<u64>(kMaxRounds - r) << 48; }

template <int W>
__device__ __forceinline__ bool stale_key(const Set<W>& cur, int want_pop) {
    return want_pop < 0 ? cur.none() : cur.count() != want_pop;
}

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

// Slot layout: W=1 {key, rank}; W=2 {key.lo, key.hi, rank, pad}.
template <int W>
__device__ __forceinline__ u64* table_slot(u64* table, u64 i) {
    return table + i * (W == 1 ? 2 : 4);
}

template <int W>
__device__ void table_insert(u64* table, u64 mask, int want_pop, const Set<W>& key, u64 rank) {
    u64 i = slot_hash<W>(key) & mask;
    for (;;) {
        u64* slot = table_slot<W>(table, i);
        if constexpr (W == 1) {
            u64 cur = *reinterpret_cast<volatile u64*>(slot);
            for (;;) {
                if (cur == key.w[0]) break;
                Set<1> c;
                c.w[0] = cur;
                if (!stale_key<1>(c, want_pop)) break;
                u64 prev = atomicCAS(slot, cur, key.w[0]);
                if (prev == cur) {
                    cur = key.w[0];
                    break;
                }
                cur = prev;
            }
            if (cur == key.w[0]) {
                atomicMin(slot + 1, rank);
                return;
            }
        } else {
            // 128-bit keys: read through a failing CAS so the view is never torn
            u64 lo, hi;
            cas128(slot, ~u64{0}, ~u64{0}, ~u64{0}, ~u64{0}, lo, hi);
            for (;;) {
                if (lo == key.w[0] && hi == key.w[1]) break;
                Set<2> c;
                c.w[0] = lo;
                c.w[1] = hi;
                if (!stale_key<2>(c, want_pop)) break;
                u64 plo, phi;
                cas128(slot, lo, hi, key.w[0], key.w[1], plo, phi);
                if (plo == lo && phi == hi) {
                    lo = key.w[0];
                    hi = key.w[1];
                    break;
                }
                lo = plo;
                hi = phi;
            }
            if (lo == key.w[0] && hi == key.w[1]) {
                atomicMin(slot + 2, rank);
                return;
            }
        }
        i = (i + 1) & mask;
    }
}

// After all inserts of the round: the rank stored with `key`.
template <int W>
__device__ __forceinline__ u64 table_rank(const u64* table, u64 mask, const Set<W>& key) {
    u64 i = slot_hash<W>(key) & mask;
    for (;;) {
        const u64* slot = table + i * (W == 1 ? 2 : 4);
        bool hit = slot[0] == key.w[0];
        if constexpr (W == 2) hit = hit && slot[1] == key.w[1];
        if (hit) return slot[W == 1 ? 1 : 2];
        i = (i + 1) & mask;
    }
}

template <int W>
__device__ __forceinline__ u64 child_rank(u64 parent_idx, int v) {
    return parent_idx * (64 * W) + static_cast<u64>(v);  // dp.cpp:66 (idx*64+v)
}

template <int W>
__global__ void __launch_bounds__(kThreads) k_exact_insert(const Params* __restrict__ P,
                                                           Control* C, Bufs B) {
    if (halted(C)) return;
    const unsigned r = C->round;
    const u64 E = C->count[r & 1];
    const u64 slots = table_slots_for(C->rs[r].offered);
    const u64 gtid = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
    if (slots > B.table_cap) {
        if (gtid == 0) {
            C->need = slots;
            C->abort = kGrowTable;
        }
        return;
    }
    const u64 mask = slots - 1;
    const int want_pop = P->any_pop ? -1 : static_cast<int>(r) + 1;
    const u64 tag = rank_tag(r);
    const int lane = threadIdx.x & 31;
    const u64 warp = gtid >> 5;
    const u64 nwarps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    const u64* in = B.keys[r & 1];
    for (u64 base = warp * 32; base < E; base += nwarps * 32) {
        const u64 idx = base + lane;
        const bool valid = idx < E;
        const Set<W> M = valid ? load_set<W>(B.cmask, idx) : Set<W>::zero();
        const Set<W> S = valid ? load_set<W>(in, idx) : Set<W>::zero();
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
                table_insert<W>(B.table, mask, want_pop, key, tag | child_rank<W>(base + src, v));
            }
        }
    }
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
// pass 2 (k_append<W,false>) turns masks into the rank-ordered next layer.
//
// Exactly-once novelty without the stripe-lock fences: an insert sets its
// 17 bits with relaxed atomicOr; if any was clear it *claims* the key in an
// epoch-tagged table with one 128-bit CAS — of several concurrent inserters
// of the same key exactly one claim succeeds (the reference's lock-based
// guarantee, bloom.cpp:86-97). W=2 keys (16 bytes + tag) do not fit a
// 16-byte CAS and use the reference's stripe locks, as does any round whose
// claim table would exceed kClaimMax.

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

template <int W, bool MMW>
__global__ void __launch_bounds__(kThreads, 3) k_bloom_dedup(const Params* __restrict__ P, Control* C,
                                                          Bufs B) {
    extern __shared__ __align__(16) u64 local_slots[];
    __shared__ Set<W> adj[64 * W];
    __shared__ unsigned novel_words[kThreads][2 * W];
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
        const Set<W> M = valid ? candidates<W, MMW>(adj, P->n, P->k, S, forbidden, pruned)
                               : Set<W>::zero();
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
    C->epoch = (C->epoch & kEpochMask) == kEpochMask ? 1 : C->epoch + 1;
    if (emitted == 0 || static_cast<int>(r) + 1 >= P->rounds) C->stop = 1;
}

template <int W, bool PROBE>
__global__ void __launch_bounds__(kThreads) k_append(const Params* __restrict__ P, Control* C,
                                                     Bufs B) {
    using BlockScan = cub::BlockScan<unsigned, kThreads>;
    __shared__ typename BlockScan::TempStorage scan_tmp;
    __shared__ unsigned win_words[kThreads][2 * W];
    __shared__ u64 s_prefix;
    __shared__ u64 s_tile;
    if (halted(C)) return;
    const unsigned r = C->round;
    const unsigned epoch = C->epoch;
    const u64 E = C->count[r & 1];
    const u64 ntiles = (E + kThreads - 1) / kThreads;
    const u64 cap = round_cap(*P, E);
    const u64 limit = cap < B.layer_cap ? cap : B.layer_cap;
    const u64 slots = PROBE ? table_slots_for(C->rs[r].offered) : 0;
    const u64 tag = rank_tag(r);
    const int lane = threadIdx.x & 31;
    const int wslot = threadIdx.x & ~31;
    const u64* in = B.keys[r & 1];
    const unsigned* hin = B.hist[r & 1];
    u64* out = B.keys[(r + 1) & 1];
    unsigned* hout = B.hist[(r + 1) & 1];

    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&C->rs[r].ticket, 1ull);
        __syncthreads();
        const u64 tile = s_tile;
        if (tile >= ntiles) break;
        const u64 idx = tile * kThreads + threadIdx.x;
        const bool valid = idx < E;
        const Set<W> S = valid ? load_set<W>(in, idx) : Set<W>::zero();
        const unsigned H = valid ? hin[idx] : 0u;
        Set<W> M = valid ? load_set<W>(B.cmask, idx) : Set<W>::zero();
        if constexpr (PROBE) {
            // winners: children whose stored min rank is their own
#pragma unroll
            for (int i = 0; i < 2 * W; ++i) win_words[threadIdx.x][i] = 0;
            __syncwarp();
            WarpFlat f;
            f.scan(M.count());
            const u64 warp_base = tile * kThreads + wslot;
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
                    const u64 mine = tag | child_rank<W>(warp_base + src, v);
                    if (table_rank<W>(B.table, slots - 1, key) == mine)
                        atomicOr(&win_words[wslot + src][v >> 5], 1u << (v & 31));
                }
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < W; ++i)
                M.w[i] = win_words[threadIdx.x][2 * i] |
                         (static_cast<u64>(win_words[threadIdx.x][2 * i + 1]) << 32);
        }
        const unsigned cnt = static_cast<unsigned>(M.count());
        unsigned excl_block, total_block;
        BlockScan(scan_tmp).ExclusiveSum(cnt, excl_block, total_block);
        if (threadIdx.x == 0) s_prefix = look_back(B.tiles, tile, total_block, epoch);
        __syncthreads();
        const u64 prefix = s_prefix;
        append_survivors<W>(M, S, H, prefix + __shfl_sync(kFull, excl_block, 0), limit, out, hout);
        if (threadIdx.x == 0 && tile == ntiles - 1) {
            // the final tile knows the round's survivor total
            const u64 unique = prefix + total_block;
            C->rs[r].unique = unique;
        }
        __syncthreads();
    }
    finish_round(P, C, B, r, E, cap);
}

// ----------------------------------------------------------------------
// table reset for a new decide (keys 0, ranks all-ones)

template <int W>
__global__ void k_table_reset(u64* table, u64 slots) {
    const u64 gtid = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
    const u64 gstride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = gtid; i < slots; i += gstride) {
        if constexpr (W == 1) {
            reinterpret_cast<ulonglong2*>(table)[i] = make_ulonglong2(0, ~u64{0});
        } else {
            reinterpret_cast<ulonglong4*>(table)[i] = make_ulonglong4(0, 0, ~u64{0}, 0);
        }
    }
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
                        int rounds, const LayerObserver* observer) {
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
        reset_control(1);
        u64 zero2[2] = {0, 0};
        unsigned root_hist = 0xFFFFFFFFu;
        copy(b_.keys[0], zero2, 16, cudaMemcpyHostToDevice, "root");
        copy(b_.hist[0], &root_hist, 4, cudaMemcpyHostToDevice, "root");
        if (cfg.dedup == DedupMode::exact_set) reset_table(W);

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
            if (s.emitted == 0) break;
        }
        res.overflowed = any_ovf;
        account(res.rounds, W, cfg);
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
        if (cfg.dedup == DedupMode::exact_set) reset_table(W);
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
    DeviceInfo info_;
    cudaStream_t stream_ = nullptr;
    Params* d_params_ = nullptr;
    Params* h_params_ = nullptr;
    Control* d_ctl_ = nullptr;
    Control* h_ctl_ = nullptr;
    Bufs b_{};
    u64 table_dirty_bytes_ = 0;  // table bytes possibly holding keys of an earlier decide
    u64 bloom_dirty_[2] = {0, 0};  // words of each Bloom filter that may hold bits
    unsigned epoch_ = 1;          // look-back epoch carried across decides
    bool bloom_round_ = false;    // current decide runs the fused Bloom round
    int grid_fused_ = 0;

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
    int table_layout_ = 0;       // slot layout (W) the clean part of the table is in
    int grid_ = 0;
    cudaEvent_t ev_[2] = {nullptr, nullptr};
    cudaEvent_t tev_[2] = {nullptr, nullptr};

    // every host<->device copy of the engine goes through here (counted)
    void copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, const char* what) {
        check(cudaMemcpyAsync(dst, src, bytes, kind, stream_), what);
        if (kind == cudaMemcpyHostToDevice) prof.t.h2d_bytes += bytes;
        if (kind == cudaMemcpyDeviceToHost) prof.t.d2h_bytes += bytes;
    }

    void init() {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            init_state_ = 2;
            return;
        }
        int dev = 0;
        if (const char* e = std::getenv("ETWG_DEVICE")) dev = std::atoi(e);
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
        p.max_states = cfg.max_layer_states;
        p.forbidden[0] = forbidden.w[0];
        p.forbidden[1] = forbidden.w[1];
        for (int v = 0; v < g.vertex_count(); ++v) {
            p.rows[v][0] = g.neighbors(v).w[0];
            p.rows[v][1] = g.neighbors(v).w[1];
        }
        copy(d_params_, h_params_, sizeof(Params), cudaMemcpyHostToDevice, "params");
    }

    void reset_control(u64 first_count) {
        Control& c = *h_ctl_;
        std::memset(&c, 0, sizeof c);
        c.count[0] = first_count;
        c.epoch = next_epoch();
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

    void ensure_table(u64 slots) {
        if (slots <= b_.table_cap && b_.table) return;
        u64 cap = std::max<u64>(slots, u64{1} << 20);
        if (b_.table) cudaFree(b_.table);
        check(cudaMalloc(&b_.table, cap * 32), "table");
        b_.table_cap = cap;
        table_dirty_bytes_ = cap * 32;  // fresh memory: reset everything before use
        table_layout_ = 0;
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

    // The "empty" pattern differs between the 16-byte (W=1) and 32-byte
    // (W=2) slot layouts, so switching layouts re-initialises the whole table.
    void reset_table(int W) {
        ensure_table(u64{1} << 20);
        if (W != table_layout_) {
            table_dirty_bytes_ = b_.table_cap * 32;
            table_layout_ = W;
        }
        if (table_dirty_bytes_ == 0) return;
        const u64 slot_bytes = W == 1 ? 16 : 32;
        u64 slots = std::min((table_dirty_bytes_ + slot_bytes - 1) / slot_bytes,
                             b_.table_cap * 32 / slot_bytes);
        int blocks = static_cast<int>(std::min<u64>((slots + 255) / 256, 4096));
        if (W == 1)
            k_table_reset<1><<<blocks, 256, 0, stream_>>>(b_.table, slots);
        else
            k_table_reset<2><<<blocks, 256, 0, stream_>>>(b_.table, slots);
        check(cudaGetLastError(), "table reset");
        prof.t.kernel_launches++;
        table_dirty_bytes_ = 0;
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
        if (!exact) {
            if (cfg.use_mmw)
                timed_launch([&] { k_bloom_dedup<W, true><<<grid_fused_, kThreads, kLocalBytes, stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.insert_ms, prof.t.insert_launches);
            else
                timed_launch([&] { k_bloom_dedup<W, false><<<grid_fused_, kThreads, kLocalBytes, stream_>>>(d_params_, d_ctl_, b_); },
                             prof.t.insert_ms, prof.t.insert_launches);
            timed_launch([&] { k_append<W, false><<<grid_, kThreads, 0, stream_>>>(d_params_, d_ctl_, b_); },
                         prof.t.append_ms, prof.t.append_launches);
            return;
        }
        if (cfg.use_mmw)
            timed_launch([&] { k_expand<W, true><<<grid_, kThreads, 0, stream_>>>(d_params_, d_ctl_, b_); },
                         prof.t.expand_ms, prof.t.expand_launches);
        else
            timed_launch([&] { k_expand<W, false><<<grid_, kThreads, 0, stream_>>>(d_params_, d_ctl_, b_); },
                         prof.t.expand_ms, prof.t.expand_launches);
        timed_launch([&] { k_exact_insert<W><<<grid_, kThreads, 0, stream_>>>(d_params_, d_ctl_, b_); },
                     prof.t.insert_ms, prof.t.insert_launches);
        timed_launch([&] { k_append<W, true><<<grid_, kThreads, 0, stream_>>>(d_params_, d_ctl_, b_); },
                     prof.t.append_ms, prof.t.append_launches);
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
        ensure_table(u64{1} << 20);
        ensure_bloom(u64{1} << 22);
        ensure_claims(u64{1} << 20);
        bloom_round_ = cfg.dedup == DedupMode::bloom;
        if (bloom_round_) clean_blooms();
        if (!prof.on) check(cudaEventRecord(ev_[0], stream_), "event");
        auto t0 = std::chrono::steady_clock::now();
        const bool sync_each = (h_params_->flags & 8) != 0;
        int chunk = observer || sync_each ? 1 : 4;
        for (;;) {
            const int start = static_cast<int>(h_ctl_->round);
            const int end = std::min(rounds, start + chunk);
            for (int r = start; r < end; ++r) {
                if (W == 1) launch_round<1>(cfg);
                else launch_round<2>(cfg);
            }
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
        if (cfg.dedup == DedupMode::exact_set) {
            const u64 slot_bytes = W == 1 ? 16 : 32;
            for (int r = 0; r < rounds; ++r)
                if (h_ctl_->rs[r].offered)
                    table_dirty_bytes_ = std::max(
                        table_dirty_bytes_, table_slots_for(h_ctl_->rs[r].offered) * slot_bytes);
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
        const unsigned r = c.round;
        switch (c.abort) {
            case kGrowLayer:
                ensure_layers(c.need + c.need / 2, static_cast<int>(r & 1), c.count[r & 1]);
                if (bloom_round_) {  // the aborted attempt left bits in filter r&1
                    bloom_dirty_[r & 1] = std::max<u64>(
                        bloom_dirty_[r & 1],
                        bloom_bits_for(host_round_cap(c.count[r & 1]), h_params_->bpe) / 32);
                    clean_blooms();
                }
                break;
            case kGrowTable:
                ensure_table(c.need);  // fresh memory, fully reset below
                reset_table(W);
                break;
            case kGrowBloom:
                ensure_bloom(c.need + c.need / 4);
                break;
            case kGrowClaims:
                ensure_claims(c.need);
                break;
            default:
                throw DeviceError("device engine: unknown abort code");
        }
        // re-arm: clear the abort and the partial statistics of round r
        c.abort = kOk;
        c.need = 0;
        c.exits = 0;
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
        const double wb = 8.0 * W + 4.0;
        const double db = cfg.dedup == DedupMode::bloom ? 4.0 * cfg.bloom_hashes : (W == 1 ? 16.0 : 24.0);
        for (const LayerStats& s : rounds) {
            prof.t.layer_bytes += wb * static_cast<double>(s.expanded + s.emitted);
            prof.t.dedup_bytes += db * static_cast<double>(s.emitted + s.duplicates);
            prof.t.expanded += s.expanded;
        }
    }
};

}  // namespace

DecideResult device_decide(const Graph& g, int k, const HostSet& forbidden, const DpConfig& cfg,
                           int rounds, const LayerObserver* observer) {
    if (k < 0) throw std::invalid_argument("k must be non-negative");
    if (cfg.max_layer_states == 0) throw std::invalid_argument("layer capacity must be positive");
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    return e.decide(g, k, forbidden, cfg, rounds, observer);
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
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    e.timer_begin();
}

double engine_timer_end() {
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
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    return e.prof.t;
}

void engine_reset_times() {
    Engine& e = Engine::instance();
    std::lock_guard<std::mutex> lock(e.mu);
    e.prof.t = KernelTimes{};
}

}  // namespace etw
