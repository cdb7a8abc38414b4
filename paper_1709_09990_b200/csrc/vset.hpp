// Fixed-width vertex set shared by host and device code.
//
// Replaces the reference's BasicVertexSet<Words> (proj/src/bitset.hpp:13-152),
// of which the reference instantiates only the one-word variant (n <= 64,
// bitset.hpp:152). Here both widths are live: Set<1> is the 8-byte state key
// for n <= 64 (bit-identical to the reference key), Set<2> the 16-byte key for
// 64 < n <= 128. Host code always stores graphs as Set<2> (HostSet) so a
// single host build covers both, and narrows to Set<1> at the device seam.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define ETW_HD __host__ __device__ __forceinline__
#else
#define ETW_HD inline
#endif

namespace etw {

ETW_HD int popc64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __popcll(x);
#else
    return __builtin_popcountll(x);
#endif
}

ETW_HD int ctz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __ffsll(static_cast<long long>(x)) - 1;
#else
    return __builtin_ctzll(x);
#endif
}

template <int W>
struct Set {
    static constexpr int kWords = W;
    static constexpr int kCapacity = 64 * W;
    uint64_t w[W];

    ETW_HD static Set zero() {
        Set s;
#pragma unroll
        for (int i = 0; i < W; ++i) s.w[i] = 0;
        return s;
    }
    // Single-bit access selects the word with constant indices (an unrolled
    // compare per word) instead of w[v >> 6]: a runtime index into w[] makes
    // nvcc keep the whole set, and every set stored next to it, in local
    // memory.
    ETW_HD static Set bit(int v) {
        Set s;
        const uint64_t b = uint64_t{1} << (v & 63);
#pragma unroll
        for (int i = 0; i < W; ++i) s.w[i] = (W == 1 || (v >> 6) == i) ? b : 0;
        return s;
    }
    // {0..n-1}
    ETW_HD static Set prefix(int n) {
        Set s;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            int lo = 64 * i;
            s.w[i] = n <= lo ? 0 : (n >= lo + 64 ? ~uint64_t{0} : (uint64_t{1} << (n - lo)) - 1);
        }
        return s;
    }
    ETW_HD uint64_t word_of(int v) const {
        uint64_t x = w[0];
#pragma unroll
        for (int i = 1; i < W; ++i)
            if ((v >> 6) == i) x = w[i];
        return x;
    }
    ETW_HD bool has(int v) const { return (word_of(v) >> (v & 63)) & 1u; }
    ETW_HD void add(int v) {
        const uint64_t b = uint64_t{1} << (v & 63);
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (W == 1 || (v >> 6) == i) w[i] |= b;
    }
    ETW_HD void del(int v) {
        const uint64_t b = uint64_t{1} << (v & 63);
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (W == 1 || (v >> 6) == i) w[i] &= ~b;
    }
    ETW_HD int count() const {
        int c = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) c += popc64(w[i]);
        return c;
    }
    ETW_HD bool any() const {
        uint64_t a = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) a |= w[i];
        return a != 0;
    }
    ETW_HD bool none() const { return !any(); }
    // smallest member; -1 when empty
    ETW_HD int lowest() const {
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (w[i]) return 64 * i + ctz64(w[i]);
        return -1;
    }
    // removes and returns the smallest member (set must be non-empty)
    ETW_HD int pop() {
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (w[i]) {
                int b = ctz64(w[i]);
                w[i] &= w[i] - 1;
                return 64 * i + b;
            }
        return -1;
    }
    ETW_HD Set operator|(const Set& o) const {
        Set r;
#pragma unroll
        for (int i = 0; i < W; ++i) r.w[i] = w[i] | o.w[i];
        return r;
    }
    ETW_HD Set operator&(const Set& o) const {
        Set r;
#pragma unroll
        for (int i = 0; i < W; ++i) r.w[i] = w[i] & o.w[i];
        return r;
    }
    // difference
    ETW_HD Set operator-(const Set& o) const {
        Set r;
#pragma unroll
        for (int i = 0; i < W; ++i) r.w[i] = w[i] & ~o.w[i];
        return r;
    }
    ETW_HD Set& operator|=(const Set& o) {
#pragma unroll
        for (int i = 0; i < W; ++i) w[i] |= o.w[i];
        return *this;
    }
    ETW_HD Set& operator&=(const Set& o) {
#pragma unroll
        for (int i = 0; i < W; ++i) w[i] &= o.w[i];
        return *this;
    }
    ETW_HD bool operator==(const Set& o) const {
        bool eq = true;
#pragma unroll
        for (int i = 0; i < W; ++i) eq = eq && (w[i] == o.w[i]);
        return eq;
    }
    ETW_HD bool operator!=(const Set& o) const { return !(*this == o); }
    ETW_HD bool subset_of(const Set& o) const { return (*this - o).none(); }
    ETW_HD bool intersects(const Set& o) const { return (*this & o).any(); }
    // numeric order, high word first (bitset.hpp:116-120)
    ETW_HD bool operator<(const Set& o) const {
        for (int i = W - 1; i >= 0; --i)
            if (w[i] != o.w[i]) return w[i] < o.w[i];
        return false;
    }
};

using HostSet = Set<2>;
constexpr int kMaxVertices = 128;

// Visit members in ascending order: for (int v : members(s)) ...
template <int W>
struct Members {
    Set<W> rest;
    struct It {
        Set<W> r;
        int cur;
        ETW_HD int operator*() const { return cur; }
        ETW_HD It& operator++() {
            cur = r.any() ? r.pop() : -1;
            return *this;
        }
        ETW_HD bool operator!=(const It& o) const { return cur != o.cur; }
    };
    ETW_HD It begin() const {
        It it{rest, -1};
        if (it.r.any()) it.cur = it.r.pop();
        return it;
    }
    ETW_HD It end() const { return It{Set<W>::zero(), -1}; }
};

template <int W>
ETW_HD Members<W> members(const Set<W>& s) {
    return Members<W>{s};
}

// Removes and returns some member (the highest) of a non-empty set. Where
// the visiting order does not matter this is the cheap pop on the device:
// one FLO per 32-bit word instead of the 64-bit ffs + borrow of pop().
template <int W>
ETW_HD int pop_any(Set<W>& s) {
#if defined(__CUDA_ARCH__)
#pragma unroll
    for (int i = W - 1; i >= 0; --i) {
        const unsigned hi = static_cast<unsigned>(s.w[i] >> 32);
        const unsigned lo = static_cast<unsigned>(s.w[i]);
        if (hi | lo) {
            const int b = hi ? 63 - __clz(hi) : 31 - __clz(lo);
            s.w[i] ^= uint64_t{1} << b;
            return 64 * i + b;
        }
    }
    return -1;
#else
    return s.pop();
#endif
}

// Calls f(v) for every member, in no particular order (descending on the
// device, 32-bit words, one FLO + one XOR per member).
template <int W, typename F>
ETW_HD void for_each_any(const Set<W>& s, F&& f) {
#if defined(__CUDA_ARCH__)
#pragma unroll
    for (int i = 2 * W - 1; i >= 0; --i) {
        unsigned x = static_cast<unsigned>(s.w[i >> 1] >> (32 * (i & 1)));
        while (x) {
            const int b = 31 - __clz(x);
            x ^= 1u << b;
            f(32 * i + b);
        }
    }
#else
    for (int v : members(s)) f(v);
#endif
}

}  // namespace etw
