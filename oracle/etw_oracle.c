/* TEST INFRASTRUCTURE ONLY — see etw_oracle.h. Plain-C restatement of the
 * reference hot path, single-threaded, 128-bit vertex sets. Each function
 * cites the reference lines it restates (paths under /root/reference/proj). */
#include "etw_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint64_t w[2];
} vs_t;

static inline int vs_has(const vs_t* s, int v) { return (int)((s->w[v >> 6] >> (v & 63)) & 1u); }
static inline void vs_add(vs_t* s, int v) { s->w[v >> 6] |= (uint64_t)1 << (v & 63); }
static inline void vs_del(vs_t* s, int v) { s->w[v >> 6] &= ~((uint64_t)1 << (v & 63)); }
static inline int vs_count(const vs_t* s) {
    return __builtin_popcountll(s->w[0]) + __builtin_popcountll(s->w[1]);
}
static inline int vs_empty(const vs_t* s) { return (s->w[0] | s->w[1]) == 0; }
static inline vs_t vs_or(vs_t a, vs_t b) { a.w[0] |= b.w[0]; a.w[1] |= b.w[1]; return a; }
static inline vs_t vs_and(vs_t a, vs_t b) { a.w[0] &= b.w[0]; a.w[1] &= b.w[1]; return a; }
static inline vs_t vs_minus(vs_t a, vs_t b) { a.w[0] &= ~b.w[0]; a.w[1] &= ~b.w[1]; return a; }
static inline int vs_eq(vs_t a, vs_t b) { return a.w[0] == b.w[0] && a.w[1] == b.w[1]; }
/* lowest member, -1 if empty (bitset.hpp:59-63) */
static inline int vs_low(const vs_t* s) {
    if (s->w[0]) return __builtin_ctzll(s->w[0]);
    if (s->w[1]) return 64 + __builtin_ctzll(s->w[1]);
    return -1;
}
static vs_t vs_first_n(int n) { /* bitset.hpp:26-38 */
    vs_t s = {{0, 0}};
    for (int i = 0; i < 2; ++i) {
        int lo = 64 * i;
        if (n <= lo) s.w[i] = 0;
        else if (n >= lo + 64) s.w[i] = ~(uint64_t)0;
        else s.w[i] = ((uint64_t)1 << (n - lo)) - 1;
    }
    return s;
}
static vs_t vs_load(const uint64_t* p) { vs_t s = {{p[0], p[1]}}; return s; }

/* iterate members ascending */
#define VS_FOR(var, set)                                                       \
    for (int var##_i = 0; var##_i < 2; ++var##_i)                              \
        for (uint64_t var##_r = (set).w[var##_i]; var##_r; var##_r &= var##_r - 1) \
            for (int var = 64 * var##_i + __builtin_ctzll(var##_r), var##_once = 1; var##_once; var##_once = 0)

typedef struct {
    int n;
    vs_t rows[ORACLE_MAXV];
} graph_t;

/* Graph::from_rows (graph.cpp:9-29): mask to universe, drop loops, symmetrize */
static void graph_init(graph_t* g, int n, const uint64_t* rows) {
    g->n = n;
    vs_t uni = vs_first_n(n);
    for (int v = 0; v < n; ++v) {
        g->rows[v] = vs_and(vs_load(rows + 2 * v), uni);
        vs_del(&g->rows[v], v);
    }
    for (int v = 0; v < n; ++v) VS_FOR(u, g->rows[v]) vs_add(&g->rows[u], v);
}

/* ------------------------------------------------------------------ */
/* Murmur3 x86_32 (bloom.cpp:27-64)                                    */
static inline uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }

uint32_t oracle_murmur3_x86_32(const void* data, size_t len, uint32_t seed) {
    const uint8_t* p = (const uint8_t*)data;
    size_t nblocks = len / 4;
    uint32_t h = seed;
    const uint32_t c1 = 0xcc9e2d51u, c2 = 0x1b873593u;
    for (size_t i = 0; i < nblocks; ++i) {
        const uint8_t* b = p + 4 * i;
        uint32_t k = (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 |
                     (uint32_t)b[3] << 24;
        k *= c1;
        k = rotl32(k, 15);
        k *= c2;
        h ^= k;
        h = rotl32(h, 13);
        h = h * 5 + 0xe6546b64u;
    }
    const uint8_t* t = p + 4 * nblocks;
    uint32_t k = 0;
    switch (len & 3) {
        case 3: k ^= (uint32_t)t[2] << 16; /* fall through */
        case 2: k ^= (uint32_t)t[1] << 8;  /* fall through */
        case 1:
            k ^= t[0];
            k *= c1;
            k = rotl32(k, 15);
            k *= c2;
            h ^= k;
    }
    h ^= (uint32_t)len;
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

/* hash_pair (bloom.cpp:66-70) with seeds bloom.hpp:24-25; words=2 is the
 * 16-byte extension for n > 64 (word 0 bytes first). */
void oracle_hash_pair(const uint64_t* key, int words, uint32_t* h1, uint32_t* h2) {
    uint8_t buf[16];
    for (int i = 0; i < 8 * words; ++i) buf[i] = (uint8_t)(key[i >> 3] >> (8 * (i & 7)));
    *h1 = oracle_murmur3_x86_32(buf, (size_t)(8 * words), 0x9747B28Cu);
    *h2 = oracle_murmur3_x86_32(buf, (size_t)(8 * words), 0x5EEDBA5Eu);
}

/* ConcurrentBloom ctor sizing (bloom.cpp:72-79) */
uint64_t oracle_bloom_bits(uint64_t expected, int bpe) {
    uint64_t bits = expected * (uint64_t)bpe;
    uint64_t m = (bits + 63) / 64 * 64;
    return m < 64 ? 64 : m;
}

typedef struct {
    uint64_t m;
    int hashes;
    uint64_t* words;
} bloom_t;

static int bloom_init(bloom_t* b, uint64_t expected, int bpe, int hashes) {
    b->m = oracle_bloom_bits(expected, bpe);
    b->hashes = hashes;
    b->words = (uint64_t*)calloc(b->m / 64, sizeof(uint64_t));
    return b->words != NULL;
}

/* insert_and_check (bloom.cpp:86-97): novel iff any probe bit was clear */
static int bloom_insert(bloom_t* b, const uint64_t* key, int words) {
    uint32_t h1, h2;
    oracle_hash_pair(key, words, &h1, &h2);
    int novel = 0;
    for (int i = 1; i <= b->hashes; ++i) {
        uint64_t pos = ((uint64_t)h1 + (uint64_t)i * (uint64_t)h2) % b->m;
        uint64_t mask = (uint64_t)1 << (pos & 63);
        if (!(b->words[pos >> 6] & mask)) novel = 1;
        b->words[pos >> 6] |= mask;
    }
    return novel;
}

uint64_t oracle_bloom_insert_seq(uint64_t expected, int bpe, int hashes, const uint64_t* keys,
                                 int words, size_t count, uint8_t* novel_out) {
    bloom_t b;
    if (!bloom_init(&b, expected, bpe, hashes)) return 0;
    for (size_t i = 0; i < count; ++i) novel_out[i] = (uint8_t)bloom_insert(&b, keys + words * i, words);
    free(b.words);
    return b.m;
}

uint64_t oracle_bloom_query(const uint32_t* bits, uint64_t m, int hashes, const uint64_t* keys,
                            int words, size_t count) {
    uint64_t hits = 0;
    for (size_t j = 0; j < count; ++j) {
        uint32_t h1, h2;
        oracle_hash_pair(keys + (size_t)words * j, words, &h1, &h2);
        int all = 1;
        for (int i = 1; i <= hashes && all; ++i) {
            uint64_t pos = ((uint64_t)h1 + (uint64_t)i * (uint64_t)h2) % m;
            if (!((bits[pos >> 5] >> (pos & 31)) & 1u)) all = 0;
        }
        hits += (uint64_t)all;
    }
    return hits;
}

/* expected_false_positive_rate (bloom.cpp:120-125) */
double oracle_bloom_expected_fp(uint64_t m, int hashes, uint64_t inserted) {
    if (inserted == 0) return 0.0;
    double k = hashes;
    return pow(1.0 - exp(-k * (double)inserted / (double)m), k);
}

/* ------------------------------------------------------------------ */
/* q_set (graph.hpp:61-78): DFS from v, walking only through members of s */
static vs_t q_set(const graph_t* g, vs_t s, int v) {
    vs_t result = {{0, 0}};
    vs_t visited = {{0, 0}};
    vs_add(&visited, v);
    int stack[ORACLE_MAXV];
    int top = 0;
    stack[top++] = v;
    while (top > 0) {
        int x = stack[--top];
        vs_t nb = vs_minus(g->rows[x], visited);
        VS_FOR(y, nb) {
            vs_add(&visited, y);
            if (vs_has(&s, y)) stack[top++] = y;
            else vs_add(&result, y);
        }
    }
    return result;
}

void oracle_q_set(int n, const uint64_t* rows, const uint64_t* s, int v, uint64_t* out) {
    graph_t g;
    graph_init(&g, n, rows);
    vs_t q = q_set(&g, vs_load(s), v);
    out[0] = q.w[0];
    out[1] = q.w[1];
}

/* ------------------------------------------------------------------ */
/* Minor-min-width over eliminate(g, s) (mmw.cpp)                       */
typedef struct {
    uint8_t parent[ORACLE_MAXV];
    uint8_t degree[ORACLE_MAXV];
    vs_t alive, eliminated;
    int n;
} view_t;

static int view_find(view_t* v, int x) { /* mmw.hpp:21-27 */
    while (v->parent[x] != x) {
        v->parent[x] = v->parent[v->parent[x]];
        x = v->parent[x];
    }
    return x;
}

static void view_init(view_t* vw, const graph_t* g, vs_t s) { /* mmw.cpp:7-18 */
    vw->n = g->n;
    vw->eliminated = s;
    vw->alive = vs_minus(vs_first_n(g->n), s);
    for (int x = 0; x < vw->n; ++x) {
        vw->parent[x] = (uint8_t)x;
        vw->degree[x] = 0;
    }
    VS_FOR(x, vw->alive) {
        vs_t q = q_set(g, s, x);
        vw->degree[x] = (uint8_t)vs_count(&q);
    }
}

/* init_view_after (mmw.cpp:20-43): rows[w] = q_set(g, s, w) for w outside s */
static void view_init_after(view_t* vw, const graph_t* g, vs_t s, int v, const vs_t* rows) {
    vw->n = g->n;
    vw->eliminated = s;
    vs_add(&vw->eliminated, v);
    vw->alive = vs_minus(vs_first_n(g->n), vw->eliminated);
    for (int x = 0; x < vw->n; ++x) {
        vw->parent[x] = (uint8_t)x;
        vw->degree[x] = 0;
    }
    VS_FOR(w, vw->alive) {
        if (vs_has(&rows[v], w)) {
            vs_t j = vs_or(rows[w], rows[v]);
            vs_del(&j, v);
            vs_del(&j, w);
            vw->degree[w] = (uint8_t)vs_count(&j);
        } else {
            vw->degree[w] = (uint8_t)vs_count(&rows[w]);
        }
    }
}

/* adjacent_roots (mmw.cpp:49-71) */
static vs_t adjacent_roots(view_t* vw, const graph_t* g, int r) {
    vs_t roots = {{0, 0}};
    vs_t visited = {{0, 0}};
    vs_add(&visited, r);
    int stack[ORACLE_MAXV];
    int top = 0;
    stack[top++] = r;
    while (top > 0) {
        int x = stack[--top];
        vs_t nb = vs_minus(g->rows[x], visited);
        VS_FOR(y, nb) {
            vs_add(&visited, y);
            if (vs_has(&vw->eliminated, y)) {
                stack[top++] = y;
                continue;
            }
            int ry = view_find(vw, y);
            if (ry == r) stack[top++] = y;
            else if (vs_has(&vw->alive, ry)) vs_add(&roots, ry);
        }
    }
    return roots;
}

static int min_alive_degree(const view_t* vw) { /* mmw.cpp:73-77 */
    int best = 1 << 30;
    VS_FOR(x, vw->alive) if (vw->degree[x] < best) best = vw->degree[x];
    return best == (1 << 30) ? 0 : best;
}

typedef struct {
    int v, u, common, min_after;
} step_t;

/* contract_step (mmw.cpp:81-116) */
static step_t contract_step(view_t* vw, const graph_t* g) {
    int v = -1, dv = 1 << 30;
    VS_FOR(x, vw->alive) if (vw->degree[x] < dv) { dv = vw->degree[x]; v = x; }
    step_t st;
    if (dv == 0) {
        vs_del(&vw->alive, v);
        st.v = v; st.u = -1; st.common = 0; st.min_after = min_alive_degree(vw);
        return st;
    }
    vs_t adj_v = adjacent_roots(vw, g, v);
    int u = -1, du = 1 << 30;
    VS_FOR(x, adj_v) if (vw->degree[x] < du) { du = vw->degree[x]; u = x; }
    vs_t adj_u = adjacent_roots(vw, g, u);
    vs_t common = vs_and(adj_v, adj_u);
    vs_del(&common, v);
    vs_del(&common, u);
    int c = vs_count(&common);
    vw->parent[u] = (uint8_t)v;
    vs_del(&vw->alive, u);
    vw->degree[v] = (uint8_t)(vw->degree[v] + vw->degree[u] - c - 2);
    VS_FOR(w, common) --vw->degree[w];
    st.v = v; st.u = u; st.common = c; st.min_after = min_alive_degree(vw);
    return st;
}

/* run_mmw (mmw.cpp:120-140); trace may be NULL */
static int run_mmw(view_t* vw, const graph_t* g, int cap, int* trace, int max_steps,
                   int* nsteps) {
    int bound = 0, steps = 0;
    while (vs_count(&vw->alive) >= 2) {
        int d1 = 1 << 30, d2 = 1 << 30;
        VS_FOR(x, vw->alive) {
            int d = vw->degree[x];
            if (d < d1) { d2 = d1; d1 = d; }
            else if (d < d2) d2 = d;
        }
        if (d2 > bound) bound = d2;
        if (bound > cap) break;
        step_t st = contract_step(vw, g);
        if (trace && steps < max_steps) {
            int* o = trace + 5 * steps;
            o[0] = st.v; o[1] = st.u; o[2] = st.common; o[3] = st.min_after; o[4] = bound;
        }
        ++steps;
    }
    if (nsteps) *nsteps = steps;
    return bound;
}

int oracle_mmw_lower_bound(int n, const uint64_t* rows, const uint64_t* s, int cap) {
    graph_t g;
    graph_init(&g, n, rows);
    view_t vw;
    view_init(&vw, &g, vs_load(s));
    return run_mmw(&vw, &g, cap, NULL, 0, NULL);
}

int oracle_mmw_trace(int n, const uint64_t* rows, const uint64_t* s, int cap, int* out,
                     int max_steps, int* bound_out) {
    graph_t g;
    graph_init(&g, n, rows);
    view_t vw;
    view_init(&vw, &g, vs_load(s));
    int steps = 0;
    int b = run_mmw(&vw, &g, cap, out, max_steps, &steps);
    if (bound_out) *bound_out = b;
    return steps;
}

/* ------------------------------------------------------------------ */
/* Layers and the DP engine (dp.hpp, dp.cpp)                            */
typedef struct {
    vs_t set;
    uint32_t hist;
} state_t;

typedef struct {
    state_t* v;
    size_t size, cap;
} layer_t;

static int layer_push(layer_t* L, state_t s) {
    if (L->size == L->cap) {
        size_t nc = L->cap ? 2 * L->cap : 16;
        state_t* p = (state_t*)realloc(L->v, nc * sizeof(state_t));
        if (!p) return 0;
        L->v = p;
        L->cap = nc;
    }
    L->v[L->size++] = s;
    return 1;
}

typedef struct {
    uint64_t k, round, expanded, emitted, duplicates, mmw_pruned;
    uint8_t overflowed;
} lstats_t;

struct oracle_run {
    int outcome;
    state_t witness;
    int overflowed;
    lstats_t* rounds;
    int nrounds;
    layer_t* layers;
    int nlayers;
    char error[160];
};

/* push_history (dp.hpp:19-21) */
static inline uint32_t push_history(uint32_t h, int v) { return (h << 8) | (uint32_t)(v & 0xFF); }

/* Exact dedup: first-emission-wins set keyed by the vertex set. Children
 * are generated in rank order (parent index major, vertex minor) in this
 * single-threaded restatement, so "keep the minimum rank per key, then
 * order by rank" (dp.cpp:130-157) is exactly "keep first occurrences in
 * generation order". */
typedef struct {
    vs_t* keys;
    uint8_t* used;
    size_t mask;
} kset_t;

static uint64_t mix64(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
    return x ^ (x >> 33);
}

static int kset_init(kset_t* h, size_t expected) {
    size_t c = 16;
    while (c < 2 * expected + 16) c <<= 1;
    h->keys = (vs_t*)malloc(c * sizeof(vs_t));
    h->used = (uint8_t*)calloc(c, 1);
    h->mask = c - 1;
    return h->keys && h->used;
}
static void kset_free(kset_t* h) { free(h->keys); free(h->used); }
/* returns 1 when newly inserted */
static int kset_insert(kset_t* h, vs_t k) {
    size_t i = (size_t)mix64(k.w[0] ^ mix64(k.w[1])) & h->mask;
    while (h->used[i]) {
        if (vs_eq(h->keys[i], k)) return 0;
        i = (i + 1) & h->mask;
    }
    h->used[i] = 1;
    h->keys[i] = k;
    return 1;
}

typedef struct {
    const graph_t* g;
    int k;
    vs_t forbidden;
    int dedup, mmw;
    uint64_t max_states;
    int bpe, hashes;
} cfg_t;

/* expand_layer (dp.cpp:73-165) with expand_range (dp.cpp:39-69) inlined. */
static int expand_layer(const cfg_t* c, const layer_t* in, layer_t* out, lstats_t* st) {
    const graph_t* g = c->g;
    int words = g->n > 64 ? 2 : 1;
    st->expanded = in->size;
    st->emitted = st->duplicates = st->mmw_pruned = 0;
    st->overflowed = 0;
    out->size = 0;
    if (in->size == 0) return 1;

    int free_count = g->n - vs_count(&c->forbidden);
    if (free_count < 0) free_count = 0;
    uint64_t upper = (uint64_t)in->size * (uint64_t)free_count;
    if (upper < 1) upper = 1;
    uint64_t cap = c->max_states < upper ? c->max_states : upper;

    /* Children of all parents, generated in rank order. */
    size_t nchild = 0, nchild_cap = 0;
    state_t* child = NULL;
    vs_t uni = vs_first_n(g->n);
    vs_t* rows = (vs_t*)malloc(sizeof(vs_t) * ORACLE_MAXV);
    if (!rows) return 0;
    for (size_t idx = 0; idx < in->size; ++idx) {
        vs_t s = in->v[idx].set;
        vs_t open = vs_minus(uni, s);
        vs_t eligible = vs_minus(open, c->forbidden);
        if (c->mmw) VS_FOR(w, open) rows[w] = q_set(g, s, w);
        VS_FOR(v, eligible) {
            vs_t q = c->mmw ? rows[v] : q_set(g, s, v);
            if (vs_count(&q) > c->k) continue;
            if (c->mmw) {
                view_t vw;
                view_init_after(&vw, g, s, v, rows);
                if (run_mmw(&vw, g, c->k, NULL, 0, NULL) > c->k) {
                    ++st->mmw_pruned;
                    continue;
                }
            }
            if (nchild == nchild_cap) {
                nchild_cap = nchild_cap ? 2 * nchild_cap : 64;
                state_t* p = (state_t*)realloc(child, nchild_cap * sizeof(state_t));
                if (!p) { free(child); free(rows); return 0; }
                child = p;
            }
            state_t ch;
            ch.set = s;
            vs_add(&ch.set, v);
            ch.hist = push_history(in->v[idx].hist, v);
            child[nchild++] = ch;
        }
    }
    free(rows);

    if (c->dedup == 0) {
        /* Bloom branch (dp.cpp:93-117) at one thread: cursor order = rank order */
        bloom_t b;
        if (!bloom_init(&b, cap, c->bpe, c->hashes)) { free(child); return 0; }
        uint64_t produced = 0;
        for (size_t i = 0; i < nchild; ++i) {
            if (!bloom_insert(&b, child[i].set.w, words)) {
                ++st->duplicates;
                continue;
            }
            if (produced < cap && !layer_push(out, child[i])) { free(b.words); free(child); return 0; }
            ++produced;
        }
        free(b.words);
        st->overflowed = produced > cap;
    } else {
        /* Exact branch (dp.cpp:118-158) */
        kset_t h;
        if (!kset_init(&h, nchild)) { free(child); return 0; }
        uint64_t unique = 0;
        for (size_t i = 0; i < nchild; ++i) {
            if (!kset_insert(&h, child[i].set)) continue;
            if (unique < cap && !layer_push(out, child[i])) { kset_free(&h); free(child); return 0; }
            ++unique;
        }
        kset_free(&h);
        st->duplicates = nchild - unique;
        st->overflowed = unique > cap;
    }
    free(child);
    st->emitted = out->size;
    return 1;
}

static oracle_run* run_new(void) {
    oracle_run* r = (oracle_run*)calloc(1, sizeof(oracle_run));
    return r;
}

static int run_add_round(oracle_run* r, lstats_t st) {
    lstats_t* p = (lstats_t*)realloc(r->rounds, (size_t)(r->nrounds + 1) * sizeof(lstats_t));
    if (!p) return 0;
    r->rounds = p;
    r->rounds[r->nrounds++] = st;
    return 1;
}

static int run_add_layer(oracle_run* r, const layer_t* L) {
    layer_t* p = (layer_t*)realloc(r->layers, (size_t)(r->nlayers + 1) * sizeof(layer_t));
    if (!p) return 0;
    r->layers = p;
    layer_t copy = {NULL, 0, 0};
    if (L->size) {
        copy.v = (state_t*)malloc(L->size * sizeof(state_t));
        if (!copy.v) return 0;
        memcpy(copy.v, L->v, L->size * sizeof(state_t));
        copy.size = copy.cap = L->size;
    }
    r->layers[r->nlayers++] = copy;
    return 1;
}

/* decide (dp.cpp:167-194). Outcome: 0 feasible, 1 infeasible, 2 indeterminate */
oracle_run* oracle_decide(int n, const uint64_t* rows, int k, const uint64_t* forbidden,
                          int dedup, int mmw, uint64_t cap, int bpe, int hashes, int rounds,
                          int keep_layers) {
    oracle_run* r = run_new();
    if (!r) return NULL;
    r->outcome = 1;
    r->witness.hist = 0xFFFFFFFFu;
    if (n < 0 || n > ORACLE_MAXV) { snprintf(r->error, sizeof r->error, "vertex count out of range"); return r; }
    if (k < 0) { snprintf(r->error, sizeof r->error, "k must be non-negative"); return r; }
    if (cap == 0) { snprintf(r->error, sizeof r->error, "layer capacity must be positive"); return r; }
    graph_t* g = (graph_t*)malloc(sizeof(graph_t));
    if (!g) { snprintf(r->error, sizeof r->error, "out of memory"); return r; }
    graph_init(g, n, rows);
    if (rounds < 0) rounds = n - k - 1 > 0 ? n - k - 1 : 0;
    cfg_t c = {g, k, forbidden ? vs_load(forbidden) : (vs_t){{0, 0}}, dedup, mmw, cap, bpe, hashes};

    layer_t cur = {NULL, 0, 0}, nxt = {NULL, 0, 0};
    state_t root = {{{0, 0}}, 0xFFFFFFFFu};
    layer_push(&cur, root);
    int done = 0;
    for (int round = 0; round < rounds && !done; ++round) {
        lstats_t st;
        memset(&st, 0, sizeof st);
        st.k = (uint64_t)k;
        st.round = (uint64_t)round;
        if (!expand_layer(&c, &cur, &nxt, &st)) { snprintf(r->error, sizeof r->error, "out of memory"); done = 2; break; }
        r->overflowed = r->overflowed || st.overflowed;
        run_add_round(r, st);
        if (keep_layers) run_add_layer(r, &nxt);
        if (nxt.size == 0) {
            r->outcome = r->overflowed ? 2 : 1;
            done = 1;
            break;
        }
        layer_t t = cur; cur = nxt; nxt = t;
    }
    if (!done) {
        r->outcome = 0;
        r->witness = cur.v[0];
    }
    free(cur.v);
    free(nxt.v);
    free(g);
    return r;
}

oracle_run* oracle_expand_layer(int n, const uint64_t* rows, int k, const uint64_t* forbidden,
                                const uint64_t* in_sets, const uint32_t* in_hist,
                                size_t in_count, int dedup, int mmw, uint64_t cap, int bpe,
                                int hashes) {
    oracle_run* r = run_new();
    if (!r) return NULL;
    graph_t* g = (graph_t*)malloc(sizeof(graph_t));
    if (!g) { snprintf(r->error, sizeof r->error, "out of memory"); return r; }
    graph_init(g, n, rows);
    cfg_t c = {g, k, forbidden ? vs_load(forbidden) : (vs_t){{0, 0}}, dedup, mmw, cap, bpe, hashes};
    layer_t in = {NULL, 0, 0}, out = {NULL, 0, 0};
    for (size_t i = 0; i < in_count; ++i) {
        state_t s = {{{in_sets[2 * i], in_sets[2 * i + 1]}}, in_hist[i]};
        layer_push(&in, s);
    }
    lstats_t st;
    memset(&st, 0, sizeof st);
    st.k = (uint64_t)k;
    if (!expand_layer(&c, &in, &out, &st)) snprintf(r->error, sizeof r->error, "out of memory");
    r->overflowed = st.overflowed;
    run_add_round(r, st);
    run_add_layer(r, &out);
    free(in.v);
    free(out.v);
    free(g);
    return r;
}

const char* oracle_run_error(const oracle_run* r) { return r->error; }
int oracle_run_outcome(const oracle_run* r) { return r->outcome; }
int oracle_run_overflowed(const oracle_run* r) { return r->overflowed; }
void oracle_run_witness(const oracle_run* r, uint64_t* set2, uint32_t* hist) {
    set2[0] = r->witness.set.w[0];
    set2[1] = r->witness.set.w[1];
    *hist = r->witness.hist;
}
int oracle_run_round_count(const oracle_run* r) { return r->nrounds; }
void oracle_run_rounds(const oracle_run* r, uint64_t* stats, uint8_t* ovf) {
    for (int i = 0; i < r->nrounds; ++i) {
        const lstats_t* s = &r->rounds[i];
        uint64_t* o = stats + 6 * i;
        o[0] = s->k; o[1] = s->round; o[2] = s->expanded; o[3] = s->emitted;
        o[4] = s->duplicates; o[5] = s->mmw_pruned;
        ovf[i] = s->overflowed;
    }
}
int oracle_run_layer_count(const oracle_run* r) { return r->nlayers; }
uint64_t oracle_run_layer_size(const oracle_run* r, int i) { return r->layers[i].size; }
void oracle_run_layer(const oracle_run* r, int i, uint64_t* sets2, uint32_t* hist) {
    const layer_t* L = &r->layers[i];
    for (size_t j = 0; j < L->size; ++j) {
        sets2[2 * j] = L->v[j].set.w[0];
        sets2[2 * j + 1] = L->v[j].set.w[1];
        hist[j] = L->v[j].hist;
    }
}
void oracle_run_free(oracle_run* r) {
    if (!r) return;
    for (int i = 0; i < r->nlayers; ++i) free(r->layers[i].v);
    free(r->layers);
    free(r->rounds);
    free(r);
}

/* deepening loop of solve_block (solver.cpp:41-65), no improvement edges */
int oracle_deepen(int n, const uint64_t* rows, const uint64_t* forbidden, int k0, int dedup,
                  int mmw, uint64_t cap, int bpe, int hashes, uint64_t* expanded_out) {
    for (int k = k0; k < (n > 0 ? n : 1); ++k) {
        oracle_run* r = oracle_decide(n, rows, k, forbidden, dedup, mmw, cap, bpe, hashes, -1, 0);
        if (!r) return -1000000;
        for (int i = 0; i < r->nrounds; ++i)
            if (expanded_out) *expanded_out += r->rounds[i].expanded;
        int oc = r->outcome;
        oracle_run_free(r);
        if (oc == 0) return k;
        if (oc == 2) return -(k + 1);
    }
    return n > 0 ? n - 1 : 0;
}

/* ------------------------------------------------------------------ */
/* std::mt19937 (32-bit MT, init_genrand) for helpers.hpp:12-32        */
typedef struct {
    uint32_t mt[624];
    int idx;
} mt_t;

static void mt_seed(mt_t* m, uint32_t seed) {
    m->mt[0] = seed;
    for (int i = 1; i < 624; ++i)
        m->mt[i] = 1812433253u * (m->mt[i - 1] ^ (m->mt[i - 1] >> 30)) + (uint32_t)i;
    m->idx = 624;
}

static uint32_t mt_next(mt_t* m) {
    if (m->idx >= 624) {
        for (int i = 0; i < 624; ++i) {
            uint32_t y = (m->mt[i] & 0x80000000u) | (m->mt[(i + 1) % 624] & 0x7fffffffu);
            m->mt[i] = m->mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        m->idx = 0;
    }
    uint32_t y = m->mt[m->idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

int oracle_random_graph(uint32_t seed, int n, double density, int connected, uint64_t* rows) {
    if (n < 0 || n > ORACLE_MAXV) return -1;
    mt_t m;
    mt_seed(&m, seed);
    uint64_t threshold = (uint64_t)(density * 4294967296.0);
    memset(rows, 0, sizeof(uint64_t) * 2 * (size_t)n);
#define ADD_EDGE(a, b)                                              \
    do {                                                            \
        rows[2 * (a) + ((b) >> 6)] |= (uint64_t)1 << ((b) & 63);    \
        rows[2 * (b) + ((a) >> 6)] |= (uint64_t)1 << ((a) & 63);    \
    } while (0)
    if (connected)
        for (int v = 0; v + 1 < n; ++v) ADD_EDGE(v, v + 1);
    for (int u = 0; u < n; ++u)
        for (int v = u + 1; v < n; ++v)
            if ((uint64_t)mt_next(&m) < threshold) ADD_EDGE(u, v);
#undef ADD_EDGE
    return n;
}
