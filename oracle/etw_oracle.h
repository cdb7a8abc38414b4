/* TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 wavefront.
 *
 * A plain-C, single-threaded restatement of the reference elimtw hot path
 * (decide -> expand_layer -> q_set, Bloom/Murmur3, minor-min-width) widened
 * to 128-bit vertex sets so it also covers the n > 64 configs the reference
 * rejects (proj/src/graph.cpp:111-113). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product library never
 * links it. Parity of this restatement is pinned against the reference
 * itself (oracle/_ref/libetwref.so, built from /root/reference sources) and
 * the golden vectors in tests/golden/ (see tests/test_oracle.py).
 *
 * Vertex sets are two little-endian u64 words; rows is n*2 words. For
 * n <= 64 every semantic matches the reference bit for bit (8-byte Bloom
 * key, rank idx*64+v); for 64 < n <= 128 the Bloom key is the 16 bytes of
 * the set (word 0 first) and the rank is idx*128+v, an extension the
 * reference does not define. */
#ifndef ETW_ORACLE_H
#define ETW_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_MAXV 128

uint32_t oracle_murmur3_x86_32(const void* data, size_t len, uint32_t seed);
/* words = 1 (8-byte key) or 2 (16-byte key) */
void oracle_hash_pair(const uint64_t* key, int words, uint32_t* h1, uint32_t* h2);
uint64_t oracle_bloom_bits(uint64_t expected, int bits_per_element);
/* Sequential inserts into a fresh filter; novel flags per key. Returns m. */
uint64_t oracle_bloom_insert_seq(uint64_t expected, int bpe, int hashes,
                                 const uint64_t* keys, int words, size_t count,
                                 uint8_t* novel_out);
double oracle_bloom_expected_fp(uint64_t m, int hashes, uint64_t inserted);
/* might_contain (bloom.cpp:99-107) against an external bit array given as
 * m/32 little-endian 32-bit words; returns how many keys test positive. */
uint64_t oracle_bloom_query(const uint32_t* bits, uint64_t m, int hashes, const uint64_t* keys,
                            int words, size_t count);

/* Q(S,v) (graph.hpp:61-78); out = 2 words. */
void oracle_q_set(int n, const uint64_t* rows, const uint64_t* s, int v, uint64_t* out);

int oracle_mmw_lower_bound(int n, const uint64_t* rows, const uint64_t* s, int cap);
/* 5 ints per step: v, u, common, min_degree_after, bound_after. */
int oracle_mmw_trace(int n, const uint64_t* rows, const uint64_t* s, int cap, int* out,
                     int max_steps, int* bound_out);

typedef struct oracle_run oracle_run;

/* decide (dp.cpp:167-194). dedup: 0 bloom, 1 exact. rounds < 0 -> n-k-1.
 * Returns NULL only on allocation failure; check oracle_run_error. */
oracle_run* oracle_decide(int n, const uint64_t* rows, int k, const uint64_t* forbidden,
                          int dedup, int mmw, uint64_t cap, int bpe, int hashes,
                          int rounds, int keep_layers);
/* one expand_layer (dp.cpp:73-165) over an explicit input list */
oracle_run* oracle_expand_layer(int n, const uint64_t* rows, int k,
                                const uint64_t* forbidden, const uint64_t* in_sets,
                                const uint32_t* in_hist, size_t in_count, int dedup,
                                int mmw, uint64_t cap, int bpe, int hashes);

const char* oracle_run_error(const oracle_run* r);
int oracle_run_outcome(const oracle_run* r); /* 0 feasible, 1 infeasible, 2 indeterminate */
int oracle_run_overflowed(const oracle_run* r);
void oracle_run_witness(const oracle_run* r, uint64_t* set2, uint32_t* hist);
int oracle_run_round_count(const oracle_run* r);
/* 6 u64 per round: k, round, expanded, emitted, duplicates, mmw_pruned */
void oracle_run_rounds(const oracle_run* r, uint64_t* stats, uint8_t* ovf);
int oracle_run_layer_count(const oracle_run* r);
uint64_t oracle_run_layer_size(const oracle_run* r, int i);
void oracle_run_layer(const oracle_run* r, int i, uint64_t* sets2, uint32_t* hist);
void oracle_run_free(oracle_run* r);

/* Deepening loop of solve_block (solver.cpp:41-65) on an already
 * preprocessed graph: decide at k = k0, k0+1, ... with forbidden clique.
 * Returns the first feasible k, or -(k+1) when indeterminate at k.
 * expanded_out accumulates LayerStats::expanded. */
int oracle_deepen(int n, const uint64_t* rows, const uint64_t* forbidden, int k0, int dedup,
                  int mmw, uint64_t cap, int bpe, int hashes, uint64_t* expanded_out);

/* mt19937 generators (proj/tests/helpers.hpp:12-32); rows n*2 words. */
int oracle_random_graph(uint32_t seed, int n, double density, int connected,
                        uint64_t* rows);

#ifdef __cplusplus
}
#endif
#endif
