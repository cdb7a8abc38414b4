/* Additive C ABI of the B200 build (libelimtw.so.1). Nothing here changes
 * elimtw.h; these entry points expose the device seam the reference keeps
 * internal, so tests and tools can drive it with plain pointers.
 *
 * Vertex sets cross the ABI as two little-endian u64 words (bits 0..127);
 * adjacency is `rows[2*v + w]`. Statuses and error buffers follow elimtw.h.
 *
 *   etwg_decide        replaces decide()        proj/src/dp.hpp:78-79
 *   etwg_expand_layer  replaces expand_layer()  proj/src/dp.hpp:68-70
 *   etwg_solve_layers  solve() with the DpConfig::observer seam
 *                      (dp.hpp:31-32) capturing every search-phase layer
 *   etwg_bloom_insert  one device insert_and_check batch (bloom.cpp:86-97)
 *   etwg_max_clique / etwg_split / etwg_disjoint_paths / etwg_improve_graph /
 *   etwg_mmw_lower_bound   host preprocessing (preprocess.hpp:23-46,
 *                      mmw.hpp:46-47) for parity tests without a GPU
 */
#ifndef ELIMTW_GPU_H
#define ELIMTW_GPU_H

#include "elimtw.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct etwg_run etwg_run;

/* 1 when a CUDA device is usable; fills name/SM count when non-NULL. */
ELIMTW_API int etwg_device_info(int* device, int* sm_count, char* name, size_t name_len);

/* One decision run tw(g) <= k? on the device. dedup: etw_dedup. rounds < 0
 * selects n-k-1. keep_layers copies every layer back (test seam). */
ELIMTW_API etw_status etwg_decide(int n, const uint64_t* rows, int k, const uint64_t* forbidden,
                                  int dedup, int use_mmw, uint64_t max_layer_states,
                                  int bloom_bits_per_element, int bloom_hashes, int rounds,
                                  int keep_layers, etwg_run** out, char* err, size_t err_len);

/* One round over an explicit input layer (sets: 2 words per state). */
ELIMTW_API etw_status etwg_expand_layer(int n, const uint64_t* rows, int k,
                                        const uint64_t* forbidden, const uint64_t* sets,
                                        const uint32_t* hist, size_t count, int dedup,
                                        int use_mmw, uint64_t max_layer_states,
                                        int bloom_bits_per_element, int bloom_hashes,
                                        etwg_run** out, char* err, size_t err_len);

/* Full etw_solve capturing every layer of the search phase in call order. */
ELIMTW_API etw_status etwg_solve_layers(const etw_graph* g, const etw_options* opts,
                                        etwg_run** out, char* err, size_t err_len);

/* 0 feasible, 1 infeasible, 2 indeterminate */
ELIMTW_API int etwg_run_outcome(const etwg_run* r);
ELIMTW_API int etwg_run_overflowed(const etwg_run* r);
ELIMTW_API void etwg_run_witness(const etwg_run* r, uint64_t* set2, uint32_t* hist);
ELIMTW_API int etwg_run_round_count(const etwg_run* r);
/* 6 u64 per round: k, round, expanded, emitted, duplicates, mmw_pruned */
ELIMTW_API void etwg_run_rounds(const etwg_run* r, uint64_t* stats, uint8_t* overflowed);
ELIMTW_API int etwg_run_layer_count(const etwg_run* r);
ELIMTW_API uint64_t etwg_run_layer_size(const etwg_run* r, int i);
/* k and round of captured layer i (etwg_solve_layers) */
ELIMTW_API void etwg_run_layer_tag(const etwg_run* r, int i, int* k, int* round);
ELIMTW_API void etwg_run_layer(const etwg_run* r, int i, uint64_t* sets2, uint32_t* hist);
ELIMTW_API void etwg_run_free(etwg_run* r);

/* Device Bloom filter sized for `expected` elements; inserts `count` keys
 * (words u64 each) concurrently, one per thread, and reports each key's
 * novelty plus the final bit array (m/8 bytes into bits_out when non-NULL).
 * Returns m, 0 on error. */
ELIMTW_API uint64_t etwg_bloom_insert(uint64_t expected, int bits_per_element, int hashes,
                                      const uint64_t* keys, int words, size_t count,
                                      uint8_t* novel_out, uint32_t* bits_out, size_t bits_words);

/* Profiling counters of the device engine (milliseconds / bytes / counts):
 * out[0..] = decide_ms, expand_ms, insert_ms, append_ms, clear_ms, fused_ms,
 * expand_launches, insert_launches, append_launches, clear_launches,
 * fused_launches, kernel_launches, layer_bytes, dedup_bytes, expanded,
 * h2d_bytes, d2h_bytes, exchange_bytes, reruns, expand_bytes, insert_bytes,
 * append_bytes, offered, unique. Returns the number of values written. */
ELIMTW_API int etwg_times(double* out, int len);
/* CUDA events on the engine stream around a region; end synchronizes and
 * returns the device milliseconds in between. */
ELIMTW_API void etwg_timer_begin(void);
ELIMTW_API double etwg_timer_end(void);
ELIMTW_API void etwg_set_profiling(int on);
ELIMTW_API void etwg_reset_times(void);

/* Owner-sharded decides. While sharding is active every decide
 * of this process — etw_solve's included — runs as one shard of G: each
 * layer state lives on shard owner(S), children are routed to their owners
 * every round and a per-round count allgather decides termination.
 *
 *   etwg_set_virtual_shards(G)   G (1..8) virtual shards on this process's
 *                                device, exchanging through device copies:
 *                                the single-GPU double of the NCCL path; 1 = off.
 *   etwg_nccl_unique_id(id)      128-byte ncclUniqueId (rank 0 makes it, the
 *                                caller distributes it, e.g. torch.distributed)
 *   etwg_shard_init(id, rank, world, device)
 *                                one shard per process over NCCL; every rank
 *                                must then make the same sequence of solves
 *   etwg_shard_release()         back to the single-device engine
 *   etwg_shard_info              world size, rank, 1 when virtual
 *   etwg_shard_exchange_p2p      1 when owners pull records over NVLink     */
ELIMTW_API etw_status etwg_set_virtual_shards(int shards, char* err, size_t err_len);
ELIMTW_API etw_status etwg_nccl_unique_id(uint8_t* id128, char* err, size_t err_len);
ELIMTW_API etw_status etwg_shard_init(const uint8_t* id128, int rank, int world, int device, char* err,
                                      size_t err_len);
ELIMTW_API void etwg_shard_release(void);
ELIMTW_API void etwg_shard_info(int* world, int* rank, int* is_virtual);
/* 1 when the NCCL path's owners read their peers' outboxes over NVLink
 * (CUDA IPC; ETWG_EXCHANGE=nccl or a failed peer mapping selects NCCL
 * grouped send/recv instead) */
ELIMTW_API int etwg_shard_exchange_p2p(void);
/* Layers of up to `states` states are expanded redundantly by every shard on
 * the single-device engine (no routing: cheaper than an exchange for small
 * layers); the first larger layer is split by owner and the decide continues
 * sharded. Default 2^19 (env ETWG_HANDOFF); 0 shards from the root. */
ELIMTW_API void etwg_set_shard_handoff(uint64_t states);
/* 1 (default): each next-layer state stays on the shard that emitted its
 * winning (min-rank) child — the owner only deduplicates and returns a mark,
 * layers stay rank-ordered per shard; 0: states move to their hash owner
 * (env ETWG_SHARD_MODE=owner). The NCCL send/recv fallback always uses 0. */
ELIMTW_API void etwg_set_shard_mode(int emitter);

/* host preprocessing (no GPU needed); rows as above. No exception crosses
 * the ABI: the etw_status ones return ETW_ERROR_INVALID_ARGUMENT (NULL
 * pointer, n outside 0..128) or ETW_ERROR_INTERNAL, the int ones -1. */
ELIMTW_API void etwg_graph_rows(const etw_graph* g, uint64_t* rows);
ELIMTW_API etw_status etwg_max_clique(int n, const uint64_t* rows, uint64_t* out2);
ELIMTW_API etw_status etwg_disjoint_paths(int n, const uint64_t* rows, uint8_t* out);
ELIMTW_API etw_status etwg_improve_graph(int n, const uint64_t* rows, int k, uint64_t* out_rows);
ELIMTW_API int etwg_mmw_lower_bound(int n, const uint64_t* rows, const uint64_t* s, int cap);
/* verts: concatenated original ids; returns block count (-1 on failure) */
ELIMTW_API int etwg_split(int n, const uint64_t* rows, int mode, int* verts, int* sizes,
                          int* cuts);

#ifdef __cplusplus
}
#endif

#endif /* ELIMTW_GPU_H */
