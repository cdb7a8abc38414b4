"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  — oracle/liboracle.so, the plain-C restatement of the
  reference hot path (oracle/etw_oracle.c), 128-bit vertex sets.
* ``RefLib``  — oracle/_ref/libetwref.so, the unmodified reference core
  compiled from /root/reference sources plus oracle/ref_harness.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(REPO, "oracle", "liboracle.so")
REF_SO = os.path.join(REPO, "oracle", "_ref", "libetwref.so")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u8p = C.POINTER(C.c_uint8)
intp = C.POINTER(C.c_int)

OUTCOMES = {0: "feasible", 1: "infeasible", 2: "indeterminate"}


@dataclass
class LayerStats:
    k: int
    round: int
    expanded: int
    emitted: int
    duplicates: int
    mmw_pruned: int
    overflowed: bool

    def tuple(self):
        return (self.k, self.round, self.expanded, self.emitted, self.duplicates,
                self.mmw_pruned, self.overflowed)


@dataclass
class DecideRun:
    outcome: str
    witness_set: int
    witness_hist: int
    overflowed: bool
    rounds: list = field(default_factory=list)
    # each layer: list of (set:int, history:int) in layer order
    layers: list = field(default_factory=list)
    error: str = ""


def _arr(ctype, values):
    values = list(values)
    return (ctype * max(1, len(values)))(*values)


def rows_words(rows, words=2):
    """Python ints (one per vertex) -> flat list of u64 words."""
    out = []
    for r in rows:
        for i in range(words):
            out.append((r >> (64 * i)) & 0xFFFFFFFFFFFFFFFF)
    return out


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle oracle`")
        L = self.lib = C.CDLL(path)
        L.oracle_murmur3_x86_32.restype = C.c_uint32
        L.oracle_murmur3_x86_32.argtypes = [C.c_void_p, C.c_size_t, C.c_uint32]
        L.oracle_hash_pair.argtypes = [u64p, C.c_int, u32p, u32p]
        L.oracle_bloom_bits.restype = C.c_uint64
        L.oracle_bloom_bits.argtypes = [C.c_uint64, C.c_int]
        L.oracle_bloom_insert_seq.restype = C.c_uint64
        L.oracle_bloom_insert_seq.argtypes = [C.c_uint64, C.c_int, C.c_int, u64p, C.c_int,
                                              C.c_size_t, u8p]
        L.oracle_bloom_expected_fp.restype = C.c_double
        L.oracle_bloom_expected_fp.argtypes = [C.c_uint64, C.c_int, C.c_uint64]
        L.oracle_bloom_query.restype = C.c_uint64
        L.oracle_bloom_query.argtypes = [u32p, C.c_uint64, C.c_int, u64p, C.c_int, C.c_size_t]
        L.oracle_q_set.argtypes = [C.c_int, u64p, u64p, C.c_int, u64p]
        L.oracle_mmw_lower_bound.restype = C.c_int
        L.oracle_mmw_lower_bound.argtypes = [C.c_int, u64p, u64p, C.c_int]
        L.oracle_mmw_trace.restype = C.c_int
        L.oracle_mmw_trace.argtypes = [C.c_int, u64p, u64p, C.c_int, intp, C.c_int, intp]
        L.oracle_decide.restype = C.c_void_p
        L.oracle_decide.argtypes = [C.c_int, u64p, C.c_int, u64p, C.c_int, C.c_int, C.c_uint64,
                                    C.c_int, C.c_int, C.c_int, C.c_int]
        L.oracle_expand_layer.restype = C.c_void_p
        L.oracle_expand_layer.argtypes = [C.c_int, u64p, C.c_int, u64p, u64p, u32p, C.c_size_t,
                                          C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int]
        L.oracle_run_error.restype = C.c_char_p
        L.oracle_run_error.argtypes = [C.c_void_p]
        for name in ("oracle_run_outcome", "oracle_run_overflowed", "oracle_run_round_count",
                     "oracle_run_layer_count"):
            getattr(L, name).restype = C.c_int
            getattr(L, name).argtypes = [C.c_void_p]
        L.oracle_run_witness.argtypes = [C.c_void_p, u64p, u32p]
        L.oracle_run_rounds.argtypes = [C.c_void_p, u64p, u8p]
        L.oracle_run_layer_size.restype = C.c_uint64
        L.oracle_run_layer_size.argtypes = [C.c_void_p, C.c_int]
        L.oracle_run_layer.argtypes = [C.c_void_p, C.c_int, u64p, u32p]
        L.oracle_run_free.argtypes = [C.c_void_p]
        L.oracle_deepen.restype = C.c_int
        L.oracle_deepen.argtypes = [C.c_int, u64p, u64p, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                    C.c_int, C.c_int, u64p]
        L.oracle_random_graph.restype = C.c_int
        L.oracle_random_graph.argtypes = [C.c_uint32, C.c_int, C.c_double, C.c_int, u64p]

    # -- hashing -------------------------------------------------------
    def murmur3(self, data: bytes, seed: int) -> int:
        return self.lib.oracle_murmur3_x86_32(data, len(data), seed)

    def hash_pair(self, key: int, words: int = 1):
        k = _arr(C.c_uint64, [(key >> (64 * i)) & (2**64 - 1) for i in range(words)])
        h1, h2 = C.c_uint32(), C.c_uint32()
        self.lib.oracle_hash_pair(k, words, C.byref(h1), C.byref(h2))
        return h1.value, h2.value

    def bloom_insert_seq(self, expected, keys, bpe=24, hashes=17, words=1):
        flat = []
        for key in keys:
            flat += [(key >> (64 * i)) & (2**64 - 1) for i in range(words)]
        out = (C.c_uint8 * max(1, len(keys)))()
        m = self.lib.oracle_bloom_insert_seq(expected, bpe, hashes, _arr(C.c_uint64, flat), words,
                                             len(keys), out)
        return m, [bool(x) for x in out[: len(keys)]]

    def bloom_query(self, bits, m, keys, hashes=17, words=1):
        flat = []
        for key in keys:
            flat += [(key >> (64 * i)) & (2**64 - 1) for i in range(words)]
        return self.lib.oracle_bloom_query(_arr(C.c_uint32, bits), m, hashes,
                                           _arr(C.c_uint64, flat), words, len(keys))

    # -- graph ---------------------------------------------------------
    def q_set(self, rows, s, v):
        out = (C.c_uint64 * 2)()
        self.lib.oracle_q_set(len(rows), _arr(C.c_uint64, rows_words(rows)),
                              _arr(C.c_uint64, rows_words([s])), v, out)
        return out[0] | (out[1] << 64)

    def mmw_lower_bound(self, rows, s=0, cap=2**31 - 1):
        return self.lib.oracle_mmw_lower_bound(len(rows), _arr(C.c_uint64, rows_words(rows)),
                                               _arr(C.c_uint64, rows_words([s])), cap)

    def mmw_trace(self, rows, s=0, cap=2**31 - 1):
        buf = (C.c_int * (5 * 130))()
        bound = C.c_int()
        m = self.lib.oracle_mmw_trace(len(rows), _arr(C.c_uint64, rows_words(rows)),
                                      _arr(C.c_uint64, rows_words([s])), cap, buf, 130,
                                      C.byref(bound))
        return bound.value, [tuple(buf[5 * i: 5 * i + 5]) for i in range(m)]

    def _collect(self, h, keep_layers=True) -> DecideRun:
        L = self.lib
        try:
            err = L.oracle_run_error(h).decode()
            ws = (C.c_uint64 * 2)()
            wh = C.c_uint32()
            L.oracle_run_witness(h, ws, C.byref(wh))
            nr = L.oracle_run_round_count(h)
            st = (C.c_uint64 * (6 * max(1, nr)))()
            ov = (C.c_uint8 * max(1, nr))()
            L.oracle_run_rounds(h, st, ov)
            rounds = [LayerStats(*[int(x) for x in st[6 * i: 6 * i + 6]], bool(ov[i]))
                      for i in range(nr)]
            layers = []
            if keep_layers:
                for i in range(L.oracle_run_layer_count(h)):
                    sz = L.oracle_run_layer_size(h, i)
                    sets = (C.c_uint64 * max(2, 2 * sz))()
                    hist = (C.c_uint32 * max(1, sz))()
                    L.oracle_run_layer(h, i, sets, hist)
                    layers.append([(sets[2 * j] | (sets[2 * j + 1] << 64), hist[j])
                                   for j in range(sz)])
            return DecideRun(OUTCOMES[L.oracle_run_outcome(h)], ws[0] | (ws[1] << 64), wh.value,
                             bool(L.oracle_run_overflowed(h)), rounds, layers, err)
        finally:
            L.oracle_run_free(h)

    def decide(self, rows, k, forbidden=0, dedup="exact", mmw=False, cap=10_000_000,
               bpe=24, hashes=17, rounds=-1, keep_layers=True) -> DecideRun:
        h = self.lib.oracle_decide(len(rows), _arr(C.c_uint64, rows_words(rows)), k,
                                   _arr(C.c_uint64, rows_words([forbidden])),
                                   1 if dedup == "exact" else 0, int(mmw), cap, bpe, hashes,
                                   rounds, int(keep_layers))
        return self._collect(h, keep_layers)

    def expand_layer(self, rows, k, states, forbidden=0, dedup="exact", mmw=False,
                     cap=10_000_000, bpe=24, hashes=17) -> DecideRun:
        sets = _arr(C.c_uint64, rows_words([s for s, _ in states]))
        hist = _arr(C.c_uint32, [h for _, h in states])
        h = self.lib.oracle_expand_layer(len(rows), _arr(C.c_uint64, rows_words(rows)), k,
                                         _arr(C.c_uint64, rows_words([forbidden])), sets, hist,
                                         len(states), 1 if dedup == "exact" else 0, int(mmw),
                                         cap, bpe, hashes)
        return self._collect(h)

    def deepen(self, rows, k0, forbidden=0, dedup="exact", mmw=False, cap=10_000_000):
        exp = C.c_uint64(0)
        k = self.lib.oracle_deepen(len(rows), _arr(C.c_uint64, rows_words(rows)),
                                   _arr(C.c_uint64, rows_words([forbidden])), k0,
                                   1 if dedup == "exact" else 0, int(mmw), cap, 24, 17,
                                   C.byref(exp))
        return k, exp.value

    def random_graph(self, seed, n, p, connected=False):
        buf = (C.c_uint64 * (2 * max(1, n)))()
        self.lib.oracle_random_graph(seed, n, p, int(connected), buf)
        return [buf[2 * v] | (buf[2 * v + 1] << 64) for v in range(n)]


class RefLib:
    """The unmodified reference (n <= 64 only)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_murmur3_x86_32.restype = C.c_uint32
        L.ref_murmur3_x86_32.argtypes = [C.c_void_p, C.c_size_t, C.c_uint32]
        L.ref_hash_pair.argtypes = [C.c_uint64, u32p, u32p]
        L.ref_bloom_insert_seq.restype = C.c_uint64
        L.ref_bloom_insert_seq.argtypes = [C.c_uint64, C.c_int, C.c_int, u64p, C.c_size_t, u8p]
        L.ref_bloom_expected_fp.restype = C.c_double
        L.ref_bloom_expected_fp.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_uint64]
        L.ref_q_set.restype = C.c_uint64
        L.ref_q_set.argtypes = [C.c_int, u64p, C.c_uint64, C.c_int]
        L.ref_decide.restype = C.c_void_p
        L.ref_decide.argtypes = [C.c_int, u64p, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                 C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_expand_layer.restype = C.c_void_p
        L.ref_expand_layer.argtypes = [C.c_int, u64p, C.c_int, C.c_uint64, u64p, u32p,
                                       C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                       C.c_int, C.c_int]
        L.ref_run_error.restype = C.c_char_p
        L.ref_run_error.argtypes = [C.c_void_p]
        for name in ("ref_run_outcome", "ref_run_overflowed", "ref_run_round_count",
                     "ref_run_layer_count"):
            getattr(L, name).restype = C.c_int
            getattr(L, name).argtypes = [C.c_void_p]
        L.ref_run_witness_set.restype = C.c_uint64
        L.ref_run_witness_set.argtypes = [C.c_void_p]
        L.ref_run_witness_hist.restype = C.c_uint32
        L.ref_run_witness_hist.argtypes = [C.c_void_p]
        L.ref_run_rounds.argtypes = [C.c_void_p, u64p, u8p]
        L.ref_run_layer_size.restype = C.c_uint64
        L.ref_run_layer_size.argtypes = [C.c_void_p, C.c_int]
        L.ref_run_layer.argtypes = [C.c_void_p, C.c_int, u64p, u32p]
        L.ref_run_free.argtypes = [C.c_void_p]
        L.ref_mmw_lower_bound.restype = C.c_int
        L.ref_mmw_lower_bound.argtypes = [C.c_int, u64p, C.c_uint64, C.c_int]
        L.ref_mmw_trace.restype = C.c_int
        L.ref_mmw_trace.argtypes = [C.c_int, u64p, C.c_uint64, C.c_int, intp, C.c_int, intp]
        L.ref_mmw_child_degrees.argtypes = [C.c_int, u64p, C.c_uint64, C.c_int, u8p]
        L.ref_max_clique.restype = C.c_uint64
        L.ref_max_clique.argtypes = [C.c_int, u64p]
        L.ref_disjoint_paths.argtypes = [C.c_int, u64p, u8p]
        L.ref_split.restype = C.c_int
        L.ref_split.argtypes = [C.c_int, u64p, C.c_int, intp, intp, intp]
        L.ref_solve.restype = C.c_int
        L.ref_solve.argtypes = [C.c_int, u64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, intp,
                                intp, intp, C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t,
                                C.c_char_p, C.c_size_t]
        L.ref_verify_order.restype = C.c_int
        L.ref_verify_order.argtypes = [C.c_int, u64p, intp, C.c_int]
        L.ref_generate.restype = C.c_int
        L.ref_generate.argtypes = [C.c_int, C.c_uint32, C.c_int, C.c_int, C.c_double, u64p]
        L.ref_solve_layers.restype = C.c_void_p
        L.ref_solve_layers.argtypes = [C.c_int, u64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_uint64, C.c_int]
        L.ref_improve_graph.argtypes = [C.c_int, u64p, C.c_int, u64p]
        L.ref_parse.restype = C.c_int
        L.ref_parse.argtypes = [C.c_char_p, C.c_size_t, intp, u64p, C.c_char_p, C.c_size_t]

    def murmur3(self, data: bytes, seed: int) -> int:
        return self.lib.ref_murmur3_x86_32(data, len(data), seed)

    def hash_pair(self, key: int):
        h1, h2 = C.c_uint32(), C.c_uint32()
        self.lib.ref_hash_pair(key, C.byref(h1), C.byref(h2))
        return h1.value, h2.value

    def bloom_insert_seq(self, expected, keys, bpe=24, hashes=17):
        out = (C.c_uint8 * max(1, len(keys)))()
        m = self.lib.ref_bloom_insert_seq(expected, bpe, hashes, _arr(C.c_uint64, keys),
                                          len(keys), out)
        return m, [bool(x) for x in out[: len(keys)]]

    def bloom_expected_fp(self, expected, inserted, bpe=24, hashes=17):
        return self.lib.ref_bloom_expected_fp(expected, bpe, hashes, inserted)

    def q_set(self, rows, s, v):
        return self.lib.ref_q_set(len(rows), _arr(C.c_uint64, rows), s, v)

    def _collect(self, h, keep_layers=True) -> DecideRun:
        L = self.lib
        try:
            err = L.ref_run_error(h).decode()
            nr = L.ref_run_round_count(h)
            st = (C.c_uint64 * (6 * max(1, nr)))()
            ov = (C.c_uint8 * max(1, nr))()
            L.ref_run_rounds(h, st, ov)
            rounds = [LayerStats(*[int(x) for x in st[6 * i: 6 * i + 6]], bool(ov[i]))
                      for i in range(nr)]
            layers = []
            if keep_layers:
                for i in range(L.ref_run_layer_count(h)):
                    sz = L.ref_run_layer_size(h, i)
                    sets = (C.c_uint64 * max(1, sz))()
                    hist = (C.c_uint32 * max(1, sz))()
                    L.ref_run_layer(h, i, sets, hist)
                    layers.append([(sets[j], hist[j]) for j in range(sz)])
            return DecideRun(OUTCOMES[L.ref_run_outcome(h)], L.ref_run_witness_set(h),
                             L.ref_run_witness_hist(h), bool(L.ref_run_overflowed(h)), rounds,
                             layers, err)
        finally:
            L.ref_run_free(h)

    def decide(self, rows, k, forbidden=0, dedup="exact", mmw=False, cap=10_000_000,
               bpe=24, hashes=17, rounds=-1, threads=1, keep_layers=True) -> DecideRun:
        h = self.lib.ref_decide(len(rows), _arr(C.c_uint64, rows), k, forbidden,
                                1 if dedup == "exact" else 0, int(mmw), threads, cap, bpe,
                                hashes, rounds, int(keep_layers))
        return self._collect(h, keep_layers)

    def expand_layer(self, rows, k, states, forbidden=0, dedup="exact", mmw=False,
                     cap=10_000_000, bpe=24, hashes=17, threads=1) -> DecideRun:
        h = self.lib.ref_expand_layer(len(rows), _arr(C.c_uint64, rows), k, forbidden,
                                      _arr(C.c_uint64, [s for s, _ in states]),
                                      _arr(C.c_uint32, [x for _, x in states]), len(states),
                                      1 if dedup == "exact" else 0, int(mmw), threads, cap, bpe,
                                      hashes)
        return self._collect(h)

    def mmw_lower_bound(self, rows, s=0, cap=2**31 - 1):
        return self.lib.ref_mmw_lower_bound(len(rows), _arr(C.c_uint64, rows), s, cap)

    def mmw_trace(self, rows, s=0, cap=2**31 - 1):
        buf = (C.c_int * (5 * 70))()
        bound = C.c_int()
        m = self.lib.ref_mmw_trace(len(rows), _arr(C.c_uint64, rows), s, cap, buf, 70,
                                   C.byref(bound))
        return bound.value, [tuple(buf[5 * i: 5 * i + 5]) for i in range(m)]

    def max_clique(self, rows):
        return self.lib.ref_max_clique(len(rows), _arr(C.c_uint64, rows))

    def disjoint_paths(self, rows):
        n = len(rows)
        out = (C.c_uint8 * max(1, n * n))()
        self.lib.ref_disjoint_paths(n, _arr(C.c_uint64, rows), out)
        return list(out[: n * n])

    def split(self, rows, mode):
        n = len(rows)
        verts = (C.c_int * (4 * n + 4))()
        sizes = (C.c_int * (2 * n + 2))()
        cuts = (C.c_int * (2 * n + 2))()
        m = self.lib.ref_split(n, _arr(C.c_uint64, rows), mode, verts, sizes, cuts)
        out, off = [], 0
        for i in range(m):
            out.append((list(verts[off: off + sizes[i]]), cuts[i]))
            off += sizes[i]
        return out

    def solve(self, rows, dedup="bloom", split=2, mmw=False, clique=True, improvement=True,
              threads=1, cap=10_000_000, bpe=24, hashes=17, start_k=-1, emit_order=False,
              json_len=1 << 24):
        n = len(rows)
        kind, value = C.c_int(), C.c_int()
        order = (C.c_int * max(1, n))()
        olen = C.c_size_t()
        js = C.create_string_buffer(json_len)
        err = C.create_string_buffer(512)
        rc = self.lib.ref_solve(n, _arr(C.c_uint64, rows), 1 if dedup == "exact" else 0, split,
                                int(mmw), int(clique), int(improvement), threads, cap, bpe,
                                hashes, start_k, int(emit_order), C.byref(kind), C.byref(value),
                                order, C.byref(olen), js, json_len, err, 512)
        if rc != 0:
            raise RuntimeError(err.value.decode())
        return {"kind": "exact" if kind.value == 0 else "lower_bound_only",
                "value": value.value, "order": list(order[: olen.value]),
                "stats": js.value.decode()}

    def solve_layers(self, rows, dedup="exact", split=2, mmw=False, clique=True,
                     improvement=True, cap=10_000_000, start_k=-1) -> DecideRun:
        """Search-phase layers of solve() via the observer; rounds[i] holds
        (k, round) of layer i."""
        h = self.lib.ref_solve_layers(len(rows), _arr(C.c_uint64, rows),
                                      1 if dedup == "exact" else 0, split, int(mmw), int(clique),
                                      int(improvement), cap, start_k)
        return self._collect(h)

    def improve_graph(self, rows, k):
        out = (C.c_uint64 * max(1, len(rows)))()
        self.lib.ref_improve_graph(len(rows), _arr(C.c_uint64, rows), k, out)
        return list(out[: len(rows)])

    def verify_order(self, rows, order):
        return self.lib.ref_verify_order(len(rows), _arr(C.c_uint64, rows),
                                         _arr(C.c_int, order), len(order))

    def generate(self, kind, seed=0, a=0, b=0, p=0.0):
        buf = (C.c_uint64 * 64)()
        n = self.lib.ref_generate(kind, seed, a, b, p, buf)
        return list(buf[:n])

    def parse(self, text: str):
        data = text.encode()
        n = C.c_int()
        rows = (C.c_uint64 * 64)()
        err = C.create_string_buffer(256)
        rc = self.lib.ref_parse(data, len(data), C.byref(n), rows, err, 256)
        if rc != 0:
            raise ValueError(err.value.decode())
        return list(rows[: n.value])
