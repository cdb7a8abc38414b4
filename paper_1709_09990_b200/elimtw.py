"""Python mirror of the elimtw C interface (include/elimtw.h, additive
include/elimtw_gpu.h) over ctypes.

Names, argument meaning and error behaviour follow the reference's C API
(proj/include/elimtw.h:51-99): ``parse_graph`` raises ``ParseError`` with the
line number for ETW_ERROR_PARSE, ``ValueError`` for ETW_ERROR_INVALID_ARGUMENT
and ``ElimtwError`` for ETW_ERROR_INTERNAL (which includes "no CUDA device").
The library is loaded from the package directory; a missing build raises
immediately — there is no Python fallback for the solver.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ETWG_LIB") or os.path.join(_HERE, "libelimtw.so")

ETW_OK, ETW_ERROR_PARSE, ETW_ERROR_INVALID_ARGUMENT, ETW_ERROR_INTERNAL = 0, 1, 2, 3
FORMATS = {"auto": 0, "gr": 1, "dimacs": 2}
DEDUP = {"bloom": 0, "exact": 1}
SPLIT = {"none": 0, "connected": 1, "biconnected": 2}
OUTCOMES = {0: "feasible", 1: "infeasible", 2: "indeterminate"}
MASK64 = (1 << 64) - 1


class ElimtwError(RuntimeError):
    """ETW_ERROR_INTERNAL (CUDA failure, no device, internal invariant)."""


class ParseError(ValueError):
    """ETW_ERROR_PARSE; the message carries 'line N: ...'."""


class etw_options(C.Structure):
    """Byte-compatible with `etw_options` (elimtw.h:51-63)."""

    _fields_ = [
        ("dedup", C.c_int),
        ("split", C.c_int),
        ("use_mmw", C.c_int),
        ("use_clique", C.c_int),
        ("use_improvement", C.c_int),
        ("thread_count", C.c_int),
        ("max_layer_states", C.c_uint64),
        ("bloom_bits_per_element", C.c_int),
        ("bloom_hashes", C.c_int),
        ("start_k", C.c_int),
        ("emit_order", C.c_int),
    ]


_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)
_ip = C.POINTER(C.c_int)

_lib = None


def library() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ElimtwError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; "
                          "g.build()'` or `make -C paper_1709_09990_b200`")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sig = {
        "etw_options_init": (None, [C.POINTER(etw_options)]),
        "etw_graph_parse": (C.c_int, [C.c_char_p, C.c_size_t, C.c_int, C.POINTER(vp), C.c_char_p,
                                      C.c_size_t]),
        "etw_graph_free": (None, [vp]),
        "etw_graph_vertex_count": (C.c_int, [vp]),
        "etw_graph_edge_count": (C.c_longlong, [vp]),
        "etw_solve": (C.c_int, [vp, C.POINTER(etw_options), C.POINTER(vp), C.c_char_p, C.c_size_t]),
        "etw_result_free": (None, [vp]),
        "etw_result_kind_of": (C.c_int, [vp]),
        "etw_result_value": (C.c_int, [vp]),
        "etw_result_order_len": (C.c_size_t, [vp]),
        "etw_result_order": (_ip, [vp]),
        "etw_result_stats_json": (C.c_char_p, [vp]),
        "etw_check_order": (C.c_int, [vp, _ip, C.c_size_t, _ip, _ip, C.c_char_p, C.c_size_t]),
        "etw_version": (C.c_char_p, []),
        "etwg_device_info": (C.c_int, [_ip, _ip, C.c_char_p, C.c_size_t]),
        "etwg_decide": (C.c_int, [C.c_int, _u64p, C.c_int, _u64p, C.c_int, C.c_int, C.c_uint64,
                                  C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp), C.c_char_p,
                                  C.c_size_t]),
        "etwg_expand_layer": (C.c_int, [C.c_int, _u64p, C.c_int, _u64p, _u64p, _u32p, C.c_size_t,
                                        C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int,
                                        C.POINTER(vp), C.c_char_p, C.c_size_t]),
        "etwg_solve_layers": (C.c_int, [vp, C.POINTER(etw_options), C.POINTER(vp), C.c_char_p,
                                        C.c_size_t]),
        "etwg_run_outcome": (C.c_int, [vp]),
        "etwg_run_overflowed": (C.c_int, [vp]),
        "etwg_run_witness": (None, [vp, _u64p, _u32p]),
        "etwg_run_round_count": (C.c_int, [vp]),
        "etwg_run_rounds": (None, [vp, _u64p, _u8p]),
        "etwg_run_layer_count": (C.c_int, [vp]),
        "etwg_run_layer_size": (C.c_uint64, [vp, C.c_int]),
        "etwg_run_layer_tag": (None, [vp, C.c_int, _ip, _ip]),
        "etwg_run_layer": (None, [vp, C.c_int, _u64p, _u32p]),
        "etwg_run_free": (None, [vp]),
        "etwg_bloom_insert": (C.c_uint64, [C.c_uint64, C.c_int, C.c_int, _u64p, C.c_int,
                                           C.c_size_t, _u8p, _u32p, C.c_size_t]),
        "etwg_times": (C.c_int, [C.POINTER(C.c_double), C.c_int]),
        "etwg_set_profiling": (None, [C.c_int]),
        "etwg_reset_times": (None, []),
        "etwg_timer_begin": (None, []),
        "etwg_timer_end": (C.c_double, []),
        "etwg_graph_rows": (None, [vp, _u64p]),
        "etwg_max_clique": (C.c_int, [C.c_int, _u64p, _u64p]),
        "etwg_disjoint_paths": (C.c_int, [C.c_int, _u64p, _u8p]),
        "etwg_improve_graph": (C.c_int, [C.c_int, _u64p, C.c_int, _u64p]),
        "etwg_mmw_lower_bound": (C.c_int, [C.c_int, _u64p, _u64p, C.c_int]),
        "etwg_split": (C.c_int, [C.c_int, _u64p, C.c_int, _ip, _ip, _ip]),
        "etwg_set_virtual_shards": (C.c_int, [C.c_int, C.c_char_p, C.c_size_t]),
        "etwg_nccl_unique_id": (C.c_int, [_u8p, C.c_char_p, C.c_size_t]),
        "etwg_shard_init": (C.c_int, [_u8p, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
        "etwg_shard_release": (None, []),
        "etwg_shard_info": (None, [_ip, _ip, _ip]),
        "etwg_shard_exchange_p2p": (C.c_int, []),
        "etwg_set_shard_handoff": (None, [C.c_uint64]),
        "etwg_set_shard_mode": (None, [C.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


# Every symbol include/elimtw.h and include/elimtw_gpu.h declare.
PUBLIC_SYMBOLS = (
    "etw_options_init", "etw_graph_parse", "etw_graph_free", "etw_graph_vertex_count",
    "etw_graph_edge_count", "etw_solve", "etw_result_free", "etw_result_kind_of",
    "etw_result_value", "etw_result_order_len", "etw_result_order", "etw_result_stats_json",
    "etw_check_order", "etw_version",
)


def _raise(status: int, err: C.Array) -> None:
    msg = err.value.decode(errors="replace")
    if status == ETW_ERROR_PARSE:
        raise ParseError(msg)
    if status == ETW_ERROR_INVALID_ARGUMENT:
        raise ValueError(msg or "invalid argument")
    raise ElimtwError(msg or "internal error")


def _words(rows: Sequence[int]) -> C.Array:
    buf = (C.c_uint64 * max(2, 2 * len(rows)))()
    for v, r in enumerate(rows):
        buf[2 * v] = r & MASK64
        buf[2 * v + 1] = (r >> 64) & MASK64
    return buf


def _set_words(s: int) -> C.Array:
    return (C.c_uint64 * 2)(s & MASK64, (s >> 64) & MASK64)


@dataclass
class Options:
    """`etw_options` with the reference defaults (capi.cpp:72-85)."""

    dedup: str = "bloom"
    split: str = "biconnected"
    use_mmw: bool = False
    use_clique: bool = True
    use_improvement: bool = True
    thread_count: int = 1
    max_layer_states: int = 10_000_000
    bloom_bits_per_element: int = 24
    bloom_hashes: int = 17
    start_k: int = -1
    emit_order: bool = False

    def to_c(self) -> etw_options:
        o = etw_options()
        library().etw_options_init(C.byref(o))
        o.dedup = DEDUP[self.dedup]
        o.split = SPLIT[self.split]
        o.use_mmw = int(self.use_mmw)
        o.use_clique = int(self.use_clique)
        o.use_improvement = int(self.use_improvement)
        o.thread_count = self.thread_count
        o.max_layer_states = self.max_layer_states
        o.bloom_bits_per_element = self.bloom_bits_per_element
        o.bloom_hashes = self.bloom_hashes
        o.start_k = self.start_k
        o.emit_order = int(self.emit_order)
        return o


class Graph:
    """Owned `etw_graph*`."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    @classmethod
    def parse(cls, text: str, fmt: str = "auto") -> "Graph":
        data = text.encode()
        out = C.c_void_p()
        err = C.create_string_buffer(512)
        st = library().etw_graph_parse(data, len(data), FORMATS[fmt], C.byref(out), err, 512)
        if st != ETW_OK:
            _raise(st, err)
        return cls(out.value)

    @classmethod
    def from_rows(cls, rows: Sequence[int]) -> "Graph":
        n = len(rows)
        lines = [f"p tw {n} 0"]
        for u in range(n):
            for v in range(u + 1, n):
                if (rows[u] >> v) & 1:
                    lines.append(f"{u + 1} {v + 1}")
        return cls.parse("\n".join(lines) + "\n", "gr")

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value and _lib is not None:
            _lib.etw_graph_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def vertex_count(self) -> int:
        return library().etw_graph_vertex_count(self._h)

    @property
    def edge_count(self) -> int:
        return library().etw_graph_edge_count(self._h)

    def rows(self) -> List[int]:
        n = self.vertex_count
        buf = (C.c_uint64 * max(2, 2 * n))()
        library().etwg_graph_rows(self._h, buf)
        return [buf[2 * v] | (buf[2 * v + 1] << 64) for v in range(n)]

    def check_order(self, order: Sequence[int]):
        """(width, decomposition_valid) — etw_check_order."""
        arr = (C.c_int * max(1, len(order)))(*order)
        width, valid = C.c_int(-1), C.c_int(0)
        err = C.create_string_buffer(512)
        st = library().etw_check_order(self._h, arr, len(order), C.byref(width), C.byref(valid),
                                       err, 512)
        if st != ETW_OK:
            _raise(st, err)
        return width.value, bool(valid.value)


@dataclass
class Result:
    kind: str
    value: int
    order: List[int]
    stats_json: str


def solve(graph: Graph, options: Optional[Options] = None) -> Result:
    """etw_solve: exact treewidth (or a lower bound on capacity overflow)."""
    opts = (options or Options()).to_c()
    out = C.c_void_p()
    err = C.create_string_buffer(1024)
    L = library()
    st = L.etw_solve(graph.handle, C.byref(opts), C.byref(out), err, 1024)
    if st != ETW_OK:
        _raise(st, err)
    try:
        kind = "exact" if L.etw_result_kind_of(out) == 0 else "lower_bound"
        n = L.etw_result_order_len(out)
        ptr = L.etw_result_order(out)
        order = [ptr[i] for i in range(n)] if n else []
        stats = L.etw_result_stats_json(out).decode()
        return Result(kind, L.etw_result_value(out), order, stats)
    finally:
        L.etw_result_free(out)


def version() -> str:
    return library().etw_version().decode()


# ---------------------------------------------------------------------------
# additive device seam (elimtw_gpu.h)

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
    layers: list = field(default_factory=list)  # [(set, hist), ...] per layer, in order
    tags: list = field(default_factory=list)    # (k, round) per captured layer


def device_info():
    dev, sms = C.c_int(-1), C.c_int(0)
    name = C.create_string_buffer(128)
    ok = library().etwg_device_info(C.byref(dev), C.byref(sms), name, 128)
    return {"available": bool(ok), "device": dev.value, "sm_count": sms.value,
            "name": name.value.decode()}


def _collect(h: C.c_void_p, keep_layers: bool = True) -> DecideRun:
    L = library()
    try:
        ws = (C.c_uint64 * 2)()
        wh = C.c_uint32()
        L.etwg_run_witness(h, ws, C.byref(wh))
        nr = L.etwg_run_round_count(h)
        st = (C.c_uint64 * (6 * max(1, nr)))()
        ov = (C.c_uint8 * max(1, nr))()
        L.etwg_run_rounds(h, st, ov)
        rounds = [LayerStats(*[int(x) for x in st[6 * i: 6 * i + 6]], bool(ov[i]))
                  for i in range(nr)]
        layers, tags = [], []
        if keep_layers:
            for i in range(L.etwg_run_layer_count(h)):
                sz = L.etwg_run_layer_size(h, i)
                sets = (C.c_uint64 * max(2, 2 * sz))()
                hist = (C.c_uint32 * max(1, sz))()
                L.etwg_run_layer(h, i, sets, hist)
                layers.append([(sets[2 * j] | (sets[2 * j + 1] << 64), hist[j]) for j in range(sz)])
                kk, rr = C.c_int(), C.c_int()
                L.etwg_run_layer_tag(h, i, C.byref(kk), C.byref(rr))
                tags.append((kk.value, rr.value))
        return DecideRun(OUTCOMES[L.etwg_run_outcome(h)], ws[0] | (ws[1] << 64), wh.value,
                         bool(L.etwg_run_overflowed(h)), rounds, layers, tags)
    finally:
        L.etwg_run_free(h)


def decide(rows: Sequence[int], k: int, forbidden: int = 0, dedup: str = "exact",
           mmw: bool = False, cap: int = 10_000_000, bpe: int = 24, hashes: int = 17,
           rounds: int = -1, keep_layers: bool = True) -> DecideRun:
    """etwg_decide: one device decision run (the reference's `decide`)."""
    out = C.c_void_p()
    err = C.create_string_buffer(1024)
    st = library().etwg_decide(len(rows), _words(rows), k, _set_words(forbidden), DEDUP[dedup],
                               int(mmw), cap, bpe, hashes, rounds, int(keep_layers), C.byref(out),
                               err, 1024)
    if st != ETW_OK:
        _raise(st, err)
    return _collect(out, keep_layers)


def expand_layer(rows: Sequence[int], k: int, states, forbidden: int = 0, dedup: str = "exact",
                 mmw: bool = False, cap: int = 10_000_000, bpe: int = 24,
                 hashes: int = 17) -> DecideRun:
    """etwg_expand_layer: one device round over an explicit input layer."""
    sets = (C.c_uint64 * max(2, 2 * len(states)))()
    hist = (C.c_uint32 * max(1, len(states)))()
    for i, (s, h) in enumerate(states):
        sets[2 * i] = s & MASK64
        sets[2 * i + 1] = (s >> 64) & MASK64
        hist[i] = h
    out = C.c_void_p()
    err = C.create_string_buffer(1024)
    st = library().etwg_expand_layer(len(rows), _words(rows), k, _set_words(forbidden), sets, hist,
                                     len(states), DEDUP[dedup], int(mmw), cap, bpe, hashes,
                                     C.byref(out), err, 1024)
    if st != ETW_OK:
        _raise(st, err)
    return _collect(out)


def solve_layers(graph: Graph, options: Optional[Options] = None) -> DecideRun:
    """etwg_solve_layers: solve with every search-phase layer captured."""
    opts = (options or Options()).to_c()
    out = C.c_void_p()
    err = C.create_string_buffer(1024)
    st = library().etwg_solve_layers(graph.handle, C.byref(opts), C.byref(out), err, 1024)
    if st != ETW_OK:
        _raise(st, err)
    return _collect(out)


def bloom_insert(expected: int, keys: Sequence[int], words: int = 1, bpe: int = 24,
                 hashes: int = 17, want_bits: bool = False):
    """Concurrent device insert_and_check batch -> (m, novel flags, bits|None)."""
    flat = (C.c_uint64 * max(1, words * len(keys)))()
    for i, key in enumerate(keys):
        for w in range(words):
            flat[words * i + w] = (key >> (64 * w)) & MASK64
    novel = (C.c_uint8 * max(1, len(keys)))()
    m_guess = max(64, (expected * bpe + 63) // 64 * 64)
    bits = (C.c_uint32 * (m_guess // 32))() if want_bits else None
    m = library().etwg_bloom_insert(expected, bpe, hashes, flat, words, len(keys), novel, bits,
                                    m_guess // 32 if want_bits else 0)
    if m == 0:
        raise ElimtwError("device bloom insert failed")
    bitlist = None
    if want_bits:
        bitlist = [bits[i] for i in range(m // 32)]
    return m, [bool(novel[i]) for i in range(len(keys))], bitlist


def timer_begin() -> None:
    library().etwg_timer_begin()


def timer_end() -> float:
    """Device ms since timer_begin (CUDA events on the engine stream)."""
    ms = library().etwg_timer_end()
    if ms < 0:
        raise ElimtwError("device timer failed")
    return ms


def set_profiling(on: bool) -> None:
    library().etwg_set_profiling(int(on))


def reset_times() -> None:
    library().etwg_reset_times()


TIME_KEYS = ("decide_ms", "expand_ms", "insert_ms", "append_ms", "clear_ms", "fused_ms",
             "expand_launches", "insert_launches", "append_launches", "clear_launches",
             "fused_launches", "kernel_launches", "layer_bytes", "dedup_bytes", "expanded",
             "h2d_bytes", "d2h_bytes", "exchange_bytes", "reruns", "expand_bytes",
             "insert_bytes", "append_bytes", "offered", "unique", "bloom_probed", "bloom_fp", "records")


def times() -> dict:
    buf = (C.c_double * len(TIME_KEYS))()
    n = library().etwg_times(buf, len(TIME_KEYS))
    return {TIME_KEYS[i]: buf[i] for i in range(n)}


# owner sharding (include/elimtw_gpu.h)

def set_virtual_shards(shards: int) -> None:
    """G virtual shards on this process's device (1 turns sharding off)."""
    err = C.create_string_buffer(1024)
    st = library().etwg_set_virtual_shards(shards, err, 1024)
    if st != ETW_OK:
        _raise(st, err)


def nccl_unique_id() -> bytes:
    out = (C.c_uint8 * 128)()
    err = C.create_string_buffer(1024)
    st = library().etwg_nccl_unique_id(out, err, 1024)
    if st != ETW_OK:
        _raise(st, err)
    return bytes(out)


def shard_init(uid: bytes, rank: int, world: int, device: int) -> None:
    """This process becomes shard `rank` of `world` over NCCL on `device`."""
    if len(uid) != 128:
        raise ValueError("ncclUniqueId must be 128 bytes")
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    err = C.create_string_buffer(1024)
    st = library().etwg_shard_init(buf, rank, world, device, err, 1024)
    if st != ETW_OK:
        _raise(st, err)


def set_shard_handoff(states: int) -> None:
    """Layers up to `states` run replicated on every shard (0: shard from the root)."""
    library().etwg_set_shard_handoff(states)


def set_shard_mode(mode: str) -> None:
    """'emitter' (default): states stay on the shard that emitted them;
    'owner': states move to their hash owner."""
    library().etwg_set_shard_mode(1 if mode == "emitter" else 0)


def shard_release() -> None:
    library().etwg_shard_release()


def shard_info() -> dict:
    w, r, v = C.c_int(), C.c_int(), C.c_int()
    library().etwg_shard_info(C.byref(w), C.byref(r), C.byref(v))
    return {"world": w.value, "rank": r.value, "virtual": bool(v.value),
            "p2p": bool(library().etwg_shard_exchange_p2p())}


# host preprocessing (no device needed)

def _prep(status: int, what: str) -> None:
    if status == ETW_ERROR_INVALID_ARGUMENT:
        raise ValueError(f"{what}: invalid argument")
    if status != ETW_OK:
        raise ElimtwError(f"{what}: internal error")


def max_clique(rows: Sequence[int]) -> int:
    out = (C.c_uint64 * 2)()
    _prep(library().etwg_max_clique(len(rows), _words(rows), out), "max_clique")
    return out[0] | (out[1] << 64)


def disjoint_paths(rows: Sequence[int]) -> List[int]:
    n = len(rows)
    out = (C.c_uint8 * max(1, n * n))()
    _prep(library().etwg_disjoint_paths(n, _words(rows), out), "disjoint_paths")
    return list(out[: n * n])


def improve_graph(rows: Sequence[int], k: int) -> List[int]:
    n = len(rows)
    out = (C.c_uint64 * max(2, 2 * n))()
    _prep(library().etwg_improve_graph(n, _words(rows), k, out), "improve_graph")
    return [out[2 * v] | (out[2 * v + 1] << 64) for v in range(n)]


def mmw_lower_bound(rows: Sequence[int], s: int = 0, cap: int = 1 << 30) -> int:
    b = library().etwg_mmw_lower_bound(len(rows), _words(rows), _set_words(s), cap)
    if b < 0:
        raise ValueError("mmw_lower_bound: invalid graph")
    return b


def split(rows: Sequence[int], mode: str = "biconnected"):
    n = len(rows)
    verts = (C.c_int * (4 * n + 4))()
    sizes = (C.c_int * (n + 2))()
    cuts = (C.c_int * (n + 2))()
    m = library().etwg_split(n, _words(rows), SPLIT[mode], verts, sizes, cuts)
    if m < 0:
        raise ValueError("split: invalid graph")
    out, off = [], 0
    for i in range(m):
        out.append((list(verts[off: off + sizes[i]]), cuts[i]))
        off += sizes[i]
    return out
