"""Host side of the drop-in boundary, CPU only: the C-ABI library loads and
exports every symbol include/*.h declares; parsing, order checking and the
host preprocessing agree with the reference (proj/tests/test_graph.cpp,
test_capi.cpp, test_preprocess.cpp); generators reproduce helpers.hpp; and the
solver refuses to run without a device instead of falling back to the CPU."""
import ctypes
import json
import os
import re
import subprocess

import pytest

from conftest import REPO, instance_text
from paper_1709_09990_b200 import generators as G

GRID = ("c 3x3 grid\np tw 9 12\n1 2\n2 3\n4 5\n5 6\n7 8\n8 9\n"
        "1 4\n4 7\n2 5\n5 8\n3 6\n6 9\n")


def declared_symbols():
    names = []
    for h in ("elimtw.h", "elimtw_gpu.h"):
        text = open(os.path.join(REPO, "include", h)).read()
        names += re.findall(r"ELIMTW_API[^;(]*?\b(etwg?_\w+)\s*\(", text, flags=re.S)
    return names


def test_library_exports_every_declared_symbol(E):
    names = declared_symbols()
    assert len([n for n in names if n.startswith("etw_")]) == 14
    lib = E.library()
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", E.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    assert set(names) <= exported
    # hidden visibility: nothing but the C ABI leaks
    assert all(s.startswith(("etw_", "etwg_")) for s in exported if not s.startswith("_"))


def test_version_and_defaults(E):
    assert E.version() == "1.0.0"
    o = E.etw_options()
    E.library().etw_options_init(ctypes.byref(o))
    assert (o.dedup, o.split, o.use_mmw, o.use_clique, o.use_improvement, o.thread_count,
            o.max_layer_states, o.bloom_bits_per_element, o.bloom_hashes, o.start_k,
            o.emit_order) == (0, 2, 0, 1, 1, 1, 10_000_000, 24, 17, -1, 0)


def test_parse_inspect_and_errors(E):
    g = E.Graph.parse(GRID)
    assert (g.vertex_count, g.edge_count) == (9, 12)
    d = E.Graph.parse("p edge 3 3\ne 1 2\ne 2 3\ne 1 3\n", "dimacs")
    assert d.vertex_count == 3 and d.edge_count == 3
    with pytest.raises(E.ParseError, match="line 2"):
        E.Graph.parse("p tw 3 1\n1 9\n", "gr")
    for bad in ("p tw 3 1\n1 two\n", "", "p edge 3 1\ne 1 2\n"):
        with pytest.raises(E.ParseError):
            E.Graph.parse(bad, "gr")
    with pytest.raises(E.ParseError):
        E.Graph.parse("hello\n")
    # 128-vertex limit (the reference stops at 64, graph.cpp:111-113)
    assert E.Graph.parse("p tw 128 1\n1 128\n").vertex_count == 128
    with pytest.raises(E.ParseError, match="limit is 128"):
        E.Graph.parse("p tw 129 0\n")


def test_parse_matches_reference(E, ref):
    for name in ("water", "myciel4", "McGeeGraph", "queen5_5", "queen6_6"):
        assert E.Graph.parse(instance_text(name)).rows() == ref.parse(instance_text(name))


def test_check_order(E):
    g = E.Graph.parse(GRID)
    w, ok = g.check_order([0, 2, 6, 8, 1, 3, 5, 7, 4])
    assert ok and w == 3
    with pytest.raises(ValueError):
        g.check_order([0, 1, 2])
    with pytest.raises(ValueError):
        g.check_order([0, 1, 2, 3, 4, 5, 6, 7, 7])


def test_check_order_matches_reference_width(E, ref):
    import random
    rng = random.Random(5)
    for seed in range(30):
        rows = G.random_graph(seed, 12, 0.35)
        g = E.Graph.from_rows(rows)
        order = list(range(12))
        rng.shuffle(order)
        w, ok = g.check_order(order)
        assert ok and w == ref.verify_order(rows, order)


def test_generators_match_reference(ref):
    for seed in range(6):
        assert G.random_graph(seed, 40, 0.3) == ref.generate(0, seed, 40, 0, 0.3)
        assert G.random_graph(seed, 30, 0.25, connected=True) == ref.generate(1, seed, 30, 0, 0.25)
    assert G.grid_graph(8, 8) == ref.generate(2, 0, 8, 8)
    assert G.petersen_graph() == ref.generate(7)
    assert G.myciel(4) == ref.parse(instance_text("myciel4"))
    assert G.queen_graph(6, 6) == ref.parse(instance_text("queen6_6"))


def test_preprocess_matches_reference(E, ref):
    """split / max_clique / disjoint paths / improvement / root MMW are host
    C++ and must be bit-identical (preprocess.cpp:188-258, mmw.cpp:148-151)."""
    for seed in range(120):
        n = 2 + seed % 22
        rows = G.random_graph(seed * 7 + 1, n, 0.1 + 0.1 * (seed % 6))
        assert E.max_clique(rows) == ref.max_clique(rows)
        for mode, name in enumerate(("none", "connected", "biconnected")):
            assert E.split(rows, name) == ref.split(rows, mode)
        assert E.disjoint_paths(rows) == ref.disjoint_paths(rows)
        for k in (1, 3, 5):
            assert E.improve_graph(rows, k) == ref.improve_graph(rows, k)
        for s, cap in ((0, 2**30), (5 & ((1 << n) - 1), 2**30), (0x1234 & ((1 << n) - 1), 3)):
            assert E.mmw_lower_bound(rows, s, cap) == ref.mmw_lower_bound(rows, s, cap)


def test_preprocess_instances_match_goldens(E, goldens):
    for name, g in goldens["instances"].items():
        rows = E.Graph.parse(instance_text(name)).rows()
        assert E.max_clique(rows) == g["max_clique"]
        assert E.mmw_lower_bound(rows) == g["mmw_root"]


def test_wide_graph_host_paths(E, oracle):
    """n > 64: host preprocessing on 128-bit rows (no reference exists)."""
    rows = G.grid_with_chords(8, 9, 6, 7)
    assert len(rows) == 72
    clique = E.max_clique(rows)
    assert bin(clique).count("1") >= 2
    assert E.mmw_lower_bound(rows) == oracle.mmw_lower_bound(rows)
    blocks = E.split(rows)
    assert sum(len(v) for v, _ in blocks) >= 72


def test_solve_without_device_fails_loudly(E):
    if E.device_info()["available"]:
        pytest.skip("a device is present")
    with pytest.raises(E.ElimtwError, match="no CUDA device"):
        E.solve(E.Graph.parse(GRID))
    with pytest.raises(E.ElimtwError):
        E.decide(G.path_graph(4), 1)


def test_option_validation_is_invalid_argument(E):
    g = E.Graph.parse(GRID)
    with pytest.raises(ValueError, match="thread count"):
        E.solve(g, E.Options(thread_count=0))
    with pytest.raises(ValueError, match="layer capacity"):
        E.solve(g, E.Options(max_layer_states=0))


def test_golden_stats_are_reference_schema(goldens):
    s = json.loads(goldens["instances"]["myciel4"]["exact_stats"])
    assert s["schema_version"] == 1 and s["result"]["value"] == 10
    assert s["totals"]["expanded"] == 86786


def test_shard_api_validates_arguments_without_a_device(E):
    """The sharding seam (elimtw_gpu.h) rejects bad arguments before touching
    a device or NCCL, with the reference's error classes; without sharding
    the process stays on the single-device engine."""
    from paper_1709_09990_b200 import distributed as D
    assert E.shard_info() == {"world": 1, "rank": 0, "virtual": False, "p2p": False}
    for bad in (0, 9, -1):
        with pytest.raises(ValueError):
            E.set_virtual_shards(bad)
    uid = E.nccl_unique_id()  # needs libnccl, not a GPU
    assert len(uid) == 128
    with pytest.raises(ValueError):
        E.shard_init(uid, 2, 2, 0)  # rank out of range
    with pytest.raises(ValueError):
        E.shard_init(uid, 0, 9, 0)  # world too large
    with pytest.raises(ValueError):
        E.shard_init(b"x" * 10, 0, 2, 0)  # not an ncclUniqueId
    E.set_virtual_shards(1)  # "off" is always accepted
    assert D.init_shards() == E.shard_info()  # world 1 (no torchrun env): a no-op
    assert E.shard_info()["world"] == 1


def test_preprocess_errors_do_not_cross_the_abi(E):
    """etwg_* preprocessing entry points map exceptions to status codes
    (graph_from_words rejects n > 128) instead of terminating the process."""
    lib = E.library()
    rows = (ctypes.c_uint64 * 512)()
    out = (ctypes.c_uint64 * 512)()
    assert lib.etwg_max_clique(200, rows, out) == E.ETW_ERROR_INVALID_ARGUMENT
    assert lib.etwg_improve_graph(-1, rows, 3, out) == E.ETW_ERROR_INVALID_ARGUMENT
    assert lib.etwg_max_clique(3, None, out) == E.ETW_ERROR_INVALID_ARGUMENT
    assert lib.etwg_mmw_lower_bound(200, rows, out, 5) == -1
    v = (ctypes.c_int * 4)()
    assert lib.etwg_split(200, rows, 2, v, v, v) == -1
    with pytest.raises(ValueError):
        E.max_clique([0] * 200)


def _embed(rows, n2, rng, triangle):
    """G (n <= 64) placed order-preservingly at sorted random positions of an
    n2-vertex graph; the other vertices are isolated fillers, or (triangle)
    three of the highest fillers form a triangle."""
    n = len(rows)
    pos = sorted(rng.sample(range(n2), n))
    fill = [p for p in range(n2) if p not in set(pos)]
    out = [0] * n2
    for u in range(n):
        for v in range(n):
            if rows[u] >> v & 1:
                out[pos[u]] |= 1 << pos[v]
    if triangle:
        a, b, c = fill[-3:]
        for x, y in ((a, b), (a, c), (b, c)):
            out[x] |= 1 << y
            out[y] |= 1 << x
    return out, pos


def _lift(mask, pos):
    return sum(1 << pos[v] for v in range(len(pos)) if mask >> v & 1)


def test_wide_preprocess_matches_reference_after_embedding(E, ref):
    """f3: the 128-bit host preprocessing keeps the
    reference's tie-breaking at n > 64. Reference graphs (n <= 64) are
    embedded order-preservingly into 72..128 vertices (positions spread over
    both 64-bit words); max_clique (preprocess.cpp:171-184), the
    vertex-disjoint path counts (:218-243), the improvement edges, the root
    MMW bound and the split blocks must be the reference's, relabelled."""
    import random
    rng = random.Random(11)
    graphs = [G.random_graph(s * 13 + 5, 20 + s % 45, 0.15 + 0.05 * (s % 5)) for s in range(14)]
    graphs += [G.queen_graph(6, 6), G.myciel(4), G.grid_graph(7, 9)]
    for i, rows in enumerate(graphs):
        n = len(rows)
        n2 = (72, 96, 128)[i % 3]
        clique = ref.max_clique(rows)
        triangle = bin(clique).count("1") >= 4
        big, pos = _embed(rows, n2, rng, triangle)
        assert any(p >= 64 for p in pos)
        assert E.max_clique(big) == _lift(clique, pos), i
        dp_small, dp_big = ref.disjoint_paths(rows), E.disjoint_paths(big)
        for u in range(n):
            for v in range(n):
                assert dp_big[pos[u] * n2 + pos[v]] == dp_small[u * n + v], (i, u, v)
        for k in (2, 4, 7):
            imp_small, imp_big = ref.improve_graph(rows, k), E.improve_graph(big, k)
            for u in range(n):
                assert imp_big[pos[u]] == _lift(imp_small[u], pos), (i, k, u)
        if not triangle:
            assert E.mmw_lower_bound(big) == ref.mmw_lower_bound(rows)
        blocks_big = {tuple(v) for v, _ in E.split(big)}
        for verts, _ in ref.split(rows, 2):
            if len(verts) > 1:
                assert tuple(pos[v] for v in verts) in blocks_big, (i, verts)
