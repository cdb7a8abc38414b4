"""Device parity on the large BASELINE configs against goldens produced by
the UNMODIFIED reference (tests/golden/make_big_goldens.py): the whole
stats JSON (every attempt, every round's expanded / emitted / duplicates /
mmw_pruned / overflowed counter, the treewidth) must be byte-identical."""
import json

import pytest

from conftest import g48_golden, instance_text
from paper_1709_09990_b200 import generators as G

pytestmark = pytest.mark.gpu


def test_g40_seed2_exact_full_sweep(E, big_goldens, gpu):
    """BASELINE cfg 3, seed 2: 8,261,454 expanded states."""
    g = big_goldens["g40_03_seed2"]
    res = E.solve(E.Graph.from_rows(G.random_graph(2, 40, 0.3)),
                  E.Options(dedup="exact", thread_count=g["threads"]))
    assert res.value == g["tw"] == 22
    assert json.loads(res.stats_json)["totals"]["expanded"] == 8_261_454
    assert res.stats_json == g["exact_stats"]


def test_myciel4_mmw_acceptance_criterion_4(E, big_goldens, gpu):
    """proj/tests/acceptance.cpp:245-286: MMW in exact mode keeps tw 10 and
    cuts the emitted states 108,207 -> 84,504; stats byte-identical and the
    order (reconstruction with MMW on) identical to the reference's."""
    g = big_goldens["myciel4_exact_mmw"]
    graph = E.Graph.parse(instance_text("myciel4"))
    plain = E.solve(graph, E.Options(dedup="exact", emit_order=True))
    mmw = E.solve(graph, E.Options(dedup="exact", use_mmw=True, emit_order=True))
    assert plain.value == mmw.value == g["tw"] == 10
    assert json.loads(plain.stats_json)["totals"]["emitted"] == 108_207
    assert json.loads(mmw.stats_json)["totals"]["emitted"] == 84_504
    assert plain.stats_json == g["plain_stats"]
    assert mmw.stats_json == g["stats"]
    assert mmw.order == g["order"]
    w, ok = graph.check_order(mmw.order)
    assert ok and w == 10


@pytest.mark.slow
def test_g48_bench_workload_matches_reference(E, gpu):
    """BASELINE cfg 4 (the bench workload): G(48,0.2) seed 1, exact dedup,
    max_layer_states 2^31 — the reference's full sweep to tw 24."""
    g = g48_golden()
    if g is None:
        pytest.skip("tests/golden/g48_ref.json not generated yet")
    res = E.solve(E.Graph.from_rows(G.random_graph(1, 48, 0.2)),
                  E.Options(dedup="exact", max_layer_states=1 << 31,
                            thread_count=g["options"]["threads"]))
    assert res.value == g["tw"] == 24
    assert res.stats_json == g["exact_stats"]
