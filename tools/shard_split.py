"""One G(48,0.2) solve on G virtual shards, for an ncu launch list (kernel
split of the sharded round). Usage: python tools/shard_split.py G"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G  # noqa: E402
E.set_virtual_shards(int(sys.argv[1]))
r = E.solve(E.Graph.from_rows(G.random_graph(1, 48, 0.2)), E.Options(dedup="exact", max_layer_states=1 << 31))
print("tw", r.value)
