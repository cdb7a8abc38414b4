"""Diagnostics (not a benchmark): the largest exact round of the bench graph's
k=22 decide (round 10: 159M parents) with and without its record emission
(ETWG_DEBUG 16384 skips the last round's emission). Run under an ncu launch
list; the last k_exact_scatter launch of each process is the one to compare.
Usage: python tools/k1_only.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G  # noqa: E402
r = E.decide(G.random_graph(1, 48, 0.2), 22, dedup="exact", cap=1 << 31, rounds=11, keep_layers=False)
print("rounds", len(r.rounds), "last expanded", r.rounds[-1].expanded)
