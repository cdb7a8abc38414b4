# Round-2 call E: abort-path trace, GPU tests, K1 A/B after the Set fix.
O=gpurun_out/r02e; mkdir -p $O
cat > /tmp/tight.py <<'PY'
import json, sys
sys.path.insert(0, ".")
from paper_1709_09990_b200 import elimtw as E, generators as G
for name, rows, k, mmw in (("g", G.random_graph(1, 40, 0.3), 21, False), ("q", G.queen_graph(5, 5), 18, True),
                           ("w", G.random_graph(9, 70, 0.07), 5, False)):
    print(name, flush=True)
    r = E.decide(rows, k, dedup="exact", mmw=mmw, rounds=8 if name == "w" else -1)
    print(name, r.outcome, [x.emitted for x in r.rounds], flush=True)
PY
ETWG_DEBUG=1024 ETWG_TRACE=1 timeout 300 python /tmp/tight.py > $O/tight.txt 2>&1; tail -30 $O/tight.txt
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.txt 2>&1; tail -5 $O/gpu_tests.txt
for v in loop1 minb4 k1old; do
  timeout 600 python tools/ab_lib.py paper_1709_09990_b200/libelimtw.so tools/ab/libelimtw_$v.so 3 > $O/ab_$v.txt 2>&1; head -3 $O/ab_$v.txt
done
