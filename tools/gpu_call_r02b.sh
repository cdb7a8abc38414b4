# Round-2 call B: reference k=24 attempt of the G(48,0.2) sweep on the box's
# host (background), GPU parity tests of the register-slot K1, A/B against the
# per-vertex-table K1, ncu capture of the new scatter's largest k=22 launch.
O=gpurun_out/r02b; mkdir -p $O
( ulimit -v 188000000; timeout 3300 python tests/golden/make_big_goldens.py g48 14 24 \
    > $O/g48_ref_k24.log 2>&1; cp tests/golden/g48_ref_k24.json $O/ 2>/dev/null ) &
REFPID=$!
timeout 900 python -m pytest tests -x -q -m gpu > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_k1old.so paper_1709_09990_b200/libelimtw.so 3 > $O/ab_k1.txt 2>&1; cat $O/ab_k1.txt
timeout 900 python tools/ncu_top.py k_exact_scatter $O/scatter_k1slots -- python tools/prof_decide.py 22 exact > $O/ncu_top.txt 2>&1; tail -2 $O/ncu_top.txt
wait $REFPID; echo "ref rc=$?"; tail -5 $O/g48_ref_k24.log
