# Round-2 call AC: sibling-sharing (rmask) buckets vs full-key buckets.
O=gpurun_out/r02ac; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py $L@ETWG_RBUCKET=0 $L 3 > $O/ab_rb.txt 2>&1; cat $O/ab_rb.txt
timeout 900 python tools/ab_lib.py $L@ETWG_RB_FRAC=35 $L@ETWG_RB_FRAC=65 3 > $O/ab_frac.txt 2>&1; cat $O/ab_frac.txt
ETWG_TRACE=1 timeout 300 python tools/prof_g48.py > $O/trace.txt 2>&1; grep -c "abort 5" $O/trace.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sibling" > $O/parity.txt 2>&1; tail -3 $O/parity.txt
for rb in 0 1; do
ETWG_RBUCKET=$rb timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_rb$rb.csv python tools/prof_g48.py > /dev/null 2>&1
python tools/summarize_launches.py $O/launches_rb$rb.csv | head -6
done
