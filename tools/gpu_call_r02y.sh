# Round-2 call Y: global open-addressing table dedup (default) vs bucket records.
O=gpurun_out/r02y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "global_table or passes or aborts or compact or g40 or myciel4 or golden" > $O/parity.txt 2>&1; tail -3 $O/parity.txt
timeout 900 python tools/ab_lib.py paper_1709_09990_b200/libelimtw.so@ETWG_GTAB=0 paper_1709_09990_b200/libelimtw.so 3 > $O/ab.txt 2>&1; cat $O/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
   --log-file $O/launches.csv python tools/prof_g48.py > $O/ncu.log 2>&1; echo ncu $?
python tools/summarize_launches.py $O/launches.csv > $O/launches_summary.txt 2>&1; head -30 $O/launches_summary.txt
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_nored.so paper_1709_09990_b200/libelimtw.so 2 bloom > $O/ab_bloom.txt 2>&1; cat $O/ab_bloom.txt
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_tab2.so tools/ab/libelimtw_tab8.so 3 > $O/ab_unroll.txt 2>&1; cat $O/ab_unroll.txt
