# Round-2 call T: TMA part kernel (register phases) vs plain; f4 passes on the bench workload.
O=gpurun_out/r02t; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 400 python tools/ab_lib.py $L tools/ab/libelimtw_notma.so 3 > $O/ab_notma.txt 2>&1; head -3 $O/ab_notma.txt
timeout 900 python tools/passes_probe.py 2 4 > $O/passes.txt 2>&1; cat $O/passes.txt
