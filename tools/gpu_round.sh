mkdir -p gpurun_out
python tools/prof_decide.py 22 exact 1 > gpurun_out/decide22_stats.txt 2>&1
python tools/ncu_top.py k_exact_scatter ncu_scatter -- python tools/prof_decide.py 22 exact 1
python tools/ncu_top.py k_exact_part ncu_part -- python tools/prof_decide.py 22 exact 1
python tools/ncu_top.py k_append ncu_append -- python tools/prof_decide.py 22 exact 1
python tools/ncu_top.py k_route ncu_route -- env VSHARDS=2 ETWG_HANDOFF=0 python tools/prof_decide.py 22 exact 1
python tools/ncu_top.py k_owner ncu_owner -- env VSHARDS=2 ETWG_HANDOFF=0 python tools/prof_decide.py 22 exact 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_g48_solve.csv python tools/prof_g48.py exact > /dev/null 2>&1
timeout 1500 python tools/configs_table.py r01_configs 2>&1 | tail -12 > gpurun_out/configs_table.md
