mkdir -p gpurun_out
python tools/prof_decide.py 22 exact > gpurun_out/decide_stats_v8.txt 2>&1; head -2 gpurun_out/decide_stats_v8.txt
for kern in k_exact_scatter k_exact_part k_append; do
  timeout 900 python tools/ncu_top.py "$kern" ${kern}_v8 -- python tools/prof_decide.py 22 exact
done
