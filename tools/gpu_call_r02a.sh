# Round-2 first GPU call: reference G(48,0.2) golden on the box's host cores
# (background, memory-bounded), GPU tests, device stats for the same solve,
# bench, compute-sanitizer on the lock-free kernels.
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
{ nproc; free -g; lscpu | head -25; nvidia-smi -L; } > $O/host.txt 2>&1
NP=$(nproc); TH=$(( NP > 4 ? NP - 2 : 1 ))
MEMKB=$(awk '/MemAvailable/{print $2}' /proc/meminfo); LIM=$(( MEMKB * 7 / 10 ))
echo "ref threads $TH vlimit_kb $LIM" >> $O/host.txt
( ulimit -v $LIM; /usr/bin/time -v timeout 9600 python tests/golden/make_big_goldens.py g48 $TH \
    > $O/g48_ref.log 2>&1; cp tests/golden/g48_ref.json $O/ 2>/dev/null ) &
REFPID=$!
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python tools/g48_stats.py $TH $O/g48_gpu_stats.json > $O/g48_gpu.log 2>&1; cat $O/g48_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
for tool in memcheck racecheck synccheck; do
  for mode in exact bloom wide shard2; do
    SAN_N=40 timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_decide.py $mode \
      > $O/san_${tool}_${mode}.txt 2>&1; echo "$tool $mode rc=$? $(tail -1 $O/san_${tool}_${mode}.txt)"
  done
done
wait $REFPID; echo "ref rc=$?"; tail -25 $O/g48_ref.log
