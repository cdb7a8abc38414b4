mkdir -p gpurun_out
timeout 900 python tests/fuzz_device.py 420 11 > gpurun_out/fuzz2.txt 2>&1; tail -5 gpurun_out/fuzz2.txt
