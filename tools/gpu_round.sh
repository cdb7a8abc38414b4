mkdir -p gpurun_out
timeout 1200 python tests/fuzz_device.py 600 7 > gpurun_out/fuzz.txt 2>&1; tail -15 gpurun_out/fuzz.txt
