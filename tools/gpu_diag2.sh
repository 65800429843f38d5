#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --layers 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/diag2_all4.json 2> gpurun_out/diag2_all4.err; echo "all4 rc=$?" >> gpurun_out/diag2_rc.txt
CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --layers 32 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/diag2_allblk.json 2> gpurun_out/diag2_allblk.err; echo "allblk rc=$?" >> gpurun_out/diag2_rc.txt
timeout 900 compute-sanitizer --tool initcheck --print-limit 10 python bench.py --workload c3 --layers 1 --steps 3 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/diag2_init_c3.txt 2>&1
