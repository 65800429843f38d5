#!/bin/bash
# session-3 state check: default bench + an ncu full capture of the fused kernel at c2 (L2 / LTS counters)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3a_smi.txt 2>&1
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 > gpurun_out/s3a_c2.json 2> gpurun_out/s3a_c2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:recon_attn -s 6 -c 1 -o gpurun_out/s3a_full_c2_recon python bench.py --workload c2 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:flash_decode -s 6 -c 1 -o gpurun_out/s3a_full_c2_dense python bench.py --workload c2 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:project -s 6 -c 1 -o gpurun_out/s3a_full_c2_proj python bench.py --workload c2 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
echo done
