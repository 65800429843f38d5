#!/bin/bash
mkdir -p gpurun_out
SALS_TC2_CG=2 timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3p_cg2_c2.json 2> gpurun_out/s3p_cg2_c2.err
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3p_c2.json 2> gpurun_out/s3p_c2.err
SALS_TC2_CG=2 timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-dense --sweep-batches 1,8,64 > gpurun_out/s3p_cg2_c5.json 2> gpurun_out/s3p_cg2_c5.err
SALS_EXTRA_NVCC=-DSALS_TC_CTATIME python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
timeout 120 python tools/cta_time.py c2 > gpurun_out/s3p_ctatime.txt 2>&1
SALS_TC2_CG=2 timeout 120 python tools/cta_time.py c2 >> gpurun_out/s3p_ctatime.txt 2>&1
SALS_EXTRA_NVCC=-DSALS_TC_TRACE python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
SALS_TC2_CG=2 timeout 120 python tools/trace_tc2.py c2 > gpurun_out/s3p_trace_cg2.txt 2>&1
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo done
