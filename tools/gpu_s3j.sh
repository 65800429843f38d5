#!/bin/bash
# host cost of the eager call (tensor-map cache) + e2e at c2 / c3; cg2 with relaxed accumulator release
mkdir -p gpurun_out
timeout 300 python tools/host_cost.py c2 > gpurun_out/s3j_host.txt 2>&1
timeout 300 python tools/host_cost.py c4 >> gpurun_out/s3j_host.txt 2>&1
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3j_c2.json 2> gpurun_out/s3j_c2.err
SALS_TC2_CG=2 timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3j_cg2_c2.json 2> gpurun_out/s3j_cg2_c2.err
SALS_TC2_CG=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_configs and c2 or ragged_requests" > gpurun_out/s3j_pytest_cg2.txt 2>&1
SALS_EXTRA_NVCC=-DSALS_TC_TRACE python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo "== cg2" > gpurun_out/s3j_trace.txt; SALS_TC2_CG=2 timeout 120 python tools/trace_tc2.py c2 >> gpurun_out/s3j_trace.txt 2>&1
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo done
