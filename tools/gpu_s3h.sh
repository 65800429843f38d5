#!/bin/bash
# cta_group::2 relay: relaxed vs release remote arrive (trace + stage times)
mkdir -p gpurun_out
SALS_EXTRA_NVCC=-DSALS_TC_TRACE python -m paper_2510_24273_b200.build --force > gpurun_out/s3h_build.txt 2>&1
echo "== cg2 relaxed" > gpurun_out/s3h_trace.txt; SALS_TC2_CG=2 timeout 120 python tools/trace_tc2.py c2 >> gpurun_out/s3h_trace.txt 2>&1
SALS_EXTRA_NVCC="-DSALS_TC_TRACE -DSALS_RELAY_RELEASE=1" python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo "== cg2 release" >> gpurun_out/s3h_trace.txt; SALS_TC2_CG=2 timeout 120 python tools/trace_tc2.py c2 >> gpurun_out/s3h_trace.txt 2>&1
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
SALS_TC2_CG=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_configs and c2 or ragged_requests or c5_grid" > gpurun_out/s3h_pytest.txt 2>&1
SALS_TC2_CG=2 timeout 300 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/s3h_c2.json 2> gpurun_out/s3h_c2.err
echo done
