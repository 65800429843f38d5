#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_configs and c2 or mha or c5_grid or ragged or head_dims or sink" > gpurun_out/s3o_pytest.txt 2>&1
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3o_c2.json 2> gpurun_out/s3o_c2.err
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-dense --sweep-batches 1,8,64 > gpurun_out/s3o_c5.json 2> gpurun_out/s3o_c5.err
SALS_EXTRA_NVCC=-DSALS_TC_TRACE python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
timeout 120 python tools/trace_tc2.py c2 > gpurun_out/s3o_trace.txt 2>&1
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo done
