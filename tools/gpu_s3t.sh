#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense or shard or full_size_configs" > gpurun_out/s3t_pytest.txt 2>&1
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3t_c4.json 2> gpurun_out/s3t_c4.err
echo done
