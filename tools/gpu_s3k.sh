#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "shard" > gpurun_out/s3k_pytest.txt 2>&1
timeout 600 python bench.py --workload c4-sharded --steps 20 --warmup 5 > gpurun_out/s3k_c4s.json 2> gpurun_out/s3k_c4s.err
timeout 300 python tools/host_cost.py c2 > gpurun_out/s3k_host.txt 2>&1
echo done
