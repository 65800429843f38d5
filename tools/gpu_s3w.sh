#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3w_pytest.txt 2>&1
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3w_c2.json 2> gpurun_out/s3w_c2.err
timeout 600 python bench.py --workload c2 --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3w_b1.json 2> gpurun_out/s3w_b1.err
echo done
