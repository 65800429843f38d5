#!/bin/bash
# cta_group::2 for MHA by default (request pairs first): full GPU suite, c2 / c5 A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3q_pytest.txt 2>&1
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3q_c2.json 2> gpurun_out/s3q_c2.err
SALS_TC2_CG=1 timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3q_cg1_c2.json 2> gpurun_out/s3q_cg1_c2.err
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/s3q_c5.json 2> gpurun_out/s3q_c5.err
SALS_TC2_CG=1 timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/s3q_cg1_c5.json 2> gpurun_out/s3q_cg1_c5.err
echo done
