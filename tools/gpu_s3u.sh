#!/bin/bash
# small-batch chain: the fused kernel's in-kernel split merge (SALS_FUSED_MERGE=1) vs the merge kernel
mkdir -p gpurun_out
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline --no-dense --sweep-batches 1,2,4 > gpurun_out/s3u_c5.json 2> gpurun_out/s3u_c5.err
SALS_FUSED_MERGE=1 timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline --no-dense --sweep-batches 1,2,4 > gpurun_out/s3u_fm_c5.json 2> gpurun_out/s3u_fm_c5.err
echo done
