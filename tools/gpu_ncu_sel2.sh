#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:shard_select -s 2 -c 1 -o gpurun_out/sel_c4c python bench.py --workload c4-sharded --steps 2 --warmup 2 --layers 2 > gpurun_out/sel_c4.log 2>&1
