#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:shard_select -c 5 --csv python bench.py --workload c4-sharded --steps 2 --warmup 2 --layers 2 > gpurun_out/sel_c4_t.csv 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "shard" 2>&1 | tail -3 > gpurun_out/sel_pytest.txt
timeout 900 python bench.py --workload c4-sharded --steps 20 --warmup 5 > gpurun_out/sel_c4s.json 2> /dev/null
