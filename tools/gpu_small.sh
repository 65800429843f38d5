#!/bin/bash
# stage times at small batches (the latency chain): c2 shape at B = 1, 2, 8 and c3 shape at B = 1
mkdir -p gpurun_out
for b in 1 2; do timeout 300 python bench.py --workload c2 --batch $b --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/small_c2_b$b.json 2>/dev/null; done
timeout 300 python bench.py --workload c3 --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/small_c3_b1.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/small_launches_b1.csv python bench.py --workload c2 --batch 1 --layers 4 --steps 2 --warmup 3 --no-cpu-baseline --no-dense > /dev/null 2>&1
