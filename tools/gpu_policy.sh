#!/bin/bash
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --policy paper --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${1:-p}_${w}_paper.json 2> gpurun_out/bench_${1:-p}_${w}_paper.err
done
