#!/bin/bash
for w in c2 c3; do
  timeout 600 python bench.py --workload $w --v-bits 4 --policy paper --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${1:-w}_${w}_v4_paper.json 2> gpurun_out/bench_${1:-w}_${w}_v4_paper.err
done
