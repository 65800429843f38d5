#!/bin/bash
for vb in 4 2; do for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --v-bits $vb --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${1:-v}_${w}_v$vb.json 2> gpurun_out/bench_${1:-v}_${w}_v$vb.err
done; done
