#!/bin/bash
# quantised-value variants: parity + c2/c3 benches (alg1 and paper policy)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/vq3_tests.txt
for w in c2 c3; do
  for pol in alg1 paper; do
    timeout 300 python bench.py --workload $w --v-bits 4 --policy $pol > gpurun_out/vq3_${w}_${pol}.json 2>gpurun_out/vq3_${w}_${pol}.err
  done
done
