#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/tk_tests.txt
for w in c3 c4; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/tk_$w.json 2> gpurun_out/tk_$w.err
done
