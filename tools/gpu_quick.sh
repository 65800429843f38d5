#!/bin/bash
# Quick GPU check: parity tests + c2/c3/c4 bench lines (no ncu).
tag=${1:-q}
mkdir -p gpurun_out
out=gpurun_out/quick_${tag}.log
: > $out
timeout 900 python -m pytest tests -m gpu -q -x >> $out 2>&1; echo "pytest rc=$?" >> $out
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${tag}_$w.json 2> gpurun_out/bench_${tag}_$w.err
  echo "bench $w rc=$?" >> $out
done
