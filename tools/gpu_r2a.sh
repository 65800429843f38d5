#!/bin/bash
# round 2, first call: microbenchmark of tcgen05 rates, full GPU test suite, c2-c4 bench lines
mkdir -p gpurun_out
./tools/exp/mma_rate.bin > gpurun_out/r2a_mma_rate.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -rA 2>&1 | tail -60 > gpurun_out/r2a_pytest.txt
for w in c2 c3 c4; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_bench_$w.json 2> gpurun_out/r2a_bench_$w.err
done
