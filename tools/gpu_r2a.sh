#!/bin/bash
# round 2, first call: tcgen05 rate microbenchmark, full GPU test suite, default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
./tools/exp/mma_rate.bin > gpurun_out/r2a_mma_rate.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -rA 2>&1 | tail -80 > gpurun_out/r2a_pytest.txt
timeout 600 python bench.py > gpurun_out/r2a_bench_default.json 2> gpurun_out/r2a_bench_default.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.txt 2>&1
