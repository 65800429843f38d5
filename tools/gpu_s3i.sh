#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense" > gpurun_out/s3i_pytest.txt 2>&1
for w in c3 c4; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3i_$w.json 2> gpurun_out/s3i_$w.err
done
echo done
