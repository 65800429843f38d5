#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size or append or c5_grid or shard or quantized" > gpurun_out/s3s_pytest.txt 2>&1
for w in c2 c3; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3s_$w.json 2> gpurun_out/s3s_$w.err
done
echo done
