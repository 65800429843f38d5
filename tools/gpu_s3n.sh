#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3n_pytest.txt 2>&1
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3n_$w.json 2> gpurun_out/s3n_$w.err
done
timeout 600 python bench.py --workload c4-sharded --steps 20 --warmup 5 > gpurun_out/s3n_c4s.json 2> gpurun_out/s3n_c4s.err
echo done
