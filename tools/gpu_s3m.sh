#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3m_pytest.txt 2>&1
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3m_$w.json 2> gpurun_out/s3m_$w.err
done
echo done
