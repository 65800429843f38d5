#!/bin/bash
# cta_group::2 MHA variant: parity first (bounded), then bench A/B
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_configs and c2" > gpurun_out/s3f_pytest0.txt 2>&1
echo "rc=$?" >> gpurun_out/s3f_pytest0.txt
if grep -q "passed" gpurun_out/s3f_pytest0.txt && ! grep -q "failed" gpurun_out/s3f_pytest0.txt; then
  timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3f_pytest.txt 2>&1
  for w in c2 c3; do
    timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/s3f_$w.json 2> gpurun_out/s3f_$w.err
    SALS_TC2_CG=1 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/s3f_cg1_$w.json 2> gpurun_out/s3f_cg1_$w.err
  done
  timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s3f_c5.json 2> gpurun_out/s3f_c5.err
fi
echo done
