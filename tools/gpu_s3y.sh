#!/bin/bash
# A-row L2 prefetch (LSU prefetch.global.L2, one line per lane) vs none
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_configs or ragged or c5_grid" > gpurun_out/s3y_pytest.txt 2>&1
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3y_pf_$w.json 2> gpurun_out/s3y_pf_$w.err
done
SALS_EXTRA_NVCC=-DSALS_A_PF=0 python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3y_nopf_$w.json 2> gpurun_out/s3y_nopf_$w.err
done
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo done
