#!/bin/bash
# dense TMA comparator: parity + bench A/B against the LSU kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense" > gpurun_out/s3b_pytest.txt 2>&1
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3b_$w.json 2> gpurun_out/s3b_$w.err
  SALS_DENSE_LSU=1 timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3b_lsu_$w.json 2> gpurun_out/s3b_lsu_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"dense|flash|merge|project" -c 40 --csv \
    python bench.py --workload c3 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > gpurun_out/s3b_launches_c3.csv 2>/dev/null
echo done
