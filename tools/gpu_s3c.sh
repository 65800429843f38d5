#!/bin/bash
# dense comparator launch list (TMA vs LSU), c2 + c3
mkdir -p gpurun_out
for w in c2 c3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"dense|flash|merge|project_kernel<.*1, 256" -c 30 --csv --log-file gpurun_out/s3c_launch_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
  SALS_DENSE_LSU=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"dense|flash|merge|project_kernel<.*1, 256" -c 30 --csv --log-file gpurun_out/s3c_launch_lsu_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/s3c_pytest.txt 2>&1
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/s3c_$w.json 2> gpurun_out/s3c_$w.err
  SALS_TC2_PAIR=0 timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/s3c_nopair_$w.json 2> gpurun_out/s3c_nopair_$w.err
done
echo done
