#!/bin/bash
# dense TMA comparator (now wired) + U multicast groups of 4
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense or group_ragged" > gpurun_out/s3d_pytest.txt 2>&1
SALS_TC2_CS=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "group_ragged or full_size or ragged" > gpurun_out/s3d_pytest_cs4.txt 2>&1
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3d_$w.json 2> gpurun_out/s3d_$w.err
  SALS_TC2_CS=4 timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/s3d_cs4_$w.json 2> gpurun_out/s3d_cs4_$w.err
  SALS_TC2_CS=1 timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/s3d_cs1_$w.json 2> gpurun_out/s3d_cs1_$w.err
done
for w in c2 c3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"dense|flash|merge|project_kernel<.*1, 256" -c 30 --csv --log-file gpurun_out/s3d_launch_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
done
echo done
