#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense" > gpurun_out/s3l_pytest.txt 2>&1
for w in c3 c4; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3l_$w.json 2> gpurun_out/s3l_$w.err
done
timeout 600 ncu --set full --clock-control none -k regex:"dense_tma" -s 2 -c 1 -o gpurun_out/s3l_full_c3_dense python bench.py --workload c3 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
echo done
