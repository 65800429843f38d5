#!/bin/bash
# dense comparator (new append / query RoPE kernels; TMA vs LSU flash) + per-CTA timing of the fused kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense" > gpurun_out/s3e_pytest.txt 2>&1
SALS_DENSE_LSU=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense" >> gpurun_out/s3e_pytest.txt 2>&1
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3e_$w.json 2> gpurun_out/s3e_$w.err
  SALS_DENSE_LSU=1 timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3e_lsu_$w.json 2> gpurun_out/s3e_lsu_$w.err
done
for w in c2 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"dense|flash|merge" -c 12 --csv --log-file gpurun_out/s3e_launch_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
done
SALS_EXTRA_NVCC=-DSALS_TC_CTATIME python -m paper_2510_24273_b200.build --force > gpurun_out/s3e_build.txt 2>&1
for w in c2 c3; do
  timeout 300 python tools/cta_time.py $w > gpurun_out/s3e_ctatime_$w.txt 2>&1
  MASK=8 timeout 300 python tools/cta_time.py $w > gpurun_out/s3e_ctatime_recon_$w.txt 2>&1
done
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo done
