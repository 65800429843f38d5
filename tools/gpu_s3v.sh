#!/bin/bash
mkdir -p gpurun_out
for b in 1 2; do
  timeout 600 python bench.py --workload c2 --batch $b --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s3v_b$b.json 2> gpurun_out/s3v_b$b.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"project|score|topk|recon|merge" -c 40 --csv --log-file gpurun_out/s3v_launches_b1.csv \
    python bench.py --workload c2 --batch 1 --steps 2 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
echo done
