#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/bench_${1:-s}_c5.json 2> gpurun_out/bench_${1:-s}_c5.err
echo "sweep rc=$?" >> gpurun_out/bench_${1:-s}_c5.err
