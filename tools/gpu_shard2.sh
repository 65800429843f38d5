#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -X faulthandler bench.py --workload c4-sharded --steps 5 --warmup 3 --layers 2 > gpurun_out/sh4.json 2> gpurun_out/sh4.err; echo "rc=$?" >> gpurun_out/sh4.err
timeout 600 compute-sanitizer --print-limit 5 python bench.py --workload c4-sharded --steps 2 --warmup 3 --layers 2 > gpurun_out/sh4_san.txt 2>&1; echo "rc=$?" >> gpurun_out/sh4_san.txt
