#!/bin/bash
mkdir -p gpurun_out
SALS_EXTRA_NVCC=-DSALS_TC_TRACE python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
timeout 120 python tools/trace_tc2.py c3 > gpurun_out/s3z_trace_c3.txt 2>&1
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo done
