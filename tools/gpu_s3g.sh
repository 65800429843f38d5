#!/bin/bash
# clock64 trace of CTA 0 of the fused kernel at c2: one-CTA kernel vs the cta_group::2 pair
mkdir -p gpurun_out
SALS_EXTRA_NVCC=-DSALS_TC_TRACE python -m paper_2510_24273_b200.build --force > gpurun_out/s3g_build.txt 2>&1
echo "== cg2" > gpurun_out/s3g_trace.txt; timeout 120 python tools/trace_tc2.py c2 >> gpurun_out/s3g_trace.txt 2>&1
echo "== cg1" >> gpurun_out/s3g_trace.txt; SALS_TC2_CG=1 timeout 120 python tools/trace_tc2.py c2 >> gpurun_out/s3g_trace.txt 2>&1
SALS_EXTRA_NVCC=-DSALS_TC_CTATIME python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo "== cg2 ctatime" >> gpurun_out/s3g_trace.txt; timeout 120 python tools/cta_time.py c2 >> gpurun_out/s3g_trace.txt 2>&1
echo "== cg1 ctatime" >> gpurun_out/s3g_trace.txt; SALS_TC2_CG=1 timeout 120 python tools/cta_time.py c2 >> gpurun_out/s3g_trace.txt 2>&1
echo done
