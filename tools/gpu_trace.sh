#!/bin/bash
# clock64 timelines (CTA 0) of the tcgen05 kernel (c2, c3) and the top-k kernel (c2, c3, c4).
mkdir -p gpurun_out
SALS_EXTRA_NVCC=-DSALS_TC_TRACE python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
for w in c2 c3; do echo "== tc2 $w"; timeout 300 python tools/trace_tc2.py $w; done > gpurun_out/trace_${1:-t}.log 2>&1
for w in c2 c3 c4; do echo "== topk $w"; timeout 300 python tools/trace_topk.py $w; done >> gpurun_out/trace_${1:-t}.log 2>&1
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
