#!/bin/bash
mkdir -p gpurun_out
for w in c3 c4; do SALS_FUSED_MERGE=1 timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/fm_bench_$w.json 2>/dev/null; done
SALS_EXTRA_NVCC="-DSALS_TC_TRACE" python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
for w in c2 c3 c4; do echo "== topk $w"; timeout 300 python tools/trace_topk.py $w; done > gpurun_out/trace_topk2.txt 2>&1
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
