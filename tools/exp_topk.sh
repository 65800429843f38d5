#!/bin/bash
for w in c2 c3 c4; do for sl in 1024 2048 4096 8192; do
  SALS_TOPK_SLICE=$sl timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-dense 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w slice=$sl', round(d['us_per_layer_step'],1), d['stages_us'])"
done; done > gpurun_out/exp_topk.log 2>&1
