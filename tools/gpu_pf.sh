#!/bin/bash
mkdir -p gpurun_out
for pf in 0 1 2; do for w in c2 c3 c4; do
  SALS_TOPK_PREFETCH=$pf timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/pf${pf}_$w.json 2>/dev/null
done; done
