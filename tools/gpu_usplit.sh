#!/bin/bash
# U-operand TMA split experiment (1 / 2 / 4 boxes per stage), A prefetch off, trace + stage times
mkdir -p gpurun_out
for u in 1 2 4; do
  SALS_EXTRA_NVCC="-DSALS_TC_TRACE -DSALS_EXP_NO_APF -DSALS_USPLIT=$u" python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
  for w in c2 c3; do echo "== usplit $u $w"; timeout 300 python tools/trace_tc2.py $w; done >> gpurun_out/us_trace.txt 2>&1
  SALS_EXTRA_NVCC="-DSALS_EXP_NO_APF -DSALS_USPLIT=$u" python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
  for w in c2 c3; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/us_bench_${u}_$w.json 2>/dev/null; done
done
