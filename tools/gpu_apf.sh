#!/bin/bash
# A-row L2 prefetch experiment: clock64 traces with / without, stage times, L2 bandwidth microbench
mkdir -p gpurun_out
./tools/exp/l2_bw.bin > gpurun_out/apf_l2bw.txt 2>&1
for v in apf noapf; do
  f=""; [ $v = noapf ] && f="-DSALS_EXP_NO_APF"
  SALS_EXTRA_NVCC="-DSALS_TC_TRACE $f" python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
  for w in c2 c3; do echo "== $v $w"; timeout 300 python tools/trace_tc2.py $w; done >> gpurun_out/apf_trace.txt 2>&1
  SALS_EXTRA_NVCC="$f" python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
  for w in c2 c3; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/apf_bench_${v}_$w.json 2>/dev/null; done
done
