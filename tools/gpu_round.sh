#!/bin/bash
# Standard GPU check: parity tests, smoke, bench lines for c2/c3/c4, launch list.
# Usage (via gpurun): bash tools/gpu_round.sh [tag]
tag=${1:-run}
mkdir -p gpurun_out
out=gpurun_out/round_${tag}.log
: > $out
timeout 900 python -m pytest tests -m gpu -q -x >> $out 2>&1; echo "pytest rc=$?" >> $out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> $out 2>&1
for w in c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/bench_${tag}_$w.json 2> gpurun_out/bench_${tag}_$w.err
  echo "bench $w rc=$?" >> $out
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'project|score|topk|recon|merge|flash|dense|owned' -c 400 --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline --no-dense \
  > /dev/null 2>&1
echo "ncu rc=$?" >> $out
