#!/bin/bash
# GPU round + one ncu --set full capture per hot kernel (c2 bench, one launch each).
tag=${1:-run}
bash tools/gpu_round.sh $tag
for k in recon_attn score topk project; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/full_${tag}_$k python bench.py --workload c2 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense \
    > gpurun_out/full_${tag}_$k.log 2>&1
  echo "ncu full $k rc=$?" >> gpurun_out/round_${tag}.log
done
