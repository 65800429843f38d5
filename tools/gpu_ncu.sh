#!/bin/bash
# ncu --set full captures of the library kernels in one bench configuration (cold, serialised).
# Usage: bash tools/gpu_ncu.sh tag workload "regex1 regex2 ..."
tag=${1:-n}; w=${2:-c2}; ks=${3:-"project latent_score|score_tma topk recon_attn merge"}
mkdir -p gpurun_out
for k in $ks; do
  safe=$(echo $k | tr -c 'a-zA-Z0-9_\n' '_')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 6 -c 2 \
    -o gpurun_out/full_${tag}_${w}_$safe python bench.py --workload $w --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense \
    > gpurun_out/full_${tag}_${w}_$safe.log 2>&1
  echo "ncu $w $k rc=$?" >> gpurun_out/ncu_${tag}.log
done
