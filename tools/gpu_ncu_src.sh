#!/bin/bash
# one ncu --set full capture (with source) of the fused kernel at c2 and c3
mkdir -p gpurun_out
for w in c3 c2; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:recon_attn -s 6 -c 1 \
    -o gpurun_out/src_$w python bench.py --workload $w --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > gpurun_out/src_$w.log 2>&1
done
