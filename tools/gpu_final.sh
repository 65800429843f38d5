#!/bin/bash
# Round-end evidence: tests, smoke, bench lines (c2 default with cpu_baseline, c3, c4, c4-sharded P=1,
# reference arm), launch list, one ncu --set full per hot kernel at c2.
tag=${1:-f}
bash tools/gpu_round.sh $tag
timeout 600 python bench.py --workload c4-sharded --steps 20 --warmup 5 > gpurun_out/bench_${tag}_c4sharded.json 2> gpurun_out/bench_${tag}_c4sharded.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${tag}_reference.json 2> gpurun_out/bench_${tag}_reference.err
bash tools/gpu_ncu.sh $tag c2 "project score_tma topk recon_attn"
bash tools/gpu_sweep.sh $tag
