#!/bin/bash
# round-2 evidence run: GPU tests, default bench (c2 + c3 + c4), c5 sweep (alg1, paper policy),
# c4-sharded, the launch list (our kernels) and ncu --set full captures of the key kernels
t=${1:-r2e}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${t}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA 2>&1 | tail -130 > gpurun_out/${t}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${t}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${t}_bench.json 2> gpurun_out/${t}_bench.err
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/${t}_c5.json 2> gpurun_out/${t}_c5.err
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --policy paper --sweep-batches 1,8,32 > gpurun_out/${t}_c5_paper.json 2> gpurun_out/${t}_c5_paper.err
timeout 600 python bench.py --workload c4-sharded --steps 20 --warmup 5 > gpurun_out/${t}_c4s.json 2> gpurun_out/${t}_c4s.err
for w in c2 c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"project|score|topk|recon|merge" -c 60 --csv \
    python bench.py --workload $w --steps 2 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > gpurun_out/${t}_launches_$w.csv 2>/dev/null
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:recon_attn -s 6 -c 1 -o gpurun_out/${t}_full_c2_recon python bench.py --workload c2 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:recon_attn -s 6 -c 1 -o gpurun_out/${t}_full_c3_recon python bench.py --workload c3 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:score_tma -s 6 -c 1 -o gpurun_out/${t}_full_c3_score python bench.py --workload c3 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:score_tma -s 6 -c 1 -o gpurun_out/${t}_full_c2_score python bench.py --workload c2 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:flash_decode -s 6 -c 1 -o gpurun_out/${t}_full_c3_dense python bench.py --workload c3 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
