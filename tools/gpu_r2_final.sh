#!/bin/bash
# round-2 final evidence: GPU tests, smoke, default bench (c2 + c3 + c4), c5 sweeps (alg1, paper policy),
# c4-sharded, launch lists (our kernels, incl. the dense step) and ncu --set full captures
t=${1:-r2f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${t}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA 2>&1 | tail -140 > gpurun_out/${t}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${t}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${t}_bench.json 2> gpurun_out/${t}_bench.err
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/${t}_c5.json 2> gpurun_out/${t}_c5.err
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --policy paper --sweep-batches 1,8,32 > gpurun_out/${t}_c5_paper.json 2> gpurun_out/${t}_c5_paper.err
timeout 600 python bench.py --workload c4-sharded --steps 20 --warmup 5 > gpurun_out/${t}_c4s.json 2> gpurun_out/${t}_c4s.err
for w in c2 c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"project|score|topk|recon|merge" -c 60 --csv --log-file gpurun_out/${t}_launches_$w.csv \
    python bench.py --workload $w --steps 2 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"dense|flash|merge" -c 12 --csv --log-file gpurun_out/${t}_dense_launches_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:recon_attn -s 6 -c 1 -o gpurun_out/${t}_full_c2_recon python bench.py --workload c2 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:recon_attn -s 6 -c 1 -o gpurun_out/${t}_full_c3_recon python bench.py --workload c3 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:recon_attn -s 6 -c 1 -o gpurun_out/${t}_full_c4_recon python bench.py --workload c4 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:score_tma -s 6 -c 1 -o gpurun_out/${t}_full_c2_score python bench.py --workload c2 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:score_tma -s 6 -c 1 -o gpurun_out/${t}_full_c3_score python bench.py --workload c3 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"dense_tma|flash_decode" -s 2 -c 1 -o gpurun_out/${t}_full_c3_dense python bench.py --workload c3 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"flash_decode" -s 2 -c 1 -o gpurun_out/${t}_full_c2_dense python bench.py --workload c2 --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
echo done
