#!/bin/bash
# GQA P V operand staged by TMA gather4 (SALS_TPV_TMA, default) vs by the epilogue's cp.async
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gqa or full_size or append_decode or ragged or shard" > gpurun_out/s4a_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/s4a_pytest.txt
for w in c3 c4; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s4a_tma_$w.json 2> gpurun_out/s4a_tma_$w.err
  SALS_TPV_TMA=0 timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/s4a_cpa_$w.json 2> gpurun_out/s4a_cpa_$w.err
done
echo done
