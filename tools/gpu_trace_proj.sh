#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "append or full_size or c5 or smoke or bulk" 2>&1 | tail -3 > gpurun_out/tp_pytest.txt
SALS_EXTRA_NVCC="-DSALS_TC_TRACE" python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
for w in c2 c3; do echo "== proj $w"; timeout 300 python tools/trace_proj.py $w; done > gpurun_out/trace_proj.txt 2>&1
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
for w in c2 c3; do timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/tp_$w.json 2>/dev/null; done
