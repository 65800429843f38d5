#!/bin/bash
# dense comparator HBM fraction at c2-c4 (tag)
tag=${1:-d}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "dense" 2>&1 | tail -3 > gpurun_out/${tag}_pytest.txt
for w in c2 c3 c4; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$w.json 2>/dev/null; done
