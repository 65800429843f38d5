#!/bin/bash
# sharded redesign: GPU tests, c4-sharded at P = 1 with phase breakdown
tag=${1:-sh}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "shard" 2>&1 | tail -15 > gpurun_out/${tag}_pytest.txt
timeout 900 python bench.py --workload c4-sharded --steps 20 --warmup 5 > gpurun_out/${tag}_c4s.json 2> gpurun_out/${tag}_c4s.err
