#!/bin/bash
# library NCCL sharded path: parity + c4-sharded bench with both exchanges
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x  2>&1 | tail -5 > gpurun_out/comm_tests.txt
timeout 300 python bench.py --workload c4-sharded --comm lib > gpurun_out/comm_lib.json 2> gpurun_out/comm_lib.err
timeout 300 python bench.py --workload c4-sharded --comm torch > gpurun_out/comm_torch.json 2> gpurun_out/comm_torch.err
