#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "topk" > gpurun_out/s3x_pytest.txt 2>&1
echo done
