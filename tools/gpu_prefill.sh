#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "bulk or calibrate or quantized" 2>&1 | tail -25 > gpurun_out/pf_pytest.txt
