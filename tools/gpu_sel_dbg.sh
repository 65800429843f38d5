#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "sharded_virtual" 2>&1 | grep -v "^$" | tail -40 > gpurun_out/sel_dbg.txt
