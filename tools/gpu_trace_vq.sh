#!/bin/bash
SALS_EXTRA_NVCC=-DSALS_TC_TRACE python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
for cfg in "0 0" "4 0" "4 64" "0 64"; do set -- $cfg; echo "== V_BITS=$1 RECENT=$2"; V_BITS=$1 RECENT=$2 timeout 300 python tools/trace_tc2.py c2 | grep -v "^v_\|^a_"; done > gpurun_out/trace_vq.log 2>&1
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
