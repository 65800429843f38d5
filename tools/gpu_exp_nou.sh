#!/bin/bash
# Is the c2 MMA starved by the U operand's L2 ingress?  Trace with and without the U fetches.
mkdir -p gpurun_out
SALS_EXTRA_NVCC=-DSALS_TC_TRACE python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo "== with U" > gpurun_out/exp_nou.log; timeout 300 python tools/trace_tc2.py c2 2>&1 | grep -v "^v_\|^a_" >> gpurun_out/exp_nou.log
SALS_EXTRA_NVCC="-DSALS_TC_TRACE -DSALS_EXP_NO_U" python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
echo "== without U" >> gpurun_out/exp_nou.log; timeout 300 python tools/trace_tc2.py c2 2>&1 | grep -v "^v_\|^a_" >> gpurun_out/exp_nou.log
echo "== without U, c3" >> gpurun_out/exp_nou.log; timeout 300 python tools/trace_tc2.py c3 2>&1 | grep -v "^v_\|^a_" >> gpurun_out/exp_nou.log
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
