#!/bin/bash
mkdir -p gpurun_out
for st in 4 8 12; do echo "== stages $st"; ./tools/exp/l2_bw_s$st.bin; done > gpurun_out/l2bw2.txt 2>&1
