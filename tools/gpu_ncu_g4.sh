#!/bin/bash
# ncu --set full of the G = 4 fused kernel (c3) and the large top-k (c4)
mkdir -p gpurun_out
bash tools/gpu_ncu.sh g4 c3 "recon_attn topk"
bash tools/gpu_ncu.sh g4 c4 "topk score_tma"
