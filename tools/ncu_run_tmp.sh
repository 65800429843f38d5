bash tools/gpu_ncu.sh n1 c3 "project score_tma recon_attn topk merge"
SALS_SCORE_LSU=1 bash tools/gpu_ncu.sh n1lsu c3 "latent_score"
