"""Algorithmic byte / FLOP accounting for the roofline figures.

Host-side arithmetic only (no kernels).  The paper's idealised model is Sec.
4.5: dense attention moves 2 s d scalars, SALS moves s r* + 2 k r,
speed-up 1 / (d_{r*}/2 + d_r k_s).  The per-stage byte counts below are what
this build's kernels must move at minimum (bf16 storage, V kept at full
precision).
"""
from __future__ import annotations


def sals_access_ratio(d_rstar: float, d_r: float, k_s: float) -> float:
    """(s r* + 2 k r) / (2 s d) = d_{r*}/2 + d_r k_s."""
    return d_rstar / 2.0 + d_r * k_s


def sals_speedup(d_rstar: float, d_r: float, k_s: float) -> float:
    """Memory-bound speed-up 1 / (d_{r*}/2 + d_r k_s)."""
    return 1.0 / sals_access_ratio(d_rstar, d_r, k_s)


def stage_bytes(*, batch, seq, num_q_heads, num_kv_heads, head_dim, rank, score_rank, top_k,
                elem=2, v_row_bytes=None, **_):
    """Algorithmic HBM bytes per layer-step of each stage (whole batch).

    seq = s (tokens incl. the decoded one); k_eff = min(k, s).
    """
    D = num_kv_heads * head_dim
    k = min(top_k, seq)
    b = {}
    b["append"] = rank * D * elem + batch * (2 * D * elem) + batch * (rank + D) * elem
    b["qproj"] = score_rank * D * elem + batch * num_q_heads * head_dim * elem
    b["score"] = batch * seq * score_rank * elem + batch * seq * 4          # latent reads + fp32 scores
    b["topk"] = batch * seq * 4 + batch * k * 4                               # scores (L2) + indices
    # fused reconstruct+attention: gathered latent rows, U once, gathered V rows, partials
    vrow = v_row_bytes if v_row_bytes else D * elem      # quantised value rows (f1) are smaller
    b["recon_attn"] = batch * k * rank * elem + rank * D * elem + batch * k * vrow
    b["total"] = b["append"] + b["qproj"] + b["score"] + b["recon_attn"]
    return b


def recon_flops(*, batch, seq, num_kv_heads, head_dim, rank, top_k, **_):
    """2 * (B k) * r * D   (Alg. 1 line 6)."""
    return 2.0 * batch * min(top_k, seq) * rank * num_kv_heads * head_dim


def dense_bytes(*, batch, seq, num_kv_heads, head_dim, elem=2, **_):
    """Full-KV flash decode: 2 s D elements per request."""
    return 2.0 * batch * seq * num_kv_heads * head_dim * elem
