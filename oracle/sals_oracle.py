"""CPU fp64 oracle for the SALS decode-attention hot path (arXiv 2510.24273).

TEST INFRASTRUCTURE ONLY.  This module is the plain, slow, obviously-correct
reference the CUDA path is checked against.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  It shares no code with
``paper_2510_24273_b200`` (no kernels, headers, helpers, tables or constants)
and never imports it.

Citations: ``P:n`` = line n of the paper's LaTeX, ``S:n`` = line n of
SPEC.md.  Every step follows Algorithm 1 in the paper's order and
notation; where the paper is silent the reading is listed in DESIGN.md §3 and
repeated at the function that applies it.

All arithmetic is float64 numpy.  Library primitives used as steps: ``@``
(matmul), ``np.lexsort`` (sorting), ``np.exp``/``np.cos``/``np.sin``.

Pins (tests/test_oracle_*.py): every function below is pinned by closed forms,
SPEC worked examples (tests/golden/), brute force on tiny inputs or the
lossless-limit identity against the independent dense attention
``dense_rope_attention``.  No function is "parity unpinned" except the
approximation *quality* for r < D, k < s, which the paper only reports on real
model data (reading R13).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ROPE_HALF = 0          # pairs (i, i + d/2): HF "rotate_half" convention (reading R6)
ROPE_INTERLEAVED = 1   # pairs (2i, 2i + 1): SPEC's convention


@dataclass(frozen=True)
class Config:
    """Problem statement of Algorithm 1: heads, head dim, rank r, r*, k, RoPE base."""
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    rank: int              # r  ("U_r in R^{nd x r}")
    score_rank: int        # r* ("leading r* coordinates"; r* = 0.5 r)
    top_k: int             # k  (Alg. 1 line 5)
    sink: int = 0          # x  (P:561-564 sink tokens; 0 = pure Alg. 1)
    recent: int = 0        # z  (P:561-564 recent window; 0 = pure Alg. 1)
    rope_base: float = 10000.0
    rope_style: int = ROPE_HALF
    softmax_scale: float = 0.0   # 0 => 1/sqrt(head_dim) (Alg. 1 line 8)

    @property
    def D(self) -> int:
        """n*d of the key cache (the paper's "nd")."""
        return self.num_kv_heads * self.head_dim

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def scale(self) -> float:
        return self.softmax_scale if self.softmax_scale > 0 else 1.0 / np.sqrt(self.head_dim)


# --------------------------------------------------------------------------
# RoPE  (Eq. 3; Alg. 1 line 7)
# --------------------------------------------------------------------------
def rope_theta(head_dim: int, base: float) -> np.ndarray:
    """theta_i = base^(-2i/d), i < d/2 (RoPE frequencies behind R_i of Eq. 3)."""
    i = np.arange(head_dim // 2, dtype=np.float64)
    return np.power(np.float64(base), -2.0 * i / head_dim)


def rope(x: np.ndarray, position, base: float, style: int = ROPE_HALF) -> np.ndarray:
    """Rotate the last axis (one head, length d) of ``x`` by R_position (Eq. 3).

    ``position`` broadcasts against ``x.shape[:-1]``.  Pair p is rotated by the
    angle position * theta_p, computed in float64 (reading R7: angles in fp64).
    """
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    theta = rope_theta(d, base)
    phi = np.asarray(position, dtype=np.float64)[..., None] * theta   # [..., d/2]
    c, s = np.cos(phi), np.sin(phi)
    out = np.empty_like(x)
    if style == ROPE_HALF:
        a, b = x[..., : d // 2], x[..., d // 2:]
        out[..., : d // 2] = a * c - b * s
        out[..., d // 2:] = a * s + b * c
    elif style == ROPE_INTERLEAVED:
        a, b = x[..., 0::2], x[..., 1::2]
        out[..., 0::2] = a * c - b * s
        out[..., 1::2] = a * s + b * c
    else:
        raise ValueError("unknown rope style")
    return out


# --------------------------------------------------------------------------
# Algorithm 1, step by step
# --------------------------------------------------------------------------
def pool_query(q: np.ndarray, cfg: Config) -> np.ndarray:
    """q [n_q*d] -> q_bar [n_kv*d]: sum of the query heads of each KV group.

    Reading R1 (P:358 assumes one q in R^{nd}; GQA is silent): summing
    the G heads makes q_bar . k the sum over all query heads of the pre-RoPE
    logits q_h . k_{g(h)}, whose rank-r approximation the latent score is
    (Eq. 2).  For G = 1 this is q itself.
    """
    q = np.asarray(q, dtype=np.float64).reshape(cfg.num_kv_heads, cfg.group, cfg.head_dim)
    return q.sum(axis=1).reshape(cfg.D)


def project_latent(U: np.ndarray, x: np.ndarray) -> np.ndarray:
    """x~ = x U  (Eq. 1; Alg. 1 line 2).  x [..., D] -> [..., r]."""
    return np.asarray(x, dtype=np.float64) @ np.asarray(U, dtype=np.float64)


def latent_scores(q_tilde: np.ndarray, K_tilde: np.ndarray, r_star: int) -> np.ndarray:
    """p'_j = q~_{:r*} . k~_{j,:r*}  (Alg. 1 line 4).  K~ [s, r] -> [s]."""
    return np.asarray(K_tilde, dtype=np.float64)[:, :r_star] @ np.asarray(q_tilde, dtype=np.float64)[:r_star]


def select_topk(scores: np.ndarray, k: int, sink: int = 0, recent: int = 0) -> np.ndarray:
    """C = TopK(p', k)  (Alg. 1 line 5) with the sink/recent policy.

    Readings: R3 (all s tokens when s <= k), R4 (sink [0,x) and recent [s-z,s)
    forced, the other y = k-x-z ranked over [x, s-z)), R5 (ties -> lower
    index).  Returns the selected indices ascending.
    """
    scores = np.asarray(scores, dtype=np.float64)
    s = scores.shape[0]
    if s <= k:
        return np.arange(s, dtype=np.int64)
    x, z = sink, recent
    y = k - x - z
    ranked = np.arange(x, s - z, dtype=np.int64)
    order = np.lexsort((ranked, -scores[ranked]))        # primary: score desc; secondary: index asc
    chosen = ranked[order[:y]]
    forced = np.concatenate([np.arange(0, x), np.arange(s - z, s)]).astype(np.int64)
    return np.sort(np.concatenate([forced, chosen]))


def reconstruct(K_tilde_C: np.ndarray, U: np.ndarray) -> np.ndarray:
    """K_C = K~_C U^T  (Alg. 1 line 6).  [|C|, r] -> [|C|, D]."""
    return np.asarray(K_tilde_C, dtype=np.float64) @ np.asarray(U, dtype=np.float64).T


def restricted_attention(qR: np.ndarray, KR: np.ndarray, V: np.ndarray, cfg: Config) -> np.ndarray:
    """Eq. 6, Alg. 1 lines 8-9: p = softmax(q^R K^R_C^T / sqrt d), y = p V_C.

    qR [n_q, d]; KR, V [|C|, n_kv, d] -> y [n_q, d].  Query head h reads KV
    head floor(h / G) (contiguous GQA groups).  Max-subtracted softmax.
    """
    y = np.empty((cfg.num_q_heads, cfg.head_dim), dtype=np.float64)
    for h in range(cfg.num_q_heads):
        g = h // cfg.group
        logits = (KR[:, g, :] @ qR[h]) * cfg.scale
        p = np.exp(logits - logits.max())
        p /= p.sum()
        y[h] = p @ V[:, g, :]
    return y


def decode_request(cfg: Config, U, q, K_tilde, V_cache, s: int, forced_selection=None) -> dict:
    """Algorithm 1 lines 2 and 4-9 for one request whose caches already hold the
    appended current token (line 3 is ``append``); s includes that token.

    q [n_q*d] pre-RoPE at position s-1; K_tilde [>=s, r]; V_cache [>=s, D].
    ``forced_selection`` replaces line 5's C (parity of the arithmetic on the
    GPU's own selection, SURVEY §8(c) check (i)).
    """
    U = np.asarray(U, dtype=np.float64)
    K_tilde = np.asarray(K_tilde, dtype=np.float64)[:s]
    V_cache = np.asarray(V_cache, dtype=np.float64)[:s]
    d, nkv, nq = cfg.head_dim, cfg.num_kv_heads, cfg.num_q_heads
    # line 2: q~ = q U_r   (after GQA pooling, reading R1)
    q_tilde = project_latent(U, pool_query(q, cfg))
    # line 4: p' = q~_{r*} K~_{r*}^T
    scores = latent_scores(q_tilde, K_tilde, cfg.score_rank)
    # line 5: C = TopK(p', k)
    if forced_selection is None:
        C = select_topk(scores, cfg.top_k, cfg.sink, cfg.recent)
    else:
        C = np.asarray(forced_selection, dtype=np.int64)
    # line 6: K_C = K~_C U_r^T, reshaped to multi-head keys
    K_C = reconstruct(K_tilde[C], U).reshape(len(C), nkv, d)
    # line 7: q^R = RoPE(q) at s-1; K^R_C = RoPE(K_C) at the original positions C (reading R8)
    qR = rope(np.asarray(q, dtype=np.float64).reshape(nq, d), s - 1, cfg.rope_base, cfg.rope_style)
    KR = rope(K_C, C[:, None], cfg.rope_base, cfg.rope_style)
    # lines 8-9
    V_C = V_cache[C].reshape(len(C), nkv, d)
    y = restricted_attention(qR, KR, V_C, cfg)
    return {"y": y.reshape(nq * d), "sel": C, "scores": scores, "q_tilde": q_tilde}


def decode(cfg: Config, U, q, latent_cache, v_cache, seq_len, forced_selection=None) -> dict:
    """Batched ``decode_request``: q [B, n_q*d], latent_cache [B, cap, r], v_cache [B, cap, D]."""
    B = len(seq_len)
    outs = []
    for b in range(B):
        fs = None if forced_selection is None else forced_selection[b]
        outs.append(decode_request(cfg, U, q[b], latent_cache[b], v_cache[b], int(seq_len[b]), fs))
    return {
        "y": np.stack([o["y"] for o in outs]),
        "sel": [o["sel"] for o in outs],
        "scores": [o["scores"] for o in outs],
        "q_tilde": np.stack([o["q_tilde"] for o in outs]),
    }


def append(cfg: Config, U, k_new, v_new, pos, latent_cache, v_cache) -> None:
    """Alg. 1 lines 2-3: k~ = k U_r; K~ <- concat(K~, k~); V <- concat(V, v).

    In place on float64 caches: row pos[b] of request b.
    """
    k_tilde = project_latent(U, np.asarray(k_new, dtype=np.float64))
    for b in range(len(pos)):
        latent_cache[b, pos[b]] = k_tilde[b]
        v_cache[b, pos[b]] = v_new[b]


# --------------------------------------------------------------------------
# Dense baseline: textbook full-KV RoPE attention (the comparator; also the
# independent side of the lossless-limit pin)
# --------------------------------------------------------------------------
def dense_rope_attention(cfg: Config, q, K_pre, V, s: int) -> np.ndarray:
    """Full causal attention of the query at position s-1 over keys 0..s-1.

    q [n_q*d] pre-RoPE; K_pre, V [>=s, D] pre-RoPE keys / values.  Written
    independently of ``restricted_attention``: explicit per-head loops over
    all tokens, no selection, no latent space.
    """
    d, nkv, nq, G = cfg.head_dim, cfg.num_kv_heads, cfg.num_q_heads, cfg.group
    q = np.asarray(q, dtype=np.float64).reshape(nq, d)
    K = np.asarray(K_pre, dtype=np.float64)[:s].reshape(s, nkv, d)
    V = np.asarray(V, dtype=np.float64)[:s].reshape(s, nkv, d)
    pos = np.arange(s)
    y = np.zeros((nq, d))
    for h in range(nq):
        g = h // G
        qr = rope(q[h], s - 1, cfg.rope_base, cfg.rope_style)
        kr = rope(K[:, g, :], pos, cfg.rope_base, cfg.rope_style)
        logits = np.array([np.dot(qr, kr[j]) for j in range(s)]) * cfg.scale
        w = np.exp(logits - np.max(logits))
        y[h] = (w[:, None] * V[:, g, :]).sum(axis=0) / w.sum()
    return y.reshape(nq * d)


def dense_decode(cfg: Config, q, k_cache_post_rope, v_cache, seq_len) -> np.ndarray:
    """Dense flash-decode comparator semantics: keys already rotated at append time."""
    d, nkv, nq, G = cfg.head_dim, cfg.num_kv_heads, cfg.num_q_heads, cfg.group
    out = []
    for b in range(len(seq_len)):
        s = int(seq_len[b])
        qr = rope(np.asarray(q[b], dtype=np.float64).reshape(nq, d), s - 1, cfg.rope_base, cfg.rope_style)
        K = np.asarray(k_cache_post_rope[b], dtype=np.float64)[:s].reshape(s, nkv, d)
        V = np.asarray(v_cache[b], dtype=np.float64)[:s].reshape(s, nkv, d)
        y = np.zeros((nq, d))
        for h in range(nq):
            logits = (K[:, h // G, :] @ qr[h]) * cfg.scale
            w = np.exp(logits - logits.max())
            y[h] = (w @ V[:, h // G, :]) / w.sum()
        out.append(y.reshape(nq * d))
    return np.stack(out)


def dense_append_key(cfg: Config, k_new, pos) -> np.ndarray:
    """Dense cache write: RoPE(k) at its position (per KV head)."""
    k = np.asarray(k_new, dtype=np.float64).reshape(-1, cfg.num_kv_heads, cfg.head_dim)
    pos = np.asarray(pos)
    return rope(k, pos[:, None], cfg.rope_base, cfg.rope_style).reshape(k.shape[0], cfg.D)


# --------------------------------------------------------------------------
# Sequence-sharded decode: the oracle of the exchange protocol
# --------------------------------------------------------------------------
def shard_candidates(scores_local: np.ndarray, shard_start: int, k: int):
    """Local top-min(k, n_local) of one shard with GLOBAL indices (ties -> lower index)."""
    n = scores_local.shape[0]
    idx = np.arange(n, dtype=np.int64)
    order = np.lexsort((idx, -scores_local))[: min(k, n)]
    return scores_local[order], idx[order] + shard_start


def global_select(cand_scores: np.ndarray, cand_idx: np.ndarray, s: int, cfg: Config) -> np.ndarray:
    """Global TopK over the gathered candidates, same policy and tie-break as ``select_topk``."""
    if s <= cfg.top_k:
        return np.arange(s, dtype=np.int64)
    x, z = cfg.sink, cfg.recent
    y = cfg.top_k - x - z
    keep = (cand_idx >= x) & (cand_idx < s - z)
    cs, ci = cand_scores[keep], cand_idx[keep]
    order = np.lexsort((ci, -cs))[:y]
    forced = np.concatenate([np.arange(0, x), np.arange(s - z, s)]).astype(np.int64)
    return np.sort(np.concatenate([forced, ci[order]]))


def shard_owned_selection(gathered_scores: np.ndarray, own_idx: np.ndarray, rank: int, lo: int, hi: int, s: int,
                          cfg: Config) -> np.ndarray:
    """One rank's part of the global selection when only the candidate SCORES are exchanged (§8(e)).

    gathered_scores [P, kc]: every rank's ranked candidates (ascending global index, -inf padded),
    in rank order; own_idx [kc]: this rank's global indices (-1 padded); this rank holds [lo, hi).
    The shards are contiguous and ascending, so the gathered order (rank, position) is the global
    index order: the global TopK of the union by (score desc, index asc) -- ``select_topk``'s rule
    -- is fixed without the other ranks' indices.  Returns this rank's selected positions plus its
    forced sink / recent ones, ascending (global indices)."""
    hi = min(hi, s)
    if s <= cfg.top_k:
        return np.arange(lo, max(lo, hi), dtype=np.int64)
    x, z = cfg.sink, cfg.recent
    y = cfg.top_k - x - z
    P, kc = gathered_scores.shape
    rk, pos = np.meshgrid(np.arange(P), np.arange(kc), indexing="ij")
    sc, rk, pos = gathered_scores.ravel(), rk.ravel(), pos.ravel()
    valid = ~np.isneginf(sc)
    sc, rk, pos = sc[valid], rk[valid], pos[valid]
    order = np.lexsort((pos, rk, -sc))[:y]
    mine = pos[order][rk[order] == rank]
    picks = own_idx[mine].astype(np.int64)
    forced = np.concatenate([np.arange(0, x), np.arange(s - z, s)]).astype(np.int64)
    forced = forced[(forced >= lo) & (forced < hi)]
    return np.sort(np.concatenate([forced, picks]))


def partial_attention(qR: np.ndarray, KR: np.ndarray, V: np.ndarray, cfg: Config):
    """Per query head (m, l, o) over a token subset: m = max logit, l = sum e^{l-m}, o = sum e^{l-m} v."""
    nq, d = cfg.num_q_heads, cfg.head_dim
    m = np.full(nq, -np.inf)
    l = np.zeros(nq)
    o = np.zeros((nq, d))
    if KR.shape[0] == 0:
        return m, l, o
    for h in range(nq):
        g = h // cfg.group
        logits = (KR[:, g, :] @ qR[h]) * cfg.scale
        m[h] = logits.max()
        w = np.exp(logits - m[h])
        l[h] = w.sum()
        o[h] = w @ V[:, g, :]
    return m, l, o


def lse_merge(ms: np.ndarray, ls: np.ndarray, os_: np.ndarray) -> np.ndarray:
    """Merge per-part (m, l, o) [P, n_q(, d)] into y [n_q, d] (log-sum-exp)."""
    M = ms.max(axis=0)
    w = np.where(np.isneginf(ms), 0.0, np.exp(ms - M))
    L = (w * ls).sum(axis=0)
    return (w[..., None] * os_).sum(axis=0) / L[:, None]


# ------------------------------------------------------------------ calibration
def calibrate(K: np.ndarray, r: int):
    """Offline calibration (Sec. 4.2): C = K^T K over the stacked
    pre-RoPE keys K [N, nd] (heads merged); C = U S U^T; U_r = the leading
    r eigenvectors.  Returns (U_r [nd, r] with columns in descending eigenvalue
    order, all eigenvalues descending).  Library primitive: ``np.linalg.eigh``.
    Eigenvectors are defined up to sign; each column is signed so that its
    largest-magnitude component is positive (first such index on ties) -- a
    convention of this build, not of the paper."""
    K = np.asarray(K, dtype=np.float64)
    C = K.T @ K
    w, V = np.linalg.eigh(C)                 # ascending
    order = np.argsort(-w, kind="stable")
    w, V = w[order], V[:, order]
    U = V[:, :r].copy()
    for j in range(r):
        i = int(np.argmax(np.abs(U[:, j])))
        if U[i, j] < 0:
            U[:, j] = -U[:, j]
    return U, w


def captured_variance(U: np.ndarray, K: np.ndarray) -> float:
    """E(U) = ||K U||_F^2 = tr(U^T K^T K U): the key energy kept by the projection (Lemma 1)."""
    KU = np.asarray(K, dtype=np.float64) @ np.asarray(U, dtype=np.float64)
    return float(np.sum(KU * KU))


# ------------------------------------------------------------------ value quantisation (f1)
def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bfloat16 (ties to even), returned as float64: the storage
    step of the quantisation parameters (a definition of the format, not arithmetic
    of the method)."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def quantize_values(v: np.ndarray, bits: int, group: int = 32):
    """Channel-wise group quantisation of the value cache (KIVI-style
    asymmetric grid; reading R15): for every token, each run of `group` consecutive
    channels shares zero = min and scale = (max - min) / (2^bits - 1), both stored
    in bfloat16; code = clamp(round((v - zero) / scale), 0, 2^bits - 1) computed
    from the stored (rounded) zero / scale; scale 0 -> code 0.

    Precision (R15): the codes are integers decided by floating point, so the
    decision is taken in the kernel's precision, IEEE fp32 with round-to-nearest-
    even: v is the stored value (bf16 / fp32, exact in fp32); hi - lo, the
    division by 2^bits - 1, v - zero and the division by scale are single fp32
    operations; the scale is rounded fp32 -> bf16 (nearest-even); round() is
    half-to-even.  v [..., D] -> (codes [..., D] int, scale [..., D/group],
    zero [..., D/group]) with scale / zero as float64 (exact bf16 values)."""
    v32 = np.asarray(v, dtype=np.float32)
    g = v32.reshape(*v32.shape[:-1], v32.shape[-1] // group, group)
    lo, hi = g.min(-1), g.max(-1)
    qmax = (1 << bits) - 1
    zero = bf16_round(lo).astype(np.float32)
    scale = bf16_round((hi - lo) / np.float32(qmax)).astype(np.float32)
    safe = np.where(scale > 0, scale, np.float32(1.0)).astype(np.float32)
    q = (g - zero[..., None]) / safe[..., None]                      # fp32 subtract, fp32 divide
    codes = np.clip(np.rint(q), 0, qmax)
    codes = np.where(scale[..., None] > 0, codes, 0).astype(np.int64)
    return codes.reshape(v32.shape), scale.astype(np.float64), zero.astype(np.float64)


def dequantize_values(codes: np.ndarray, scale: np.ndarray, zero: np.ndarray, group: int = 32) -> np.ndarray:
    """v^ = zero + scale * code per group (the V^ of Alg. 1)."""
    c = np.asarray(codes, dtype=np.float64)
    g = c.reshape(*c.shape[:-1], c.shape[-1] // group, group)
    return (np.asarray(zero, np.float64)[..., None] + np.asarray(scale, np.float64)[..., None] * g).reshape(c.shape)


def value_hat(v_rows: np.ndarray, bits: int, recent: int, s: int, group: int = 32) -> np.ndarray:
    """The V^ of Algorithm 1 as the quantised cache holds it for a request of
    s tokens (reading R15): positions j >= s - z (the recent window, whose
    tokens "are compressed by only 50%" = 8-bit codes on the same grid
    rule) are reconstructed from 8-bit codes, all earlier positions from `bits`-bit
    codes; bits = 16 keeps the stored values (no quantisation).  v_rows [>= s, D] ->
    [s, D] float64."""
    v = np.asarray(v_rows, dtype=np.float64)[:s]
    if bits == 16:
        return v.copy()
    out = dequantize_values(*quantize_values(v, bits, group), group)
    z = min(max(recent, 0), s)
    if z > 0:
        out[s - z:] = dequantize_values(*quantize_values(v[s - z:], 8, group), group)
    return out
