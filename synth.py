"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests,
``smoke()`` and ``bench.py``.

Holds none of the method's arithmetic (no projection, scoring, selection,
RoPE or attention): only random draws, a QR for a random orthonormal basis,
and fixed scalings.  Recipe:

* U = Q of the QR of an N(0,1) [D, r] matrix (orthonormal columns).
* Latent key cache K~[b, j, i] = c * sigma_i * N(0,1), sigma_i = 0.5^(i / (r/8))
  (PCA-like decaying spectrum, so the leading r* coordinates carry most of the
  energy); c normalises E||U k~||^2 to D.
* Query: a latent direction w (same spectrum); q_h = 0.8 N(0,1) + 0.6 sqrt(d)
  (U w)_g / ||(U w)_g|| for every head h of KV group g.
* Planted heavy hitters: max(1, s/64) random positions per request get
  K~ += 3 c ||sigma|| w/||w|| (peaked attention, as the paper relies on).
* V, k_new, v_new ~ N(0, 1).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 24273


def orthonormal(rng: np.random.Generator, D: int, r: int) -> np.ndarray:
    q, _ = np.linalg.qr(rng.standard_normal((D, r)))
    return q


def spectrum(r: int) -> np.ndarray:
    return 0.5 ** (np.arange(r) / max(r / 8.0, 1.0))


def gen_problem(*, num_q_heads, num_kv_heads, head_dim, rank, batch, seq_lens, cap=None,
                seed=SEED_BASE, plant=True, U=None):
    """Return float32 numpy arrays for one layer of a decode step.

    seq_lens[b] = s_b, the length INCLUDING the token being decoded; the caches
    are filled for positions < s_b - 1 (the appended token is k_new / v_new,
    written at position s_b - 1 by ``append``).
    """
    rng = np.random.default_rng(seed)
    D = num_kv_heads * head_dim
    G = num_q_heads // num_kv_heads
    seq_lens = np.asarray(seq_lens, dtype=np.int64)
    cap = int(cap if cap is not None else seq_lens.max())
    if U is None:
        U = orthonormal(rng, D, rank)
    sig = spectrum(rank)
    c = np.sqrt(D / np.sum(sig ** 2))
    latent = (rng.standard_normal((batch, cap, rank), dtype=np.float32) * (c * sig).astype(np.float32))
    w = rng.standard_normal(rank) * sig
    u = (U.astype(np.float64) @ w).reshape(num_kv_heads, head_dim)
    u /= np.linalg.norm(u, axis=1, keepdims=True) + 1e-30
    q = 0.8 * rng.standard_normal((batch, num_q_heads, head_dim))
    q += 0.6 * np.sqrt(head_dim) * np.repeat(u, G, axis=0)[None]
    if plant:
        wn = (w / np.linalg.norm(w)).astype(np.float32)
        amp = np.float32(3.0 * c * np.linalg.norm(sig))
        for b in range(batch):
            s = int(seq_lens[b])
            n = max(1, s // 64)
            pos = rng.choice(max(s - 1, 1), size=min(n, max(s - 1, 1)), replace=False)
            latent[b, pos] += amp * wn
    v = rng.standard_normal((batch, cap, D), dtype=np.float32)
    k_new = rng.standard_normal((batch, D), dtype=np.float32)
    v_new = rng.standard_normal((batch, D), dtype=np.float32)
    return {
        "U": U.astype(np.float32),
        "latent": latent,
        "v": v,
        "q": q.reshape(batch, num_q_heads * head_dim).astype(np.float32),
        "k_new": k_new,
        "v_new": v_new,
        "seq_len": seq_lens.astype(np.int32),
    }


def gen_full_keys(rng: np.random.Generator, n: int, D: int, rank_hint: int) -> np.ndarray:
    """Pre-RoPE full keys with a low-rank-dominated covariance (for definition-mode pins)."""
    basis = orthonormal(rng, D, min(rank_hint, D)).astype(np.float64)
    z = rng.standard_normal((n, basis.shape[1])) * spectrum(basis.shape[1])
    return (z @ basis.T + 0.05 * rng.standard_normal((n, D))).astype(np.float32)


# Paper-shaped configurations (BASELINE.json "configs")
CONFIGS = {
    "c1": dict(num_q_heads=4, num_kv_heads=4, head_dim=16, rank=16, score_rank=8, top_k=32,
               batch=1, seq=256, rope_base=10000.0, dtype="f32"),
    "c2": dict(num_q_heads=32, num_kv_heads=32, head_dim=128, rank=512, score_rank=256, top_k=512,
               batch=8, seq=4096, rope_base=10000.0, dtype="bf16"),
    "c3": dict(num_q_heads=32, num_kv_heads=8, head_dim=128, rank=512, score_rank=256, top_k=4096,
               batch=4, seq=32768, rope_base=1.0e6, dtype="bf16"),
    "c4": dict(num_q_heads=32, num_kv_heads=8, head_dim=128, rank=512, score_rank=256, top_k=16384,
               batch=1, seq=131072, rope_base=500000.0, dtype="bf16"),
    "c5": dict(num_q_heads=32, num_kv_heads=32, head_dim=128, rank=512, score_rank=256, top_k=None,
               batch=None, seq=None, rope_base=10000.0, dtype="bf16"),
}


def gen_layer_torch(*, num_q_heads, num_kv_heads, head_dim, rank, batch, seq, cap=None, generator=None,
                    device="cuda", dtype=None, dense=False):
    """The same recipe as ``gen_problem`` drawn directly on the device with torch
    (bench-sized problems: 32 layers x hundreds of MiB).  Returns a dict of
    device tensors; ``dense`` adds a full pre-RoPE key cache K for the dense
    comparator."""
    import torch
    dtype = dtype or torch.bfloat16
    g = generator
    D = num_kv_heads * head_dim
    G = num_q_heads // num_kv_heads
    cap = cap or seq
    U, _ = torch.linalg.qr(torch.randn(D, rank, device=device, generator=g, dtype=torch.float32))
    sig = torch.tensor(spectrum(rank), device=device, dtype=torch.float32)
    c = float(np.sqrt(D / float((sig ** 2).sum())))
    # per-request draws (fp32 temporaries of one request at a time: bench-sized batches
    # of 32 layers fill most of HBM)
    latent = torch.empty(batch, cap, rank, device=device, dtype=dtype)
    for b in range(batch):
        latent[b] = (torch.randn(cap, rank, device=device, generator=g, dtype=torch.float32) * (c * sig)).to(dtype)
    w = torch.randn(rank, device=device, generator=g) * sig
    u = (U @ w).view(num_kv_heads, head_dim)
    u = u / u.norm(dim=1, keepdim=True)
    q = 0.8 * torch.randn(batch, num_q_heads, head_dim, device=device, generator=g)
    q = q + 0.6 * float(np.sqrt(head_dim)) * u.repeat_interleave(G, dim=0)[None]
    n = max(1, seq // 64)
    pos = torch.randint(0, max(seq - 1, 1), (batch, n), device=device, generator=g)
    amp = 3.0 * c * float(sig.norm())
    hit = (amp * w / w.norm())
    for b in range(batch):   # planted heavy hitters (fp32 add, one rounding to the storage type)
        rows = latent[b, pos[b]].float() + hit
        latent[b, pos[b]] = rows.to(dtype)
    v = torch.empty(batch, cap, D, device=device, dtype=dtype)
    for b in range(batch):
        v[b] = torch.randn(cap, D, device=device, generator=g, dtype=torch.float32).to(dtype)
    out = {
        "U": U.to(dtype).contiguous(),
        "latent": latent,
        "v": v,
        "q": q.reshape(batch, num_q_heads * head_dim).to(dtype),
        "k_new": torch.randn(batch, D, device=device, generator=g).to(dtype),
        "v_new": torch.randn(batch, D, device=device, generator=g).to(dtype),
    }
    if dense:   # dense comparator's key cache: independent N(0,1) draws (timing only)
        kd = torch.empty(batch, cap, D, device=device, dtype=dtype)
        for b in range(batch):
            kd[b] = torch.randn(cap, D, device=device, generator=g, dtype=torch.float32).to(dtype)
        out["k_dense"] = kd
    return out
