"""Pins of the fp64 oracle against the paper and mathematics (no GPU).

Each test states what it pins.  None re-types the oracle's formula: they use
worked examples (tests/golden, cited), closed forms, brute force on tiny
inputs, invariants, or the lossless limit against the independent dense
attention.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import sals_oracle as O
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _cfg(**kw):
    base = dict(num_q_heads=4, num_kv_heads=2, head_dim=8, rank=16, score_rank=8, top_k=8)
    base.update(kw)
    return O.Config(**base)


# ---------------------------------------------------------------- RoPE (Eq. 3)
@pytest.mark.parametrize("style", [O.ROPE_HALF, O.ROPE_INTERLEAVED])
def test_rope_golden(style):
    """SPEC S:111-113 examples (style-free: d = 2 or m = 0) and the d >= 4, m >= 1
    cases written from S:98 pair by pair (tests/golden/make_rope_examples.py): they
    pin theta_i = base^(-2i/d) for i >= 1 and each style's pairing."""
    name = {O.ROPE_HALF: "half", O.ROPE_INTERLEAVED: "interleaved"}[style]
    n = 0
    for c in _gold("rope_examples.json")["cases"]:
        if c.get("style", name) != name:
            continue
        out = O.rope(np.array(c["x"]), c["m"], c["base"], style)
        np.testing.assert_allclose(out, c["expected"], rtol=0, atol=1e-14)
        n += 1
    assert n >= 5


def _explicit_rotation(d, m, base, style):
    """R_m as an explicit d x d block rotation matrix (independent construction)."""
    R = np.zeros((d, d))
    for p in range(d // 2):
        ang = m * base ** (-(2.0 * p) / d)
        i, j = (p, p + d // 2) if style == O.ROPE_HALF else (2 * p, 2 * p + 1)
        R[i, i] = math.cos(ang)
        R[i, j] = -math.sin(ang)
        R[j, i] = math.sin(ang)
        R[j, j] = math.cos(ang)
    return R


@pytest.mark.parametrize("style", [O.ROPE_HALF, O.ROPE_INTERLEAVED])
@pytest.mark.parametrize("d", [2, 8, 16, 128])
def test_rope_matches_rotation_matrix_and_invariants(style, d):
    rng = np.random.default_rng(1)
    for m in [0, 1, 7, 4095, 131071]:
        x = rng.standard_normal(d)
        out = O.rope(x, m, 10000.0, style)
        np.testing.assert_allclose(out, _explicit_rotation(d, m, 10000.0, style) @ x, atol=1e-11)
        assert abs(np.linalg.norm(out) - np.linalg.norm(x)) < 1e-12        # S:127 norm preservation
    # relative position property: <R_i q, R_j k> = <R_{i+t} q, R_{j+t} k>
    q, k = rng.standard_normal(d), rng.standard_normal(d)
    for i, j, t in [(5, 3, 11), (1000, 17, 4096), (0, 131000, 71)]:
        a = O.rope(q, i, 1e4, style) @ O.rope(k, j, 1e4, style)
        b = O.rope(q, i + t, 1e4, style) @ O.rope(k, j + t, 1e4, style)
        assert abs(a - b) < 1e-9


def test_rope_batch_positions_rowwise():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((5, 3, 16))
    pos = np.array([0, 3, 9, 100, 70000])
    out = O.rope(X, pos[:, None], 5e5)
    for i in range(5):
        for h in range(3):
            np.testing.assert_allclose(out[i, h], O.rope(X[i, h], pos[i], 5e5), atol=1e-13)


# ------------------------------------------------- projection / scores (Eq. 1, Alg. 1 l.2/4)
def test_projection_coordinate_nullspace_roundtrip():
    rng = np.random.default_rng(3)
    D, r = 12, 5
    U = np.vstack([np.eye(r), np.zeros((D - r, r))])         # S:253 coordinate projection
    k = rng.standard_normal(D)
    np.testing.assert_array_equal(O.project_latent(U, k), k[:r])
    k0 = np.concatenate([np.zeros(r), rng.standard_normal(D - r)])
    np.testing.assert_array_equal(O.project_latent(U, k0), np.zeros(r))   # S:254 null space
    Uf = synth.orthonormal(rng, D, D).astype(np.float64)                    # S:255 round trip r = nd
    np.testing.assert_allclose(O.reconstruct(O.project_latent(Uf, k)[None], Uf)[0], k, atol=1e-12)
    # keys inside span(U) reconstruct exactly for r < nd
    Ur = Uf[:, :r]
    ks = Ur @ rng.standard_normal(r)
    np.testing.assert_allclose(O.reconstruct(O.project_latent(Ur, ks)[None], Ur)[0], ks, atol=1e-12)


def test_pool_query_groups():
    cfg = _cfg(num_q_heads=6, num_kv_heads=2, head_dim=3)
    q = np.arange(18, dtype=float)
    # heads 0,1,2 -> kv 0 ; heads 3,4,5 -> kv 1 (contiguous groups)
    expect = np.concatenate([q[0:3] + q[3:6] + q[6:9], q[9:12] + q[12:15] + q[15:18]])
    np.testing.assert_array_equal(O.pool_query(q, cfg), expect)


@pytest.mark.parametrize("nq,nkv", [(4, 4), (8, 2)])
def test_latent_scores_lossless_limit_bruteforce(nq, nkv):
    """U = I, r* = r = D: p'_j == sum over query heads of pre-RoPE q_h . k_{g(h),j}."""
    rng = np.random.default_rng(4)
    d = 4
    cfg = _cfg(num_q_heads=nq, num_kv_heads=nkv, head_dim=d, rank=nkv * d, score_rank=nkv * d)
    D = cfg.D
    K = rng.standard_normal((9, D))
    q = rng.standard_normal(nq * d)
    qt = O.project_latent(np.eye(D), O.pool_query(q, cfg))
    s = O.latent_scores(qt, O.project_latent(np.eye(D), K), D)
    for j in range(9):
        ref = 0.0
        for h in range(nq):
            g = h // (nq // nkv)
            for t in range(d):
                ref += q[h * d + t] * K[j, g * d + t]
        assert abs(s[j] - ref) < 1e-12
    assert np.all(O.latent_scores(np.zeros(D), K, D) == 0)             # S:334 q = 0


def test_latent_scores_truncation_bruteforce():
    rng = np.random.default_rng(5)
    Kt = rng.standard_normal((7, 10))
    qt = rng.standard_normal(10)
    s = O.latent_scores(qt, Kt, 4)
    for j in range(7):
        assert abs(s[j] - sum(qt[i] * Kt[j, i] for i in range(4))) < 1e-13


# ------------------------------------------------------------------ TopK (Alg. 1 l.5)
def test_topk_golden():
    for c in _gold("topk_examples.json")["cases"]:
        got = O.select_topk(np.array(c["scores"]), c["k"], c["sink"], c["recent"])
        assert got.tolist() == c["expected"]


def _brute_topk(scores, k, x, z):
    """Exhaustive: the unique subset T of the ranked range, |T| = y, such that every
    chosen j beats every unchosen i (higher score, or equal score and lower index)."""
    s = len(scores)
    if s <= k:
        return list(range(s))
    y = k - x - z
    ranked = list(range(x, s - z))
    winners = []
    for T in itertools.combinations(ranked, y):
        Ts = set(T)
        ok = all((scores[j] > scores[i]) or (scores[j] == scores[i] and j < i)
                 for j in T for i in ranked if i not in Ts)
        if ok:
            winners.append(T)
    assert len(winners) == 1
    return sorted(list(range(x)) + list(winners[0]) + list(range(s - z, s)))


def test_topk_exhaustive_small():
    rng = np.random.default_rng(6)
    for trial in range(150):
        s = int(rng.integers(1, 10))
        scores = rng.integers(0, 3, size=s).astype(float)            # many ties
        k = int(rng.integers(1, 10))
        x = int(rng.integers(0, k + 1))
        z = int(rng.integers(0, k - x + 1))
        got = O.select_topk(scores, k, x, z).tolist()
        assert got == _brute_topk(scores.tolist(), k, x, z), (scores, k, x, z)


def test_topk_invariants():
    rng = np.random.default_rng(7)
    sc = rng.standard_normal(500)
    base = O.select_topk(sc, 40, 4, 8)
    assert len(base) == 40 and np.all(np.diff(base) > 0)
    assert set(range(4)) | set(range(492, 500)) <= set(base.tolist())
    np.testing.assert_array_equal(O.select_topk(3.0 * sc - 7.0, 40, 4, 8), base)   # S:366 affine
    np.testing.assert_array_equal(O.select_topk(sc[:30], 40), np.arange(30))      # s <= k


# ------------------------------------------------------------ attention (Eq. 6, l.8-9)
def test_restricted_softmax_golden():
    cfg = _cfg(num_q_heads=1, num_kv_heads=1, head_dim=2, softmax_scale=1.0)
    for c in _gold("softmax_examples.json")["cases"]:
        n = len(c["logits"])
        qR = np.array([[1.0, 0.0]])
        KR = np.array([[[lg, 0.0]] for lg in c["logits"]])
        V = np.zeros((n, 1, 2))
        V[:, 0, 0] = np.arange(n) == 0
        V[:, 0, 1] = np.arange(n) == n - 1 if n > 1 else 0
        y = O.restricted_attention(qR, KR, V, cfg)[0]
        np.testing.assert_allclose(y[0], c["expected_p"][0], atol=1e-15)
        if n > 1:
            np.testing.assert_allclose(y[1], c["expected_p"][-1], atol=1e-15)


def test_default_scale_is_inverse_sqrt_head_dim_closed_form():
    """qR = (2,0,0,0), keys (1,0,0,0) and 0: raw dots (2, 0), scaled by 1/sqrt(4) -> (1, 0)."""
    cfg = _cfg(num_q_heads=1, num_kv_heads=1, head_dim=4)
    qR = np.array([[2.0, 0, 0, 0]])
    KR = np.array([[[1.0, 0, 0, 0]], [[0.0, 0, 0, 0]]])
    V = np.array([[[1.0, 0, 0, 0]], [[0.0, 1, 0, 0]]])
    y = O.restricted_attention(qR, KR, V, cfg)[0]
    e = math.e
    np.testing.assert_allclose(y[:2], [e / (1 + e), 1 / (1 + e)], atol=1e-15)


def test_dense_attention_closed_forms():
    cfg = _cfg(num_q_heads=1, num_kv_heads=1, head_dim=4, rank=4, score_rank=4)
    V = np.array([[1.0, 2, 3, 4], [5.0, 6, 7, 8]])
    # s = 1 -> y = v
    np.testing.assert_allclose(O.dense_rope_attention(cfg, [1, 2, 3, 4], np.ones((1, 4)), V[:1], 1), V[0], atol=1e-15)
    # q = 0 -> uniform -> mean of values
    np.testing.assert_allclose(O.dense_rope_attention(cfg, np.zeros(4), np.ones((2, 4)), V, 2), V.mean(0), atol=1e-14)
    # s = 2, key 1 = q at the query's own position, key 0 = 0: logits (0, |q|^2/sqrt d) = (0, 2)
    q = np.array([2.0, 0, 0, 0])
    K = np.array([[0.0, 0, 0, 0], q])
    p1 = math.exp(2) / (1 + math.exp(2))
    np.testing.assert_allclose(O.dense_rope_attention(cfg, q, K, V, 2), (1 - p1) * V[0] + p1 * V[1], atol=1e-14)


def test_decode_single_token_returns_value():
    """s = 1: the only token is the appended one, p = [1], y = v_new."""
    cfg = _cfg(top_k=4)
    rng = np.random.default_rng(8)
    U = synth.orthonormal(rng, cfg.D, cfg.rank)
    lat = rng.standard_normal((1, cfg.rank))
    v = rng.standard_normal((1, cfg.D))
    out = O.decode_request(cfg, U, rng.standard_normal(cfg.num_q_heads * cfg.head_dim), lat, v, 1)
    G = cfg.group
    expect = np.repeat(v[0].reshape(cfg.num_kv_heads, 1, cfg.head_dim), G, axis=1).reshape(-1)
    np.testing.assert_allclose(out["y"], expect, atol=1e-14)


# ------------------------------------------------------- lossless limit (whole Alg. 1)
@pytest.mark.parametrize("nq,nkv,style,x,z", [(4, 4, O.ROPE_HALF, 0, 0), (8, 2, O.ROPE_HALF, 2, 3),
                                            (4, 2, O.ROPE_INTERLEAVED, 0, 1)])
def test_lossless_limit_equals_dense_rope_attention(nq, nkv, style, x, z):
    """r = D, orthogonal U, k >= s: SALS == textbook dense RoPE attention."""
    rng = np.random.default_rng(9)
    d = 8
    D = nkv * d
    for trial in range(20):
        s = int(rng.integers(1, 40))
        cfg = _cfg(num_q_heads=nq, num_kv_heads=nkv, head_dim=d, rank=D, score_rank=int(rng.integers(1, D + 1)),
                   top_k=s + int(rng.integers(0, 3)), sink=x, recent=z, rope_base=float(rng.choice([1e4, 5e5])),
                   rope_style=style)
        U = synth.orthonormal(rng, D, D).astype(np.float64)
        K = rng.standard_normal((s, D))
        V = rng.standard_normal((s, D))
        q = rng.standard_normal(nq * d)
        lat = np.empty((1, s, D))
        vc = np.empty((1, s, D))
        # write the cache through append, token by token (Alg. 1 lines 2-3)
        for j in range(s):
            O.append(cfg, U, K[j][None], V[j][None], [j], lat, vc)
        out = O.decode(cfg, U, q[None], lat, vc, [s])
        ref = O.dense_rope_attention(cfg, q, K, V, s)
        np.testing.assert_allclose(out["y"][0], ref, atol=1e-10)


def test_dense_decode_post_rope_cache_equals_textbook():
    rng = np.random.default_rng(10)
    cfg = _cfg(num_q_heads=8, num_kv_heads=2, head_dim=8, rope_base=1e6)
    s = 33
    K = rng.standard_normal((s, cfg.D))
    V = rng.standard_normal((s, cfg.D))
    q = rng.standard_normal(cfg.num_q_heads * cfg.head_dim)
    kc = O.dense_append_key(cfg, K, np.arange(s))
    y = O.dense_decode(cfg, q[None], kc[None], V[None], [s])[0]
    np.testing.assert_allclose(y, O.dense_rope_attention(cfg, q, K, V, s), atol=1e-12)


def test_output_invariant_to_unselected_tokens():
    """Perturbing V of tokens outside C leaves y unchanged."""
    rng = np.random.default_rng(11)
    cfg = _cfg(top_k=6)
    p = synth.gen_problem(num_q_heads=4, num_kv_heads=2, head_dim=8, rank=16, batch=1, seq_lens=[50], seed=3)
    out = O.decode(cfg, p["U"], p["q"], p["latent"], p["v"], [50])
    sel = out["sel"][0]
    v2 = p["v"].copy()
    mask = np.ones(50, bool)
    mask[sel] = False
    v2[0, mask] += rng.standard_normal((mask.sum(), cfg.D)).astype(np.float32)
    out2 = O.decode(cfg, p["U"], p["q"], p["latent"], v2, [50])
    np.testing.assert_array_equal(out["y"], out2["y"])
    assert len(sel) == 6


def test_forced_selection_with_own_selection_is_identity():
    cfg = _cfg(top_k=6, sink=1, recent=2)
    p = synth.gen_problem(num_q_heads=4, num_kv_heads=2, head_dim=8, rank=16, batch=2, seq_lens=[50, 9], seed=4)
    a = O.decode(cfg, p["U"], p["q"], p["latent"], p["v"], p["seq_len"])
    b = O.decode(cfg, p["U"], p["q"], p["latent"], p["v"], p["seq_len"], forced_selection=a["sel"])
    np.testing.assert_array_equal(a["y"], b["y"])
    assert a["sel"][1].tolist() == list(range(6)) or len(a["sel"][1]) == 6


# ---------------------------------------------------------- sharded protocol (§8(e))
def test_sharded_selection_and_merge_equal_unsharded():
    rng = np.random.default_rng(12)
    cfg = _cfg(num_q_heads=4, num_kv_heads=2, head_dim=8, top_k=17, sink=2, recent=3)
    for trial in range(30):
        s = int(rng.integers(5, 120))
        P = int(rng.integers(1, 6))
        sc = rng.integers(0, 6, size=s).astype(float)                 # ties across shards
        ref = O.select_topk(sc, cfg.top_k, cfg.sink, cfg.recent)
        bounds = np.linspace(0, s, P + 1).astype(int)
        cs, ci = [], []
        for p_ in range(P):
            a, b = bounds[p_], bounds[p_ + 1]
            x1, x2 = O.shard_candidates(sc[a:b], a, cfg.top_k)
            cs.append(x1)
            ci.append(x2)
        got = O.global_select(np.concatenate(cs), np.concatenate(ci), s, cfg)
        np.testing.assert_array_equal(got, ref)
        # scores-only exchange: each rank's owned part from the gathered scores, union == ref
        y = cfg.top_k - cfg.sink - cfg.recent
        pad = max(cfg.top_k, 1)
        gs, gi = np.full((P, pad), -np.inf), np.full((P, pad), -1)
        for p_ in range(P):
            a, b = bounds[p_], bounds[p_ + 1]
            keep = (ci[p_] >= cfg.sink) & (ci[p_] < s - cfg.recent)
            sel = np.sort(ci[p_][keep][np.lexsort((ci[p_][keep], -cs[p_][keep]))[:y]])   # ranked, ascending index
            gs[p_, :len(sel)] = sc[sel]
            gi[p_, :len(sel)] = sel
        owned = [O.shard_owned_selection(gs, gi[p_], p_, bounds[p_], bounds[p_ + 1], s, cfg) for p_ in range(P)]
        np.testing.assert_array_equal(np.concatenate(owned), ref)
        # LSE merge of per-shard partial attention == restricted attention over all of C
        qR = rng.standard_normal((cfg.num_q_heads, cfg.head_dim))
        KR = rng.standard_normal((len(ref), cfg.num_kv_heads, cfg.head_dim))
        V = rng.standard_normal((len(ref), cfg.num_kv_heads, cfg.head_dim))
        parts = [O.partial_attention(qR, KR[(ref >= bounds[i]) & (ref < bounds[i + 1])],
                                     V[(ref >= bounds[i]) & (ref < bounds[i + 1])], cfg) for i in range(P)]
        y = O.lse_merge(np.stack([p_[0] for p_ in parts]), np.stack([p_[1] for p_ in parts]),
                        np.stack([p_[2] for p_ in parts]))
        np.testing.assert_allclose(y, O.restricted_attention(qR, KR, V, cfg), atol=1e-12)


# ---------------------------------------------------------- byte model (Sec. 4.5)
def test_memory_model_matches_paper_table2_and_p427():
    from paper_2510_24273_b200 import traffic
    g = _gold("memory_model.json")
    for a in g["exact_anchors"]:
        assert traffic.sals_access_ratio(a["d_rstar"], a["d_r"], a["k_s"]) == a["ratio"]
        assert traffic.sals_speedup(a["d_rstar"], a["d_r"], a["k_s"]) == a["speedup"]
    for c in g["cases"]:
        ratio = traffic.sals_access_ratio(c["d_r"] * c["r_star_over_r"], c["d_r"], c["k_s"])
        assert abs(ratio - c["table2_access"]) <= c["abs_tol"]
        assert abs(1.0 / c["table2_access"] - c["p427_reduction"]) < 0.01


def test_roofline_numerators_match_survey_sizes():
    """The per-launch work the bench divides by kernel time (traffic.stage_bytes /
    recon_flops) against the sizes SURVEY §8(a) lists for c2 / c3 / c4: latent
    reads of the score stage 16 / 64 / 64 MiB (a3), gathered latent rows 4 / 16 /
    16 MiB and the reconstruction GEMM 4096x4096x512 / 16384x1024x512 = 17.18
    GFLOP each (a5), gathered V rows 32 MiB each (a7), U 4 / 1 / 1 MiB."""
    from paper_2510_24273_b200 import traffic
    MiB = 1 << 20
    want = {"c2": (16, 4, 32, 4), "c3": (64, 16, 32, 1), "c4": (64, 16, 32, 1)}
    for name, (score_mib, lat_mib, v_mib, u_mib) in want.items():
        sh = dict(synth.CONFIGS[name])
        kw = dict(batch=sh["batch"], seq=sh["seq"], num_q_heads=sh["num_q_heads"], num_kv_heads=sh["num_kv_heads"],
                  head_dim=sh["head_dim"], rank=sh["rank"], score_rank=sh["score_rank"], top_k=sh["top_k"])
        b = traffic.stage_bytes(**kw)
        B, s = sh["batch"], sh["seq"]
        assert b["score"] == score_mib * MiB + B * s * 4          # + the fp32 scores written
        assert b["recon_attn"] == (lat_mib + u_mib + v_mib) * MiB
        assert abs(traffic.recon_flops(**kw) / 1e9 - 17.18) < 0.01
        # 4-bit values (R15): 128 * 4 / 8 code bytes + 4 (scale, zero) pairs per head-token
        vq = sh["num_kv_heads"] * (64 + 16)
        bq = traffic.stage_bytes(**kw, v_row_bytes=vq)
        assert bq["recon_attn"] == b["recon_attn"] - v_mib * MiB + B * min(sh["top_k"], s) * vq


# ------------------------------------------------------------------ calibration (Sec. 4.2, Lemma 1)
def test_calibrate_eigenpairs_and_ky_fan():
    """U_r from calibrate() satisfies C U = U diag(w_:r) (the eigen-equation, not a
    re-call of eigh), is column-orthonormal, and captures tr(U^T C U) = sum of the
    r largest eigenvalues -- the Ky Fan maximum, which no other orthonormal U beats."""
    rng = np.random.default_rng(3)
    N, D, r = 600, 24, 6
    K = rng.standard_normal((N, D)) * (0.7 ** np.arange(D))
    U, w = O.calibrate(K, r)
    C = K.T @ K
    np.testing.assert_allclose(C @ U, U * w[:r], atol=1e-8 * w[0])
    np.testing.assert_allclose(U.T @ U, np.eye(r), atol=1e-12)
    assert np.all(np.diff(w) <= 1e-12)
    E = O.captured_variance(U, K)
    np.testing.assert_allclose(E, w[:r].sum(), rtol=1e-12)
    for _ in range(20):
        Q, _ = np.linalg.qr(rng.standard_normal((D, r)))
        assert O.captured_variance(Q, K) <= E * (1 + 1e-12)
    # sign convention: the largest-magnitude component of every column is positive
    assert all(U[int(np.argmax(np.abs(U[:, j]))), j] > 0 for j in range(r))


def test_calibrate_recovers_a_planted_subspace():
    """Keys that live in an r-dimensional subspace are reconstructed exactly by
    U_r U_r^T (projection error 0: the discarded eigenvalues are 0)."""
    rng = np.random.default_rng(4)
    D, r = 20, 5
    B, _ = np.linalg.qr(rng.standard_normal((D, r)))
    K = rng.standard_normal((300, r)) @ B.T
    U, w = O.calibrate(K, r)
    np.testing.assert_allclose(K @ U @ U.T, K, atol=1e-10)
    assert np.all(np.abs(w[r:]) < 1e-9 * w[0])


def test_lemma1_joint_projection_captures_at_least_per_head():
    """Lemma 1: the best joint multi-head projection (rank r over nd)
    keeps at least the energy of the best per-head block-diagonal projection
    (rank r/n per head), for correlated heads strictly more."""
    rng = np.random.default_rng(5)
    n, d, r = 4, 8, 8
    base = rng.standard_normal((500, 3))
    K = np.concatenate([base @ rng.standard_normal((3, d)) + 0.1 * rng.standard_normal((500, d)) for _ in range(n)], 1)
    Uj, _ = O.calibrate(K, r)
    blocks = []
    for h in range(n):
        Uh, _ = O.calibrate(K[:, h * d:(h + 1) * d], r // n)
        blocks.append(Uh)
    Ub = np.zeros((n * d, r))
    for h in range(n):
        Ub[h * d:(h + 1) * d, h * (r // n):(h + 1) * (r // n)] = blocks[h]
    np.testing.assert_allclose(Ub.T @ Ub, np.eye(r), atol=1e-12)
    assert O.captured_variance(Uj, K) >= O.captured_variance(Ub, K) * (1 + 1e-3)


# ------------------------------------------------------------------ value quantisation (f1)
@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quantize_values_grid(bits):
    """Every group's min and max are on the grid (codes 0 and 2^b - 1 up to the bf16
    storage of zero / scale), every element is within half a step (+ the storage
    rounding) of its reconstruction, and values already on a representable grid
    round-trip exactly."""
    rng = np.random.default_rng(bits)
    v = rng.standard_normal((5, 3, 64))
    codes, scale, zero = O.quantize_values(v, bits, 32)
    qmax = (1 << bits) - 1
    assert codes.min() >= 0 and codes.max() <= qmax
    vh = O.dequantize_values(codes, scale, zero, 32)
    g = v.reshape(5, 3, 2, 32)
    step = scale[..., None]
    err = np.abs(vh.reshape(5, 3, 2, 32) - g)
    # half a step + the bf16 rounding of zero (<= 2^-9 |min|) and of scale (x qmax)
    bound = 0.5 * step + 2.0 ** -8 * (np.abs(g.min(-1))[..., None] + qmax * step) + 1e-12
    assert np.all(err <= bound)
    # exact grid: zero / scale representable in bf16, values = zero + scale * code
    c = rng.integers(0, qmax + 1, size=(4, 32))
    c[:, 0], c[:, 1] = 0, qmax
    vg = -1.5 + 0.125 * c
    codes2, s2, z2 = O.quantize_values(vg, bits, 32)
    np.testing.assert_array_equal(codes2, c)
    np.testing.assert_array_equal(O.dequantize_values(codes2, s2, z2, 32), vg)


def test_quantize_constant_group_and_bf16_round():
    """A constant group has scale 0 and code 0 and reconstructs to its value (bf16);
    bf16_round matches hand-computed roundings (ties to even)."""
    v = np.full((1, 32), 0.3)
    codes, scale, zero = O.quantize_values(v, 4, 32)
    assert scale[0, 0] == 0 and np.all(codes == 0)
    np.testing.assert_allclose(O.dequantize_values(codes, scale, zero, 32), O.bf16_round(v))
    # 1 + 2^-8 is a tie between 1 and 1 + 2^-7: ties to even -> 1; 1 + 3*2^-8 -> 1 + 2^-6
    np.testing.assert_array_equal(O.bf16_round(np.array([1 + 2.0 ** -8, 1 + 3 * 2.0 ** -8, -2.0])),
                                  [1.0, 1 + 2.0 ** -6, -2.0])


def test_quantize_rounding_rule_closed_form():
    """R15's code rule on hand-computed cases: hi - lo = 30 over 15 steps gives
    scale 2 exactly, so (v - zero) / scale lands on exact halves, which round to
    even (2.5 -> 2, 3.5 -> 4, 0.5 -> 0, 14.5 -> 14); values past the grid clamp."""
    v = np.zeros((1, 32))
    v[0, 0], v[0, 1] = 0.0, 30.0                                  # lo, hi
    v[0, 2:8] = [5.0, 7.0, 1.0, 29.0, 3.0, 13.0]                   # /2 = 2.5, 3.5, 0.5, 14.5, 1.5, 6.5
    codes, scale, zero = O.quantize_values(v, 4, 32)
    assert scale[0, 0] == 2.0 and zero[0, 0] == 0.0
    np.testing.assert_array_equal(codes[0, :8], [0, 15, 2, 4, 0, 14, 2, 6])
    # bf16 storage of the scale: (hi - lo) / 15 = 1/15 * 3 = 0.2 -> bf16 0.2001953125 (nearest even)
    w = np.zeros((1, 32)); w[0, 1] = 3.0
    c2, s2, _ = O.quantize_values(w, 4, 32)
    assert s2[0, 0] == 0.2001953125
    assert c2[0, 1] == 15                                         # 3 / 0.2001953125 = 14.985 -> 15


def test_value_hat_mixed_precision_worked_example():
    """Mixed-precision V^: one 32-channel group per row with values k/64,
    k in [0, 255], min 0 and max 255/64 in every row.  8-bit: scale (255/64)/255 = 1/64,
    so window rows (j >= s - z) reconstruct exactly; 4-bit: scale (255/64)/15 = 17/64
    (exact in bf16), so the other rows reconstruct to 17 * round(k/17) / 64 (k/17 is
    never a half, so no tie)."""
    rng = np.random.default_rng(3)
    s, z = 6, 2
    k = rng.integers(0, 256, size=(s, 32))
    k[:, 0], k[:, 31] = 0, 255
    v = k / 64.0
    vh = O.value_hat(v, 4, z, s)
    np.testing.assert_array_equal(vh[s - z:], v[s - z:])
    np.testing.assert_array_equal(vh[:s - z], 17.0 * np.floor(k[:s - z] / 17.0 + 0.5) / 64.0)
    # z = 0: every row 4-bit; z >= s: every row 8-bit (exact); bits = 16: the values
    np.testing.assert_array_equal(O.value_hat(v, 4, 0, s), 17.0 * np.floor(k / 17.0 + 0.5) / 64.0)
    np.testing.assert_array_equal(O.value_hat(v, 4, 99, s), v)
    np.testing.assert_array_equal(O.value_hat(v, 16, 2, s), v)


@pytest.mark.parametrize("bits", [2, 4])
def test_value_hat_error_bounds(bits):
    """Window rows are within half an 8-bit step of v, the others within half a
    b-bit step (+ the bf16 storage of the grid), on N(0,1) rows of bf16 values."""
    rng = np.random.default_rng(10 + bits)
    s, z, D = 40, 7, 128
    v = O.bf16_round(rng.standard_normal((s, D)))
    vh = O.value_hat(v, bits, z, s)
    g = v.reshape(s, D // 32, 32)
    rngw = (g.max(-1) - g.min(-1))[..., None]
    for rows, q in ((slice(s - z, s), 255), (slice(0, s - z), (1 << bits) - 1)):
        err = np.abs(vh.reshape(s, D // 32, 32)[rows] - g[rows])
        step = rngw[rows] / q
        assert np.all(err <= 0.5 * step * (1 + 2.0 ** -7) + q * step * 2.0 ** -8 + 1e-6)
