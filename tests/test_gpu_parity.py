"""GPU parity of the CUDA path (through the C ABI) against the fp64 oracle.

Small cases span several tiles / clusters and ragged tails; the paper-shaped
configs c2-c4 run at BASELINE.json's full sizes with the launch configuration
bench.py times (every output element is compared: the oracle is fast enough).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import sals_oracle as O
from tests import harness as H

pytestmark = pytest.mark.gpu

C = synth.CONFIGS


def _shape(name, **over):
    s = dict(C[name])
    s.update(over)
    return s


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2510_24273_b200 import build
    build.build()
    assert torch.cuda.is_available()


# ------------------------------------------------------------------ small / edge
def test_c1_tiny_fp32():
    r = H.full_check(_shape("c1"), 1, [256])
    assert r["swaps"] == 0


@pytest.mark.parametrize("path", [1, 0])
def test_mha_ragged_batch(path):
    sh = _shape("c2", num_q_heads=8, num_kv_heads=8, rank=256, score_rank=128, top_k=96)
    H.full_check(sh, 5, [1, 37, 96, 97, 1500], path=path, seed=11)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_gqa_groups(G):
    sh = _shape("c3", num_q_heads=4 * G, num_kv_heads=4, rank=256, score_rank=128, top_k=200)
    H.full_check(sh, 3, [700, 2049, 300], seed=12 + G)


def test_sink_recent_policy():
    sh = _shape("c2", num_q_heads=8, num_kv_heads=8, rank=128, score_rank=64, top_k=128)
    H.full_check(sh, 2, [3000, 129], sink=16, recent=32, seed=13)


def test_interleaved_rope_and_long_positions():
    sh = _shape("c4", num_q_heads=8, num_kv_heads=2, rank=128, score_rank=64, top_k=256)
    H.full_check(sh, 1, [70001], rope_style=1, seed=14)


@pytest.mark.parametrize("hd", [64, 256])
def test_head_dims(hd):
    sh = _shape("c2", num_q_heads=4, num_kv_heads=4, head_dim=hd, rank=128, score_rank=64, top_k=64)
    H.full_check(sh, 2, [500, 64], seed=15)


def test_single_token_returns_value():
    sh = _shape("c2", num_q_heads=4, num_kv_heads=4, rank=64, score_rank=32, top_k=16)
    cfg, host, gpu = H.run_sals(sh, 1, [1], seed=16)
    expect = host["v_new"][0]
    assert np.max(np.abs(gpu["out"][0] - expect)) <= 2 ** -8 * np.abs(expect).max()
    assert gpu["sel"][0][0] == 0 and np.all(gpu["sel"][0][1:] == -1)


def test_topk_ties_lower_index():
    """All-equal latent rows: every score ties, selection must be the first k tokens."""
    from paper_2510_24273_b200 import sals
    sh = _shape("c2", num_q_heads=4, num_kv_heads=4, rank=64, score_rank=32, top_k=40)
    cfg = sals.make_config(**sh)
    B, s = 2, 5000
    U = torch.from_numpy(synth.orthonormal(np.random.default_rng(0), 512, 64).astype(np.float32)).cuda().bfloat16()
    lat = torch.ones(B, s, 64, dtype=torch.bfloat16, device="cuda")
    v = torch.randn(B, s, 512, device="cuda").bfloat16()
    q = torch.randn(B, 512, device="cuda").bfloat16()
    seq = torch.tensor([s, 3000], dtype=torch.int32, device="cuda")
    ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s), "cuda")
    out = torch.empty(B, 512, dtype=torch.bfloat16, device="cuda")
    sel = torch.empty(B, 40, dtype=torch.int32, device="cuda")
    sals.sals_decode(cfg, U, q, lat, v, seq, s, out, ws, sel_idx_out=sel)
    assert sel.cpu().numpy().tolist() == [list(range(40))] * 2


@pytest.mark.parametrize("s,npat,sink,recent,k", [
    (5000, 7, 0, 0, 512),        # few distinct scores: threshold bin > survivor limit -> radix passes
    (5000, 1000, 4, 64, 512),    # many distinct values: survivor select
    (40000, 3, 0, 0, 4096),      # > candidate capacity: cluster-wide overflow passes
    (131072, 2, 16, 128, 16384), # c4 geometry, two score values
    (70001, 50000, 8, 32, 4096), # ragged, mostly distinct
])
def test_topk_exact_on_kernel_scores(s, npat, sink, recent, k):
    """Selection is bit-exact given the scores: compare the kernel's C with the
    oracle's select_topk (R3-R5) applied to the kernel's own p' (scores_out).
    Latent rows are drawn from npat patterns so equal scores are frequent."""
    from paper_2510_24273_b200 import sals
    sh = _shape("c2", num_q_heads=4, num_kv_heads=4, rank=64, score_rank=32, top_k=k)
    sh.update(sink=sink, recent=recent)
    cfg = sals.make_config(**sh)
    B = 2
    g = torch.Generator(device="cuda"); g.manual_seed(7 + s + npat)
    U = torch.from_numpy(synth.orthonormal(np.random.default_rng(1), 512, 64).astype(np.float32)).cuda().bfloat16()
    pats = torch.randn(npat, 64, device="cuda", generator=g).bfloat16()
    which = torch.randint(0, npat, (B, s), device="cuda", generator=g)
    lat = pats[which].contiguous()
    v = torch.randn(B, s, 512, device="cuda", generator=g).bfloat16()
    q = torch.randn(B, 512, device="cuda", generator=g).bfloat16()
    seq = torch.tensor([s, s - s // 3], dtype=torch.int32, device="cuda")
    ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s), "cuda")
    out = torch.empty(B, 512, dtype=torch.bfloat16, device="cuda")
    sel = torch.empty(B, k, dtype=torch.int32, device="cuda")
    scores = torch.empty(B, s, dtype=torch.float32, device="cuda")
    sals.sals_decode(cfg, U, q, lat, v, seq, s, out, ws, sel_idx_out=sel, scores_out=scores)
    torch.cuda.synchronize()
    sc = scores.cpu().numpy()
    got = sel.cpu().numpy()
    for b in range(B):
        sb = int(seq[b])
        want = O.select_topk(sc[b, :sb].astype(np.float64), k, sink=sink, recent=recent)
        n = len(want)
        assert np.array_equal(got[b, :n], want), f"request {b}"
        assert (got[b, n:] == -1).all()


@pytest.mark.parametrize("s,k,sink,recent", [(4096, 512, 0, 0), (5000, 512, 4, 64), (8000, 1000, 16, 128)])
def test_topk_threshold_bin_fully_taken(s, k, sink, recent):
    """Exactly k - x - z ranked tokens share the top score (the rest share a lower one),
    so the top-digit threshold bin is taken whole and the single-CTA top-k stops its radix
    passes early (topk_cta.cu): the selection must still equal the oracle's select_topk on
    the kernel's own scores."""
    from paper_2510_24273_b200 import sals
    sh = _shape("c2", num_q_heads=4, num_kv_heads=4, rank=64, score_rank=32, top_k=k)
    sh.update(sink=sink, recent=recent)
    cfg = sals.make_config(**sh)
    B = 2
    g = torch.Generator(device="cuda"); g.manual_seed(99 + s)
    U = torch.from_numpy(synth.orthonormal(np.random.default_rng(2), 512, 64).astype(np.float32)).cuda().bfloat16()
    q = torch.randn(B, 512, device="cuda", generator=g).bfloat16()
    qt = (q.float() @ U.float())[:, :32]                      # the latent query direction (r* columns)
    hi = (qt / qt.norm(dim=1, keepdim=True)).repeat(1, 2)     # [B, 64]: large positive score
    lat = torch.empty(B, s, 64, device="cuda")
    rng = np.random.default_rng(s)
    for b in range(B):
        lat[b] = -0.5 * hi[b]
        ranked = np.arange(sink, s - recent)
        pick = rng.choice(ranked, size=k - sink - recent, replace=False)
        lat[b, torch.from_numpy(pick).cuda()] = 2.0 * hi[b]
    lat = lat.bfloat16()
    v = torch.randn(B, s, 512, device="cuda", generator=g).bfloat16()
    seq = torch.tensor([s, s], dtype=torch.int32, device="cuda")
    ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s), "cuda")
    out = torch.empty(B, 512, dtype=torch.bfloat16, device="cuda")
    sel = torch.empty(B, k, dtype=torch.int32, device="cuda")
    scores = torch.empty(B, s, dtype=torch.float32, device="cuda")
    sals.sals_decode(cfg, U, q, lat, v, seq, s, out, ws, sel_idx_out=sel, scores_out=scores)
    torch.cuda.synchronize()
    sc = scores.cpu().numpy()
    got = sel.cpu().numpy()
    for b in range(B):
        want = O.select_topk(sc[b].astype(np.float64), k, sink=sink, recent=recent)
        assert np.array_equal(got[b, :len(want)], want), f"request {b}"


def test_graph_capture_replay_is_deterministic():
    from paper_2510_24273_b200 import sals
    sh = _shape("c3", rank=256, score_rank=128, top_k=512)
    cfg = sals.make_config(**sh)
    B, s = 2, 4000
    p = synth.gen_problem(num_q_heads=32, num_kv_heads=8, head_dim=128, rank=256, batch=B, seq_lens=[s, s], seed=3)
    dev = lambda a: torch.from_numpy(a).cuda().bfloat16()
    U, lat, v, q = dev(p["U"]), dev(p["latent"]), dev(p["v"]), dev(p["q"])
    seq = torch.tensor([s, s], dtype=torch.int32, device="cuda")
    ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s), "cuda")
    out = torch.empty(B, 32 * 128, dtype=torch.bfloat16, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        sals.sals_decode(cfg, U, q, lat, v, seq, s, out, ws)
        st.synchronize()
        ref = out.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            sals.sals_decode(cfg, U, q, lat, v, seq, s, out, ws)
        for _ in range(3):
            out.zero_()
            g.replay()
        st.synchronize()
    assert torch.equal(out, ref)


# ------------------------------------------------------------------ full sizes
@pytest.mark.parametrize("fused", [False, True], ids=["two_calls", "append_decode"])
@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_full_size_configs(name, fused):
    """c2-c4 at BASELINE.json's full sizes, every output element against the oracle;
    ``append_decode`` is the exact call bench.py times (sals_append_decode, bf16 V)."""
    sh = _shape(name)
    s = sh["seq"]
    B = sh["batch"]
    r = H.full_check(sh, B, [s] * B, seed=synth.SEED_BASE + int(name[1]) + (100 if fused else 0), fused=fused)
    print(name, fused, r)


@pytest.mark.parametrize("B,n", [(1, 4096), (16, 4096), (64, 4096), (1, 32768), (16, 32768), (64, 32768)])
def test_c5_grid_points(B, n):
    """c5 (LLaMA2-7B-shaped MHA 32/32 x 128, r 512, r* 256, k = n/8; BASELINE configs[4],
    the batched-decode shapes of Table 7 P:705-711 at sparsity 1/8 P:692): one layer in
    the bench's launch configuration (device-drawn inputs, sals_append_decode); append
    rows of every request and sampled requests (first, middle, last: the projection's
    batch passes and the last chunk) element by element against the oracle."""
    sh = _shape("c5", batch=B, seq=n, top_k=n // 8)
    sample = sorted({0, B // 2, B - 1})
    stats = H.sampled_check(sh, B, n, sample=sample, seed=synth.SEED_BASE + 5000 + B + n)
    print(B, n, stats)


@pytest.mark.parametrize("B,seqs", [(4, [4096, 100, 2000, 1]), (8, [4096, 4000, 1, 1, 700, 4096, 129, 3000])])
def test_ragged_requests_c2_heads(B, seqs):
    """MHA at c2's head shape (D = 4096, one chunk per request in the fused kernel)
    with very different selection counts per request (1 to 4 tiles, one-token
    requests), every output element against the oracle."""
    sh = _shape("c2")
    H.full_check(sh, B, seqs, seed=61 + B)


def test_full_size_ragged_c3():
    sh = _shape("c3")
    H.full_check(sh, 4, [32768, 17, 4096, 30001], seed=21)


# ------------------------------------------------------------------ dense comparator
@pytest.mark.parametrize("dtype,G", [("bf16", 1), ("bf16", 4), ("f32", 2)])
def test_dense_decode(dtype, G):
    """Dense flash decode over a post-RoPE cache (cache rows written by the oracle's
    dense append and rounded to the storage dtype) vs the oracle's dense decode."""
    from paper_2510_24273_b200 import sals
    nkv, d = 4, (128 if dtype == "bf16" else 64)
    sh = dict(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=64, score_rank=32, top_k=64,
              rope_base=5e5, dtype=dtype)
    cfg = sals.make_config(**sh)
    oc = O.Config(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=64, score_rank=32, top_k=64, rope_base=5e5)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rng = np.random.default_rng(5)
    B, cap = 3, 3000
    seq_lens = np.array([3000, 1, 1777], dtype=np.int32)
    D = nkv * d
    K = rng.standard_normal((B, cap, D))
    kc_ref = np.stack([O.dense_append_key(oc, K[b], np.arange(cap)) for b in range(B)])
    kc = torch.from_numpy(kc_ref.astype(np.float32)).cuda().to(tdt)
    vc = torch.from_numpy(rng.standard_normal((B, cap, D)).astype(np.float32)).cuda().to(tdt)
    qt = torch.from_numpy(rng.standard_normal((B, nkv * G * d)).astype(np.float32)).cuda().to(tdt)
    seq = torch.from_numpy(seq_lens).cuda()
    ws = sals.alloc_workspace(sals.sals_dense_workspace_bytes(cfg, B, cap), "cuda")
    out = torch.empty(B, nkv * G * d, dtype=tdt, device="cuda")
    sals.sals_dense_decode(cfg, qt, kc, vc, seq, cap, out, ws)
    torch.cuda.synchronize()
    y = O.dense_decode(oc, H.widen(qt), H.widen(kc), H.widen(vc), seq_lens)
    H.check_output(H.widen(out), y, dtype)


@pytest.mark.parametrize("nkv,G,B,cap,lens", [
    (8, 4, 4, 3000, [3000, 1, 1777, 9]),        # D = 1024 (c3 / c4 heads): TMA kernel, 8 tokens per stage
    (8, 2, 3, 2051, [2051, 2, 1000]),
    (8, 8, 2, 999, [999, 31]),                  # G = 8: flash_decode_kernel
    (8, 1, 2, 40000, [40000, 33333]),           # long rows: many stages per CTA
    (32, 1, 3, 1025, [1025, 1, 513]),           # D = 4096 (c2 heads): flash_decode_kernel
])
def test_dense_decode_full_shapes(nkv, G, B, cap, lens):
    """The dense comparator at the paper's head shapes (dense_tma.cu for 8 KV heads,
    flash_decode_kernel otherwise) vs the oracle's dense decode, ragged lengths
    (partial stages, one-token requests, empty splits)."""
    from paper_2510_24273_b200 import sals
    d = 128
    sh = dict(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=64, score_rank=32, top_k=64, rope_base=1e4)
    cfg = sals.make_config(**sh)
    oc = O.Config(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=64, score_rank=32, top_k=64, rope_base=1e4)
    rng = np.random.default_rng(50 + nkv + G)
    seq_lens = np.array(lens, dtype=np.int32)
    D = nkv * d
    kc = torch.from_numpy(rng.standard_normal((B, cap, D)).astype(np.float32)).cuda().bfloat16()
    vc = torch.from_numpy(rng.standard_normal((B, cap, D)).astype(np.float32)).cuda().bfloat16()
    qt = torch.from_numpy((2.0 * rng.standard_normal((B, nkv * G * d))).astype(np.float32)).cuda().bfloat16()
    seq = torch.from_numpy(seq_lens).cuda()
    ws = sals.alloc_workspace(sals.sals_dense_workspace_bytes(cfg, B, cap), "cuda")
    out = torch.empty(B, nkv * G * d, dtype=torch.bfloat16, device="cuda")
    sals.sals_dense_decode(cfg, qt, kc, vc, seq, cap, out, ws)
    torch.cuda.synchronize()
    y = O.dense_decode(oc, H.widen(qt), H.widen(kc), H.widen(vc), seq_lens)
    H.check_output(H.widen(out), y, "bf16")


def test_dense_append_positions():
    from paper_2510_24273_b200 import sals
    sh = dict(num_q_heads=8, num_kv_heads=2, head_dim=128, rank=64, score_rank=32, top_k=64, rope_base=5e5)
    cfg = sals.make_config(**sh)
    rng = np.random.default_rng(6)
    B, cap = 4, 140000
    pos = np.array([0, 1, 70000, 131071], dtype=np.int32)
    k = torch.from_numpy(rng.standard_normal((B, 256)).astype(np.float32)).cuda().bfloat16()
    v = torch.from_numpy(rng.standard_normal((B, 256)).astype(np.float32)).cuda().bfloat16()
    kc = torch.zeros(B, cap, 256, dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    sals.sals_dense_append(cfg, k, v, torch.from_numpy(pos).cuda(), kc, vc)
    oc = O.Config(num_q_heads=8, num_kv_heads=2, head_dim=128, rank=64, score_rank=32, top_k=64, rope_base=5e5)
    ref = O.dense_append_key(oc, H.widen(k), pos)
    got = np.stack([H.widen(kc[b, pos[b]]) for b in range(B)])
    ulp = 2.0 ** (np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
    assert np.all(np.abs(got - ref) <= ulp + 1e-5)


# ------------------------------------------------------------------ sharded (virtual ranks)
@pytest.mark.parametrize("P,sink,recent", [(2, 0, 0), (4, 16, 64), (3, 0, 8)])
def test_sharded_virtual_ranks_equal_unsharded(P, sink, recent):
    from paper_2510_24273_b200 import sals
    sh = _shape("c4", rank=256, score_rank=128, top_k=1024)
    B, s = 2, 20000
    cfg, host, gpu = H.run_sals(sh, B, [s, s - 3333], sink=sink, recent=recent, seed=31)
    oc = H.oracle_cfg(sh, sink, recent)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()
    U, q = dev(host["U"]), dev(host["q"])
    seq = torch.from_numpy(host["seq_len"]).cuda()
    k = sh["top_k"]
    bounds = np.linspace(0, s, P + 1).astype(int)
    cands_s, cands_i, wss, shards = [], [], [], []
    for p in range(P):
        a, b_ = bounds[p], bounds[p + 1]
        lat = dev(host["latent"][:, a:b_])
        vv = dev(host["v"][:, a:b_])
        loc = np.clip(host["seq_len"] - a, 0, b_ - a).astype(np.int32)
        locd = torch.from_numpy(loc).cuda()
        ws = sals.alloc_workspace(sals.sals_shard_workspace_bytes(cfg, B, b_ - a, P), "cuda")
        cs = torch.empty(B, k, dtype=torch.float32, device="cuda")
        ci = torch.empty(B, k, dtype=torch.int32, device="cuda")
        sals.sals_shard_candidates(cfg, U, q, lat, int(a), locd, b_ - a, seq, cs, ci, ws)
        cands_s.append(cs); cands_i.append(ci); wss.append(ws); shards.append((a, b_, lat, vv, locd))
    all_s = torch.stack(cands_s).contiguous()    # the scores-only exchange
    parts = []
    for p in range(P):
        a, b_, lat, vv, locd = shards[p]
        part = torch.empty(B, sh["num_q_heads"], sh["head_dim"] + 2, dtype=torch.float32, device="cuda")
        sals.sals_shard_attend(cfg, U, q, lat, vv, int(a), locd, b_ - a, seq, all_s, cands_i[p], P, p, part, wss[p])
        parts.append(part)
    out = torch.empty(B, sh["num_q_heads"] * sh["head_dim"], dtype=torch.bfloat16, device="cuda")
    sals.sals_merge_partials(cfg, torch.stack(parts).contiguous(), P, B, out)
    torch.cuda.synchronize()
    # same selection as the unsharded GPU decode => output equal up to fp32 merge order
    forced = [gpu["sel"][b][gpu["sel"][b] >= 0].astype(np.int64) for b in range(B)]
    orc = O.decode(oc, host["U"], host["q"], host["latent"], host["v"], host["seq_len"], forced_selection=forced)
    H.check_output(H.widen(out), orc["y"], "bf16")
    assert np.max(np.abs(H.widen(out) - gpu["out"])) <= 2 ** -6


@pytest.mark.parametrize("P,sink,recent", [(2, 0, 0), (4, 0, 0), (3, 8, 16)])
def test_sharded_select_cross_shard_ties(P, sink, recent):
    """Shards holding IDENTICAL latent / value rows, so every score appears P times, bitwise
    (the per-token reduction order is shard-invariant): the scores-only exchange must split the
    ties at the (k-x-z)-th score between the ranks exactly as the unsharded top-k does (lower
    global index first, R5).  Checked: the union of the owned selections against the unsharded
    GPU selection index by index, and the merged output against the oracle forced to it."""
    from paper_2510_24273_b200 import sals
    sh = _shape("c4", rank=256, score_rank=128, top_k=1024)
    n1, B = 1500, 1
    s = P * n1
    pr = synth.gen_problem(num_q_heads=sh["num_q_heads"], num_kv_heads=sh["num_kv_heads"], head_dim=sh["head_dim"],
                           rank=sh["rank"], batch=B, seq_lens=[n1], cap=n1, seed=43)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()
    U, q = dev(pr["U"]), dev(pr["q"])
    lat = dev(np.concatenate([pr["latent"]] * P, axis=1))
    vv = dev(np.concatenate([pr["v"]] * P, axis=1))
    cfg = sals.make_config(**sh, sink=sink, recent=recent)
    seq = torch.full((B,), s, dtype=torch.int32, device="cuda")
    k = sh["top_k"]
    ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s), "cuda")
    ref_out = torch.empty(B, sh["num_q_heads"] * sh["head_dim"], dtype=torch.bfloat16, device="cuda")
    ref_sel = torch.full((B, k), -7, dtype=torch.int32, device="cuda")
    sals.sals_decode(cfg, U, q, lat, vv, seq, s, ref_out, ws, sel_idx_out=ref_sel)
    cands_s, cands_i, wss = [], [], []
    for p in range(P):
        a = p * n1
        locd = torch.full((B,), n1, dtype=torch.int32, device="cuda")
        w = sals.alloc_workspace(sals.sals_shard_workspace_bytes(cfg, B, n1, P), "cuda")
        cs = torch.empty(B, k, dtype=torch.float32, device="cuda")
        ci = torch.empty(B, k, dtype=torch.int32, device="cuda")
        sals.sals_shard_candidates(cfg, U, q, lat[:, a:a + n1].contiguous(), a, locd, n1, seq, cs, ci, w)
        cands_s.append(cs); cands_i.append(ci); wss.append(w)
    all_s = torch.stack(cands_s).contiguous()
    owned, parts = [], []
    for p in range(P):
        a = p * n1
        locd = torch.full((B,), n1, dtype=torch.int32, device="cuda")
        part = torch.empty(B, sh["num_q_heads"], sh["head_dim"] + 2, dtype=torch.float32, device="cuda")
        sals.sals_shard_attend(cfg, U, q, lat[:, a:a + n1].contiguous(), vv[:, a:a + n1].contiguous(), a, locd, n1,
                               seq, all_s, cands_i[p], P, p, part, wss[p])
        torch.cuda.synchronize()
        parts.append(part)
        own, cnt = sals.shard_owned_list(cfg, wss[p], B, n1)   # (debug view of the workspace)
        owned.append(own[0, :cnt[0]].astype(np.int64) + a)
    out = torch.empty_like(ref_out)
    sals.sals_merge_partials(cfg, torch.stack(parts).contiguous(), P, B, out)
    torch.cuda.synchronize()
    gsel = ref_sel[0].cpu().numpy()
    gsel = gsel[gsel >= 0].astype(np.int64)
    np.testing.assert_array_equal(np.concatenate(owned), gsel)
    assert np.max(np.abs(H.widen(out) - H.widen(ref_out))) <= 2 ** -6
    oc = H.oracle_cfg(sh, sink, recent)
    full_lat = np.concatenate([pr["latent"]] * P, axis=1)
    full_v = np.concatenate([pr["v"]] * P, axis=1)
    orc = O.decode(oc, H.widen(U), H.widen(q), H.widen(dev(full_lat)), H.widen(dev(full_v)), np.array([s]),
                   forced_selection=[gsel])
    H.check_output(H.widen(out), orc["y"], "bf16")


@pytest.mark.parametrize("sink,recent", [(0, 0), (16, 64)])
def test_decode_sharded_nccl_one_rank(sink, recent):
    """sals_decode_sharded (phases + in-place NCCL all-gathers inside the library)
    on a one-rank communicator: the selection of the unsharded decode, the output
    against the oracle forced to it, and equal to the unsharded output up to the
    fp32 merge order; also graph-capturable."""
    from paper_2510_24273_b200 import sals
    sh = _shape("c4", rank=256, score_rank=128, top_k=1024)
    B, s = 2, 20000
    cfg, host, gpu = H.run_sals(sh, B, [s, s - 3333], sink=sink, recent=recent, seed=37)
    oc = H.oracle_cfg(sh, sink, recent)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()
    U, q, lat, vv = dev(host["U"]), dev(host["q"]), dev(host["latent"]), dev(host["v"])
    seq = torch.from_numpy(host["seq_len"]).cuda()
    comm = sals.sals_comm_init(sals.sals_comm_unique_id(), 1, 0)
    try:
        ws = sals.alloc_workspace(sals.sals_decode_sharded_workspace_bytes(cfg, B, s, 1), "cuda")
        out = torch.empty(B, sh["num_q_heads"] * sh["head_dim"], dtype=torch.bfloat16, device="cuda")
        sals.sals_decode_sharded(cfg, comm, U, q, lat, vv, 0, seq, s, seq, out, ws)
        torch.cuda.synchronize()
        forced = [gpu["sel"][b][gpu["sel"][b] >= 0].astype(np.int64) for b in range(B)]
        orc = O.decode(oc, host["U"], host["q"], host["latent"], host["v"], host["seq_len"], forced_selection=forced)
        H.check_output(H.widen(out), orc["y"], "bf16")
        assert np.max(np.abs(H.widen(out) - gpu["out"])) <= 2 ** -6
        first = out.clone()
        st = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            with torch.cuda.graph(g, stream=st):
                sals.sals_decode_sharded(cfg, comm, U, q, lat, vv, 0, seq, s, seq, out, ws, stream=st)
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, first)
    finally:
        sals.sals_comm_destroy(comm)


def test_append_decode_sharded_one_rank():
    """sals_append_decode_sharded on a one-rank communicator: the appended latent row
    (U^T k_new, 1 bf16 ulp) and value row (bit-exact) against the oracle, the output
    against the oracle forced to the selection of the unsharded fused call on the same
    problem; a shard that does not hold position s - 1 writes nothing."""
    from paper_2510_24273_b200 import sals
    sh = _shape("c4", rank=256, score_rank=128, top_k=1024)
    B, s = 2, 20000
    seqs = [s, s - 3333]
    cfg, host, gpu = H.run_sals(sh, B, seqs, seed=41, fused=True)
    oc = H.oracle_cfg(sh, 0, 0)
    p = synth.gen_problem(num_q_heads=sh["num_q_heads"], num_kv_heads=sh["num_kv_heads"], head_dim=sh["head_dim"],
                          rank=sh["rank"], batch=B, seq_lens=seqs, cap=s, seed=41)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()
    U, q, kn, vn = dev(p["U"]), dev(p["q"]), dev(p["k_new"]), dev(p["v_new"])
    lat, vv = dev(p["latent"]), dev(p["v"])
    seq = torch.tensor(seqs, dtype=torch.int32, device="cuda")
    comm = sals.sals_comm_init(sals.sals_comm_unique_id(), 1, 0)
    try:
        ws = sals.alloc_workspace(sals.sals_decode_sharded_workspace_bytes(cfg, B, s, 1), "cuda")
        out = torch.empty(B, sh["num_q_heads"] * sh["head_dim"], dtype=torch.bfloat16, device="cuda")
        sals.sals_append_decode_sharded(cfg, comm, U, kn, vn, q, lat, vv, 0, seq, s, seq, out, ws)
        torch.cuda.synchronize()
        hl, hv = H.widen(lat), H.widen(vv)
        H.check_append(dict(U=H.widen(U), k_new=H.widen(kn), v_new=H.widen(vn), latent=hl, v=hv,
                            seq_len=np.asarray(seqs)), "bf16")
        forced = [gpu["sel"][b][gpu["sel"][b] >= 0].astype(np.int64) for b in range(B)]
        orc = O.decode(oc, H.widen(U), H.widen(q), hl, hv, np.asarray(seqs), forced_selection=forced)
        H.check_output(H.widen(out), orc["y"], "bf16")
        # a shard holding positions [0, s_b - 100) is not the newest token's owner: no write
        lat2, v2 = dev(p["latent"]), dev(p["v"])
        loc = (seq - 100).to(torch.int32)
        sals.sals_append_decode_sharded(cfg, comm, U, kn, vn, q, lat2, v2, 0, loc, s, seq, out, ws)
        torch.cuda.synchronize()
        assert torch.equal(lat2, dev(p["latent"])) and torch.equal(v2, dev(p["v"]))
    finally:
        sals.sals_comm_destroy(comm)


# ------------------------------------------------------------------ fused append + decode
@pytest.mark.parametrize("nkv,G,d,B,seqs", [(8, 4, 128, 3, [3000, 1777, 2048]),   # D = 1024
                                          (32, 1, 128, 2, [4096, 2500])])         # D = 4096
def test_append_decode_against_oracle(nkv, G, d, B, seqs):
    """sals_append_decode (append + decode in one call) against the oracle, and its
    cache rows identical to sals_append_latent's (the append writes the same rows
    whichever call does it; the output is checked against the oracle, never against
    the other GPU call)."""
    from paper_2510_24273_b200 import sals
    sh = dict(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=256, score_rank=128, top_k=384,
              rope_base=1e6, dtype="bf16")
    H.full_check(sh, B, seqs, seed=11, fused=True)
    cfg = sals.make_config(**sh)
    p = synth.gen_problem(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=256, batch=B, seq_lens=seqs, seed=11)
    dev = lambda a: torch.from_numpy(a).cuda().bfloat16()
    U, q, kn, vn = dev(p["U"]), dev(p["q"]), dev(p["k_new"]), dev(p["v_new"])
    lat1, v1 = dev(p["latent"]), dev(p["v"])
    lat2, v2 = lat1.clone(), v1.clone()
    s_max = max(seqs)
    seq = torch.tensor(seqs, dtype=torch.int32, device="cuda")
    ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s_max), "cuda")
    o2 = torch.empty(B, nkv * G * d, dtype=torch.bfloat16, device="cuda")
    sals.sals_append_latent(cfg, U, kn, vn, (seq - 1).to(torch.int32), lat1, v1)
    sals.sals_append_decode(cfg, U, kn, vn, q, lat2, v2, seq, s_max, o2, ws)
    torch.cuda.synchronize()
    assert torch.equal(lat1, lat2) and torch.equal(v1, v2)


# ------------------------------------------------------------------ prefill (bulk append)
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_append_latent_bulk(dtype):
    """Prefill rows [start, start + n) == U^T k (fp64 oracle, one rounding of the stored
    type), value rows copied; rows outside the block untouched; a decode after a bulk
    prefill equals the oracle as usual."""
    from paper_2510_24273_b200 import sals
    nkv, G, d, r, B, n, start, cap = 4, 2, 64, 128, 3, 300, 17, 400
    sh = dict(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=r, score_rank=64, top_k=96, rope_base=1e4,
              dtype=dtype)
    cfg = sals.make_config(**sh)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rng = np.random.default_rng(5)
    D = nkv * d
    U = torch.from_numpy(synth.orthonormal(rng, D, r)).cuda().to(tdt)
    k = torch.from_numpy(rng.normal(size=(B, n, D))).cuda().to(tdt)
    v = torch.from_numpy(rng.normal(size=(B, n, D))).cuda().to(tdt)
    lat = torch.full((B, cap, r), 7.0, dtype=tdt, device="cuda")
    vc = torch.full((B, cap, D), 7.0, dtype=tdt, device="cuda")
    sals.sals_append_latent_bulk(cfg, U, k, v, start, lat, vc)
    torch.cuda.synchronize()
    ref = O.project_latent(H.widen(U), H.widen(k).reshape(B * n, D)).reshape(B, n, r)
    got = H.widen(lat[:, start:start + n])
    tol = (2.0 ** -7 if dtype == "bf16" else 1e-5) * np.abs(ref) + 1e-3 * (1 if dtype == "bf16" else 1e-2)
    assert np.all(np.abs(got - ref) <= tol), np.max(np.abs(got - ref))
    assert torch.equal(vc[:, start:start + n], v)
    assert bool((lat[:, :start] == 7.0).all()) and bool((lat[:, start + n:] == 7.0).all())
    assert bool((vc[:, :start] == 7.0).all()) and bool((vc[:, start + n:] == 7.0).all())


@pytest.mark.parametrize("nkv,r,B,n,start", [(32, 512, 2, 1000, 3000), (8, 512, 1, 4096, 0), (8, 256, 3, 77, 5)])
def test_append_latent_bulk_tcgen05(nkv, r, B, n, start):
    """The tcgen05 bulk-append GEMM (prefill_tc.cu) at model sizes (D = 4096 / 1024, r = 512,
    ragged n): latent rows == U^T k (fp64 oracle, one bf16 rounding + fp32-accumulation
    allowance), rows outside the block untouched."""
    from paper_2510_24273_b200 import sals
    d = 128
    D = nkv * d
    sh = dict(num_q_heads=nkv, num_kv_heads=nkv, head_dim=d, rank=r, score_rank=r // 2, top_k=128, rope_base=1e4,
              dtype="bf16")
    cfg = sals.make_config(**sh)
    rng = np.random.default_rng(11)
    cap = start + n + 50
    U = torch.from_numpy(synth.orthonormal(rng, D, r)).cuda().bfloat16()
    k = torch.from_numpy(rng.normal(size=(B, n, D))).cuda().bfloat16()
    v = torch.from_numpy(rng.normal(size=(B, n, D))).cuda().bfloat16()
    lat = torch.full((B, cap, r), 7.0, dtype=torch.bfloat16, device="cuda")
    vc = torch.full((B, cap, D), 7.0, dtype=torch.bfloat16, device="cuda")
    sals.sals_launch_count(reset=True)
    sals.sals_append_latent_bulk(cfg, U, k, v, start, lat, vc)
    torch.cuda.synchronize()
    assert sals.sals_launch_count(reset=True) >= 1          # the in-build kernel ran (no cuBLAS fallback)
    ref = O.project_latent(H.widen(U), H.widen(k).reshape(B * n, D)).reshape(B, n, r)
    got = H.widen(lat[:, start:start + n])
    tol = 2.0 ** -7 * np.abs(ref) + 2e-3
    assert np.all(np.abs(got - ref) <= tol), np.max(np.abs(got - ref) - tol)
    assert torch.equal(vc[:, start:start + n], v)
    assert bool((lat[:, :start] == 7.0).all()) and bool((lat[:, start + n:] == 7.0).all())


@pytest.mark.parametrize("bits,z", [(4, 0), (2, 0), (4, 64), (2, 100)])
def test_append_latent_bulk_quantized(bits, z):
    """Bulk prefill of a quantised value cache: every row of the block BYTE-identical to
    the oracle's quantiser (R15), the 8-bit recent-window ring holding the last z tokens of
    the block at slot pos % z, rows outside the block untouched."""
    from paper_2510_24273_b200 import sals
    nkv, d, r, B, n, start = 8, 128, 256, 2, 700, 40
    D = nkv * d
    sh = dict(num_q_heads=nkv * 4, num_kv_heads=nkv, head_dim=d, rank=r, score_rank=128, top_k=256, rope_base=1e6,
              dtype="bf16")
    cfg = sals.make_config(**sh, v_bits=bits, recent=z)
    rng = np.random.default_rng(13)
    cap = start + n + 9
    U = torch.from_numpy(synth.orthonormal(rng, D, r)).cuda().bfloat16()
    k = torch.from_numpy(rng.normal(size=(B, n, D))).cuda().bfloat16()
    v = torch.from_numpy(rng.normal(size=(B, n, D))).cuda().bfloat16()
    lat = torch.zeros(B, cap, r, dtype=torch.bfloat16, device="cuda")
    rb = sals.sals_v_row_bytes(cfg)
    total = sals.sals_v_cache_bytes(cfg, B, cap)
    vq = torch.full((total,), 0xA5, dtype=torch.uint8, device="cuda")
    sals.sals_append_latent_bulk(cfg, U, k, v, start, lat, vq)
    torch.cuda.synchronize()
    rows = vq[:B * cap * rb].view(B, cap, rb).cpu().numpy()
    vh = H.widen(v)
    np.testing.assert_array_equal(rows[:, start:start + n], _pack_values(vh, bits, nkv))
    assert (rows[:, :start] == 0xA5).all() and (rows[:, start + n:] == 0xA5).all()
    if z:
        ring = vq[B * cap * rb:].view(B, z, nkv * 144).cpu().numpy()
        for b in range(B):
            for t in range(n - z, n):
                pos = start + t
                np.testing.assert_array_equal(ring[b, pos % z], _pack8(vh[b, t][None], nkv)[0])


# ------------------------------------------------------------------ calibration
def test_calibrate_matches_oracle():
    """sals_calibrate (cuBLAS Gram + cuSOLVER syevd, fp32) == oracle calibrate (fp64
    eigh) on keys with a decaying spectrum: same eigenvalues (fp32-relative) and the
    same signed leading eigenvectors (well separated eigenvalues)."""
    from paper_2510_24273_b200 import sals
    rng = np.random.default_rng(6)
    N, nkv, d, r = 4096, 2, 64, 32
    D = nkv * d
    K = rng.standard_normal((N, D)) * (0.93 ** np.arange(D))[None]
    cfg = sals.make_config(num_q_heads=nkv, num_kv_heads=nkv, head_dim=d, rank=r, score_rank=16, top_k=8,
                           dtype="f32")
    Kd = torch.from_numpy(K).float().cuda()
    U = torch.empty(D, r, dtype=torch.float32, device="cuda")
    w = torch.empty(D, dtype=torch.float32, device="cuda")
    sals.sals_calibrate(cfg, Kd, U, w)
    torch.cuda.synchronize()
    Uo, wo = O.calibrate(H.widen(Kd), r)
    np.testing.assert_allclose(H.widen(w), wo, rtol=2e-4, atol=1e-3 * wo[0] * 1e-3)
    np.testing.assert_allclose(H.widen(U), Uo, atol=2e-3)


# ------------------------------------------------------------------ quantised value cache (f1)
def _pack_values(v, bits, nkv):
    """The library's quantised row format (include/sals.h, cfg.v_bits), written with the
    oracle's quantiser: per KV head 128*bits/8 code bytes (low bits first) + 4 x (bf16
    scale, bf16 zero)."""
    codes, scale, zero = O.quantize_values(v, bits, 32)          # [..., D], [..., D/32]
    lead = v.shape[:-1]
    per = 8 // bits
    c = codes.reshape(*lead, nkv, 128 // per, per)
    packed = np.zeros((*lead, nkv, 128 // per), dtype=np.uint8)
    for e in range(per):
        packed |= (c[..., e] << (e * bits)).astype(np.uint8)
    sb = torch.from_numpy(scale.astype(np.float32)).bfloat16().view(torch.int16).numpy().view(np.uint16)
    zb = torch.from_numpy(zero.astype(np.float32)).bfloat16().view(torch.int16).numpy().view(np.uint16)
    par = np.stack([sb, zb], -1).reshape(*lead, nkv, 4, 2).view(np.uint8).reshape(*lead, nkv, 16)
    return np.concatenate([packed, par], -1).reshape(*lead, -1)


@pytest.mark.parametrize("bits,nkv,G", [(4, 8, 4), (2, 8, 4), (4, 4, 1)])
def test_quantized_values_decode(bits, nkv, G):
    """Quantised value cache: the append's row of the new token is BYTE-identical to the
    oracle's quantisation of v_new (R15's exact fp32 code rule: codes, bf16 scale and
    zero), and the decode equals the oracle's Algorithm 1 with V replaced by the
    oracle's own V^ (O.value_hat of the bf16 values; nothing read back from the GPU
    cache feeds the oracle): selection in the band, bf16 output tolerances."""
    from paper_2510_24273_b200 import sals
    d, B, seqs, k = 128, 2, [3000, 2311], 384
    D = nkv * d
    sh = dict(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=256, score_rank=128, top_k=k,
              rope_base=1e6, dtype="bf16")
    cfg = sals.make_config(**sh, v_bits=bits)
    row_bytes = sals.sals_v_row_bytes(cfg)
    assert row_bytes == nkv * (128 * bits // 8 + 16)
    p = synth.gen_problem(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=256, batch=B, seq_lens=seqs, seed=21)
    dev = lambda a: torch.from_numpy(a).cuda().bfloat16()
    U, q, kn, vn, lat = dev(p["U"]), dev(p["q"]), dev(p["k_new"]), dev(p["v_new"]), dev(p["latent"])
    v_host = H.widen(dev(p["v"]))                                   # the bf16 values the cache quantises
    vq = torch.from_numpy(_pack_values(v_host, bits, nkv)).cuda()    # [B, cap, row_bytes] uint8
    s_max = max(seqs)
    seq = torch.tensor(seqs, dtype=torch.int32, device="cuda")
    ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s_max), "cuda")
    out = torch.empty(B, nkv * G * d, dtype=torch.bfloat16, device="cuda")
    sel = torch.full((B, k), -7, dtype=torch.int32, device="cuda")
    scores = torch.zeros(B, s_max, dtype=torch.float32, device="cuda")
    sals.sals_append_decode(cfg, U, kn, vn, q, lat, vq, seq, s_max, out, ws, sel_idx_out=sel, scores_out=scores)
    torch.cuda.synchronize()
    rows = vq.cpu().numpy()
    vn_host = H.widen(vn)
    v_full = v_host.copy()
    for b in range(B):   # append: the new token's row, byte for byte
        np.testing.assert_array_equal(rows[b, seqs[b] - 1], _pack_values(vn_host[b:b + 1], bits, nkv)[0])
        v_full[b, seqs[b] - 1] = vn_host[b]
    oc = H.oracle_cfg(sh)
    host_lat = H.widen(lat)
    vhat = np.zeros_like(v_full)
    for b in range(B):
        vhat[b, :seqs[b]] = O.value_hat(v_full[b], bits, 0, seqs[b])
    orc = O.decode(oc, H.widen(U), H.widen(q), host_lat, vhat, np.array(seqs))
    forced = []
    for b in range(B):
        H.check_selection(orc["scores"][b], orc["sel"][b], sel.cpu().numpy()[b], seqs[b], k, 0, 0)
        srow = sel.cpu().numpy()[b]
        forced.append(srow[srow >= 0].astype(np.int64))
    orc_f = O.decode(oc, H.widen(U), H.widen(q), host_lat, vhat, np.array(seqs), forced_selection=forced)
    H.check_output(H.widen(out), orc_f["y"], "bf16")


def _pack8(v, nkv):
    """8-bit rows of the recent-window ring: per KV head 128 code bytes + 4 (bf16 scale, bf16 zero)."""
    codes, scale, zero = O.quantize_values(v, 8, 32)
    lead = v.shape[:-1]
    c = codes.reshape(*lead, nkv, 128).astype(np.uint8)
    sb = torch.from_numpy(scale.astype(np.float32)).bfloat16().view(torch.int16).numpy().view(np.uint16)
    zb = torch.from_numpy(zero.astype(np.float32)).bfloat16().view(torch.int16).numpy().view(np.uint16)
    par = np.stack([sb, zb], -1).reshape(*lead, nkv, 4, 2).view(np.uint8).reshape(*lead, nkv, 16)
    return np.concatenate([c, par], -1).reshape(*lead, -1)


@pytest.mark.parametrize("bits,nkv,G,z", [(4, 8, 4, 64), (2, 4, 1, 100), (4, 8, 2, 20), (2, 8, 4, 128)])
def test_quantized_values_recent_window(bits, nkv, G, z):
    """Quantised values with the high-precision recent window: the forced
    recent z tokens are read from the 8-bit ring, the rest from the b-bit rows; the
    append writes both formats.  Checked against the oracle over the stored V^."""
    _quantized_window_case(bits, nkv, G, z, seqs=[3000, 2311], k=384, rank=256, rstar=128, seed=23)


def test_quantized_values_recent_window_c3_size():
    """The same at c3's shape (Mistral-7B GQA 32/8, r 512, r* 256, k 4096, 32K tokens)
    with the paper's Mistral recent window z = 128, 4-bit values."""
    _quantized_window_case(4, 8, 4, 128, seqs=[32768, 30001], k=4096, rank=512, rstar=256, seed=29)


def _quantized_window_case(bits, nkv, G, z, seqs, k, rank, rstar, seed):
    """The cache holds the oracle's b-bit rows and 8-bit recent-window ring for the old
    tokens; the append writes the new token's b-bit row and ring slot, which must be
    byte-identical to the oracle's; the decode is compared with the oracle's
    Algorithm 1 over O.value_hat (mixed precision V^) of the bf16 values."""
    from paper_2510_24273_b200 import sals
    d, B = 128, len(seqs)
    sh = dict(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=rank, score_rank=rstar, top_k=k,
              rope_base=1e6, dtype="bf16")
    cfg = sals.make_config(**sh, v_bits=bits, recent=z)
    p = synth.gen_problem(num_q_heads=nkv * G, num_kv_heads=nkv, head_dim=d, rank=rank, batch=B, seq_lens=seqs,
                          seed=seed)
    cap = max(seqs)
    dev = lambda a: torch.from_numpy(a).cuda().bfloat16()
    U, q, kn, vn, lat = dev(p["U"]), dev(p["q"]), dev(p["k_new"]), dev(p["v_new"]), dev(p["latent"])
    v_host = H.widen(dev(p["v"]))
    rb = sals.sals_v_row_bytes(cfg)
    total = sals.sals_v_cache_bytes(cfg, B, cap)
    assert total == B * cap * rb + B * z * nkv * 144
    main = _pack_values(v_host, bits, nkv)                               # [B, cap, rb]
    ring = np.zeros((B, z, nkv * 144), dtype=np.uint8)
    for b in range(B):
        for pos in range(seqs[b] - z, seqs[b] - 1):                      # the new token's slot: the append's
            ring[b, pos % z] = _pack8(v_host[b, pos][None], nkv)[0]
    vq = torch.from_numpy(np.concatenate([main.reshape(-1), ring.reshape(-1)])).cuda()
    seq = torch.tensor(seqs, dtype=torch.int32, device="cuda")
    ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, cap), "cuda")
    out = torch.empty(B, nkv * G * d, dtype=torch.bfloat16, device="cuda")
    sel = torch.full((B, k), -7, dtype=torch.int32, device="cuda")
    sals.sals_append_decode(cfg, U, kn, vn, q, lat, vq, seq, cap, out, ws, sel_idx_out=sel)
    torch.cuda.synchronize()
    allb = vq.cpu().numpy()
    rows = allb[:B * cap * rb].reshape(B, cap, rb)
    ringg = allb[B * cap * rb:].reshape(B, z, nkv * 144)
    vn_host = H.widen(vn)
    v_full = v_host.copy()
    for b in range(B):
        s = seqs[b]
        np.testing.assert_array_equal(rows[b, s - 1], _pack_values(vn_host[b:b + 1], bits, nkv)[0])
        np.testing.assert_array_equal(ringg[b, (s - 1) % z], _pack8(vn_host[b:b + 1], nkv)[0])
        v_full[b, s - 1] = vn_host[b]
    vhat = np.zeros_like(v_full)
    for b in range(B):
        vhat[b, :seqs[b]] = O.value_hat(v_full[b], bits, z, seqs[b])
    oc = H.oracle_cfg(sh, recent=z)
    host_lat = H.widen(lat)
    orc = O.decode(oc, H.widen(U), H.widen(q), host_lat, vhat, np.array(seqs))
    forced = []
    for b in range(B):
        srow = sel.cpu().numpy()[b]
        H.check_selection(orc["scores"][b], orc["sel"][b], srow, seqs[b], k, 0, z)
        assert np.all(np.isin(np.arange(seqs[b] - z, seqs[b]), srow))
        forced.append(srow[srow >= 0].astype(np.int64))
    orc_f = O.decode(oc, H.widen(U), H.widen(q), host_lat, vhat, np.array(seqs), forced_selection=forced)
    H.check_output(H.widen(out), orc_f["y"], "bf16")
