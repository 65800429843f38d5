"""Test / smoke harness: seeded synthetic problems on the GPU through the C ABI,
and the acceptance checks against the fp64 oracle (north_star tolerances)."""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle import sals_oracle as O

# north_star: selection band 1e-3 relative of the k-th score; bf16 output
# within 2e-2 max-abs and 1e-2 mean-rel; fp32 (c1) 1e-4 max-abs.
SEL_BAND = 1e-3
BF16_MAX_ABS, BF16_MEAN_REL = 2e-2, 1e-2
F32_MAX_ABS = 1e-4


def oracle_cfg(shape: dict, sink=0, recent=0, top_k=None, rope_style=0) -> O.Config:
    return O.Config(num_q_heads=shape["num_q_heads"], num_kv_heads=shape["num_kv_heads"],
                    head_dim=shape["head_dim"], rank=shape["rank"], score_rank=shape["score_rank"],
                    top_k=top_k if top_k is not None else shape["top_k"], sink=sink, recent=recent,
                    rope_base=shape["rope_base"], rope_style=rope_style)


def widen(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def run_sals(shape: dict, batch: int, seq_lens, *, seed=synth.SEED_BASE, cap=None, sink=0, recent=0,
             top_k=None, path=0, rope_style=0, dtype=None, fused=False):
    """Generate, append the new token, decode (``fused``: the one call
    sals_append_decode that bench.py times, else sals_append_latent + sals_decode).
    Returns (cfg, stored host tensors, gpu results)."""
    from paper_2510_24273_b200 import sals
    dtype = dtype or shape["dtype"]
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    seq_lens = np.asarray(seq_lens, dtype=np.int32)
    cap = int(cap or seq_lens.max())
    k = top_k if top_k is not None else shape["top_k"]
    cfg = sals.make_config(**{**shape, "top_k": k, "dtype": dtype}, sink=sink, recent=recent, path=path,
                           rope_style=rope_style)
    p = synth.gen_problem(num_q_heads=shape["num_q_heads"], num_kv_heads=shape["num_kv_heads"],
                          head_dim=shape["head_dim"], rank=shape["rank"], batch=batch, seq_lens=seq_lens,
                          cap=cap, seed=seed)
    dev = "cuda"
    U = torch.from_numpy(p["U"]).to(dev).to(tdt)
    latent = torch.from_numpy(p["latent"]).to(dev).to(tdt)
    v = torch.from_numpy(p["v"]).to(dev).to(tdt)
    q = torch.from_numpy(p["q"]).to(dev).to(tdt)
    k_new = torch.from_numpy(p["k_new"]).to(dev).to(tdt)
    v_new = torch.from_numpy(p["v_new"]).to(dev).to(tdt)
    seq = torch.from_numpy(seq_lens).to(dev)
    pos = (seq - 1).to(torch.int32)
    D = shape["num_kv_heads"] * shape["head_dim"]
    max_s = int(seq_lens.max())
    ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, batch, max_s), dev)
    out = torch.empty(batch, shape["num_q_heads"] * shape["head_dim"], dtype=tdt, device=dev)
    sel = torch.full((batch, k), -7, dtype=torch.int32, device=dev)
    scores = torch.zeros(batch, max_s, dtype=torch.float32, device=dev)
    if fused:
        sals.sals_append_decode(cfg, U, k_new, v_new, q, latent, v, seq, max_s, out, ws, sel_idx_out=sel,
                                scores_out=scores)
    else:
        sals.sals_append_latent(cfg, U, k_new, v_new, pos, latent, v)
        sals.sals_decode(cfg, U, q, latent, v, seq, max_s, out, ws, sel_idx_out=sel, scores_out=scores)
    torch.cuda.synchronize()
    host = dict(U=widen(U), q=widen(q), k_new=widen(k_new), v_new=widen(v_new), latent=widen(latent), v=widen(v),
                seq_len=seq_lens, D=D)
    gpu = dict(out=widen(out), sel=sel.cpu().numpy(), scores=scores.cpu().numpy())
    return cfg, host, gpu


def check_append(host, dtype):
    """Row pos_b of the latent cache == bf16/fp32 rounding of U^T k_new (1 ulp)."""
    ref = O.project_latent(host["U"], host["k_new"])                      # [B, r] fp64
    rows = np.stack([host["latent"][b, host["seq_len"][b] - 1] for b in range(len(host["seq_len"]))])
    if dtype == "bf16":
        ulp = 2.0 ** (np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
        assert np.all(np.abs(rows - ref) <= ulp + 1e-6), np.max(np.abs(rows - ref) / ulp)
    else:
        assert np.max(np.abs(rows - ref)) <= 1e-5 * (1 + np.abs(ref).max())
    vrows = np.stack([host["v"][b, host["seq_len"][b] - 1] for b in range(len(host["seq_len"]))])
    np.testing.assert_array_equal(vrows, host["v_new"])


def check_selection(orc_scores, orc_sel, gpu_sel_row, s, k, sink, recent):
    """|C_gpu| = |C_orc| and C_gpu ^ C_orc within the 1e-3 band of the y-th score."""
    gsel = gpu_sel_row[gpu_sel_row >= 0]
    n = min(k, s)
    assert len(gsel) == n, (len(gsel), n)
    assert np.all(np.diff(gsel) > 0), "selection must be ascending"
    assert np.all(gpu_sel_row[n:] == -1)
    diff = set(gsel.tolist()) ^ set(orc_sel.tolist())
    if not diff:
        return 0
    ranked = orc_scores[sink:s - recent]
    y = k - sink - recent
    sy = np.sort(ranked)[::-1][y - 1]
    band = SEL_BAND * max(abs(sy), np.mean(np.abs(orc_scores[:s])))
    for j in diff:
        assert sink <= j < s - recent, j
        assert abs(orc_scores[j] - sy) <= band, (j, orc_scores[j], sy, band)
    return len(diff)


def check_output(y_gpu, y_orc, dtype):
    err = np.abs(y_gpu - y_orc)
    if dtype == "bf16":
        assert err.max() <= BF16_MAX_ABS, err.max()
        assert err.sum() / np.abs(y_orc).sum() <= BF16_MEAN_REL, err.sum() / np.abs(y_orc).sum()
    else:
        assert err.max() <= F32_MAX_ABS, err.max()
    return float(err.max()), float(err.sum() / max(np.abs(y_orc).sum(), 1e-30))


def full_check(shape, batch, seq_lens, **kw):
    """append parity, score parity, selection parity, output parity (forced to C_gpu and,
    when equal, the oracle's own C)."""
    dtype = kw.get("dtype") or shape["dtype"]
    cfg, host, gpu = run_sals(shape, batch, seq_lens, **kw)
    oc = oracle_cfg(shape, kw.get("sink", 0), kw.get("recent", 0), kw.get("top_k"), kw.get("rope_style", 0))
    check_append(host, dtype)
    orc = O.decode(oc, host["U"], host["q"], host["latent"], host["v"], host["seq_len"])
    nswap = 0
    forced = []
    for b in range(batch):
        s = int(host["seq_len"][b])
        sc_err = np.abs(gpu["scores"][b, :s] - orc["scores"][b])
        assert sc_err.max() <= 1e-4 * max(1.0, np.abs(orc["scores"][b]).max()), sc_err.max()
        nswap += check_selection(orc["scores"][b], orc["sel"][b], gpu["sel"][b], s, oc.top_k, oc.sink, oc.recent)
        forced.append(gpu["sel"][b][gpu["sel"][b] >= 0].astype(np.int64))
    orc_forced = O.decode(oc, host["U"], host["q"], host["latent"], host["v"], host["seq_len"],
                          forced_selection=forced)
    stats = check_output(gpu["out"], orc_forced["y"], dtype)
    if nswap == 0:
        check_output(gpu["out"], orc["y"], dtype)
    return dict(swaps=nswap, max_abs=stats[0], mean_rel=stats[1])


def sampled_check(shape: dict, batch: int, seq: int, *, sample, seed=synth.SEED_BASE, sink=0, recent=0):
    """Bench-sized parity: one layer drawn on the device with the bench's generator
    (synth.gen_layer_torch), the whole batch through sals_append_decode in the launch
    configuration bench.py times; the append rows of EVERY request against the oracle,
    and the requests in ``sample`` one by one through the oracle (scores, selection
    band, output forced to the GPU's C and, when equal, the oracle's own C).  Only the
    sampled requests' rows are widened to fp64 on the host."""
    from paper_2510_24273_b200 import sals
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    ly = synth.gen_layer_torch(num_q_heads=shape["num_q_heads"], num_kv_heads=shape["num_kv_heads"],
                               head_dim=shape["head_dim"], rank=shape["rank"], batch=batch, seq=seq, generator=g)
    cfg = sals.make_config(**shape, sink=sink, recent=recent)
    oc = oracle_cfg(shape, sink, recent)
    k = shape["top_k"]
    seqd = torch.full((batch,), seq, dtype=torch.int32, device="cuda")
    ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, batch, seq), "cuda")
    out = torch.empty(batch, shape["num_q_heads"] * shape["head_dim"], dtype=torch.bfloat16, device="cuda")
    sel = torch.full((batch, k), -7, dtype=torch.int32, device="cuda")
    scores = torch.zeros(batch, seq, dtype=torch.float32, device="cuda")
    sals.sals_append_decode(cfg, ly["U"], ly["k_new"], ly["v_new"], ly["q"], ly["latent"], ly["v"], seqd, seq, out,
                            ws, sel_idx_out=sel, scores_out=scores)
    torch.cuda.synchronize()
    U = widen(ly["U"])
    # append rows of every request (1 bf16 ulp of the fp64 projection; value rows bit-exact)
    ref = O.project_latent(U, widen(ly["k_new"]))
    rows = widen(ly["latent"][:, seq - 1])
    ulp = 2.0 ** (np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
    assert np.all(np.abs(rows - ref) <= ulp + 1e-6), np.max(np.abs(rows - ref) / ulp)
    assert torch.equal(ly["v"][:, seq - 1], ly["v_new"])
    stats = []
    gsel = sel.cpu().numpy()
    gout = widen(out)
    for b in sample:
        lat_b = widen(ly["latent"][b, :seq])
        v_b = widen(ly["v"][b, :seq])
        q_b = widen(ly["q"][b])
        orc = O.decode_request(oc, U, q_b, lat_b, v_b, seq)
        sc = scores[b].cpu().numpy().astype(np.float64)
        assert np.abs(sc - orc["scores"]).max() <= 1e-4 * max(1.0, np.abs(orc["scores"]).max())
        nswap = check_selection(orc["scores"], orc["sel"], gsel[b], seq, k, sink, recent)
        forced = gsel[b][gsel[b] >= 0].astype(np.int64)
        orc_f = O.decode_request(oc, U, q_b, lat_b, v_b, seq, forced_selection=forced)
        st = check_output(gout[b], orc_f["y"], "bf16")
        if nswap == 0:
            check_output(gout[b], orc["y"], "bf16")
        stats.append(dict(b=int(b), swaps=nswap, max_abs=st[0], mean_rel=st[1]))
    del ly
    torch.cuda.empty_cache()
    return stats
