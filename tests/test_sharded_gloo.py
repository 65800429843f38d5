"""World-size-2/3 gloo tests (CPU) of the sequence-sharded exchange protocol.

The orchestration under test is paper_2510_24273_b200.sharded.ShardedDecoder
(what is all-gathered, in which layout, the merge order) with its device phases
replaced by fp64 oracle phases; the result must equal the unsharded oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_phases(cfg, U, q, s):
    """CPU phases with the same tensor contract as sharded.gpu_phases."""
    import sys
    sys.path.insert(0, ROOT)
    from oracle import sals_oracle as O
    B = q.shape[0]
    k, x, z = cfg.top_k, cfg.sink, cfg.recent
    y = k - x - z
    nq, d, nkv = cfg.num_q_heads, cfg.head_dim, cfg.num_kv_heads

    def candidates(lat, start, local_len):
        cs = torch.full((B, k), float("-inf"), dtype=torch.float32)
        ci = torch.full((B, k), -1, dtype=torch.int32)
        for b in range(B):
            n = int(local_len[b])
            qt = O.project_latent(U, O.pool_query(q[b], cfg))
            sc = O.latent_scores(qt, lat[b, :n], cfg.score_rank)
            gidx = np.arange(n) + start
            keep = (gidx >= x) & (gidx < s - z)
            sc, gidx = sc[keep], gidx[keep]
            order = np.lexsort((gidx, -sc))[: min(y, len(sc))]
            sel = np.sort(gidx[order])                      # ascending global index
            cs[b, : len(sel)] = torch.from_numpy(sc[np.searchsorted(gidx, sel)].astype(np.float32))
            ci[b, : len(sel)] = torch.from_numpy(sel.astype(np.int32))
        return cs, ci

    def attend(lat, v, start, local_len, all_s, own_i):
        rank = dist.get_rank()
        part = torch.zeros(B, nq, d + 2, dtype=torch.float64)
        for b in range(B):
            n = int(local_len[b])
            own = O.shard_owned_selection(all_s[:, b].double().numpy(), own_i[b].numpy().astype(np.int64), rank,
                                          start, start + n, s, cfg)
            loc = own - start
            KC = O.reconstruct(lat[b, loc], U).reshape(len(loc), nkv, d)
            KR = O.rope(KC, own[:, None], cfg.rope_base)
            qR = O.rope(np.asarray(q[b], dtype=np.float64).reshape(nq, d), s - 1, cfg.rope_base)
            m, l, o = O.partial_attention(qR, KR, v[b, loc].reshape(len(loc), nkv, d), cfg)
            part[b, :, 0] = torch.from_numpy(m)
            part[b, :, 1] = torch.from_numpy(l)
            part[b, :, 2:] = torch.from_numpy(o)
        return part

    def merge(part_all):
        pa = part_all.numpy()
        return np.stack([O.lse_merge(pa[:, b, :, 0], pa[:, b, :, 1], pa[:, b, :, 2:]).reshape(-1)
                         for b in range(pa.shape[1])])

    from paper_2510_24273_b200.sharded import Phases
    return Phases(candidates, attend, merge)


def _worker(rank, world, port, sink, recent, result_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from oracle import sals_oracle as O
        from paper_2510_24273_b200.sharded import ShardedDecoder, shard_bounds
        cfg = O.Config(num_q_heads=8, num_kv_heads=2, head_dim=16, rank=24, score_rank=16, top_k=23,
                       sink=sink, recent=recent, rope_base=5e5)
        s = 301
        p = synth.gen_problem(num_q_heads=8, num_kv_heads=2, head_dim=16, rank=24, batch=2, seq_lens=[s, s], seed=5)
        U = p["U"].astype(np.float64)
        # identical scores across shards for some tokens -> exercise cross-shard tie-breaking
        p["latent"][:, 40] = p["latent"][:, 200]
        start, end = shard_bounds(s, world, rank)
        lat = p["latent"][:, start:end].astype(np.float64)
        v = p["v"][:, start:end].astype(np.float64)
        loc = np.full(2, end - start)
        dec = ShardedDecoder(oracle_phases(cfg, U, p["q"], s))
        y = dec.decode(lat, v, start, loc)
        ref = O.decode(cfg, U, p["q"], p["latent"], p["v"], [s, s])["y"]
        result_q.put((rank, float(np.max(np.abs(y - ref)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,sink,recent", [(2, 0, 0), (2, 4, 8), (3, 1, 5)])
def test_sharded_protocol_gloo(world, sink, recent):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sink, recent, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
        assert pr.exitcode == 0
    res = dict(q.get() for _ in range(world))
    assert all(err < 1e-10 for err in res.values()), res


def test_shard_bounds_cover():
    from paper_2510_24273_b200.sharded import shard_bounds
    for s in [1, 7, 131072, 131071]:
        for P in [1, 2, 3, 8]:
            spans = [shard_bounds(s, P, r) for r in range(P)]
            assert spans[0][0] == 0 and spans[-1][1] == s
            assert all(spans[i][1] == spans[i + 1][0] for i in range(P - 1))
