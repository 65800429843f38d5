"""Sequence-sharded SALS decode over P GPUs: one process per GPU,
contiguous shards of every request's tokens, two all-gathers per layer.

    rank p:  local q~, p' over its shard, local top-(k-x-z) candidates with
             GLOBAL indices, ascending (sals_shard_candidates)
    all-gather #1: candidate SCORES only -> [P, B, k]   (NCCL over NVLink); the
             gathered order (rank, position) is the global index order
    rank p:  exact global TopK over the union (radix select of the (k-x-z)-th
             score + tie quota, ranks in order) fused with its owned list,
             reconstruct + RoPE + attention over the OWNED selected tokens
             -> one (m, l, o) partial per (request, query head)   (sals_shard_attend)
    all-gather #2: partials -> [P, B, n_q, d+2]
    every rank: log-sum-exp merge -> y   (sals_merge_partials)

The exchange plumbing (what is gathered, in which layout, and the merge order)
lives in ``ShardedDecoder``; the device phases are injectable so the same
orchestration runs on CPU with gloo and the fp64 oracle in the tests.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist


def shard_bounds(seq_len: int, world: int, rank: int):
    """Contiguous shard [start, end) of positions 0..seq_len-1 held by `rank`."""
    per = math.ceil(seq_len / world)
    start = min(rank * per, seq_len)
    return start, min(start + per, seq_len)


@dataclass
class Phases:
    """Device (or oracle) implementations of the three local phases."""
    candidates: callable    # (latent_shard, start, local_len) -> (cand_score [B,k] f32, cand_idx [B,k] i32)
    attend: callable        # (latent_shard, v_shard, start, local_len, all_score [P,B,k], own cand_idx) -> partial
    merge: callable         # (partial_all [P,B,n_q,d+2]) -> y [B, n_q*d]


class ShardedDecoder:
    def __init__(self, phases: Phases, group=None):
        self.ph = phases
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def _gather(self, t: torch.Tensor) -> torch.Tensor:
        """All-gather along a new leading rank axis ([P, *t.shape], rank order)."""
        t = t.contiguous()
        out = torch.empty((self.world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out.view((self.world,) + tuple(t.shape))

    def decode(self, latent_shard, v_shard, start, local_len):
        cs, ci = self.ph.candidates(latent_shard, start, local_len)
        all_s = self._gather(cs)            # [P, B, k], rank order = ascending global index
        part = self.ph.attend(latent_shard, v_shard, start, local_len, all_s, ci)
        part_all = self._gather(part)       # [P, B, n_q, d+2]
        return self.ph.merge(part_all)


def gpu_phases(cfg, U, q, seq_len, max_local_len, ws, world, rank):
    """Phases backed by the C ABI (libsals.so) on the current CUDA stream."""
    from . import sals
    B = q.shape[0]
    k = cfg.top_k
    n_q, d = cfg.num_q_heads, cfg.head_dim
    cs = torch.empty(B, k, dtype=torch.float32, device=q.device)
    ci = torch.empty(B, k, dtype=torch.int32, device=q.device)
    part = torch.empty(B, n_q, d + 2, dtype=torch.float32, device=q.device)
    out = torch.empty(B, n_q * d, dtype=q.dtype, device=q.device)

    def candidates(lat, start, local_len):
        sals.sals_shard_candidates(cfg, U, q, lat, start, local_len, max_local_len, seq_len, cs, ci, ws)
        return cs, ci

    def attend(lat, v, start, local_len, all_s, own_i):
        sals.sals_shard_attend(cfg, U, q, lat, v, start, local_len, max_local_len, seq_len, all_s, own_i, world,
                               rank, part, ws)
        return part

    def merge(part_all):
        sals.sals_merge_partials(cfg, part_all, world, B, out)
        return out

    return Phases(candidates, attend, merge)


# ---------------------------------------------------------------------------
# bench: c4 sequence-sharded over torchrun ranks (strong scaling)
# ---------------------------------------------------------------------------
def bench(args, rank, world):
    import json
    import sys
    import time

    import synth
    from . import build, sals
    build.build()
    sys_shape = dict(synth.CONFIGS["c4"])
    B, s, L = sys_shape["batch"], sys_shape["seq"], args.layers
    cfg = sals.make_config(**sys_shape, path=args.path)
    start, end = shard_bounds(s, world, rank)
    n_loc = end - start
    g = torch.Generator(device="cuda")
    g.manual_seed(synth.SEED_BASE + 7)
    layers = []
    for _ in range(L):
        ly = synth.gen_layer_torch(num_q_heads=sys_shape["num_q_heads"], num_kv_heads=sys_shape["num_kv_heads"],
                                   head_dim=sys_shape["head_dim"], rank=sys_shape["rank"], batch=B, seq=n_loc,
                                   generator=g)
        layers.append(ly)
    seq = torch.full((B,), s, dtype=torch.int32, device="cuda")
    loc = torch.full((B,), n_loc, dtype=torch.int32, device="cuda")
    ws = sals.alloc_workspace(sals.sals_shard_workspace_bytes(cfg, B, n_loc, world), "cuda")
    owner = rank == world - 1                       # holds position s-1, appends the new token
    pos_local = (loc - 1).to(torch.int32)
    comm = None
    if args.comm == "lib":   # the library's one-call path with its own NCCL communicator
        uid = [sals.sals_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = sals.sals_comm_init(uid[0], world, rank)
        ws = sals.alloc_workspace(sals.sals_decode_sharded_workspace_bytes(cfg, B, n_loc, world), "cuda")
        outs = [torch.empty(B, ly["q"].shape[1], dtype=ly["q"].dtype, device="cuda") for ly in layers]
    else:
        decs = [ShardedDecoder(gpu_phases(cfg, ly["U"], ly["q"], seq, n_loc, ws, world, rank)) for ly in layers]

    def step():
        for i, ly in enumerate(layers):
            if comm is not None:   # the append runs inside the call, on the rank holding position s - 1
                sals.sals_append_decode_sharded(cfg, comm, ly["U"], ly["k_new"], ly["v_new"], ly["q"], ly["latent"],
                                                ly["v"], start, loc, n_loc, seq, outs[i], ws)
            else:
                if owner:
                    sals.sals_append_latent(cfg, ly["U"], ly["k_new"], ly["v_new"], pos_local, ly["latent"], ly["v"])
                decs[i].decode(ly["latent"], ly["v"], start, loc)

    stream = torch.cuda.Stream()
    graph = None
    torch.cuda.synchronize()   # inputs were made on the default stream
    with torch.cuda.stream(stream):
        step()
        stream.synchronize()
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step()
        except Exception:
            graph = None
        for _ in range(args.warmup):
            graph.replay() if graph else step()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            graph.replay() if graph else step()
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # per-phase us per layer-step (library path): a graph of the same step with only one
    # phase enabled (sals_profile_stage_mask), max over ranks; the phases' sum vs the step
    # shows how much the chain overlaps
    phases = {}
    if comm is not None and graph is not None:
        bits = dict(sals.STAGE_BITS)
        bits.pop("flash", None)
        bits.update(exchange=sals.EXCHANGE_BIT, shard_select=sals.SHARD_SELECT_BIT)
        for name, bit in bits.items():
            print(f"[sharded bench] phase {name}", file=sys.stderr, flush=True)
            sals.sals_profile_stage_mask(1 << bit)
            try:
                with torch.cuda.stream(stream):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
                        step()
            finally:
                sals.sals_profile_stage_mask(0xffffffff)
            with torch.cuda.stream(stream):
                step()
                for _ in range(3):
                    g.replay()
                torch.cuda.synchronize()
                dist.barrier()
                f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                f0.record(stream)
                for _ in range(max(5, args.steps)):
                    g.replay()
                f1.record(stream)
                torch.cuda.synchronize()
                step()
            pt = torch.tensor([f0.elapsed_time(f1) / max(5, args.steps)], dtype=torch.float64, device="cuda")
            dist.all_reduce(pt, op=dist.ReduceOp.MAX)
            us = float(pt.item()) * 1e3 / L
            if us > 0.05:
                phases[name] = round(us, 2)
            del g
    if rank == 0:
        line = {"metric": "decode attention tokens/s (32-layer attention step)", "value": B / (ms / 1e3),
                "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic",
                "config": {"workload": f"c4-sharded: B={B} n={s} sequence-sharded over {world} GPUs x{L} layers",
                           "batch": B, "seq_len": s, "layers": L, "parallelism": f"sequence-shard x{world}",
                           "graph": graph is not None,
                           "exchange": "sals_append_decode_sharded (library NCCL; the append in the query projection's launch)" if comm is not None
                           else "torch.distributed all_gather_into_tensor"},
                "us_per_layer_step": ms * 1e3 / L,
                "phases_us_per_layer": phases,
                "phases_note": "graph of the step with one phase enabled (others skipped), max over ranks; "
                               "'qproj_rope' includes the owner rank's append (one launch), 'exchange' the two NCCL all-gathers"}
        print(json.dumps(line), flush=True)
    if comm is not None:
        torch.cuda.synchronize()
        sals.sals_comm_destroy(comm)
