"""Thin ctypes binding of the C ABI in include/sals.h (argument marshalling only).

Every function has the C name and forwards torch tensors as raw device
pointers plus the current CUDA stream; all compute runs in libsals.so.  There
is no fallback: importing this module without the in-tree library raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsals.so")

SALS_F32, SALS_BF16 = 0, 1
SALS_ROPE_HALF, SALS_ROPE_INTERLEAVED = 0, 1
SALS_PATH_AUTO, SALS_PATH_SIMT, SALS_PATH_TCGEN05 = 0, 1, 2
STATUS = {0: "SALS_OK", 1: "SALS_ERR_INVALID_ARGUMENT", 2: "SALS_ERR_UNSUPPORTED",
          3: "SALS_ERR_WORKSPACE_TOO_SMALL", 4: "SALS_ERR_CUDA", 5: "SALS_ERR_NCCL"}

EXPORTED = ["sals_workspace_bytes", "sals_append_latent", "sals_decode", "sals_decode_profile", "sals_dense_append",
            "sals_dense_workspace_bytes", "sals_dense_decode", "sals_shard_candidates", "sals_shard_attend",
            "sals_merge_partials", "sals_shard_workspace_bytes", "sals_status_string", "sals_last_error",
            "sals_launch_count", "sals_profile_stage_mask", "sals_append_decode",
            "sals_append_latent_bulk", "sals_calibrate_workspace_bytes", "sals_calibrate",
            "sals_v_row_bytes", "sals_v_cache_bytes", "sals_comm_unique_id", "sals_comm_init",
            "sals_comm_destroy", "sals_decode_sharded_workspace_bytes", "sals_decode_sharded",
            "sals_workspace_selection_offsets", "sals_append_decode_sharded"]


class SalsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class sals_config(ctypes.Structure):
    _fields_ = [("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("score_rank", ctypes.c_int32), ("top_k", ctypes.c_int32),
                ("sink", ctypes.c_int32), ("recent", ctypes.c_int32), ("rope_base", ctypes.c_float),
                ("rope_style", ctypes.c_int32), ("dtype", ctypes.c_int32), ("softmax_scale", ctypes.c_float),
                ("path", ctypes.c_int32), ("v_bits", ctypes.c_int32)]


def make_config(*, num_q_heads, num_kv_heads, head_dim, rank, score_rank, top_k, sink=0, recent=0,
                rope_base=10000.0, rope_style=SALS_ROPE_HALF, dtype="bf16", softmax_scale=0.0,
                path=SALS_PATH_AUTO, v_bits=0, **_unused) -> sals_config:
    dt = {"bf16": SALS_BF16, "f32": SALS_F32, torch.bfloat16: SALS_BF16, torch.float32: SALS_F32}[dtype]
    return sals_config(num_q_heads, num_kv_heads, head_dim, rank, score_rank, top_k, sink, recent,
                       float(rope_base), rope_style, dt, float(softmax_scale), path, int(v_bits))


def torch_dtype(cfg: sals_config):
    return torch.bfloat16 if cfg.dtype == SALS_BF16 else torch.float32


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2510_24273_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    C = ctypes.POINTER(sals_config)
    sig = {
        "sals_workspace_bytes": (SZ, [C, I32, I32]),
        "sals_append_latent": (I32, [C, P, P, P, I32, P, P, P, I64, P]),
        "sals_decode": (I32, [C, P, P, P, P, I64, I32, P, I32, P, P, P, P, SZ, P]),
        "sals_append_decode": (I32, [C, P, P, P, P, P, P, I64, I32, P, I32, P, P, P, P, SZ, P]),
        "sals_append_latent_bulk": (I32, [C, P, P, P, I32, I32, I64, P, P, I64, P]),
        "sals_calibrate_workspace_bytes": (SZ, [C]),
        "sals_v_row_bytes": (SZ, [C]),
        "sals_v_cache_bytes": (SZ, [C, I32, I64]),
        "sals_calibrate": (I32, [C, P, I64, P, P, P, SZ, P]),
        "sals_decode_profile": (I32, [C, P, P, P, P, I64, I32, P, I32, P, P, SZ, I32, P, P]),
        "sals_dense_append": (I32, [C, P, P, I32, P, P, P, I64, P]),
        "sals_dense_workspace_bytes": (SZ, [C, I32, I32]),
        "sals_dense_decode": (I32, [C, P, P, P, I64, I32, P, I32, P, P, SZ, P]),
        "sals_shard_candidates": (I32, [C, P, P, P, I64, I32, I64, P, I32, P, P, P, P, SZ, P]),
        "sals_shard_attend": (I32, [C, P, P, P, P, I64, I32, I64, P, I32, P, P, P, I32, I32, P, P, SZ, P]),
        "sals_workspace_selection_offsets": (I32, [C, I32, I32, P, P]),
        "sals_merge_partials": (I32, [C, P, I32, I32, P, P]),
        "sals_shard_workspace_bytes": (SZ, [C, I32, I32, I32]),
        "sals_comm_unique_id": (I32, [P]),
        "sals_comm_init": (I32, [P, I32, I32, ctypes.POINTER(P)]),
        "sals_comm_destroy": (I32, [P]),
        "sals_decode_sharded_workspace_bytes": (SZ, [C, I32, I32, I32]),
        "sals_decode_sharded": (I32, [C, P, P, P, P, P, I64, I32, I64, P, I32, P, P, P, SZ, P]),
        "sals_append_decode_sharded": (I32, [C, P, P, P, P, P, P, P, I64, I32, I64, P, I32, P, P, P, SZ, P]),
        "sals_status_string": (ctypes.c_char_p, [I32]),
        "sals_last_error": (ctypes.c_char_p, []),
        "sals_launch_count": (ctypes.c_uint64, [I32]),
        "sals_profile_stage_mask": (ctypes.c_uint32, [ctypes.c_uint32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


_lib = _load()


def _p(t):
    return None if t is None else t.data_ptr()   # (argtypes c_void_p: an int is passed as the pointer)


# the caller's current stream as a raw handle: torch's C-level accessors when present
# (~0.3 us instead of ~3.4 us for torch.cuda.current_stream() per call), else the public API
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_cur_dev = getattr(torch._C, "_cuda_getDevice", None)


def _stream(stream=None):
    if stream is not None:
        return stream.cuda_stream
    if _raw_stream is not None and _cur_dev is not None:
        return _raw_stream(_cur_dev())
    return torch.cuda.current_stream().cuda_stream


def _check(status: int):
    if status != 0:
        raise SalsError(status, _lib.sals_last_error().decode())


def sals_workspace_bytes(cfg: sals_config, batch: int, max_seq_len: int) -> int:
    return int(_lib.sals_workspace_bytes(ctypes.byref(cfg), batch, max_seq_len))


def sals_dense_workspace_bytes(cfg: sals_config, batch: int, max_seq_len: int) -> int:
    return int(_lib.sals_dense_workspace_bytes(ctypes.byref(cfg), batch, max_seq_len))


def sals_shard_workspace_bytes(cfg: sals_config, batch: int, max_local_len: int, world: int) -> int:
    return int(_lib.sals_shard_workspace_bytes(ctypes.byref(cfg), batch, max_local_len, world))


def alloc_workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)


def sals_append_latent(cfg, U, k_new, v_new, pos, latent_cache, v_cache, stream=None):
    B = k_new.shape[0]
    _check(_lib.sals_append_latent(ctypes.byref(cfg), _p(U), _p(k_new), _p(v_new), B, _p(pos),
                                   _p(latent_cache), _p(v_cache), latent_cache.shape[1], _stream(stream)))


def sals_decode(cfg, U, q, latent_cache, v_cache, seq_len, max_seq_len, out, workspace,
                sel_idx_out=None, scores_out=None, stream=None):
    B = q.shape[0]
    _check(_lib.sals_decode(ctypes.byref(cfg), _p(U), _p(q), _p(latent_cache), _p(v_cache), latent_cache.shape[1],
                            B, _p(seq_len), int(max_seq_len), _p(out), _p(sel_idx_out), _p(scores_out),
                            _p(workspace), workspace.numel(), _stream(stream)))


STAGES = ["qproj_rope", "score", "topk", "recon_attn", "flash", "merge"]


def sals_v_row_bytes(cfg) -> int:
    """Bytes of one token's value-cache row (D * dtype size, or the quantised layout of cfg.v_bits)."""
    return int(_lib.sals_v_row_bytes(ctypes.byref(cfg)))


def sals_v_cache_bytes(cfg, batch: int, cap: int) -> int:
    """Bytes of a value cache (rows + the quantised values' 8-bit recent-window ring)."""
    return int(_lib.sals_v_cache_bytes(ctypes.byref(cfg), int(batch), int(cap)))


def sals_calibrate_workspace_bytes(cfg) -> int:
    return int(_lib.sals_calibrate_workspace_bytes(ctypes.byref(cfg)))


def sals_calibrate(cfg, K, U_out, eigvals_out=None, stream=None):
    """Offline calibration: U_out [D, r] = leading eigenvectors of K^T K (K [N, D] pre-RoPE keys)."""
    ws = alloc_workspace(sals_calibrate_workspace_bytes(cfg), K.device)
    _check(_lib.sals_calibrate(ctypes.byref(cfg), _p(K), K.shape[0], _p(U_out), _p(eigvals_out), _p(ws),
                               ws.numel(), _stream(stream)))


def sals_append_latent_bulk(cfg, U, k, v, start, latent_cache, v_cache, stream=None):
    """Prefill: latent/value rows [start, start + n) of every request from k, v [B, n, D]."""
    _check(_lib.sals_append_latent_bulk(ctypes.byref(cfg), _p(U), _p(k), _p(v), k.shape[0], k.shape[1], int(start),
                                        _p(latent_cache), _p(v_cache), latent_cache.shape[1], _stream(stream)))


def sals_append_decode(cfg, U, k_new, v_new, q, latent_cache, v_cache, seq_len, max_seq_len, out, workspace,
                       sel_idx_out=None, scores_out=None, stream=None):
    """sals_append_latent (slot seq_len - 1) + sals_decode in one call (one projection launch)."""
    _check(_lib.sals_append_decode(ctypes.byref(cfg), _p(U), _p(k_new), _p(v_new), _p(q), _p(latent_cache),
                                   _p(v_cache), latent_cache.shape[1], q.shape[0], _p(seq_len), int(max_seq_len),
                                   _p(out), _p(sel_idx_out), _p(scores_out), _p(workspace), workspace.numel(),
                                   _stream(stream)))


def sals_decode_profile(cfg, U, q, latent_cache, v_cache, seq_len, max_seq_len, out, workspace, iters=10,
                        stream=None) -> dict:
    ms = (ctypes.c_float * 6)()
    _check(_lib.sals_decode_profile(ctypes.byref(cfg), _p(U), _p(q), _p(latent_cache), _p(v_cache),
                                    latent_cache.shape[1], q.shape[0], _p(seq_len), int(max_seq_len), _p(out),
                                    _p(workspace), workspace.numel(), int(iters), ms, _stream(stream)))
    return {k: float(v) for k, v in zip(STAGES, ms)}


def sals_dense_append(cfg, k_new, v_new, pos, k_cache, v_cache, stream=None):
    _check(_lib.sals_dense_append(ctypes.byref(cfg), _p(k_new), _p(v_new), k_new.shape[0], _p(pos), _p(k_cache),
                                  _p(v_cache), k_cache.shape[1], _stream(stream)))


def sals_dense_decode(cfg, q, k_cache, v_cache, seq_len, max_seq_len, out, workspace, stream=None):
    _check(_lib.sals_dense_decode(ctypes.byref(cfg), _p(q), _p(k_cache), _p(v_cache), k_cache.shape[1], q.shape[0],
                                  _p(seq_len), int(max_seq_len), _p(out), _p(workspace), workspace.numel(),
                                  _stream(stream)))


def sals_shard_candidates(cfg, U, q, latent_shard, shard_start, local_len, max_local_len, seq_len,
                          cand_score, cand_idx, workspace, stream=None):
    _check(_lib.sals_shard_candidates(ctypes.byref(cfg), _p(U), _p(q), _p(latent_shard), latent_shard.shape[1],
                                      q.shape[0], int(shard_start), _p(local_len), int(max_local_len), _p(seq_len),
                                      _p(cand_score), _p(cand_idx), _p(workspace), workspace.numel(),
                                      _stream(stream)))


def sals_shard_attend(cfg, U, q, latent_shard, v_shard, shard_start, local_len, max_local_len, seq_len,
                      cand_all_score, cand_idx, world, rank, partial, workspace, stream=None):
    _check(_lib.sals_shard_attend(ctypes.byref(cfg), _p(U), _p(q), _p(latent_shard), _p(v_shard),
                                  latent_shard.shape[1], q.shape[0], int(shard_start), _p(local_len),
                                  int(max_local_len), _p(seq_len), _p(cand_all_score), _p(cand_idx), int(world),
                                  int(rank), _p(partial), _p(workspace), workspace.numel(), _stream(stream)))


def sals_workspace_selection_offsets(cfg, batch, max_seq_len):
    """Byte offsets (selection list, counts) inside a decode / shard workspace."""
    o_sel, o_cnt = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(_lib.sals_workspace_selection_offsets(ctypes.byref(cfg), int(batch), int(max_seq_len),
                                                 ctypes.byref(o_sel), ctypes.byref(o_cnt)))
    return o_sel.value, o_cnt.value


def shard_owned_list(cfg, workspace, batch, max_local_len):
    """(inspection) the owned local rows [B, k] and counts [B] a completed
    sals_shard_attend left in `workspace` (host numpy copies)."""
    o_sel, o_cnt = sals_workspace_selection_offsets(cfg, batch, max_local_len)
    k = cfg.top_k
    sel = workspace[o_sel:o_sel + batch * k * 4].view(torch.int32).view(batch, k).cpu().numpy()
    cnt = workspace[o_cnt:o_cnt + batch * 4].view(torch.int32).cpu().numpy()
    return sel, cnt


def sals_merge_partials(cfg, partial_all, world, batch, out, stream=None):
    _check(_lib.sals_merge_partials(ctypes.byref(cfg), _p(partial_all), int(world), int(batch), _p(out),
                                    _stream(stream)))


def sals_comm_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.sals_comm_unique_id(buf))
    return buf.raw


def sals_comm_init(unique_id: bytes, world: int, rank: int) -> ctypes.c_void_p:
    """Blocking over the `world` ranks; returns the opaque communicator handle."""
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    comm = ctypes.c_void_p()
    _check(_lib.sals_comm_init(buf, int(world), int(rank), ctypes.byref(comm)))
    return comm


def sals_comm_destroy(comm) -> None:
    _check(_lib.sals_comm_destroy(comm))


def sals_decode_sharded_workspace_bytes(cfg: sals_config, batch: int, max_local_len: int, world: int) -> int:
    return int(_lib.sals_decode_sharded_workspace_bytes(ctypes.byref(cfg), batch, max_local_len, world))


def sals_decode_sharded(cfg, comm, U, q, latent_shard, v_shard, shard_start, local_len, max_local_len, seq_len, out,
                        workspace, stream=None):
    _check(_lib.sals_decode_sharded(ctypes.byref(cfg), comm, _p(U), _p(q), _p(latent_shard), _p(v_shard),
                                    latent_shard.shape[1], q.shape[0], int(shard_start), _p(local_len),
                                    int(max_local_len), _p(seq_len), _p(out), _p(workspace), workspace.numel(),
                                    _stream(stream)))


def sals_append_decode_sharded(cfg, comm, U, k_new, v_new, q, latent_shard, v_shard, shard_start, local_len,
                               max_local_len, seq_len, out, workspace, stream=None):
    """sals_decode_sharded with the new token's append in the same call (the rank whose shard
    holds position seq_len - 1 writes its latent / value rows in the query projection's launch)."""
    _check(_lib.sals_append_decode_sharded(ctypes.byref(cfg), comm, _p(U), _p(k_new), _p(v_new), _p(q),
                                           _p(latent_shard), _p(v_shard), latent_shard.shape[1], q.shape[0],
                                           int(shard_start), _p(local_len), int(max_local_len), _p(seq_len), _p(out),
                                           _p(workspace), workspace.numel(), _stream(stream)))


def sals_launch_count(reset: bool = False) -> int:
    return int(_lib.sals_launch_count(1 if reset else 0))


STAGE_BITS = {"qproj_rope": 0, "score": 1, "topk": 2, "recon_attn": 3, "flash": 4, "merge": 5, "append": 6}
EXCHANGE_BIT = 7   # (sharded) the NCCL all-gathers inside sals_decode_sharded
SHARD_SELECT_BIT = 8   # (sharded) global selection + owned list (shard_select_kernel)


def sals_profile_stage_mask(mask: int) -> int:
    """Profiling only: restrict this thread's calls to the stages in `mask` (STAGE_BITS)."""
    return int(_lib.sals_profile_stage_mask(mask & 0xffffffff))


def sals_status_string(status: int) -> str:
    return _lib.sals_status_string(status).decode()


def sals_last_error() -> str:
    return _lib.sals_last_error().decode()
