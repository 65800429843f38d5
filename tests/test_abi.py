"""C-ABI boundary checks that need no GPU: the library builds / loads, exports
every symbol include/sals.h declares, and validates arguments on the host."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sals.h")


@pytest.fixture(scope="module")
def lib_path():
    from paper_2510_24273_b200 import build
    return build.build()


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sals_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ["sals_append_latent", "sals_decode", "sals_workspace_bytes", "sals_dense_decode",
              "sals_shard_candidates", "sals_shard_attend", "sals_merge_partials"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (sals_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing


def test_binding_names_match_header(lib_path):
    from paper_2510_24273_b200 import sals
    for n in _declared():
        assert hasattr(sals, n), n
    assert sorted(sals.EXPORTED) == _declared()


def test_sm100a_code_only(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def _cfg(sals, **kw):
    base = dict(num_q_heads=32, num_kv_heads=8, head_dim=128, rank=512, score_rank=256, top_k=4096,
                rope_base=1e6, dtype="bf16")
    base.update(kw)
    return sals.make_config(**base)


def test_host_validation_without_gpu(lib_path):
    from paper_2510_24273_b200 import sals
    c = _cfg(sals)
    assert sals.sals_workspace_bytes(c, 4, 32768) > 0
    bad = [dict(score_rank=1024), dict(rank=12), dict(num_q_heads=30), dict(head_dim=96),
           dict(sink=4000, recent=200), dict(top_k=0), dict(rope_base=0.0)]
    for b in bad:
        cb = _cfg(sals, **b)
        assert sals.sals_workspace_bytes(cb, 4, 32768) == 0, b
        st = sals._lib.sals_decode(ctypes.byref(cb), None, None, None, None, 1, 1, None, 1, None, None, None,
                                   None, 0, None)
        assert st in (1, 2), (b, st)
        assert sals.sals_last_error()
    # NULL tensors are rejected synchronously
    st = sals._lib.sals_decode(ctypes.byref(c), None, None, None, None, 1, 1, None, 1, None, None, None, None, 0, None)
    assert st == 1
    st = sals._lib.sals_append_latent(ctypes.byref(c), None, None, None, 1, None, None, None, 1, None)
    assert st == 1
    assert sals.sals_status_string(3) == "SALS_ERR_WORKSPACE_TOO_SMALL"
    assert sals.sals_status_string(5) == "SALS_ERR_NCCL"
    # sharded one-call path: NULL communicator / bad rank rejected before any NCCL or CUDA work
    st = sals._lib.sals_decode_sharded(ctypes.byref(c), None, None, None, None, None, 1, 1, 0, None, 1, None, None,
                                       None, 0, None)
    assert st == 1 and "communicator" in sals.sals_last_error()
    # the window of quantised values is not sharded: refused before anything is enqueued
    cw = _cfg(sals, v_bits=4, recent=64)
    fake = ctypes.c_void_p(256)
    st = sals._lib.sals_decode_sharded(ctypes.byref(cw), fake, fake, fake, fake, fake, 4096, 1, 0, fake, 4096, fake,
                                       fake, fake, 1 << 30, None)
    assert st == 2 and "window" in sals.sals_last_error()
    # the fused sharded append: NULL k_new / v_new, or a NULL communicator, rejected up front
    st = sals._lib.sals_append_decode_sharded(ctypes.byref(c), fake, fake, None, None, fake, fake, fake, 4096, 1, 0,
                                              fake, 4096, fake, fake, fake, 1 << 30, None)
    assert st == 1
    st = sals._lib.sals_append_decode_sharded(ctypes.byref(c), None, fake, fake, fake, fake, fake, fake, 4096, 1, 0,
                                              fake, 4096, fake, fake, fake, 1 << 30, None)
    assert st == 1 and "communicator" in sals.sals_last_error()
    h = ctypes.c_void_p()
    assert sals._lib.sals_comm_init(ctypes.create_string_buffer(128), 2, 2, ctypes.byref(h)) == 1
    assert sals._lib.sals_comm_destroy(None) == 0
    w1 = sals.sals_decode_sharded_workspace_bytes(c, 1, 16384, 1)
    w8 = sals.sals_decode_sharded_workspace_bytes(c, 1, 16384, 8)
    assert w8 > w1 > sals.sals_shard_workspace_bytes(c, 1, 16384, 1) > 0


def test_workspace_monotone(lib_path):
    from paper_2510_24273_b200 import sals
    c = _cfg(sals)
    a = sals.sals_workspace_bytes(c, 1, 4096)
    b = sals.sals_workspace_bytes(c, 4, 131072)
    assert 0 < a < b
