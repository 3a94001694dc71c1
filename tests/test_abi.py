"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/tm.h declares, and its host logic (config validation, the
closed-form cache size) works without a GPU."""
import ctypes
import os
import re

import pytest

from paper_2506_03099_b200 import tm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "tm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(tm_[a-z_0-9]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert "tm_chunk_attention" in names and "tm_flow_euler_step" in names
    lib = ctypes.CDLL(tm.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), f"libtm.so does not export {n}"
    assert set(names) == set(tm.EXPORTED)


def test_version():
    assert tm.tm_version() == 102


def wan512(**kw):
    base = dict(heads=40, head_dim=128, ref_tokens=1024, chunk_tokens=3072, num_layers=40,
                num_steps=2)
    base.update(kw)
    return tm.make_config(**base)


def test_cache_bytes_closed_form():
    """Constant memory: ref + 2 slots of K and V per
    (layer, step); 10.94 GiB / P at 512^2."""
    c = wan512()
    per_tok = 40 * 128 * 2
    expect = 40 * 2 * (2 * 1024 * per_tok + 4 * 3072 * per_tok)
    assert tm.tm_kvcache_bytes(c) == expect
    assert abs(expect / 2**30 - 10.9375) < 1e-9
    for P in (2, 4, 8):
        assert tm.tm_kvcache_bytes(wan512(world_size=P)) == expect // P


def test_cache_bytes_720_and_alignment():
    c = tm.make_config(40, 128, 2025, 6075, 40, 2)
    per_tok = 40 * 128 * 2
    al = lambda x: (x + 1023) // 1024 * 1024
    assert tm.tm_kvcache_bytes(c) == 80 * (2 * al(2025 * per_tok) + 4 * al(6075 * per_tok))


@pytest.mark.parametrize("bad", [
    dict(head_dim=96), dict(head_dim=0), dict(heads=0), dict(ref_tokens=0), dict(chunk_tokens=-1),
    dict(world_size=3), dict(world_size=2, rank=2), dict(dtype=5), dict(num_steps=0),
    dict(batch=0), dict(softmax_scale=-1.0), dict(transport=2),
    dict(transport=tm.TM_TRANSPORT_PEER, dtype=tm.TM_FP32),
    dict(transport=tm.TM_TRANSPORT_PEER, heads=40, world_size=10)])
def test_invalid_configs_are_rejected(bad):
    c = wan512(**bad)
    assert tm.tm_kvcache_bytes(c) == 0
    assert tm.tm_workspace_bytes(c) == 0
    with pytest.raises(tm.TMError) as e:
        tm.tm_attn_init(c, None, 1024, 1 << 40, 1024, 1 << 20)
    assert e.value.status in (1, 2, 7)


def test_workspace_sizes():
    # bf16: debug flag + split-KV scratch: 1 partial slot per (schedule block <= 8, persistent
    # CTA <= 160; three fp16 tile partials fit it) + two 64-bit contributor masks (one per Q tile)
    scratch = 8 * 160 * (256 * 128 + 512) * 4 + 8 * 160 * 2 * 8
    assert tm.tm_workspace_bytes(wan512()) == 1024 + (scratch + 1023) // 1024 * 1024
    assert tm.tm_workspace_bytes(wan512(dtype=tm.TM_FP32)) == 1024
    ws8 = tm.tm_workspace_bytes(wan512(world_size=8))
    shard = 384 * 40 * 128 * 2          # [Lc/8][H][d] bf16
    assert ws8 >= 1024 + 2 * 3 * shard + 2 * 3072 * 5 * 128 * 2


def test_null_and_error_paths_without_gpu():
    with pytest.raises(tm.TMError):
        tm.tm_attn_init(wan512(), None, 0, 0, 0, 0)
    # Euler argument validation happens before any launch
    with pytest.raises(tm.TMError):
        tm.tm_flow_euler_step(None, 0, 0, tm.TM_FP32, 10, 0.5)
    with pytest.raises(tm.TMError):
        tm.tm_flow_euler_step(None, 16, 16, 7, 10, 0.5)
    tm.tm_flow_euler_step(None, 0, 0, tm.TM_FP32, 0, 0.5)   # n == 0 is a no-op
    assert tm.tm_last_launch_count(None) == -1


def test_init_without_device_reports_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(tm.TMError) as e:
        tm.tm_attn_init(wan512(), None, 1024, 1 << 40, 1024, 1 << 30)
    assert e.value.status == 8


def test_cache_bytes_table1_variants():
    """f3: chunk 7 x 4 steps at 512^2: ref + 2 slots per (layer, step)."""
    c = tm.make_config(40, 128, 1024, 7168, 40, 4)
    per_tok = 40 * 128 * 2
    assert tm.tm_kvcache_bytes(c) == 160 * (2 * 1024 * per_tok + 4 * 7168 * per_tok)


def test_peer_workspace_layout():
    """TM_TRANSPORT_PEER: the workspace ends in the peer window: 4 KiB of
    counters, Q/K/V windows [B][max(Lc,Lr)][H/P][d] and the O window
    [B][ceil(Lc/P)][H][d], each 1024-B aligned; no NCCL staging."""
    al = lambda x: (x + 1023) // 1024 * 1024
    scratch = 1024 + al(8 * 160 * (256 * 128 + 512) * 4 + 8 * 160 * 2 * 8)
    for P in (1, 2, 8):
        c = wan512(world_size=P, transport=tm.TM_TRANSPORT_PEER)
        win = 4096 + 3 * al(3072 * (40 // P) * 128 * 2) + al(-(-3072 // P) * 40 * 128 * 2)
        assert tm.tm_workspace_bytes(c) == scratch + win
    c = tm.make_config(40, 128, 2025, 6075, 40, 2, world_size=8, transport=tm.TM_TRANSPORT_PEER)
    win = 4096 + 3 * al(6075 * 5 * 128 * 2) + al(760 * 40 * 128 * 2)
    assert tm.tm_workspace_bytes(c) == scratch + win
    # Lr > Lc: the K/V windows also carry the reference push
    c = tm.make_config(4, 64, 500, 100, 1, 1, world_size=2, transport=tm.TM_TRANSPORT_PEER)
    scratch64 = 1024 + al(8 * 160 * (256 * 64 + 512) * 4 + 8 * 160 * 2 * 8)
    assert tm.tm_workspace_bytes(c) == scratch64 + 4096 + 3 * al(500 * 2 * 64 * 2) + al(50 * 4 * 64 * 2)


def test_sched_heads_validation_host():
    """tm_config.sched_heads must be 0 or divide the heads per rank."""
    assert tm.tm_kvcache_bytes(tm.make_config(40, 128, 1024, 3072, 1, 1, sched_heads=5)) > 0
    assert tm.tm_kvcache_bytes(tm.make_config(40, 128, 1024, 3072, 1, 1, sched_heads=3)) == 0
    assert tm.tm_kvcache_bytes(tm.make_config(40, 128, 1024, 3072, 1, 1, world_size=8,
                                              sched_heads=5)) > 0
    assert tm.tm_kvcache_bytes(tm.make_config(40, 128, 1024, 3072, 1, 1, world_size=8,
                                              sched_heads=10)) == 0
    assert tm.tm_kvcache_bytes(tm.make_config(40, 128, 1024, 3072, 1, 1, sched_heads=-1)) == 0
