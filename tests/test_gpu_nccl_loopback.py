"""GPU tests of the NCCL transport's data path at P > 1 on ONE device (rows
a2 / a6, the Ulysses exchange of P:171, "NCCL + CUDA streams" P:183;
SURVEY Sec 4.3 T2):

P virtual ranks in one process form a LOOPBACK group
(tm_nccl_connect_local): every call runs exactly as with a communicator --
pack kernel (seq -> per-peer blocks), all-to-all, unpack kernel (received
blocks -> head shard; K/V straight into the cache slot), head-sharded
attention, pack of O, all-to-all, unpack to the sequence shard -- except that
the all-to-all itself is the same block permutation done with device copies
between the ranks' workspaces (NCCL cannot hold several ranks on one GPU).

Checked: every rank's head block of the assembled output equals a direct
one-GPU context over those heads bit for bit (the same kernel, schedule and
split), shard padding rows are zero, and the whole output is within the bf16
alarm (fp32: the 1e-4 bar) of the fp64 oracle.
"""
import numpy as np
import pytest
import torch

import oracle
from gpu_util import BF16_ALARM, FP32_TOL, from_dev, rel_err, sample_rows, to_dev
from paper_2506_03099_b200 import tm
from synthetic import inputs as syn

pytestmark = pytest.mark.gpu

NCCL = tm.TM_TRANSPORT_NCCL


def bits(x):
    if x.dtype == torch.bfloat16:
        return x.view(torch.int16).cpu().numpy()
    return x.view(torch.int32).cpu().numpy()


def shard(x, L, P, r, fill=float("nan")):
    """Rows [r*Ls, r*Ls+Ls) of a [..., L, H, d] tensor (token axis -3), padded
    to Ls rows with NaN (padding must never be read)."""
    Ls = -(-L // P)
    shape = list(x.shape)
    shape[-3] = Ls
    out = torch.full(shape, fill, dtype=x.dtype, device=x.device)
    lo, hi = r * Ls, min(r * Ls + Ls, L)
    if hi > lo:
        out[..., : hi - lo, :, :] = x[..., lo:hi, :, :]
    return out


def make_inputs(H, d, Lr, Lc, chunks, seed, dtype="bf16"):
    si = syn.StreamInputs(H, d, Lr, Lc, dtype, "D0", seed)
    host = [si.chunk(0, 0, t) for t in range(chunks + 1)]
    dev = [tuple(None if x is None else to_dev(x) for x in c) for c in host]
    return host, dev


def direct_stream(H, d, Lr, Lc, inputs, heads, dtype=tm.TM_BF16):
    Hh = heads.stop - heads.start
    ca = tm.ChunkAttention(Hh, d, Lr, Lc, 1, 1, dtype=dtype)
    _, kr, vr = inputs[0]
    ca.put_reference(0, 0, kr[:, heads].contiguous(), vr[:, heads].contiguous())
    outs = []
    for t, (q, k, v) in enumerate(inputs[1:], start=1):
        o = torch.empty(Lc, Hh, d, dtype=q.dtype, device="cuda")
        ca.attend(0, 0, t, q[:, heads].contiguous(), k[:, heads].contiguous(),
                  v[:, heads].contiguous(), o)
        outs.append(o)
    torch.cuda.synchronize()
    ca.close()
    return outs


def run_loopback(P, H, d, Lr, Lc, dev, dtype=tm.TM_BF16):
    """The stream of chunks 1.. through a P-rank loopback group; returns the
    assembled [Lc][H][d] outputs (and checks the shard padding rows)."""
    cas = [tm.ChunkAttention(H, d, Lr, Lc, 1, 1, dtype=dtype, world_size=P, rank=r,
                             transport=NCCL) for r in range(P)]
    tm.ChunkAttention.nccl_connect_local(cas)
    _, kr, vr = dev[0]
    for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
        for r in range(P):
            cas[r].put_reference_phases(0, 0, shard(kr, Lr, P, r), shard(vr, Lr, P, r), ph)
    outs = []
    for t in range(1, len(dev)):
        q, k, v = dev[t]
        qs, ks, vs = ([shard(x, Lc, P, r) for r in range(P)] for x in (q, k, v))
        os_ = [torch.full_like(qs[r], 7.0) for r in range(P)]
        for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
            for r in range(P):
                cas[r].attend_phases(0, 0, t, qs[r], ks[r], vs[r], os_[r], ph)
        torch.cuda.synchronize()
        full = torch.cat(os_, dim=0)
        assert (bits(full[Lc:]) == 0).all(), "shard padding rows must be zero"
        outs.append(full[:Lc].contiguous())
    for c in cas:
        c.check()
        c.close()
    return outs


def oracle_check(host, outs, tol):
    so = oracle.StreamOracle()
    _, kr, vr = host[0]
    so.put_reference(0, 0, kr.f64, vr.f64)
    for t, o in enumerate(outs, start=1):
        q, k, v = host[t]
        L = q.f64.shape[0]
        rows = sample_rows(L, k=48) if L > 1024 else None
        ref = so.attend(0, 0, t, q.f64, k.f64, v.f64, rows=rows)
        got = from_dev(o)
        assert rel_err(got if rows is None else got[rows], ref) <= tol


@pytest.mark.parametrize("P,Lr,Lc", [(2, 200, 333), (3, 97, 400), (4, 300, 1000), (8, 300, 1000),
                                    (8, 1024, 3072)])
def test_nccl_loopback_bitwise_per_head_block(P, Lr, Lc):
    """P = 2/3/4/8 virtual ranks, NCCL transport: the pack -> all-to-all ->
    unpack -> attention -> pack -> all-to-all -> unpack path reproduces, per
    head block, the direct one-GPU path bit for bit.  (8, 300, 1000): 125-row
    shards; (8, 1024, 3072): the WAN-512 config at one node's P = 8."""
    H = 40 if Lc >= 3072 else (6 if P == 3 else 8)
    d = 128
    host, dev = make_inputs(H, d, Lr, Lc, 3, syn.seed_for(21, P))
    outs = run_loopback(P, H, d, Lr, Lc, dev)
    Hl = H // P
    for r in range(P):
        hb = slice(r * Hl, (r + 1) * Hl)
        ref = direct_stream(H, d, Lr, Lc, dev, hb)
        for a, b in zip(outs, ref):
            assert (bits(a[:, hb].contiguous()) == bits(b)).all(), f"rank {r}"
    oracle_check(host, outs, BF16_ALARM)


@pytest.mark.parametrize("P", [2, 4])
def test_nccl_loopback_fp32_validation_mode(P):
    """The fp32 validation mode uses the NCCL transport at P > 1: loopback
    P = 2 / 4 against the direct fp32 path (bitwise per head block) and the
    1e-4 bar of the fp64 oracle."""
    H, d, Lr, Lc = 8, 64, 100, 250
    host, dev = make_inputs(H, d, Lr, Lc, 2, syn.seed_for(22, P), dtype="fp32")
    outs = run_loopback(P, H, d, Lr, Lc, dev, dtype=tm.TM_FP32)
    Hl = H // P
    for r in range(P):
        hb = slice(r * Hl, (r + 1) * Hl)
        ref = direct_stream(H, d, Lr, Lc, dev, hb, dtype=tm.TM_FP32)
        for a, b in zip(outs, ref):
            assert (bits(a[:, hb].contiguous()) == bits(b)).all(), f"rank {r}"
    oracle_check(host, outs, FP32_TOL)


def test_nccl_loopback_equals_peer_transport():
    """Both transports shard heads identically: the loopback NCCL group and a
    peer-transport group of the same size give the same output bit for bit."""
    P, H, d, Lr, Lc = 4, 8, 128, 256, 1000
    _, dev = make_inputs(H, d, Lr, Lc, 2, syn.seed_for(23, 0))
    a = run_loopback(P, H, d, Lr, Lc, dev)
    cas = [tm.ChunkAttention(H, d, Lr, Lc, 1, 1, world_size=P, rank=r,
                             transport=tm.TM_TRANSPORT_PEER) for r in range(P)]
    tm.ChunkAttention.connect_local(cas)
    _, kr, vr = dev[0]
    for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
        for r in range(P):
            cas[r].put_reference_phases(0, 0, shard(kr, Lr, P, r), shard(vr, Lr, P, r), ph)
    for t in (1, 2):
        q, k, v = dev[t]
        os_ = [torch.empty_like(shard(q, Lc, P, r)) for r in range(P)]
        for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
            for r in range(P):
                cas[r].attend_phases(0, 0, t, shard(q, Lc, P, r), shard(k, Lc, P, r),
                                     shard(v, Lc, P, r), os_[r], ph)
        torch.cuda.synchronize()
        b = torch.cat(os_, dim=0)[:Lc].contiguous()
        assert (bits(a[t - 1]) == bits(b)).all(), t
    for c in cas:
        c.check()
        c.close()


def test_nccl_loopback_batch_layers_steps_shared_reference():
    """Loopback P = 4, batch 2, d = 64, Lr > Lc, 2 layers x 2 steps, a shared
    reference (step = -1, exchanged once then aliased) and a redo of chunk 2:
    every output equals, per head block, a direct context over those heads."""
    P, H, d, Lr, Lc, B, L_, S_ = 4, 8, 64, 700, 300, 2, 2, 2
    g = torch.Generator(device="cuda").manual_seed(9)
    mk = lambda L: torch.randn(B, L, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
    cas = [tm.ChunkAttention(H, d, Lr, Lc, L_, S_, batch=B, world_size=P, rank=r, transport=NCCL)
           for r in range(P)]
    tm.ChunkAttention.nccl_connect_local(cas)
    Hl = H // P
    dirs = [tm.ChunkAttention(Hl, d, Lr, Lc, L_, S_, batch=B) for _ in range(P)]
    for l in range(L_):
        kr, vr = mk(Lr), mk(Lr)
        for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
            for r in range(P):
                cas[r].put_reference_phases(l, -1, shard(kr, Lr, P, r), shard(vr, Lr, P, r), ph)
        for r in range(P):
            hb = slice(r * Hl, (r + 1) * Hl)
            dirs[r].put_reference(l, -1, kr[:, :, hb].contiguous(), vr[:, :, hb].contiguous())
    for t in (1, 2, 2, 3):
        for st in range(S_):
            for l in range(L_):
                q, k, v = mk(Lc), mk(Lc), mk(Lc)
                os_ = [torch.empty(B, -(-Lc // P), H, d, dtype=torch.bfloat16, device="cuda")
                       for _ in range(P)]
                for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
                    for r in range(P):
                        cas[r].attend_phases(l, st, t, shard(q, Lc, P, r), shard(k, Lc, P, r),
                                             shard(v, Lc, P, r), os_[r], ph)
                full = torch.cat(os_, dim=1)[:, :Lc]
                for r in range(P):
                    hb = slice(r * Hl, (r + 1) * Hl)
                    o = torch.empty(B, Lc, Hl, d, dtype=torch.bfloat16, device="cuda")
                    dirs[r].attend(l, st, t, q[:, :, hb].contiguous(), k[:, :, hb].contiguous(),
                                   v[:, :, hb].contiguous(), o)
                    assert (bits(full[:, :, hb].contiguous()) == bits(o)).all(), (t, st, l, r)
    for c in cas + dirs:
        c.close()


def test_nccl_loopback_errors():
    """Unconnected loopback contexts refuse to exchange; phased calls are
    accepted only once the group is connected; connect checks the ranks."""
    H, d, Lr, Lc, P = 4, 64, 64, 128, 2
    cas = [tm.ChunkAttention(H, d, Lr, Lc, 1, 1, world_size=P, rank=r, transport=NCCL)
           for r in range(P)]
    kr = torch.zeros(Lr // P, H, d, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(tm.TMError) as e:
        cas[0].put_reference(0, 0, kr, kr)
    assert e.value.status == 4
    with pytest.raises(tm.TMError) as e:            # wrong rank order
        tm.tm_nccl_connect_local([cas[1].ctx, cas[0].ctx])
    assert e.value.status == 1
    tm.ChunkAttention.nccl_connect_local(cas)
    with pytest.raises(tm.TMError) as e:            # already connected
        tm.ChunkAttention.nccl_connect_local(cas)
    assert e.value.status == 4
    for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
        for r in range(P):
            cas[r].put_reference_phases(0, 0, kr, kr, ph)
    for c in cas:
        c.close()
