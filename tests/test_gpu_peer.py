"""GPU tests of the peer-memory Ulysses transport (TM_TRANSPORT_PEER; rows
a2/a6 over NVLink peer memory) on ONE device:

- a one-rank group runs the FUSED kernel (in-kernel push of Q/K/V into its
  own window, counter waits, epilogue scatter into the O window, done
  signal, receive kernel): bitwise equal to the direct single-GPU path;
- P = 2, 4, 8 virtual ranks in one process (tm_peer_connect_local), their
  phases enqueued rank by rank (SEND, ATTEND, RECV): every rank's head block
  of the assembled output is bitwise equal to a direct single-GPU context
  over those heads (the same kernel schedule), and the whole output is
  within the bf16 bar of the fp64 oracle;
- two PROCESSES on the one device, windows mapped with CUDA IPC, every call
  fused and collective (the multi-GPU code path; the GPU time-slices the two
  contexts, so each rank's waits are met by the other's pushes).
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from gpu_util import BF16_ALARM, from_dev, rel_err, sample_rows, to_dev
from paper_2506_03099_b200 import tm
from synthetic import inputs as syn

pytestmark = pytest.mark.gpu

PEER = tm.TM_TRANSPORT_PEER


def bits(x):
    return x.view(torch.int16).cpu().numpy()


def shard(x, L, P, r, fill=float("nan")):
    """Rows [r*Ls, r*Ls+Ls) of a [L][H][d] device tensor, padded to Ls rows
    with NaN (the padding must never be read)."""
    Ls = -(-L // P)
    out = torch.full((Ls,) + tuple(x.shape[1:]), fill, dtype=x.dtype, device=x.device)
    lo, hi = r * Ls, min(r * Ls + Ls, L)
    if hi > lo:
        out[: hi - lo] = x[lo:hi]
    return out


def direct_stream(H, d, Lr, Lc, inputs, heads=None):
    """Outputs of the direct single-GPU path for chunks 1.. of `inputs`
    (list of (q, k, v) full tensors; inputs[0] = reference), optionally over
    a head sub-range."""
    hs = slice(None) if heads is None else heads
    Hh = H if heads is None else heads.stop - heads.start
    ca = tm.ChunkAttention(Hh, d, Lr, Lc, 1, 1)
    _, kr, vr = inputs[0]
    ca.put_reference(0, 0, kr[:, hs].contiguous(), vr[:, hs].contiguous())
    outs = []
    for t, (q, k, v) in enumerate(inputs[1:], start=1):
        o = torch.empty(Lc, Hh, d, dtype=torch.bfloat16, device="cuda")
        ca.attend(0, 0, t, q[:, hs].contiguous(), k[:, hs].contiguous(), v[:, hs].contiguous(), o)
        outs.append(o)
    torch.cuda.synchronize()
    ca.close()
    return outs


def make_inputs(H, d, Lr, Lc, chunks, seed):
    si = syn.StreamInputs(H, d, Lr, Lc, "bf16", "D0", seed)
    host = [si.chunk(0, 0, t) for t in range(chunks + 1)]
    dev = [tuple(None if x is None else to_dev(x) for x in c) for c in host]
    return host, dev


def oracle_check(host, outs):
    so = oracle.StreamOracle()
    _, kr, vr = host[0]
    so.put_reference(0, 0, kr.f64, vr.f64)
    for t, o in enumerate(outs, start=1):
        q, k, v = host[t]
        L = q.f64.shape[0]
        rows = sample_rows(L, k=48) if L > 1024 else None
        ref = so.attend(0, 0, t, q.f64, k.f64, v.f64, rows=rows)
        got = from_dev(o)
        assert rel_err(got if rows is None else got[rows], ref) <= BF16_ALARM


@pytest.mark.parametrize("separate", [False, True])
@pytest.mark.parametrize("Lr,Lc", [(200, 333), (1024, 3072)])
def test_peer_one_rank_bitwise_equals_direct(separate, Lr, Lc, monkeypatch):
    """P = 1 peer group: the fused kernel (or, with TM_PEER_SEPARATE_PUSH=1,
    push kernel + attention) through the window must reproduce the direct
    path bit for bit, including c_{t-1} appended from the window."""
    if separate:
        monkeypatch.setenv("TM_PEER_SEPARATE_PUSH", "1")
    H, d = 8, 128
    host, dev = make_inputs(H, d, Lr, Lc, 3, syn.seed_for(11, 0))
    ref = direct_stream(H, d, Lr, Lc, dev)
    ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1, transport=PEER)
    _, kr, vr = dev[0]
    ca.put_reference(0, 0, kr, vr)
    outs = []
    for t in (1, 2, 3):
        q, k, v = dev[t]
        o = torch.empty_like(q)
        ca.attend(0, 0, t, q, k, v, o)
        assert ca.launches == (3 if separate else 2)
        outs.append(o)
    ca.check()
    for a, b in zip(outs, ref):
        assert (bits(a) == bits(b)).all()
    oracle_check(host, outs)
    ca.close()


def _run_virtual(P, H, d, Lr, Lc, dev, layers=1):
    cas = [tm.ChunkAttention(H, d, Lr, Lc, layers, 1, world_size=P, rank=r, transport=PEER)
           for r in range(P)]
    tm.ChunkAttention.connect_local(cas)
    _, kr, vr = dev[0]
    krs = [shard(kr, Lr, P, r) for r in range(P)]
    vrs = [shard(vr, Lr, P, r) for r in range(P)]
    for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
        for r in range(P):
            cas[r].put_reference_phases(0, 0, krs[r], vrs[r], ph)
    outs = []
    for t in range(1, len(dev)):
        q, k, v = dev[t]
        qs, ks, vs = ([shard(x, Lc, P, r) for r in range(P)] for x in (q, k, v))
        os_ = [torch.full_like(qs[r], 7.0) for r in range(P)]
        for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
            for r in range(P):
                cas[r].attend_phases(0, 0, t, qs[r], ks[r], vs[r], os_[r], ph)
        torch.cuda.synchronize()
        Ls = -(-Lc // P)
        full = torch.cat(os_, dim=0)
        assert (bits(full[Lc:]) == 0).all(), "shard padding rows must be zero"
        outs.append(full[:Lc].contiguous())
    for c in cas:
        c.check()
        c.close()
    return outs


@pytest.mark.parametrize("P,Lr,Lc", [(2, 200, 333), (3, 97, 400), (4, 1024, 3072), (8, 300, 1000),
                                    (8, 2025, 6075)])
def test_peer_virtual_ranks_bitwise_per_head_block(P, Lr, Lc):
    """P virtual ranks on one device: rank r's heads [r*Hl, (r+1)*Hl) of the
    assembled output equal a direct context over those heads bit for bit
    (same kernel, same schedule); the whole output is within the bf16 bar of
    the oracle.  (8, 300, 1000): shards of 125 rows, so Q and K/V tiles span
    two source ranks; (8, 2025, 6075): the 720^2 shape, ragged shards, also
    checked against the oracle on sampled rows."""
    H, d = 40 if Lc >= 3072 else (6 if P == 3 else 8), 128
    host, dev = make_inputs(H, d, Lr, Lc, 3, syn.seed_for(12, P))
    outs = _run_virtual(P, H, d, Lr, Lc, dev)
    Hl = H // P
    for r in range(P):
        hb = slice(r * Hl, (r + 1) * Hl)
        ref = direct_stream(H, d, Lr, Lc, dev, heads=hb)
        for a, b in zip(outs, ref):
            assert (bits(a[:, hb].contiguous()) == bits(b)).all(), f"rank {r}"
    oracle_check(host, outs)             # row-sampled at the large shapes (incl. 720^2)


def test_peer_virtual_ranks_batch_layers_steps_d64():
    """Virtual P = 4 with batch 2, head_dim 64, Lr > Lc (the K/V windows carry
    the longer reference push), 2 layers x 2 steps (separate cache regions and
    epochs interleaved), a shared reference (step = -1) and a redo of chunk 2:
    every output equals, per head block, a direct context over those heads."""
    P, H, d, Lr, Lc, B, L_, S_ = 4, 8, 64, 700, 300, 2, 2, 2
    g = torch.Generator(device="cuda").manual_seed(7)
    mk = lambda L: torch.randn(B, L, H, d, device="cuda", dtype=torch.bfloat16, generator=g)

    def shard_b(x, L, r):
        return torch.stack([shard(x[b], L, P, r) for b in range(B)])

    cas = [tm.ChunkAttention(H, d, Lr, Lc, L_, S_, batch=B, world_size=P, rank=r, transport=PEER)
           for r in range(P)]
    tm.ChunkAttention.connect_local(cas)
    Hl = H // P
    dirs = [tm.ChunkAttention(Hl, d, Lr, Lc, L_, S_, batch=B) for _ in range(P)]
    refs = {l: (mk(Lr), mk(Lr)) for l in range(L_)}
    for l in range(L_):
        kr, vr = refs[l]
        for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
            for r in range(P):
                cas[r].put_reference_phases(l, -1, shard_b(kr, Lr, r), shard_b(vr, Lr, r), ph)
        for r in range(P):
            hb = slice(r * Hl, (r + 1) * Hl)
            dirs[r].put_reference(l, -1, kr[:, :, hb].contiguous(), vr[:, :, hb].contiguous())
    for t in (1, 2, 2, 3):                       # chunk 2 twice: a redo (same c_{t-1})
        for st in range(S_):
            for l in range(L_):
                q, k, v = mk(Lc), mk(Lc), mk(Lc)
                os_ = [torch.empty(B, -(-Lc // P), H, d, dtype=torch.bfloat16, device="cuda")
                       for _ in range(P)]
                for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
                    for r in range(P):
                        cas[r].attend_phases(l, st, t, shard_b(q, Lc, r), shard_b(k, Lc, r),
                                             shard_b(v, Lc, r), os_[r], ph)
                full = torch.cat(os_, dim=1)[:, :Lc]
                for r in range(P):
                    hb = slice(r * Hl, (r + 1) * Hl)
                    o = torch.empty(B, Lc, Hl, d, dtype=torch.bfloat16, device="cuda")
                    dirs[r].attend(l, st, t, q[:, :, hb].contiguous(), k[:, :, hb].contiguous(),
                                   v[:, :, hb].contiguous(), o)
                    assert (bits(full[:, :, hb].contiguous()) == bits(o)).all(), (t, st, l, r)
    for c in cas + dirs:
        if c in cas:
            c.check()
        c.close()


def test_peer_phase_order_errors():
    """Phased operations: must start with SEND, continue in order with the
    same arguments, and nothing else may start in between (host errors, no
    launch)."""
    H, d, Lr, Lc, P = 4, 64, 64, 128, 2
    cas = [tm.ChunkAttention(H, d, Lr, Lc, 1, 1, world_size=P, rank=r, transport=PEER)
           for r in range(P)]
    kr = torch.zeros(Lr // P, H, d, dtype=torch.bfloat16, device="cuda")
    q = torch.zeros(Lc // P, H, d, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(tm.TMError) as e:          # not connected yet
        cas[0].put_reference(0, 0, kr, kr)
    assert e.value.status == 4
    tm.ChunkAttention.connect_local(cas)
    with pytest.raises(tm.TMError) as e:
        cas[0].put_reference_phases(0, 0, kr, kr, tm.TM_PHASE_ATTEND)
    assert e.value.status == 4
    with pytest.raises(tm.TMError) as e:
        cas[0].put_reference_phases(0, 0, kr, kr, tm.TM_PHASE_SEND | tm.TM_PHASE_RECV)
    assert e.value.status == 1
    for r in range(P):
        cas[r].put_reference_phases(0, 0, kr, kr, tm.TM_PHASE_SEND)
    with pytest.raises(tm.TMError) as e:          # a chunk while the reference is in flight
        cas[0].attend_phases(0, 0, 1, q, q, q, q, tm.TM_PHASE_SEND)
    assert e.value.status == 4
    with pytest.raises(tm.TMError) as e:          # skipping ATTEND
        cas[0].put_reference_phases(0, 0, kr, kr, tm.TM_PHASE_RECV)
    assert e.value.status == 4
    for ph in (tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
        for r in range(P):
            cas[r].put_reference_phases(0, 0, kr, kr, ph)
    o = [torch.empty_like(q) for _ in range(P)]
    for r in range(P):
        cas[r].attend_phases(0, 0, 1, q, q, q, o[r], tm.TM_PHASE_SEND)
    with pytest.raises(tm.TMError) as e:          # a later phase with other arguments
        cas[0].attend_phases(0, 0, 1, q, q, q, o[1], tm.TM_PHASE_ATTEND)
    assert e.value.status == 4
    for ph in (tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
        for r in range(P):
            cas[r].attend_phases(0, 0, 1, q, q, q, o[r], ph)
    for c in cas:
        c.check()
        c.close()


# ------------------------------------------------------------------ two processes, CUDA IPC

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, H, d, Lr, Lc, outdir, errq, zero_copy=False):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        host, dev = make_inputs(H, d, Lr, Lc, 3, syn.seed_for(13, 0))
        ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1, world_size=world, rank=rank, transport=PEER)
        ca.connect_dist()
        _, kr, vr = dev[0]
        ca.put_reference(0, 0, shard(kr, Lr, world, rank), shard(vr, Lr, world, rank))
        for t in (1, 2, 3):
            q, k, v = dev[t]
            o = ca.output_window()[0] if zero_copy else torch.full_like(shard(q, Lc, world, rank), 7.0)
            ca.attend(0, 0, t, shard(q, Lc, world, rank), shard(k, Lc, world, rank),
                      shard(v, Lc, world, rank), o)
            if zero_copy:
                assert ca.launches == 1        # the fused kernel waits for every rank itself
            torch.cuda.synchronize()
            ob = bits(o)
            if zero_copy:                      # shard padding rows are unspecified there
                n = min(-(-Lc // world), Lc - rank * (-(-Lc // world)))
                ob[n:] = 0
            np.save(os.path.join(outdir, f"o_r{rank}_t{t}.npy"), ob)
        ca.check()
        dist.barrier()
        ca.close()
        dist.destroy_process_group()
    except BaseException as e:
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


@pytest.mark.parametrize("P,zero_copy", [(2, False), (4, False), (8, False), (2, True), (8, True)])
def test_peer_two_processes_ipc_fused(tmp_path, P, zero_copy):
    """World size 2 (and 4) as processes sharing the device: windows exchanged
    as CUDA IPC handles over torch.distributed (gloo), every call fused (push
    in the attention kernel, epilogue scatter, receive).  Each rank's shard of
    the output equals the direct path's rows bit for bit per head block.  At
    P = 4 and 8 the shards are 250 and 125 rows, so Q and K/V tiles span two
    source ranks; P = 8 is the node-size group of the multi-GPU benchmark.
    zero_copy: o is the rank's O window (as bench.py runs it), so the fused
    kernel's last CTA waits for every rank and no receive kernel follows."""
    import torch.multiprocessing as mp
    H, d, Lr, Lc = 8, 128, 256, 1000
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker,
                         args=(r, P, port, H, d, Lr, Lc, str(tmp_path), errq, zero_copy))
             for r in range(P)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=400)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    for p in procs:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), errs
    _, dev = make_inputs(H, d, Lr, Lc, 3, syn.seed_for(13, 0))
    Hl, Ls = H // P, -(-Lc // P)
    for r in range(P):
        ref = direct_stream(H, d, Lr, Lc, dev, heads=slice(r * Hl, (r + 1) * Hl))
        for t in (1, 2, 3):
            full = np.concatenate([np.load(tmp_path / f"o_r{s}_t{t}.npy") for s in range(P)])
            assert (full[Lc:] == 0).all()
            assert (full[:Lc, r * Hl:(r + 1) * Hl] == bits(ref[t - 1])).all(), (r, t)


def test_peer_zero_copy_output_window():
    """tm_peer_output_ptr: passing the O window as `o` skips the receive copy;
    the valid rows equal the copying path's output bit for bit."""
    P, H, d, Lr, Lc = 2, 8, 128, 300, 333
    host, dev = make_inputs(H, d, Lr, Lc, 2, syn.seed_for(14, 0))
    ref = _run_virtual(P, H, d, Lr, Lc, dev)
    cas = [tm.ChunkAttention(H, d, Lr, Lc, 1, 1, world_size=P, rank=r, transport=PEER)
           for r in range(P)]
    tm.ChunkAttention.connect_local(cas)
    _, kr, vr = dev[0]
    for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
        for r in range(P):
            cas[r].put_reference_phases(0, 0, shard(kr, Lr, P, r), shard(vr, Lr, P, r), ph)
    wins = [c.output_window() for c in cas]
    Ls = -(-Lc // P)
    for t in (1, 2):
        q, k, v = dev[t]
        for ph in (tm.TM_PHASE_SEND, tm.TM_PHASE_ATTEND, tm.TM_PHASE_RECV):
            for r in range(P):
                cas[r].attend_phases(0, 0, t, shard(q, Lc, P, r), shard(k, Lc, P, r),
                                     shard(v, Lc, P, r), wins[r][0], ph)
        torch.cuda.synchronize()
        full = torch.cat([w[0] for w in wins], dim=0)[:Lc]
        assert cas[0].launches == 1            # the wait kernel only, no copy
        assert (bits(full.contiguous()) == bits(ref[t - 1])).all(), t
    for c in cas:
        c.check()
        c.close()
