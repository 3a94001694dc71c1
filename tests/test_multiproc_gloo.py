"""The N>1 (Ulysses) host logic at world size 2 over gloo on CPU.

Each rank holds a sequence shard of Q/K/V (padded to ceil(L/P) rows), packs it
with the library's own layout code (tm_ulysses_shuffle_host: the index map the
device pack/unpack kernels use), exchanges blocks with a real
torch.distributed all_to_all (gloo), unpacks to its head shard, runs the fp64
oracle on its heads, and sends O back the same way.  The result must equal
the unsharded oracle exactly (attention heads are independent), and the
unpacked head shards must equal the corresponding slices bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2506_03099_b200 import tm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _a2a(x: np.ndarray) -> np.ndarray:
    """Block p of x (first axis) goes to rank p; block q of the result came from rank q."""
    t = torch.from_numpy(np.ascontiguousarray(x))
    out = torch.empty_like(t)
    dist.all_to_all_single(out, t)
    return out.numpy()


def _seq_to_heads(shard, L, Ls, Hl, P, d):
    send = np.zeros((P, 1, Ls, Hl, d), dtype=np.float32)
    tm.tm_ulysses_shuffle_host(0, shard, send, 1, Ls, L, Hl, P, d, 4)
    recv = _a2a(send)
    heads = np.zeros((1, L, Hl, d), dtype=np.float32)
    tm.tm_ulysses_shuffle_host(1, recv, heads, 1, Ls, L, Hl, P, d, 4)
    return heads[0]


def _heads_to_seq(heads, L, Ls, Hl, P, d):
    send = np.zeros((P, 1, Ls, Hl, d), dtype=np.float32)
    tm.tm_ulysses_shuffle_host(2, np.ascontiguousarray(heads[None]), send, 1, Ls, L, Hl, P, d, 4)
    recv = _a2a(send)
    shard = np.zeros((1, Ls, Hl * P, d), dtype=np.float32)
    tm.tm_ulysses_shuffle_host(3, recv, shard, 1, Ls, L, Hl, P, d, 4)
    return shard[0]


def _worker(rank, world, port, H, d, Lr, Lc, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        rng = np.random.default_rng(2506030990)
        q, k, v = (rng.standard_normal((Lc, H, d)).astype(np.float32) for _ in range(3))
        kr, vr = (rng.standard_normal((Lr, H, d)).astype(np.float32) for _ in range(2))
        P, Hl = world, H // world
        Ls, Lrs = -(-Lc // P), -(-Lr // P)

        def shard(x, L, S):
            out = np.zeros((S, H, d), dtype=np.float32)
            lo, hi = rank * S, min(rank * S + S, L)
            if hi > lo:
                out[: hi - lo] = x[lo:hi]
            return out

        qh, kh, vh = (_seq_to_heads(shard(x, Lc, Ls), Lc, Ls, Hl, P, d) for x in (q, k, v))
        krh, vrh = (_seq_to_heads(shard(x, Lr, Lrs), Lr, Lrs, Hl, P, d) for x in (kr, vr))
        hs = slice(rank * Hl, rank * Hl + Hl)
        for got, full in ((qh, q), (kh, k), (vh, v), (krh, kr), (vrh, vr)):
            assert (got == full[:, hs]).all(), "head shard layout mismatch"
        # t = 1: attend {c_0, c_1}; t = 2 also c_{t-1} (here: reuse k/v as prev)
        for prev in (None, (kh, vh)):
            oh = oracle.stream_attention(qh, krh, vrh, None if prev is None else prev[0],
                                         None if prev is None else prev[1], kh, vh)
            o_shard = _heads_to_seq(oh.astype(np.float32), Lc, Ls, Hl, P, d)
            ref = oracle.stream_attention(q, kr, vr, None if prev is None else k,
                                          None if prev is None else v, k, v)
            lo, hi = rank * Ls, min(rank * Ls + Ls, Lc)
            assert np.abs(o_shard[: hi - lo] - ref[lo:hi].astype(np.float32)).max() == 0.0
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # report to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


@pytest.mark.parametrize("H,d,Lr,Lc", [(4, 8, 5, 7), (2, 4, 3, 8), (6, 16, 17, 33)])
def test_ulysses_exchange_world2_gloo(H, d, Lr, Lc):
    oracle.build()
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, H, d, Lr, Lc, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert all(p.exitcode == 0 for p in procs), errs


def test_shuffle_host_roundtrip_and_padding():
    """mode 0 then mode 3 is the identity on valid rows (single process, P=3,
    ragged L); mode 2 writes zero into pad rows."""
    rng = np.random.default_rng(1)
    B, P, Hl, d, L = 2, 3, 2, 4, 10
    Ls = -(-L // P)
    x = rng.standard_normal((B, Ls, P * Hl, d)).astype(np.float32)
    blk = np.zeros((P, B, Ls, Hl, d), dtype=np.float32)
    tm.tm_ulysses_shuffle_host(0, x, blk, B, Ls, L, Hl, P, d, 4)
    y = np.zeros_like(x)
    tm.tm_ulysses_shuffle_host(3, blk, y, B, Ls, L, Hl, P, d, 4)
    assert (y == x).all()
    heads = rng.standard_normal((B, L, Hl, d)).astype(np.float32)
    blk2 = np.full((P, B, Ls, Hl, d), 7.0, dtype=np.float32)
    tm.tm_ulysses_shuffle_host(2, heads, blk2, B, Ls, L, Hl, P, d, 4)
    assert (blk2[P - 1, :, L - (P - 1) * Ls:] == 0).all()   # the padded tail rows
    with pytest.raises(tm.TMError):
        tm.tm_ulysses_shuffle_host(0, x, blk, B, Ls, L, Hl, P, 3, 4)   # 12-byte rows


# ------------------------------------------------------------------ peer transport (TM_TRANSPORT_PEER)

def _peer_worker(rank, world, port, H, d, Lr, Lc, errq):
    """The peer transport's routing at world size 2 over gloo: each rank
    routes its sequence shard into P window images with the library's own
    index map (tm_peer_route_host mode 0 = the device push), the images go to
    their owners (all_to_all) and are overlaid; the oracle runs on the
    owned heads; the output rows are routed to their token owners (mode 1 =
    the attention epilogue's scatter) and overlaid again.  Every rank's O
    shard must equal the unsharded oracle rows exactly."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        rng = np.random.default_rng(2506030991)
        q, k, v = (rng.standard_normal((Lc, H, d)).astype(np.float32) for _ in range(3))
        kr, vr = (rng.standard_normal((Lr, H, d)).astype(np.float32) for _ in range(2))
        P, Hl = world, H // world
        Ls, Lrs = -(-Lc // P), -(-Lr // P)
        Lw = max(Lc, Lr)

        def shard(x, L, S):
            out = np.full((S, H, d), np.nan, dtype=np.float32)    # padding must never be read
            lo, hi = rank * S, min(rank * S + S, L)
            if hi > lo:
                out[: hi - lo] = x[lo:hi]
            return out

        def push(x, L, S):
            img = np.zeros((P, 1, Lw, Hl, d), dtype=np.float32)
            tm.tm_peer_route_host(0, shard(x, L, S), img, 1, S, L, Lw, Hl, P, rank, d, 4)
            return _a2a(img).sum(axis=0)[0]          # disjoint rows from each source

        qw, kw, vw = (push(x, Lc, Ls) for x in (q, k, v))
        hs = slice(rank * Hl, rank * Hl + Hl)
        for got, full in ((qw, q), (kw, k), (vw, v)):
            assert (got[:Lc] == full[:, hs]).all(), "window layout mismatch"
        krw, vrw = (push(x, Lr, Lrs)[:Lr] for x in (kr, vr))
        assert (krw == kr[:, hs]).all() and (vrw == vr[:, hs]).all()
        for prev in (None, (kw[:Lc], vw[:Lc])):
            oh = oracle.stream_attention(qw[:Lc], krw, vrw, None if prev is None else prev[0],
                                         None if prev is None else prev[1], kw[:Lc], vw[:Lc])
            img = np.zeros((P, 1, Ls, H, d), dtype=np.float32)
            tm.tm_peer_route_host(1, np.ascontiguousarray(oh.astype(np.float32)[None]), img, 1, Ls,
                                  Lc, Lw, Hl, P, rank, d, 4)
            o_shard = _a2a(img).sum(axis=0)[0]     # disjoint head blocks from each source
            ref = oracle.stream_attention(q, kr, vr, None if prev is None else k,
                                          None if prev is None else v, k, v)
            lo, hi = rank * Ls, min(rank * Ls + Ls, Lc)
            assert np.abs(o_shard[: hi - lo] - ref[lo:hi].astype(np.float32)).max() == 0.0
            assert (o_shard[hi - lo:] == 0).all()
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # report to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


@pytest.mark.parametrize("H,d,Lr,Lc", [(4, 8, 5, 7), (2, 4, 9, 4), (6, 16, 17, 33)])
def test_peer_routes_world2_gloo(H, d, Lr, Lc):
    oracle.build()
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, H, d, Lr, Lc, errq))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert all(p.exitcode == 0 for p in procs), errs


def test_peer_route_host_single_process():
    """mode 0 over every source rank rebuilds each owner's head slice exactly
    (P=3, ragged L, padding never routed); mode 1 over every source fills
    each owner's O window exactly once."""
    rng = np.random.default_rng(3)
    B, P, Hl, d, L = 2, 3, 2, 8, 10
    Ls, H, Lw = -(-L // P), P * Hl, 12
    full = rng.standard_normal((B, L, H, d)).astype(np.float32)
    win = np.zeros((P, B, Lw, Hl, d), dtype=np.float32)
    for r in range(P):
        sh = np.full((B, Ls, H, d), np.nan, dtype=np.float32)
        n = min(Ls, L - r * Ls)
        sh[:, :n] = full[:, r * Ls: r * Ls + n]
        tm.tm_peer_route_host(0, sh, win, B, Ls, L, Lw, Hl, P, r, d, 4)
    for p in range(P):
        assert (win[p][:, :L] == full[:, :, p * Hl:(p + 1) * Hl]).all()
        assert (win[p][:, L:] == 0).all()
    out = np.full((P, B, Ls, H, d), -1.0, dtype=np.float32)
    for r in range(P):
        tm.tm_peer_route_host(1, np.ascontiguousarray(full[:, :, r * Hl:(r + 1) * Hl]), out, B, Ls,
                              L, Lw, Hl, P, r, d, 4)
    flat = out.transpose(1, 0, 2, 3, 4).reshape(B, P * Ls, H, d)
    assert (flat[:, :L] == full).all()
    assert (flat[:, L:] == -1.0).all()          # pad rows are the receive kernel's job
