#!/usr/bin/env python
"""Projected Ulysses scaling from one GPU (no multi-GPU box this round).

Measures, on one B200: the attention kernel for one rank's heads (H/P of 40)
at P = 1, 2, 4, 8 for WAN-512 and WAN-720 (zero-copy calls, kernel only), and
the peer receive kernel's cost; then models
    t(P) = t_kernel(H/P) + t_Q(P) + t_done
with t_done ~1 us: with the zero-copy output bench.py uses, the fused kernel's
last CTA waits for every rank's done signal itself (one round of system-scope
acquires), no receive kernel.  The copying receive kernel is measured too.
with t_Q the exposed Q push (the remote share of this rank's Q shard over
NVLink at 900 GB/s; K/V are pushed while the cached segments are attended)
and prints E(P) = t(1) / (P t(P)).  A model, not a measurement: the driver's
multi-GPU run is the number that counts.
    python tools/scale_model.py [out.json]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

NVLINK_GBS = 900.0


def kernel_us(H, d, Lr, Lc, reps=40):
    NL = 8
    ca = tm.ChunkAttention(H, d, Lr, Lc, NL, 1)
    mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16)
    kr, vr, ks, vs = mk(Lr), mk(Lr), mk(Lc), mk(Lc)
    qs = [mk(Lc) for _ in range(4)]
    o = torch.empty_like(qs[0])
    for l in range(NL):
        ca.put_reference(l, 0, kr, vr)
    chunk = [0] * NL
    for r in range(2):
        for l in range(NL):
            chunk[l] += 1
            ca.attend(l, 0, chunk[l], qs[0], ks, vs, o)
    ev = []
    for i in range(reps + 8):
        l = i % NL
        chunk[l] += 1
        kp, vp = ca.slot_ptr(l, 0, chunk[l])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ca.attend(l, 0, chunk[l], qs[i % 4], kp, vp, o)
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    ca.close()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev[8:])


def recv_us(H, d, Lr, Lc, P, zero_copy=False):
    """One rank's receive kernel (waits already met): the O-window copy, or with
    zero_copy (o = the window, as bench.py runs it) only the wait."""
    cas = [tm.ChunkAttention(H, d, Lr, Lc, 1, 1, world_size=P, rank=r, transport=tm.TM_TRANSPORT_PEER)
           for r in range(P)]
    tm.ChunkAttention.connect_local(cas)
    Ls, Lrs = -(-Lc // P), -(-Lr // P)
    mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16)
    for ph in (1, 2, 4):
        for r in range(P):
            cas[r].put_reference_phases(0, 0, mk(Lrs), mk(Lrs), ph)
    q = mk(Ls)
    os_ = [c.output_window()[0] if zero_copy else torch.empty_like(q) for c in cas]
    times = []
    for t in range(1, 4):
        for ph in (1, 2):
            for r in range(P):
                cas[r].attend_phases(0, 0, t, q, q, q, os_[r], ph)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for r in range(P):
            cas[r].attend_phases(0, 0, t, q, q, q, os_[r], 4)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) * 1e3 / P)
    for c in cas:
        c.close()
    return statistics.median(times)


out = {"note": "model from one-GPU measurements (see docstring); not a multi-GPU measurement",
       "nvlink_gbs_assumed": NVLINK_GBS, "configs": {}}
for name, Lr, Lc in (("wan512", 1024, 3072), ("wan720", 2025, 6075)):
    H, d = 40, 128
    rows = {}
    t1 = None
    for P in (1, 2, 4, 8):
        tk = kernel_us(H // P, d, Lr, Lc)
        Ls = -(-Lc // P)
        q_remote = Ls * H * d * 2 * (P - 1) / P if P > 1 else 0.0
        tq = q_remote / (NVLINK_GBS * 1e3)                     # us
        tr = recv_us(H, d, Lr, Lc, P) if P > 1 else 0.0
        tz = 1.0 if P > 1 else 0.0
        t = tk + tq + tz           # bench.py passes the O window (zero-copy, in-kernel wait)
        if P == 1:
            t1 = t
        rows[P] = {"kernel_us": round(tk, 1), "q_push_us": round(tq, 1), "recv_copy_us": round(tr, 1),
                   "done_wait_us_assumed": tz,
                   "t_us": round(t, 1), "E": round(t1 / (P * t), 3)}
        print(name, P, rows[P], flush=True)
    out["configs"][name] = rows
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "scale_model.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
