#!/usr/bin/env python
"""Loop timing (one event pair around K back-to-back calls, repeated R times,
median) of the WAN-512 t>=2 chunk attention at the head counts of one rank's
share (SWEEP_HS, default "5,10,20,40"), fused append or zero-copy
(SWEEP_APPEND=1/0), for the env-selected variant (TM_SCHED_ITEM_COST, ...).
    TM_SCHED_ITEM_COST=1.5 python tools/shard_sweep.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

d, Lr, Lc = 128, 1024, 3072
K, R, NL, NB = 40, 5, 8, 4
APPEND = os.environ.get("SWEEP_APPEND", "1") == "1"
SH = int(os.environ.get("SWEEP_SCHED_HEADS", "0"))
tag = os.environ.get("SWEEP_TAG", "")
out = []
for H in [int(x) for x in os.environ.get("SWEEP_HS", "5,10,20,40").split(",")]:
    g = torch.Generator(device="cuda").manual_seed(2506030990 + H)
    ca = tm.ChunkAttention(H, d, Lr, Lc, NL, 1, sched_heads=SH if H % max(SH, 1) == 0 else 0)
    sets = [[torch.randn(Lc, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3)]
            for _ in range(NB)]
    o = torch.empty(Lc, H, d, device="cuda", dtype=torch.bfloat16)
    kr = torch.randn(Lr, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
    for l in range(NL):
        ca.put_reference(l, 0, kr, kr)
    chunk = [0] * NL

    def call(i):
        l = i % NL
        chunk[l] += 1
        q, k, v = sets[i % NB]
        if not APPEND and chunk[l] >= 2:
            k, v = ca.slot_ptr(l, 0, chunk[l])
        ca.attend(l, 0, chunk[l], q, k, v, o)

    for i in range(3 * NL):
        call(i)
    torch.cuda.synchronize()
    ts = []
    for r in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(K):
            call(i)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / K)
    fl = 4.0 * Lc * (Lr + 2 * Lc) * d * H
    med = statistics.median(ts)
    out.append(f"H={H}: {med:6.1f} us ({fl / med / 1e6:6.1f} TFLOP/s) [{min(ts):.1f}..{max(ts):.1f}]")
    ca.close()
    del sets
    torch.cuda.empty_cache()
print(f"{tag:24s} append={int(APPEND)} " + "  ".join(out), flush=True)
