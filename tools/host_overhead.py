#!/usr/bin/env python
"""Host-side cost of one tm_chunk_attention call (argument checks, segment
schedule, tensor-map encoding, launch) through the ctypes binding, measured
as CPU time per call while the GPU queue is kept busy.  At P = 8 a call's GPU
time is ~56 us, so the host must enqueue faster than that.
    python tools/host_overhead.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

for H in (40, 5):
    d, Lr, Lc, NL = 128, 1024, 3072, 8
    ca = tm.ChunkAttention(H, d, Lr, Lc, NL, 1)
    mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16)
    kr, vr, q, k, v = mk(Lr), mk(Lr), mk(Lc), mk(Lc), mk(Lc)
    o = torch.empty_like(q)
    for l in range(NL):
        ca.put_reference(l, 0, kr, vr)
    chunk = [0] * NL
    n = 400
    for i in range(50):
        chunk[i % NL] += 1
        ca.attend(i % NL, 0, chunk[i % NL], q, k, v, o)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        chunk[i % NL] += 1
        ca.attend(i % NL, 0, chunk[i % NL], q, k, v, o)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    # raw ctypes call without the Python wrapper layers
    ctx, qp, kp, vp, op = ca.ctx, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr()
    t3 = time.perf_counter()
    for i in range(n):
        chunk[i % NL] += 1
        tm.lib.tm_chunk_attention(ctx, i % NL, 0, chunk[i % NL], qp, kp, vp, op, None)
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"H={H}: host {1e6 * (t1 - t0) / n:.1f} us/call (binding), "
          f"{1e6 * (t4 - t3) / n:.1f} us/call (raw ctypes); GPU {1e6 * (t2 - t0) / n:.1f} us/call")
    ca.close()
