#!/usr/bin/env python
"""f1 (full 21-frame window, 7 chunks x 3072 tokens, 40 heads) standalone:
the single window launch vs the same work as 7 streaming calls (reference
attention for chunk 0, then chunks 1..6), both as loops between one event pair.
    python tools/f1_timing.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

H, d, Lc, n = 40, 128, 3072, 7
bf = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(5)
L = n * Lc
q, k, v = (torch.randn(L, H, d, device="cuda", dtype=bf, generator=g) for _ in range(3))
o = torch.empty_like(q)
fl = 4.0 * d * H * Lc * Lc * (1 + 2 + 3 * (n - 2))
ca = tm.ChunkAttention(H, d, Lc, Lc, 1, 1)


def loop(fn, reps=20, R=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    return statistics.median(ts)


ms = loop(lambda: ca.window(q, k, v, o, [Lc] * n))
print(f"f1 window, one launch: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s  (launches {ca.launches})")
sc = tm.ChunkAttention(H, d, Lc, Lc, 1, 1)
ob = torch.empty(Lc, H, d, device="cuda", dtype=bf)


def seven():
    sc.reset()
    sc.reference_attend(0, 0, q[:Lc], k[:Lc], v[:Lc], ob)
    for t in range(1, n):
        s = slice(t * Lc, (t + 1) * Lc)
        sc.attend(0, 0, t, q[s], k[s], v[s], ob)


ms7 = loop(seven)
print(f"same work as 7 streaming calls:  {ms7:.3f} ms  {fl / ms7 / 1e9:.1f} TFLOP/s")
