#!/usr/bin/env python
"""Kernel-only timing of the WAN-512 t>=2 chunk attention for the env-selected
variant (e.g. TM_POLY); prints one line.  Used for tuning sweeps:
    for v in 0 1 3 4; do TM_POLY=$v python tools/sweep.py; done   (0 = default split)
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

cfg = os.environ.get("SWEEP_CFG", "512")
H, d, Lr, Lc = (40, 128, 1024, 3072) if cfg == "512" else (40, 128, 2025, 6075)
H = int(os.environ.get("SWEEP_H", H))     # e.g. 20/10/5: one rank's heads at P = 2/4/8
NL = int(os.environ.get("SWEEP_NL", 8))   # layer caches rotated (8: operands from HBM)
ca = tm.ChunkAttention(H, d, Lr, Lc, NL, 1)
g = torch.Generator(device="cuda").manual_seed(1)
mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
kr, vr = mk(Lr), mk(Lr)
qs = [mk(Lc) for _ in range(4)]
o = torch.empty_like(qs[0])
for l in range(NL):
    ca.put_reference(l, 0, kr, vr)
chunk = [0] * NL


APPEND = os.environ.get("SWEEP_APPEND") == "1"     # fused c_t append (as in bench's step)


def call(i):
    l = i % NL
    chunk[l] += 1
    if APPEND:
        kp, vp = ks, vs
    else:
        kp, vp = ca.slot_ptr(l, 0, chunk[l])
    ca.attend(l, 0, chunk[l], qs[i % 4], kp, vp, o)


# Fill every layer's cache slots with real (random) K/V via the fused append
# first: timing zero-copy calls on never-written (zero) slots is optimistic.
ks, vs = mk(Lc), mk(Lc)
for rnd in range(2):
    for l in range(NL):
        chunk[l] += 1
        ca.attend(l, 0, chunk[l], qs[0], ks, vs, o)
for i in range(3 * NL):
    call(i)
torch.cuda.synchronize()
ev = []
for i in range(60):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    call(i)
    b.record()
    ev.append((a, b))
torch.cuda.synchronize()
ms = [a.elapsed_time(b) for a, b in ev]
fl = 4.0 * Lc * (Lr + 2 * Lc) * d * H
med = statistics.median(ms)
print(f"{os.environ.get('TM_POLY', '-'):>3} append={int(APPEND)} "
      f"cfg={cfg} H={H} median {med * 1e3:7.1f} us  "
      f"{fl / med / 1e9:7.1f} TFLOP/s  min {min(ms) * 1e3:7.1f} us")
