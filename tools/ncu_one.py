#!/usr/bin/env python
"""A few fused-append WAN-512 t>=2 chunk-attention calls at SWEEP_H heads (one
layer cache set per call, 8 rotated), for one `ncu --set full` capture of a
steady-state launch:
    SWEEP_H=5 ncu --set full --clock-control none --import-source on \
        -k regex:fmha_sm100_kernel --launch-skip 12 --launch-count 1 \
        -o gpurun_out/h5 python tools/ncu_one.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

H = int(os.environ.get("SWEEP_H", "40"))
d, Lr, Lc, NL = 128, 1024, 3072, 8
g = torch.Generator(device="cuda").manual_seed(2506030990 + H)
ca = tm.ChunkAttention(H, d, Lr, Lc, NL, 1)
mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
kr = mk(Lr)
for l in range(NL):
    ca.put_reference(l, 0, kr, kr)
q, k, v = mk(Lc), mk(Lc), mk(Lc)
o = torch.empty_like(q)
chunk = [0] * NL
for i in range(16):
    l = i % NL
    chunk[l] += 1
    ca.attend(l, 0, chunk[l], q, k, v, o)
torch.cuda.synchronize()
print("ok")
