#!/usr/bin/env python
"""Burst A/B of the 40-head WAN-512 t>=2 call (the bench's main shape): loops of
40 calls, each after a 1 s idle (so neither library runs power-capped),
median of 5; fused append and zero-copy.  Run once per library:
    TM_LIB_PATH=... AB_TAG=x python tools/ab_h40.py"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_03099_b200 import tm  # noqa: E402

s = torch.cuda.current_stream()
out = []
for zc in (False, True):
    ts = [bench.attention_loop(tm, torch, 40, 128, 1024, 3072, 40, s, zero_copy=zc, R=1, idle=1.0)
          for _ in range(5)]
    fl = 4.0 * 3072 * 7168 * 128 * 40
    m = statistics.median(ts)
    out.append(f"{'zc' if zc else 'fused'} {m * 1e3:6.1f} us ({fl / m / 1e9:6.1f} TFLOP/s) "
               f"[{min(ts) * 1e3:.1f}..{max(ts) * 1e3:.1f}]")
print(f"{os.environ.get('AB_TAG', ''):10s} " + "  ".join(out), flush=True)
