#!/usr/bin/env python
"""Item-switch bubbles of CTA 0 (TM_TRACE build): the per-tile period of the
softmax warpgroups (code 20 = S_i(j) seen) and the gaps at item boundaries,
for one WAN-512 t>=2 call with SWEEP_H heads (5 = one rank's share at P = 8).
Rebuilds libtm.so with -DTM_TRACE_ENABLED (run last in a GPU session).
    SWEEP_H=5 python tools/item_gaps.py"""
import os
import statistics
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PATH = "/tmp/tm_trace.bin"
if os.path.exists(PATH):
    os.unlink(PATH)
os.environ["TM_TRACE"] = PATH
os.environ["TM_TRACE_BUILD"] = "1"
subprocess.check_call([sys.executable, "-m", "paper_2506_03099_b200.build"], cwd=ROOT,
                      stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

H = int(os.environ.get("SWEEP_H", "5"))
d, Lr, Lc = 128, 1024, 3072
ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1)
g = torch.Generator(device="cuda").manual_seed(1)
mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
ca.put_reference(0, 0, mk(Lr), mk(Lr))
for t in (1, 2, 3):
    q, k, v = mk(Lc), mk(Lc), mk(Lc)
    o = torch.empty_like(q)
    ca.attend(0, 0, t, q, k, v, o)
torch.cuda.synchronize()
W = 13 * 4096 + 8 * 160
raw = np.fromfile(PATH, dtype=np.uint64).reshape(-1, W)[-1][:13 * 4096].reshape(13, 4096)
names = ["prod", "mma", "store", "mmapv", "obs"] + [f"w{k}" for k in range(8)]
by = {}
t0 = None
for r in range(13):
    x = raw[r]
    x = x[x != 0]
    for v in x:
        t, c = int(v >> 8), int(v & 0xFF)
        by.setdefault((names[r], c), []).append(t)
allt = [t for v in by.values() for t in v]
t0 = min(allt)
for wname in ("w0", "w4"):
    s = sorted(by.get((wname, 20), []))
    p = sorted(by.get((wname, 24), []))
    if len(s) < 3:
        continue
    gaps = [b - a for a, b in zip(s, s[1:])]
    med = statistics.median(gaps)
    print(f"{wname}: {len(s)} tiles, first S seen at {s[0] - t0} cyc, last p_full at {p[-1] - t0} cyc, "
          f"median period {med:.0f} cyc")
    big = sorted(range(len(gaps)), key=lambda i: -gaps[i])[:4]
    for i in sorted(big):
        print(f"   gap after tile {i}: {gaps[i]} cyc ({gaps[i] / med:.1f} periods) at {s[i] - t0}")
end = max(allt)
print(f"CTA 0 span {end - t0} cyc; sum of tiles x median period = {len(by.get(('w0', 20), [])) * med:.0f}")
