#!/usr/bin/env python
"""Run one WAN-512 chunk attention (t>=2) with a TM_TRACE build and print CTA 0's
kernel timeline (debug aid; clock64 cycles).  Rebuilds libtm.so with
-DTM_TRACE_ENABLED first (run it last in a GPU session).

Events: producer 1/2 = K/V slot acquired; MMA 10 = K_j full, 15/16 = s_free
(+q_full) seen before S_i, 13/14 = S_i issued, 11/12 = p_full_i seen before
PV_i; softmax_i 20 = s_full seen, 21 = S loaded (s_free arrived), 22 = max
decision, 25 = previous PV done (first P store), 23 = exps done, 24 = p_full.
"""
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

H, d, Lr, Lc = 40, 128, 1024, 3072
ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1)
g = torch.Generator(device="cuda").manual_seed(1)
mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
ca.put_reference(0, 0, mk(Lr), mk(Lr))
for t in (1, 2, 3):
    q, k, v = mk(Lc), mk(Lc), mk(Lc)
    o = torch.empty_like(q)
    ca.attend(0, 0, t, q, k, v, o)
torch.cuda.synchronize()
raw = np.fromfile(PATH, dtype=np.uint64).reshape(-1, 4, 4096)[-1]   # last call
names = ["prod", "mma", "sm0", "sm1"]
ev = []
for r in range(4):
    x = raw[r]
    x = x[x != 0]
    ev += [(int(v >> 8), names[r], int(v & 0xFF)) for v in x]
ev.sort()
t0 = ev[0][0]
# print a window in the middle of the first item
mid = [e for e in ev if e[1] == "sm0" and e[2] == 20]
lo = mid[20][0] if len(mid) > 24 else ev[0][0]
hi = mid[24][0] if len(mid) > 24 else ev[-1][0]
print("time(rel)  role  code")
for t, r, c in ev:
    if lo <= t <= hi:
        print(f"{t - lo:8d}  {r:5s} {c}")
by = {}
for t, r, c in ev:
    by.setdefault((r, c), []).append(t)


def per(r, c):
    x = by.get((r, c), [])
    return statistics.median([b - a for a, b in zip(x, x[1:])]) if len(x) > 2 else float("nan")


print("period sm0 s_full", per("sm0", 20), " sm1", per("sm1", 20), " mma K", per("mma", 10))
