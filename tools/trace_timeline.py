#!/usr/bin/env python
"""Run one WAN-512 chunk attention (t>=2) with TM_TRACE and print CTA 0's
kernel timeline (debug aid; clock64 cycles).

Roles: 0 producer (1=K slot acquired, 2=V slot acquired), 1 MMA (10=K full,
11/12=p_full[i] seen, 13/14=S_i issued+committed), 2/3 softmax tile 0/1
(20=s_full seen, 21=S loaded, 22=max done, 23=exp done, 24=p_full arrived).
"""
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PATH = "/tmp/tm_trace.bin"
if os.path.exists(PATH):
    os.unlink(PATH)
os.environ["TM_TRACE"] = PATH

import subprocess  # noqa: E402
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
names = ["producer", "mma", "softmax0", "softmax1"]
ev = {}
for r in range(4):
    x = raw[r]
    x = x[x != 0]
    ev[r] = [(int(v >> 8), int(v & 0xFF)) for v in x]
t0 = min(e[0][0] for e in ev.values() if e)
for r in range(4):
    print(f"== {names[r]}: {len(ev[r])} events")
    print("   ", " ".join(f"{c}@{t - t0}" for t, c in ev[r][:60]))


def gaps(r, a, b):
    """durations from each code-a event to the next code-b event of role r."""
    out, last = [], None
    for t, c in ev[r]:
        if c == a:
            last = t
        elif c == b and last is not None:
            out.append(t - last)
            last = None
    return out


def period(r, a):
    ts = [t for t, c in ev[r] if c == a]
    return [y - x for x, y in zip(ts, ts[1:])]


for r in (2, 3):
    print(f"{names[r]}: period(s_full) median {statistics.median(period(r, 20)):.0f} cycles")
    for a, b, what in [(20, 21, "ld S"), (21, 22, "max"), (22, 23, "exp+st"), (23, 24, "wait_st+arrive"),
                       (24, 20, "wait for next S")]:
        gg = gaps(r, a, b)
        if gg:
            print(f"   {what:18s} median {statistics.median(gg):7.0f}  mean {statistics.mean(gg):7.0f}")
for a, b, what in [(10, 11, "K full -> p_full0"), (11, 13, "PV0+S0 issue"), (13, 12, "-> p_full1"),
                   (12, 14, "PV1+S1 issue")]:
    gg = gaps(1, a, b)
    if gg:
        print(f"mma {what:20s} median {statistics.median(gg):7.0f}")
print("mma period(K full)", statistics.median(period(1, 10)))
