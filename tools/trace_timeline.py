#!/usr/bin/env python
"""Run one WAN-512 chunk attention (t>=2) with a TM_TRACE build and print CTA 0's
kernel timeline (debug aid; clock64 cycles).  Rebuilds libtm.so with
-DTM_TRACE_ENABLED first (run it last in a GPU session).

Events: producer 3/4 = waiting for a K/V slot, 1/2 = K/V slot acquired (TMA issued),
5 = waited for an append store; store warp 40/41 = K/V tile landed (kv_full, in order);
S-issuer (mma) 10 = K_j full, 15/16 = s_free
(+q_full) seen before S_i, 13/14 = S_i issued; PV-issuer (mmapv) 11/12 = p_full_i seen before
PV_i; softmax_i 20 = s_full seen, 21 = S loaded (s_free arrived), 22 = max
decision, 25 = previous PV done (first P store), 23 = exps done, 24 = p_full;
w0..w7: per-softmax-warp 20/21/24 (lane 0 of each warp);
observer (warp 10 lane 1) 30/31 = S_0/S_1 commit landed.
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
W = 13 * 4096 + 8 * 160        # role timelines + per-CTA span words (csrc/internal.h kTraceWords)
raw = np.fromfile(PATH, dtype=np.uint64).reshape(-1, W)[-1][:13 * 4096].reshape(13, 4096)   # last call
names = ["prod", "mma", "store", "mmapv", "obs"] + [f"w{k}" for k in range(8)]
ev = []
for r in range(13):
    x = raw[r]
    x = x[x != 0]
    ev += [(int(v >> 8), names[r], int(v & 0xFF)) for v in x]
ev.sort()
t0 = ev[0][0]
# print a window in the middle of the first item
mid = [e for e in ev if e[1] == "w0" and e[2] == 20]
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


print("period obs S0", per("obs", 30))
print("period w0 s_full", per("w0", 20), " w4", per("w4", 20), " mma K", per("mma", 10))

# per-warp skew inside each softmax warpgroup (events of the same tile index)
for wg in range(2):
    ws = [f"w{wg * 4 + k}" for k in range(4)]
    for code, label in ((20, "s_full seen"), (21, "S loaded"), (24, "p_full arrive")):
        lists = [by.get((w, code), []) for w in ws]
        n = min(len(x) for x in lists)
        if n < 4:
            continue
        spread = [max(x[t] for x in lists) - min(x[t] for x in lists) for t in range(n)]
        late = [max(range(4), key=lambda k: lists[k][t]) for t in range(n)]
        print(f"WG{wg} {label:14s}: median spread {statistics.median(spread):6.0f} cyc, "
              f"latest warp histogram {[late.count(k) for k in range(4)]}")
    for k, w in enumerate(ws):
        c = {code: by.get((w, code), []) for code in (20, 21, 22, 25, 23, 24)}
        n = min(len(v) for v in c.values())
        if n > 2:
            med = lambda a, b: statistics.median([c[b][t] - c[a][t] for t in range(n)])
            print(f"  {w}: 20->21 {med(20, 21):5.0f}  21->22 {med(21, 22):5.0f}  22->25 {med(22, 25):5.0f}"
                  f"  25->23 {med(25, 23):5.0f}  23->24 {med(23, 24):5.0f}")
        a, b = by.get((w, 20), []), by.get((w, 24), [])
        n = min(len(a), len(b))
        if n > 2:
            print(f"  {w}: median s_full->p_full {statistics.median([b[t] - a[t] for t in range(n)]):6.0f} cyc")

# TMA latency: n-th acquire (1/2) of the producer vs n-th landing (40/41) seen by the store warp
acq = [t for t, r, c in ev if r == "prod" and c in (1, 2)]
land = [t for t, r, c in ev if r == "store" and c in (40, 41)]
n = min(len(acq), len(land))
if n > 8:
    lat = [land[k] - acq[k] for k in range(n)]
    print(f"TMA issue->landed (in-order view): median {statistics.median(lat):.0f} cyc, p90 {sorted(lat)[int(0.9 * n)]:.0f}")
    waits = by.get(("prod", 3), []) + by.get(("prod", 4), [])
    print(f"producer slot waits: {len(waits)}; store_done waits: {len(by.get(('prod', 5), []))}")
mk = by.get(("mma", 10), [])
