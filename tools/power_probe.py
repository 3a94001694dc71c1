#!/usr/bin/env python
"""Sustained WAN-512 chunk-attention loop (~3 s, random data in every cache
slot) with nvidia-smi sampling: SM clock, power and throttle reasons under
load, to tell power-capped from clock-capped behaviour."""
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

H, d, Lr, Lc, NL = 40, 128, 1024, 3072, 8
ca = tm.ChunkAttention(H, d, Lr, Lc, NL, 1)
g = torch.Generator(device="cuda").manual_seed(1)
mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
kr, vr = mk(Lr), mk(Lr)
qs = [mk(Lc) for _ in range(4)]
ks, vs = mk(Lc), mk(Lc)
o = torch.empty_like(qs[0])
for l in range(NL):
    ca.put_reference(l, 0, kr, vr)
chunk = [0] * NL
for rnd in range(2):
    for l in range(NL):
        chunk[l] += 1
        ca.attend(l, 0, chunk[l], qs[0], ks, vs, o)
torch.cuda.synchronize()
tmp = tempfile.NamedTemporaryFile("w+", delete=False)
proc = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw,temperature.gpu,"
                         "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
                         "clocks_event_reasons.sw_thermal_slowdown", "--format=csv,noheader,nounits",
                         "-lms", "50"], stdout=tmp, stderr=subprocess.DEVNULL)
time.sleep(1.5)
n = int(os.environ.get("PROBE_CALLS", "8000"))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(n):
    l = i % NL
    chunk[l] += 1
    if os.environ.get("PROBE_APPEND") == "1":      # fused c_t append (bench's step)
        kp, vp = ks, vs
    else:
        kp, vp = ca.slot_ptr(l, 0, chunk[l])
    ca.attend(l, 0, chunk[l], qs[i % 4], kp, vp, o)
b.record()
torch.cuda.synchronize()
time.sleep(0.2)
proc.terminate()
proc.wait()
tmp.seek(0)
rows = [r.split(",") for r in tmp.read().strip().splitlines()]
load = [r for r in rows if float(r[1]) > 300]
us = a.elapsed_time(b) * 1e3 / n
fl = 4.0 * Lc * (Lr + 2 * Lc) * d * H
print(f"TM_POLY={os.environ.get('TM_POLY', '-')} append={os.environ.get('PROBE_APPEND', '0')}: {n} calls, {us:.1f} us/call, {fl / us / 1e6:.1f} TFLOP/s")
if load:
    print("under load: sm MHz median", statistics.median(float(r[0]) for r in load),
          " power W median", statistics.median(float(r[1]) for r in load),
          " max", max(float(r[1]) for r in load), " temp", max(float(r[2]) for r in load),
          " sw_power_cap active in", sum("Active" in r[3] and "Not" not in r[3] for r in load),
          "of", len(load), "samples")
