#!/usr/bin/env python
"""HBM-bound kernels at 12.6 M elements (64 WAN-512 chunk latents): a7 Euler
step and the f2 sampler step, each timed as K calls back to back between one
event pair with NS operand sets rotated (> the 126 MB L2), GB/s of the
algorithmic bytes and the fraction of MEASURED_PEAKS.json hbm_gbs.
    python tools/hbm_bench.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

n = int(os.environ.get("HBM_N", 64 * 16 * 3 * 64 * 64))
NS, K = 4, 40
try:
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    peak = 6650.0
g = torch.Generator(device="cuda").manual_seed(5)
xs = [torch.randn(n, device="cuda", generator=g) for _ in range(NS)]
vs = [torch.randn(n, device="cuda", generator=g).to(torch.bfloat16) for _ in range(NS)]
xbs = [torch.empty(n, device="cuda", dtype=torch.bfloat16) for _ in range(NS)]
es = [torch.randn(n, device="cuda", generator=g) for _ in range(NS)]
cnt = [0]


def loop(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / K)
    return sorted(ts)[1]


def euler():
    i = cnt[0] % NS
    cnt[0] += 1
    tm.tm_flow_euler_step(None, xs[i], vs[i], tm.TM_BF16, n, 0.5)


def sampler():
    i = cnt[0] % NS
    cnt[0] += 1
    tm.tm_flow_sampler_step(None, xs[i], vs[i], tm.TM_BF16, n, 0.0, 0.5, seed=1, x_bf16_out=xbs[i])


def sampler_eps():
    i = cnt[0] % NS
    cnt[0] += 1
    tm.tm_flow_sampler_step(None, xs[i], vs[i], tm.TM_BF16, n, 0.0, 0.5, eps=es[i], x_bf16_out=xbs[i])


def copy():
    i = cnt[0] % NS
    cnt[0] += 1
    xs[(i + 1) % NS].copy_(xs[i])


tag = os.environ.get("HBM_TAG", "")
for name, fn, byts in (("euler", euler, 10 * n), ("sampler", sampler, 12 * n),
                       ("sampler eps", sampler_eps, 16 * n), ("torch copy fp32", copy, 8 * n)):
    ms = loop(fn)
    gbs = byts / (ms * 1e-3) / 1e9
    print(f"{tag:10s} {name:16s} n={n}: {ms * 1e3:6.1f} us  {gbs:7.1f} GB/s  {gbs / peak:.3f} of {peak:.0f}")
