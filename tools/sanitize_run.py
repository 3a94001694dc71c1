#!/usr/bin/env python
"""Small workload for compute-sanitizer: every entry point
once on tiny / ragged shapes through the C ABI.
    compute-sanitizer --tool memcheck python tools/sanitize_run.py
    (also racecheck, synccheck, initcheck)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402


def stream(H, d, Lr, Lc, dtype, transport=tm.TM_TRANSPORT_NCCL, zero_copy=False, sched_heads=0):
    dt = torch.bfloat16 if dtype == tm.TM_BF16 else torch.float32
    ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1, dtype=dtype, transport=transport,
                           sched_heads=sched_heads)
    mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=dt)
    ca.put_reference(0, 0, mk(Lr), mk(Lr))
    for t in (1, 2, 3):
        q, k, v = mk(Lc), mk(Lc), mk(Lc)
        if zero_copy:
            kp, vp = ca.slot_ptr(0, 0, t)
            torch.cuda.synchronize()
            k, v = kp, vp
        o = torch.empty(Lc, H, d, device="cuda", dtype=dt)
        ca.attend(0, 0, t, q, k, v, o)
    torch.cuda.synchronize()
    if transport == tm.TM_TRANSPORT_PEER:
        ca.check()
    ca.close()


stream(2, 128, 200, 300, tm.TM_BF16)
stream(2, 64, 17, 130, tm.TM_BF16)
stream(2, 128, 200, 300, tm.TM_BF16, zero_copy=True)
stream(2, 128, 130, 70, tm.TM_FP32)
stream(2, 128, 200, 300, tm.TM_BF16, transport=tm.TM_TRANSPORT_PEER)
# stream-K merges: 3 partials (six column-half copies through three buffers), 16 partials
stream(1, 128, 1024, 512, tm.TM_BF16)
stream(1, 64, 1024, 512, tm.TM_BF16)
stream(1, 128, 8192, 256, tm.TM_BF16)
# schedule blocks (tm_config.sched_heads): 4 blocks of one head in one launch
stream(4, 128, 1024, 512, tm.TM_BF16, sched_heads=1)
# f1 window, f4 audio, a7 Euler, f2 sampler
H, d = 2, 128
ca = tm.ChunkAttention(H, d, 16, 16, 1, 1)
lens = [100, 37, 130]
L = sum(lens)
q, k, v = (torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
ca.window(q, k, v, o, lens)
frames, T, A = 3, 64, 16
qa = torch.randn(frames, T, H, d, device="cuda", dtype=torch.bfloat16)
ka, va = (torch.randn(frames, A, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(2))
oa = torch.empty_like(qa)
ca.audio(qa, ka, va, oa, torch.arange(0, 40, device="cuda", dtype=torch.int32), window=5)
x = torch.randn(1003, device="cuda")
vv = torch.randn(1003, device="cuda").to(torch.bfloat16)
ca.euler(x, vv, tm.TM_BF16, 0.5)
xb = torch.empty(1003, device="cuda", dtype=torch.bfloat16)
tm.tm_flow_sampler_step(ca.ctx, x, vv, tm.TM_BF16, 1003, 0.0, 0.5, seed=3, x_bf16_out=xb)
torch.cuda.synchronize()
ca.close()
print("sanitize_run: done")
