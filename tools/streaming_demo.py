#!/usr/bin/env python
"""How a caller drives the library through a TalkingMachines-style stream
(P:130-153): chunk by chunk, each chunk denoised in 2 steps (NFE), and
every step running the DiT's attention layers over {c_0, c_{t-1}, c_t}
 from the per-(layer, step) KV cache, then the few-step
sampler update (x1_hat, Eq 1 re-noise, bf16 cast).

The DiT itself (projections, MLPs, VAE) is out of scope; random tensors
stand in for its Q/K/V and velocity.  K/V are written straight into the cache
slot (tm_kvcache_slot_ptr), as a fused QKV projection would, so the append is
zero-copy.  Prints ms per chunk.
    python tools/streaming_demo.py [--layers 40] [--chunks 8] [--res 512]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=40)
ap.add_argument("--chunks", type=int, default=8)
ap.add_argument("--res", type=int, default=512, choices=[512, 720])
a = ap.parse_args()

H, d = 40, 128
tok = 1024 if a.res == 512 else 2025                 # tokens per latent frame
Lr, Lc = tok, 3 * tok                                # reference frame, 3-frame chunks
side = 64 if a.res == 512 else 90
n_lat = 16 * 3 * side * side                         # latent elements per chunk
steps = [(0.0, 0.5), (0.5, 1.0)]                     # 2-NFE schedule (t_cur, t_next), reading Q10

ca = tm.ChunkAttention(H, d, Lr, Lc, num_layers=a.layers, num_steps=len(steps))
bf = torch.bfloat16
mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=bf)
for layer in range(a.layers):                        # a1: reference K/V once per stream
    ca.put_reference(layer, -1, mk(Lr), mk(Lr))
# Stand-in for the projection writing K/V into the slots: random contents in
# every slot once (all-zero operands would run ~12 % faster: power).
for layer in range(a.layers):
    for s_ in range(len(steps)):
        for t in (1, 2):
            for ptr in ca.slot_ptr(layer, s_, t):
                tm._wrap_device_ptr(ptr, Lc * H * d, bf, 0).copy_(mk(Lc).view(-1))
q, o = mk(Lc), torch.empty(Lc, H, d, device="cuda", dtype=bf)
x = torch.randn(n_lat, device="cuda")                # latent state (fp32 master)
v = torch.randn(n_lat, device="cuda").to(bf)         # stand-in for the DiT's velocity
xb = torch.empty(n_lat, device="cuda", dtype=bf)     # next NFE's model input
ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.chunks + 1)]
for t in range(1, a.chunks + 1):
    ev[t - 1].record()
    x.normal_()                                      # the new chunk starts from noise
    for s, (t_cur, t_next) in enumerate(steps):
        for layer in range(a.layers):
            kslot, vslot = ca.slot_ptr(layer, s, t)  # the projection writes K/V here
            ca.attend(layer, s, t, q, kslot, vslot, o)
        tm.tm_flow_sampler_step(ca.ctx, x, v, tm.TM_BF16, n_lat, t_cur, t_next,
                                seed=2506030990, offset=2 * t + s, x_bf16_out=xb)
ev[a.chunks].record()
torch.cuda.synchronize()
ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.chunks)]
print(f"{a.res}^2, {a.layers} layers x {len(steps)} steps: ms per chunk "
      + " ".join(f"{m:.1f}" for m in ms))
ca.close()
