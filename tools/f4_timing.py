#!/usr/bin/env python
"""f4 audio cross-attention at the bench's WAN-512 chunk shape (3 latent frames x
1024 tokens, 16x16 face region, 5 x 32 audio keys, 40 heads): loop time between
one event pair.  Under ncu --metrics gpu__time_duration.sum it gives the
per-kernel split (prep gather/zero-fill vs attention).
    python tools/f4_timing.py [reps]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
H, d = 40, 128
frames, T, A = 3, 1024, 32
bf = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(3)
ca = tm.ChunkAttention(H, d, 16, 16, 1, 1)
qa = torch.randn(frames, T, H, d, device="cuda", dtype=bf, generator=g)
ka = torch.randn(frames, A, H, d, device="cuda", dtype=bf, generator=g)
va = torch.randn(frames, A, H, d, device="cuda", dtype=bf, generator=g)
oa = torch.empty_like(qa)
face = torch.tensor([r * 32 + c for r in range(8, 24) for c in range(8, 24)], dtype=torch.int32,
                    device="cuda")
for _ in range(3):
    ca.audio(qa, ka, va, oa, face)
torch.cuda.synchronize()
import time  # noqa: E402
ts, hs = [], []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    for _ in range(reps):
        ca.audio(qa, ka, va, oa, face)
    hs.append((time.perf_counter() - t0) * 1e6 / reps)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3 / reps)
print(f"f4 audio: {statistics.median(ts):.1f} us/call ({ca.launches} launches/call), eager loop; "
      f"host enqueue {statistics.median(hs):.1f} us/call")
# the same calls captured in a CUDA graph: no host work between launches
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=s):
    for _ in range(reps):
        ca.audio(qa, ka, va, oa, face)
graph.replay()
torch.cuda.synchronize()
gt = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    graph.replay()
    b.record()
    torch.cuda.synchronize()
    gt.append(a.elapsed_time(b) * 1e3 / reps)
print(f"f4 audio: {statistics.median(gt):.1f} us/call, CUDA graph replay")
