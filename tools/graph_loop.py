#!/usr/bin/env python
"""Per-call time of the WAN-512 t>=2 chunk attention at one rank's head count,
three ways: an eager loop (one event pair around K calls, as bench.py's
attention loop), the same K calls captured once in a CUDA graph and replayed
(no host work between launches), and the host's enqueue time per call.  A
small-H call (~50 us on the GPU) can be host-bound in an eager loop.
    GL_HS=5,40 python tools/graph_loop.py"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

d, Lr, Lc, NL, NB, K = 128, 1024, 3072, 8, 4, 40
APPEND = os.environ.get("GL_APPEND", "1") == "1"
for H in [int(x) for x in os.environ.get("GL_HS", "5,10,20,40").split(",")]:
    g = torch.Generator(device="cuda").manual_seed(2506030990 + H)
    ca = tm.ChunkAttention(H, d, Lr, Lc, NL, 1)
    sets = [[torch.randn(Lc, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3)]
            for _ in range(NB)]
    o = torch.empty(Lc, H, d, device="cuda", dtype=torch.bfloat16)
    kr = torch.randn(Lr, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
    for l in range(NL):
        ca.put_reference(l, 0, kr, kr)
    chunk = [0] * NL

    def call(i):
        l = i % NL
        chunk[l] += 1
        q, k, v = sets[i % NB]
        if not APPEND and chunk[l] >= 2:
            k, v = ca.slot_ptr(l, 0, chunk[l])
        ca.attend(l, 0, chunk[l], q, k, v, o)

    for i in range(3 * NL):
        call(i)
    torch.cuda.synchronize()
    eager = []
    for r in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t0 = time.perf_counter()
        for i in range(K):
            call(i)
        t1 = time.perf_counter()
        b.record()
        torch.cuda.synchronize()
        eager.append((a.elapsed_time(b) * 1e3 / K, (t1 - t0) * 1e6 / K))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for i in range(K):
            call(i)
    torch.cuda.synchronize()
    graph.replay()
    torch.cuda.synchronize()
    gt = []
    for r in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        torch.cuda.synchronize()
        gt.append(a.elapsed_time(b) * 1e3 / K)
    fl = 4.0 * Lc * (Lr + 2 * Lc) * d * H
    em = statistics.median(x for x, _ in eager)
    hm = statistics.median(y for _, y in eager)
    gm = statistics.median(gt)
    print(f"H={H:2d} append={int(APPEND)}: eager {em:6.1f} us ({fl / em / 1e6:6.1f} TFLOP/s), host enqueue "
          f"{hm:5.1f} us/call; graph replay {gm:6.1f} us ({fl / gm / 1e6:6.1f} TFLOP/s)", flush=True)
    del graph
    ca.close()
    del sets
    torch.cuda.empty_cache()
