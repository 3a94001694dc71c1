import os, sys, statistics, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2506_03099_b200 import tm
H, d, Lr, Lc = 40, 128, 1024, 3072
NL = 8
ca = tm.ChunkAttention(H, d, Lr, Lc, NL, 1)
g = torch.Generator(device="cuda").manual_seed(1)
mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
kr, vr = mk(Lr), mk(Lr)
qs = [mk(Lc) for _ in range(4)]
outs = [torch.empty_like(qs[0]) for _ in range(4)]
for l in range(NL): ca.put_reference(l, 0, kr, vr)
chunk = [0] * NL
cur = torch.cuda.current_stream()
def run(n, stream_arg, multi_out, tag):
    ev = []
    for i in range(n):
        l = i % NL; chunk[l] += 1
        kp, vp = ca.slot_ptr(l, 0, chunk[l])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        ca.attend(l, 0, chunk[l], qs[i % 4], kp, vp, outs[i % 4] if multi_out else outs[0], stream_arg)
        b.record(cur)
        ev.append((a, b))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev][5:]
    print(f"{tag:30s} mean {statistics.mean(ms)*1e3:7.1f} us  median {statistics.median(ms)*1e3:7.1f}")
for rep in range(2):
    run(40, None, False, "stream=None, one out")
    run(40, cur, False, "stream=current, one out")
    run(40, cur, True, "stream=current, 4 outs")
    run(40, None, True, "stream=None, 4 outs")
