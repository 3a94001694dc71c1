# Synced-call stress over many head counts / shapes (stream-K tails with 1..16
# pieces per unit, d = 64 and 128, fused append and zero-copy): any kernel trap
# or non-finite output is reported with its shape.
import os, sys, time, itertools
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2506_03099_b200 import tm
bf = torch.bfloat16
shapes = [(H, d, Lr, Lc) for H in (1, 2, 3, 5, 7, 12, 40) for d in (64, 128) for (Lr, Lc) in ((1024, 3072), (300, 1000), (8192, 256))]
for (H, d, Lr, Lc) in shapes:
    for zc in (False, True):
        g = torch.Generator(device="cuda").manual_seed(H * 1000 + d + Lc)
        ca = tm.ChunkAttention(H, d, Lr, Lc, 4, 1)
        mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=bf, generator=g)
        kr, vr = mk(Lr), mk(Lr)
        for l in range(4):
            ca.put_reference(l, 0, kr, vr)
        q, k, v = mk(Lc), mk(Lc), mk(Lc)
        o = torch.empty(Lc, H, d, device="cuda", dtype=bf)
        chunk = [0] * 4
        t0 = time.time()
        try:
            for i in range(24):
                l = i % 4
                chunk[l] += 1
                kk, vv = (ca.slot_ptr(l, 0, chunk[l]) if zc and chunk[l] >= 2 else (k, v))
                ca.attend(l, 0, chunk[l], q, kk, vv, o)
                torch.cuda.synchronize()
            ok = bool(torch.isfinite(o.float()).all())
        except Exception as e:
            print(f"FAIL H={H} d={d} Lr={Lr} Lc={Lc} zc={zc} after {time.time()-t0:.2f}s: {str(e).splitlines()[0]}", flush=True)
            sys.exit(1)
        if not ok:
            print(f"NONFINITE H={H} d={d} Lr={Lr} Lc={Lc} zc={zc}", flush=True)
        ca.close()
print("all shapes ok", flush=True)
