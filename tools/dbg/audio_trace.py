import os, subprocess, sys
import numpy as np
PATH = "/tmp/tm_trace.bin"
if os.path.exists(PATH): os.unlink(PATH)
os.environ["TM_TRACE"] = PATH
os.environ["TM_TRACE_BUILD"] = "1"
subprocess.check_call([sys.executable, "-m", "paper_2506_03099_b200.build"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
sys.path.insert(0, '.')
import torch
from paper_2506_03099_b200 import tm
H, d = 40, 128
frames, T, A = 3, 1024, 32
bf = torch.bfloat16
qa = torch.randn(frames, T, H, d, device="cuda", dtype=bf)
ka = torch.randn(frames, A, H, d, device="cuda", dtype=bf)
va = torch.randn(frames, A, H, d, device="cuda", dtype=bf)
oa = torch.empty_like(qa)
face = torch.tensor([r * 32 + cc for r in range(8, 24) for cc in range(8, 24)], dtype=torch.int32, device="cuda")
ca = tm.ChunkAttention(H, d, 16, 16, 1, 1)
for _ in range(3): ca.audio(qa, ka, va, oa, face)
torch.cuda.synchronize()
W = 13 * 4096 + 8 * 160
raw = np.fromfile(PATH, dtype=np.uint64).reshape(-1, W)[-1][:13 * 4096].reshape(13, 4096)
names = ["prod", "mma", "store", "mmapv", "obs"] + [f"w{k}" for k in range(8)]
ev = []
for r in range(13):
    x = raw[r]; x = x[x != 0]
    ev += [(int(v >> 8), names[r], int(v & 0xFF)) for v in x]
ev.sort()
t0 = ev[0][0]
for t, r, c in ev:
    if r in ("prod", "mma", "mmapv", "obs", "w0", "w4"):
        print(f"{t - t0:8d} {r:6s} {c}")
