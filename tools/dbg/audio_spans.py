#!/usr/bin/env python
"""Per-CTA spans (entry, first S, exit) of the f4 audio attention launch at the
bench's shape, from a TM_SPANS build (rebuilds libtm.so; rebuild normally
afterwards).  TM_DBG_AUDIO_PART=2 times the attention launch without the prep."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
PATH = "/tmp/tm_spans.bin"
if os.path.exists(PATH): os.unlink(PATH)
os.environ["TM_TRACE"] = PATH
os.environ["TM_TRACE_BUILD"] = "spans"
subprocess.check_call([sys.executable, "-m", "paper_2506_03099_b200.build"], cwd=ROOT, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
sys.path.insert(0, ROOT)
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
for _ in range(5): ca.audio(qa, ka, va, oa, face)
torch.cuda.synchronize()
W = 13 * 4096 + 8 * 160
allw = np.fromfile(PATH, dtype=np.uint64).reshape(-1, W)[-1][13 * 4096:].reshape(160, 8)
allw = allw[allw[:, 0] != 0].astype(np.int64)
raw = allw[:, :6]
t0 = raw[:, 0].min()
rel = np.where(raw != 0, (raw - t0) / 1000.0, np.nan)
items = allw[:, 7] & 0xFFFF
for j, name in enumerate(["entry", "first S", "item2", "exit", "prologue", "dep wait"]):
    col = rel[:, j][raw[:, j] != 0]
    if len(col): print(f"{name:8s} min {col.min():6.1f} med {np.median(col):6.1f} max {col.max():6.1f} us  n {len(col)}")
act = items > 0
print("CTAs with items", act.sum(), "exit of working CTAs: med", np.median(rel[act, 3]), "max", rel[act, 3].max(),
      "; idle CTAs exit med", np.median(rel[~act, 3]) if (~act).any() else None)
