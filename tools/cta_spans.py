#!/usr/bin/env python
"""Per-CTA spans of one chunk-attention launch (TM_TRACE build: globaltimer at
CTA entry, first S seen by the softmax, second item start, exit).  Shows the
fixed per-launch costs (prologue latency, tail spread) at a given head count:
    SWEEP_H=5 python tools/cta_spans.py      (one rank's heads at P = 8)
Rebuilds libtm.so with -DTM_SPANS_ENABLED; rebuild normally afterwards.

Per-CTA words: 0 entry, 1 first S seen, 2 second item start, 3 exit,
4 merge wait begin, 5 merge go (globaltimer ns), 6 tiles, 7 items | smid << 16.
Extra A/B instrumentation via TM_EXTRA_DEFINES (same slots, other meanings):
  TM_SPANS_MERGE  2 = start of each item's epilogue (the last one survives),
                  1 = O loaded from TMEM in the row store, 4 = softmax loop left,
                  5 = merge go (mergers) / row store done (others)
  TM_SPANS_PROD   1 = producer clock64 cycles waiting on store_done,
                  5 = producer cycles waiting on kv_empty (raw values in "raw")
"""
import os
import statistics
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PATH = "/tmp/tm_spans.bin"
if os.path.exists(PATH):
    os.unlink(PATH)
os.environ["TM_TRACE"] = PATH
os.environ["TM_TRACE_BUILD"] = "spans"      # per-CTA stamps only (no role timeline)
subprocess.check_call([sys.executable, "-m", "paper_2506_03099_b200.build"], cwd=ROOT,
                      stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
import torch  # noqa: E402

from paper_2506_03099_b200 import tm  # noqa: E402

cfg = os.environ.get("SWEEP_CFG", "512")
H, d, Lr, Lc = (40, 128, 1024, 3072) if cfg == "512" else (40, 128, 2025, 6075)
H = int(os.environ.get("SWEEP_H", H))
ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1)
g = torch.Generator(device="cuda").manual_seed(1)
mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
ca.put_reference(0, 0, mk(Lr), mk(Lr))
ZC = os.environ.get("SPANS_ZC") == "1"     # zero-copy calls (K/V already in the cache slot)
for t in range(1, 6):
    q, k, v = mk(Lc), mk(Lc), mk(Lc)
    o = torch.empty_like(q)
    if ZC:
        k, v = ca.slot_ptr(0, 0, t)
    ca.attend(0, 0, t, q, k, v, o)
torch.cuda.synchronize()
W = 13 * 4096 + 8 * 160
allw = np.fromfile(PATH, dtype=np.uint64).reshape(-1, W)[-1][13 * 4096:].reshape(160, 8)
allw = allw[allw[:, 0] != 0].astype(np.int64)
raw = allw[:, :6]
t0 = raw[:, 0].min()
rel = np.where(raw != 0, (raw - t0) / 1000.0, np.nan)          # us
print(f"cfg={cfg} H={H}: {len(raw)} CTAs, kernel span {rel[:, 3].max():.1f} us")
for j, name in enumerate(["entry", "first S", "item 2 start", "exit", "merge wait", "merge go"]):
    col = rel[:, j][raw[:, j] != 0]
    if len(col):
        print(f"  {name:13s} min {col.min():7.1f}  median {statistics.median(col):7.1f}  max {col.max():7.1f} us")
busy = rel[:, 3] - rel[:, 0]
print(f"  CTA busy     min {busy.min():7.1f}  median {statistics.median(busy):7.1f}  max {busy.max():7.1f} us")
wait = rel[:, 5] - rel[:, 4]
ok = ~np.isnan(wait)
if ok.any():
    print(f"  merge wait   n {ok.sum()}  median {np.median(wait[ok]):6.1f}  max {wait[ok].max():6.1f} us")
tiles, items, smid = allw[:, 6], allw[:, 7] & 0xFFFF, allw[:, 7] >> 16
print(f"  tiles/CTA min {tiles.min()} max {tiles.max()}; items/CTA {sorted(set(items.tolist()))}")
order = np.argsort(rel[:, 3])
print("  slowest 8 CTAs: (cta, smid, tiles, items, exit us, merge wait us)")
for c in order[-8:]:
    print(f"    {c:4d} {smid[c]:4d} {tiles[c]:4d} {items[c]:3d} {rel[c, 3]:7.1f} {wait[c] if ok[c] else float('nan'):6.1f}")
rate_all = tiles / (rel[:, 3] - rel[:, 1])
print("  rate by smid (tiles/us), 148 values in smid order:")
by = sorted(zip(smid.tolist(), rate_all.tolist()))
print("   " + " ".join(f"{r:.3f}" for _, r in by))
rate = tiles / (rel[:, 3] - rel[:, 1])
print(f"  tiles/us per CTA: min {rate.min():.3f} median {np.median(rate):.3f} max {rate.max():.3f}")

# Per-CTA table (host replica of the stream-K item math) -> gpurun_out/spans_<H>.json
import json  # noqa: E402
n_tiles = sum(-(-L // 128) for L in (Lr, Lc, Lc))
qpairs = -(-(-(-Lc // 128)) // 2)
U = H * qpairs
C = len(allw)
R, T = U // C, U % C
G = 0
if T:
    G = min(C, max(T, T * n_tiles // 4))
W = T * n_tiles
rows = []
for c in range(C):
    items = [("whole", n_tiles)] * R
    if T and c < G:
        s, e = c * W // G, (c + 1) * W // G
        u = s // n_tiles
        while u * n_tiles < e:
            lo, hi = max(s, u * n_tiles) - u * n_tiles, min(e, (u + 1) * n_tiles) - u * n_tiles
            items.append((f"u{u}[{lo},{hi})", hi - lo))
            u += 1
    rows.append({"cta": c, "raw": [int(x) for x in allw[c]], "smid": int(smid[c]), "exit": float(rel[c, 3]), "first_s": float(rel[c, 1]),
                 "merge_wait": float(rel[c, 4]) if raw[c, 4] else None,
                 "merge_go": float(rel[c, 5]) if raw[c, 5] else None,
                 "item2": float(rel[c, 2]) if raw[c, 2] else None, "rate": float(rate_all[c]),
                 "items": items})
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", f"spans_{cfg}_{H}.json"), "w") as f:
    json.dump(rows, f)
