#!/usr/bin/env python
"""Writes tests/golden/sampler_u_one.json: Philox counters (offset, seed) of
the f2 sampler whose Box-Muller radius word w0 or w2 lies in the top 128
values, where the fp32 uniform (w + 0.5) 2^-32 rounds to exactly 1 (ln u = 0).
Calls only oracle/ (its own Philox4x32-10, KAT-pinned in test_oracle_pins).
    python tests/golden/make_sampler_u_one.py"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

SEED = 2506030990
TOP = np.uint32(0xFFFFFFFF - 127)
hits = []
chunk = 1 << 22
for base in range(0, 1 << 28, chunk):
    off = np.arange(base, base + chunk, dtype=np.uint64)
    ctr = np.zeros((chunk, 4), dtype=np.uint32)
    ctr[:, 2] = (off & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    key = np.tile(np.array([[SEED & 0xFFFFFFFF, SEED >> 32]], dtype=np.uint32), (chunk, 1))
    w = oracle.philox4x32_10(ctr, key)
    for word in (0, 2):
        for i in np.nonzero(w[:, word] >= TOP)[0][:2]:
            hits.append({"offset": int(off[i]), "word": word, "w": int(w[i, word])})
    if len({h["word"] for h in hits}) == 2:
        break
with open(os.path.join(HERE, "sampler_u_one.json"), "w") as f:
    json.dump({"seed": SEED, "note": "counter (0, 0, offset, 0), key = seed; word w >= 2^32 - 128: "
               "the kernel's fp32 uniform rounds to 1 (S:221-224 sampler, DESIGN Q18)",
               "hits": hits}, f, indent=1)
print(hits)
