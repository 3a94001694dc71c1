#!/usr/bin/env python
"""Accuracy of the CUDA path against the fp64 oracle at WAN sizes, every
query row (not sampled): max|O - O_ref| / max|O_ref| (the BJ.north_star
measure, bound 2e-2 for bf16 and 1e-4 for the fp32 mode) and the mean
relative error, per value distribution, chunks 1 and 2.
    python tools/accuracy_report.py [out.json]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import oracle  # noqa: E402
from gpu_util import from_dev, to_dev  # noqa: E402
from paper_2506_03099_b200 import tm  # noqa: E402
from synthetic import inputs as syn  # noqa: E402

CASES = [  # (name, H, Lr, Lc, dtype, dist, rows)
    ("wan512_bf16_D0", 40, 1024, 3072, "bf16", "D0", None),
    ("wan512_bf16_D1_peaky", 40, 1024, 3072, "bf16", "D1", None),
    ("wan512_bf16_D2_ref_dominant", 40, 1024, 3072, "bf16", "D2", None),
    ("wan512_bf16_D6_large_logits", 40, 1024, 3072, "bf16", "D6", None),
    ("wan512_fp32_D0", 40, 1024, 3072, "fp32", "D0", None),
    ("wan720_bf16_D0_sampled", 40, 2025, 6075, "bf16", "D0", 512),
    # one P = 8 rank's heads: every unit is cut into 3 pieces and co-merged from fp16 partials
    ("wan512_h5_bf16_D0", 5, 1024, 3072, "bf16", "D0", None),
    ("wan512_h5_bf16_D1_peaky", 5, 1024, 3072, "bf16", "D1", None),
    ("wan512_h5_bf16_D6_large_logits", 5, 1024, 3072, "bf16", "D6", None),
]

out = {"measure": "max|O-O_ref|/max|O_ref| over all rows and heads (rows: sampled where noted)",
       "oracle": "fp64 two-pass softmax over the literal concatenation (oracle/tm_oracle.c)",
       "cases": {}}
for name, H, Lr, Lc, dtype, dist, nrows in CASES:
    t0 = time.time()
    si = syn.StreamInputs(H, 128, Lr, Lc, dtype, dist, syn.seed_for(20, hash(name) % 97))
    ca = tm.ChunkAttention(H, 128, Lr, Lc, 1, 1, dtype=tm.TM_BF16 if dtype == "bf16" else tm.TM_FP32)
    so = oracle.StreamOracle()
    _, kr, vr = si.chunk(0, 0, 0)
    ca.put_reference(0, 0, to_dev(kr), to_dev(vr))
    so.put_reference(0, 0, kr.f64, vr.f64)
    rows = None
    if nrows:
        rows = np.sort(np.random.default_rng(1).choice(Lc, nrows, replace=False))
    res = {}
    for t in (1, 2):
        q, k, v = si.chunk(0, 0, t)
        o = torch.empty_like(to_dev(q))
        ca.attend(0, 0, t, to_dev(q), to_dev(k), to_dev(v), o)
        torch.cuda.synchronize()
        got = from_dev(o)
        ref = so.attend(0, 0, t, q.f64, k.f64, v.f64, rows=rows)
        if rows is not None:
            got = got[rows]
        err = np.abs(got - ref)
        res[f"chunk{t}"] = {"max_err_over_max_abs": float(err.max() / np.abs(ref).max()),
                            "mean_abs_err_over_mean_abs": float(err.mean() / np.abs(ref).mean()),
                            "rows": int(ref.shape[0])}
    ca.close()
    res["seconds"] = round(time.time() - t0, 1)
    out["cases"][name] = res
    print(name, json.dumps(res), flush=True)
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "accuracy.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
