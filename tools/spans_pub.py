#!/usr/bin/env python
"""Stream-K merge chain from a TM_SPANS_MERGE2 + TM_SPANS_PUB spans build
(tools/cta_spans.py with TM_EXTRA_DEFINES="TM_SPANS_MERGE2 TM_SPANS_PUB"):
partners stamp 4 = tiles done, 6 = partial published; mergers stamp 4 = own
tiles done, 5 = all partials counted in, 1 = weights ready, 2 = merged, 3 = exit.
    python tools/spans_pub.py gpurun_out/spans_512_5.json"""
import json
import statistics as st
import sys

rows = json.load(open(sys.argv[1]))
t0 = min(r["raw"][0] for r in rows)
us = lambda r, j: (r["raw"][j] - t0) / 1e3 if r["raw"][j] else None
mer = [r for r in rows if r["raw"][5]]
par = [r for r in rows if r["raw"][6] and not r["raw"][5]]  # (mergers stamp 6 = last buffer landed)
both = []
med = lambda v: f"median {st.median(v):6.2f} min {min(v):6.2f} max {max(v):6.2f}" if v else "-"
print(f"{len(rows)} CTAs: {len(mer)} mergers, {len(par)} partner-only, {len(both)} partner+merger")
print("  partner write (tiles done -> published)", med([us(r, 6) - us(r, 4) for r in par if r["raw"][4]]))
print("  partner published (abs)                ", med([us(r, 6) for r in par + both]))
print("  merger own done (abs)                  ", med([us(r, 4) for r in mer]))
print("  merger wait (own done -> counted in)   ", med([us(r, 5) - us(r, 4) for r in mer]))
print("  weights (counted in -> weights)        ", med([us(r, 1) - us(r, 5) for r in mer if r["raw"][1]]))
print("  merge loop (weights -> merged)         ", med([us(r, 2) - us(r, 1) for r in mer if r["raw"][2]]))
print("  last buffer landed (counted in -> 6)   ", med([us(r, 6) - us(r, 5) for r in mer if r["raw"][6]]))
print("  merge after landing (6 -> merged)      ", med([us(r, 2) - us(r, 6) for r in mer if r["raw"][6] and r["raw"][2]]))
print("  store+exit (merged -> exit)            ", med([us(r, 3) - us(r, 2) for r in mer if r["raw"][2]]))
print("  exit: mergers", med([us(r, 3) for r in mer]), "| others", med([us(r, 3) for r in rows if not r["raw"][5]]))
# per merger: its partners are the following CTAs that published, up to the next merger's CTA
idx = {r["cta"]: r for r in rows}
lag = []
for r in mer:
    c = r["cta"] + 1
    last = None
    while c in idx and idx[c]["raw"][6]:
        last = us(idx[c], 6)
        if idx[c]["raw"][5]:
            break
        c += 1
    if last is not None:
        lag.append(us(r, 5) - last)
print("  poll lag (last following partner published -> counted in)", med(lag))
