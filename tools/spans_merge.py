#!/usr/bin/env python
"""Merge-phase spans of the stream-K mergers from a TM_SPANS_MERGE2 spans build
(tools/cta_spans.py with TM_EXTRA_DEFINES=TM_SPANS_MERGE2 writes
gpurun_out/spans_<cfg>_<H>.json; slots: 4 merge wait begin, 5 merge go,
2 partials merged, 3 exit; 4 = the merger's own compute done, 5 = the last
remote partial's m/l landed).  Prints per-phase medians/maxima:
    python tools/spans_merge.py gpurun_out/spans_512_5.json"""
import json
import statistics
import sys

rows = json.load(open(sys.argv[1]))
t0 = min(r["raw"][0] for r in rows)
us = lambda r, j: (r["raw"][j] - t0) / 1e3 if r["raw"][j] else None
m = [r for r in rows if r["raw"][5]]
ph = {"to last (4->5)": [us(r, 5) - us(r, 4) for r in m],
      "merge (5->2)": [us(r, 2) - us(r, 5) for r in m if r["raw"][2]],
      "store+exit (2->3)": [us(r, 3) - us(r, 2) for r in m if r["raw"][2]]}
print(f"{len(m)} mergers of {len(rows)} CTAs; kernel end {max(us(r, 3) for r in rows):.1f} us")
for k, v in ph.items():
    if v:
        print(f"  {k:18s} median {statistics.median(v):5.2f}  max {max(v):5.2f} us")
nm = [us(r, 3) for r in rows if not r["raw"][5]]
print(f"  non-merger exit median {statistics.median(nm):.1f} max {max(nm):.1f}; "
      f"merger exit median {statistics.median(us(r, 3) for r in m):.1f} max {max(us(r, 3) for r in m):.1f}")
