import json, statistics, sys
rows = json.load(open(sys.argv[1]))
m = [r for r in rows if r['merge_wait'] is not None]
def d(a, b): return [r[b] - r[a] for r in m if r[a] is not None and r[b] is not None]
# raw: 0 entry,1 weights ready,2 merged,3 exit,4 wait begin,5 go
import numpy as np
t0 = min(r['raw'][0] for r in rows)
def t(r, j): return (r['raw'][j] - t0) / 1000.0
wait = [t(r,5)-t(r,4) for r in m]; wts = [t(r,1)-t(r,5) for r in m]; mer = [t(r,2)-t(r,1) for r in m]; st = [t(r,3)-t(r,2) for r in m]
for name, x in (("wait", wait), ("m/l+weights", wts), ("merge loop", mer), ("store+exit", st)):
    print(f"{name:12s} median {statistics.median(x):5.2f} max {max(x):5.2f} us")
print("merger exits", statistics.median([t(r,3) for r in m]), "non-merger exits", statistics.median([t(r,3) for r in rows if r['merge_wait'] is None]))
