#!/usr/bin/env python
"""SASS census of libtm.so: per kernel, the instruction counts that prove the
Blackwell-native path (/opt/skills/guides/B200_PROFILING.md table): tcgen05.mma
-> UTC*MMA, tcgen05.ld/st -> LDTM/STTM, TMA -> UTMALDG/UTMASTG/UBLKCP, plus
the legacy tensor path (HMMA) that must NOT appear, and MUFU.EX2 / FFMA2 of
the softmax.  Runs here (no GPU): cuobjdump -sass on the built library.
    python tools/sass_census.py [out.txt]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2506_03099_b200", "libtm.so")
PATTERNS = [("UTC*MMA", r"\bUTC\w*MMA\b"), ("LDTM", r"\bLDTM\b"), ("STTM", r"\bSTTM\b"),
            ("UTMALDG", r"\bUTMALDG\b"), ("UTMASTG", r"\bUTMASTG\b"), ("UBLKCP", r"\bUBLKCP\b"),
            ("UTMAPF", r"\bUTMAPF\b"), ("HMMA", r"\bHMMA\b"), ("MUFU.EX2", r"\bMUFU\.EX2\b"),
            ("FFMA2", r"\bFFMA2\b"), ("FMNMX3", r"\bFMNMX3\b"), ("SYNCS", r"\bSYNCS\.\w+"),
            ("ST.E(global)", r"\bSTG\.E\w*"), ("LD.E(global)", r"\bLDG\.E\w*")]


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        return name


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    arch = sorted(set(re.findall(r"arch = (sm_\w+)", sass)))
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        for nm, pat in PATTERNS:
            if re.search(pat, line):
                counts[cur][nm] += 1
    lines = [f"# SASS census of {os.path.relpath(LIB, ROOT)} (cuobjdump -sass); arch {arch}",
             "# columns: " + " ".join(nm for nm, _ in PATTERNS)]
    for fn, c in counts.items():
        dn = demangle(fn)
        dn = dn.replace("(anonymous namespace)::", "").replace("void ", "")
        short = re.sub(r"\(.*", "", dn)
        lines.append(f"{short[:60]:60s} " + " ".join(f"{nm}={c[nm]}" for nm, _ in PATTERNS if c[nm]))
    txt = "\n".join(lines) + "\n"
    if out:
        with open(out, "w") as f:
            f.write(txt)
    print(txt)


if __name__ == "__main__":
    main()
