#!/bin/bash
# Per-CTA spans at one head count for the working tree and for the A/B base tree
# in .ab_base/ (a copy of the baseline commit's sources):  tools/spans_ab.sh 5 [EXTRA_DEFINES]
H=${1:-5}
for tree in .ab_base .; do
  (cd $tree && TM_EXTRA_DEFINES="$2" SWEEP_H=$H python tools/cta_spans.py 2>&1 | grep -v "^   [0-9]" | sed "s|^|[$tree] |")
  if [ -n "$2" ]; then python tools/spans_merge.py $tree/gpurun_out/spans_512_$H.json | sed "s|^|[$tree] |"; fi
  (cd $tree && python -m paper_2506_03099_b200.build > /dev/null 2>&1)   # back to the production build
done
