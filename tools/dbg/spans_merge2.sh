TM_EXTRA_DEFINES="TM_SPANS_MERGE2" SWEEP_H=5 python tools/cta_spans.py > gpurun_out/spans5m.txt 2>&1
head -12 gpurun_out/spans5m.txt
python tools/dbg/merge_spans.py gpurun_out/spans_512_5.json
TM_EXTRA_DEFINES="TM_SPANS_MERGE2" SWEEP_H=40 python tools/cta_spans.py > gpurun_out/spans40m.txt 2>&1
python tools/dbg/merge_spans.py gpurun_out/spans_512_40.json
