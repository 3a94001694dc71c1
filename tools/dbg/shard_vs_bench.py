# Why does bench.py's H=5 loop read slower than tools/shard_sweep.py?  Same loop,
# with/without the nvidia-smi clock sampler running, inside one process.
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2506_03099_b200 import tm
stream = torch.cuda.current_stream()
for rep in range(2):
    ms = bench.attention_loop(tm, torch, 5, 128, 1024, 3072, 40, stream)
    print(f"attention_loop H=5 no sampler: {ms*1e3:.1f} us", flush=True)
    ck = bench.ClockSampler(0); ck.start()
    ms = bench.attention_loop(tm, torch, 5, 128, 1024, 3072, 40, stream)
    ck.stop()
    print(f"attention_loop H=5 with nvidia-smi sampler: {ms*1e3:.1f} us  {ck.summary()}", flush=True)
    nv = bench.NvmlSampler(0); nv.start()
    ms = bench.attention_loop(tm, torch, 5, 128, 1024, 3072, 40, stream)
    nv.stop()
    print(f"attention_loop H=5 with NVML thread: {ms*1e3:.1f} us", flush=True)
    ms = bench.attention_loop(tm, torch, 40, 128, 1024, 3072, 40, stream)
    print(f"attention_loop H=40: {ms*1e3:.1f} us", flush=True)
