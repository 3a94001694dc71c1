# One bench attention_loop at H heads (fresh context), repeated R times.
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2506_03099_b200 import tm
H = int(os.environ.get("H", "20")); R = int(os.environ.get("R", "1")); K = int(os.environ.get("K", "40"))
for i in range(R):
    ms = bench.attention_loop(tm, torch, H, 128, 1024, 3072, K, torch.cuda.current_stream(), R=1)
    print(f"H={H} rep {i}: {ms*1e3:.1f} us", flush=True)
