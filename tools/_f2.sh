# f2 sampler A/B: libtm_old.so vs libtm.so, back-to-back calls (bench.py's _time_ms) and with an L2 flush between calls
for rep in 1 2 3; do for v in old new; do
  L=paper_2506_03099_b200/libtm.so; [ $v = old ] && L=paper_2506_03099_b200/libtm_old.so
  TM_LIB_PATH=$L python - <<'PY'
import os, sys, torch, statistics
sys.path.insert(0, '.')
from paper_2506_03099_b200 import tm
n = 64*16*3*64*64
g = torch.Generator(device='cuda').manual_seed(1)
x = torch.randn(n, device='cuda', generator=g); v = torch.randn(n, device='cuda', generator=g).to(torch.bfloat16)
xb = torch.empty(n, device='cuda', dtype=torch.bfloat16)
ca = tm.ChunkAttention(40, 128, 16, 16, 1, 1)
f = lambda: tm.tm_flow_sampler_step(ca.ctx, x, v, tm.TM_BF16, n, 0.0, 0.5, seed=1, x_bf16_out=xb)
big = torch.empty(256*1024*1024, dtype=torch.uint8, device='cuda')
def run(flush):
    ts = []
    for i in range(30):
        if flush: big.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record()
        if flush: torch.cuda.synchronize()
        ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ts[5:]) * 1e3
print(os.environ['TM_LIB_PATH'].split('/')[-1], 'b2b %.1f us  flush %.1f us' % (run(False), run(True)))
PY
done; done > gpurun_out/f2ab2.txt 2>&1
