timeout 300 python -m pytest tests -m gpu -q -x -k "sampler" > gpurun_out/g22.log 2>&1
for rep in 1 2 3; do for v in old a new; do
  L=paper_2506_03099_b200/libtm.so; case $v in old) L=paper_2506_03099_b200/libtm_old.so;; a) L=paper_2506_03099_b200/libtm_a.so;; esac
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
ts = []
for i in range(30):
    big.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ms = statistics.median(ts[5:])
print(os.environ['TM_LIB_PATH'].split('/')[-1], os.environ.get('TM_SAMPLER_GRID','res'), 'sampler %.1f us  %.0f GB/s' % (ms*1e3, n*12/(ms*1e-3)/1e9))
PY
done; done > gpurun_out/f2ab.txt 2>&1
