# f1 window A/B of the L2 prefetch (TM_L2_PREFETCH=0 vs 2), bench's measure_extras f1 code
for rep in 1 2 3; do for v in 0 2; do
TM_L2_PREFETCH=$v python - <<'PY'
import os, sys, torch, statistics
sys.path.insert(0, '.')
import bench
from paper_2506_03099_b200 import tm
H, d = 40, 128
bf = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(2506030990 + 77)
lens = [3 * 1024] * 7
L = sum(lens)
q, k, v = (torch.randn(L, H, d, device="cuda", dtype=bf, generator=g) for _ in range(3))
o = torch.empty_like(q)
ca = tm.ChunkAttention(H, d, 16, 16, 1, 1)
ms = bench._time_ms(torch, lambda: ca.window(q, k, v, o, lens))
fl = 4.0 * d * H * 3072 * 3072 * 18
print('pf=' + os.environ['TM_L2_PREFETCH'], 'f1 %.3f ms %.1f TFLOP/s' % (ms, fl / (ms * 1e-3) / 1e12))
PY
done; done > gpurun_out/ab31.txt 2>&1
