import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2506_03099_b200 import tm
torch.manual_seed(0)
H, d = int(sys.argv[1]), 128
n = int(sys.argv[2]); Lc = int(sys.argv[3])
lens = [Lc] * n
L = sum(lens)
q, k, v = (torch.randn(L, H, d, device='cuda', dtype=torch.bfloat16) for _ in range(3))
ca = tm.ChunkAttention(H, d, Lc, Lc, 1, 1)
ow = torch.empty_like(q)
ca.window(q, k, v, ow, lens)
print("launches", ca.launches)
ca.put_reference(0, 0, k[:Lc].contiguous(), v[:Lc].contiguous())
for t in range(1, n):
    sl = slice(t * Lc, (t + 1) * Lc)
    os_ = torch.empty_like(q[sl])
    ca.attend(0, 0, t, q[sl].contiguous(), k[sl].contiguous(), v[sl].contiguous(), os_)
    torch.cuda.synchronize()
    diff = (os_.float() - ow[sl].float()).abs()
    bad = diff.amax(dim=2) > 1e-2     # [Lc][H]
    nb = int(bad.sum())
    print(f"chunk {t}: bad (row,head) pairs {nb} of {Lc*H}; bitwise equal {torch.equal(os_.view(torch.int16), ow[sl].view(torch.int16))}")
    if nb:
        rows, heads = torch.nonzero(bad, as_tuple=True)
        qp = (rows // 256).cpu().numpy(); hh = heads.cpu().numpy()
        units = sorted(set(zip(hh.tolist(), qp.tolist())))
        print("  bad (head, qpair) units:", units[:40], "count", len(units))
        print("  rows per unit sample:", [(int(h), int(p_), int(((hh==h)&(qp==p_)).sum())) for h,p_ in units[:8]])
