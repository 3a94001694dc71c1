import sys, torch
sys.path.insert(0, '.')
from paper_2506_03099_b200 import tm

def run(H, lens, label):
    d = 128
    torch.manual_seed(0)
    L = sum(lens)
    q, k, v = (torch.randn(L, H, d, device='cuda', dtype=torch.bfloat16) for _ in range(3))
    ca = tm.ChunkAttention(H, d, lens[0], lens[1], 1, 1)
    ow = torch.empty_like(q)
    ca.window(q, k, v, ow, lens)
    nl = ca.launches
    ca.put_reference(0, 0, k[:lens[0]].contiguous(), v[:lens[0]].contiguous())
    res = []
    s0 = lens[0]
    for t in range(1, len(lens)):
        sl = slice(s0, s0 + lens[t]); s0 += lens[t]
        os_ = torch.empty_like(q[sl])
        ca.attend(0, 0, t, q[sl].contiguous(), k[sl].contiguous(), v[sl].contiguous(), os_)
        torch.cuda.synchronize()
        diff = (os_.float() - ow[sl].float()).abs().max().item()
        res.append((t, round(diff, 4), torch.equal(os_.view(torch.int16), ow[sl].view(torch.int16))))
    print(label, "H", H, "lens", lens[:3], "...", len(lens), "launches", nl, res, flush=True)
    ca.close()

run(4, [200] + [384] * 4, "small-pass")
run(8, [3072] * 2, "A")
run(8, [1024] * 3, "B")
run(8, [512] * 3, "C")
run(2, [3072] * 2, "D")
run(1, [3072] * 2, "E")
run(8, [384] * 3, "F")
run(4, [384] * 3, "G")
