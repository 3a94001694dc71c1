import sys, torch
sys.path.insert(0, '.')
from paper_2506_03099_b200 import tm

def ref_attn(q, k, v):   # [L][H][d] fp32
    s = torch.einsum('qhd,khd->hqk', q.float(), k.float()) / (q.shape[-1] ** 0.5)
    p = torch.softmax(s, dim=-1)
    return torch.einsum('hqk,khd->qhd', p, v.float())

def run(H, lens, label):
    d = 128
    torch.manual_seed(0)
    L = sum(lens)
    st = [0]
    for x in lens: st.append(st[-1] + x)
    q, k, v = (torch.randn(L, H, d, device='cuda', dtype=torch.bfloat16) for _ in range(3))
    ca = tm.ChunkAttention(H, d, lens[0], lens[1], 1, 1)
    ow = torch.empty_like(q)
    ca.window(q, k, v, ow, lens)
    ca.put_reference(0, 0, k[:lens[0]].contiguous(), v[:lens[0]].contiguous())
    res = []
    for t in range(0, len(lens)):
        sl = slice(st[t], st[t + 1])
        kc = sorted({0, max(t - 1, 0), t})
        kk = torch.cat([k[st[c]:st[c + 1]] for c in kc]); vv = torch.cat([v[st[c]:st[c + 1]] for c in kc])
        r = ref_attn(q[sl], kk, vv)
        ew = (ow[sl].float() - r).abs().max().item()
        es = None
        if t >= 1:
            os_ = torch.empty_like(q[sl])
            ca.attend(0, 0, t, q[sl].contiguous(), k[sl].contiguous(), v[sl].contiguous(), os_)
            torch.cuda.synchronize()
            es = round((os_.float() - r).abs().max().item(), 4)
        res.append((t, round(ew, 4), es))
    print(label, "H", H, "lens", lens[:2], len(lens), "(chunk, window err, stream err)", res, flush=True)
    ca.close()

run(4, [200] + [384] * 4, "small")
run(1, [3072] * 2, "E")
run(8, [384] * 3, "F")
run(8, [3072] * 2, "A")
