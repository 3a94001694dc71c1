import sys, time, torch
sys.path.insert(0, '.')
from paper_2506_03099_b200 import tm
H, d = 40, 128
frames, T, A = 3, 1024, 32
bf = torch.bfloat16
qa = torch.randn(frames, T, H, d, device="cuda", dtype=bf)
ka = torch.randn(frames, A, H, d, device="cuda", dtype=bf)
va = torch.randn(frames, A, H, d, device="cuda", dtype=bf)
oa = torch.empty_like(qa)
face = torch.tensor([r * 32 + cc for r in range(8, 24) for cc in range(8, 24)], dtype=torch.int32, device="cuda")
ca = tm.ChunkAttention(H, d, 16, 16, 1, 1)
n = face.numel()
nb = tm.tm_audio_scratch_bytes(ca.ctx, frames, n)
scratch = torch.empty(nb + 1024, dtype=torch.uint8, device="cuda")
ptr = (scratch.data_ptr() + 1023) // 1024 * 1024
s = torch.cuda.current_stream().cuda_stream
def call():
    tm.lib.tm_audio_cross_attention(ca.ctx, qa.data_ptr(), ka.data_ptr(), va.data_ptr(), oa.data_ptr(), frames, T, A, face.data_ptr(), n, 5, ptr, nb, s)
for _ in range(20): call()
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N): call()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"audio: host {1e6*(t1-t0)/N:.1f} us/call, wall incl. GPU {1e6*(t2-t0)/N:.1f} us/call")
# chunk attention H=5 zero-copy
for Hs in (5, 40):
    c2 = tm.ChunkAttention(Hs, d, 1024, 3072, 2, 1)
    q = torch.randn(3072, Hs, d, device="cuda", dtype=bf)
    c2.put_reference(0, 0, q[:1024].contiguous(), q[:1024].contiguous())
    c2.put_reference(1, 0, q[:1024].contiguous(), q[:1024].contiguous())
    o = torch.empty_like(q)
    ch = [0, 0]
    def call2(i):
        l = i % 2; ch[l] += 1
        tm.lib.tm_chunk_attention(c2.ctx, l, 0, ch[l], q.data_ptr(), q.data_ptr(), q.data_ptr(), o.data_ptr(), s)
    for i in range(10): call2(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(N): call2(i)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"chunk H={Hs}: host {1e6*(t1-t0)/N:.1f} us/call, wall {1e6*(t2-t0)/N:.1f} us/call")
