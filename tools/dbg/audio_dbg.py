import sys, torch, statistics
sys.path.insert(0, '.')
from paper_2506_03099_b200 import tm
H, d = 40, 128
frames, T, A = 3, 1024, 32
g = torch.Generator(device="cuda").manual_seed(1)
bf = torch.bfloat16
qa = torch.randn(frames, T, H, d, device="cuda", dtype=bf, generator=g)
ka = torch.randn(frames, A, H, d, device="cuda", dtype=bf, generator=g)
va = torch.randn(frames, A, H, d, device="cuda", dtype=bf, generator=g)
oa = torch.empty_like(qa)
face = torch.tensor([r * 32 + cc for r in range(8, 24) for cc in range(8, 24)], dtype=torch.int32, device="cuda")
ca = tm.ChunkAttention(H, d, 16, 16, 1, 1)
n = face.numel()
nb = tm.tm_audio_scratch_bytes(ca.ctx, frames, n)
scratch = torch.empty(nb + 1024, dtype=torch.uint8, device="cuda")
ptr = (scratch.data_ptr() + 1023) // 1024 * 1024
def call():
    tm.tm_audio_cross_attention(ca.ctx, qa, ka, va, oa, frames, T, A, face, n, 5, ptr, nb)
for _ in range(10): call()
torch.cuda.synchronize()
for mode in range(3):
    ts = []
    for r in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if mode == 2:
            torch.empty(64 << 20, dtype=torch.uint8, device="cuda").fill_(1)   # flush L2
        a.record()
        if mode == 0:
            call()
        else:
            call()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print("mode", mode, "median us", statistics.median(ts), "launches", ca.launches)
# loop timing
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): call()
b.record(); torch.cuda.synchronize()
print("loop per call us", a.elapsed_time(b) * 1e3 / 50)
