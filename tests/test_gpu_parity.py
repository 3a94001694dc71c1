"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 oracle on the
same seeded inputs.  Tolerances (BJ.north_star): bf16 max|err| <= 2e-2 *
max|O| (internal alarm 8e-3), fp32 validation mode <= 1e-4, Euler fp32
<= 1e-6 * max|x|."""
import os

import numpy as np
import pytest
import torch

import oracle
from gpu_util import (BF16_ALARM, BF16_TOL, FP32_TOL, dev_copy, from_dev, rel_err, sample_rows,
                      to_dev)
from paper_2506_03099_b200 import tm
from synthetic import inputs as syn

pytestmark = pytest.mark.gpu

DT = {"bf16": tm.TM_BF16, "fp32": tm.TM_FP32}


def run_stream(H, d, Lr, Lc, dtype, dist="D0", chunks=2, layers=1, steps=1, rows=None,
               seed=syn.SEED_BASE, batch_check=True):
    """Stream `chunks` chunks through every (layer, step) and compare each
    call with the oracle's own streaming replay.  Returns the worst error."""
    si = syn.StreamInputs(H, d, Lr, Lc, dtype, dist, seed)
    ca = tm.ChunkAttention(H, d, Lr, Lc, layers, steps, dtype=DT[dtype])
    so = oracle.StreamOracle()
    for layer in range(layers):
        for step in range(steps):
            _, k, v = si.chunk(layer, step, 0)
            ca.put_reference(layer, step, to_dev(k), to_dev(v))
            so.put_reference(layer, step, k.f64, v.f64)
    worst = 0.0
    for t in range(1, chunks + 1):
        for step in range(steps):
            for layer in range(layers):
                q, k, v = si.chunk(layer, step, t)
                qd, kd, vd = to_dev(q), to_dev(k), to_dev(v)
                o = torch.empty_like(qd)
                ca.attend(layer, step, t, qd, kd, vd, o)
                ref = so.attend(layer, step, t, q.f64, k.f64, v.f64, rows=rows)
                got = from_dev(o)
                if rows is not None:
                    got = got[rows]
                worst = max(worst, rel_err(got, ref))
    ca.close()
    return worst


# ------------------------------------------------------------------ tiny (BJ.configs[0])

def test_tiny_config_fp32():
    """BJ.configs[0]: 2 heads, d=64, ref 16 tokens, 2 chunks x 32, fp32, 1 step."""
    err = run_stream(2, 64, 16, 32, "fp32", chunks=2)
    assert err <= FP32_TOL, err


@pytest.mark.parametrize("d", [64, 128])
def test_tiny_config_bf16(d):
    err = run_stream(2, d, 16, 32, "bf16", chunks=3)
    assert err <= BF16_ALARM, err


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("Lr,Lc", [(1, 1), (1, 130), (130, 1), (127, 129), (256, 128), (5, 300)])
def test_ragged_segments(dtype, Lr, Lc):
    """D5: segments of 1..300 tokens: partial KV tiles (masked keys must not
    leak: SURVEY Sec 4.4 shows 5 unmasked zero keys cost 4.6e-4, caught by
    the fp32 bar) and partial Q tiles (pad rows must not be stored)."""
    err = run_stream(3, 128, Lr, Lc, dtype, chunks=3)
    assert err <= (FP32_TOL if dtype == "fp32" else BF16_ALARM), err


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("H,Lr,Lc", [(1, 7000, 200), (1, 2000, 256), (2, 5000, 130)])
def test_few_units_long_kv_many_pieces(dtype, H, Lr, Lc):
    """Few work units with long KV ranges: the stream-K tail cuts one unit into
    up to 14 pieces over 14 CTAs (1 x 1 x 59 tiles at Lr=7000), so the merger
    accumulates 13 partials (two batches of weight loads, 13 bulk copies)."""
    err = run_stream(H, 128, Lr, Lc, dtype, chunks=2)
    assert err <= (FP32_TOL if dtype == "fp32" else BF16_ALARM), err


@pytest.mark.parametrize("Lr,Lc", [(7000, 200), (1024, 512)])
def test_many_pieces_d64_bf16(Lr, Lc):
    """d = 64 merges: the partials' column halves are 32 KB, three in flight
    over the Q tiles and the ring (13 partials at Lr=7000, 3 at Lr=1024)."""
    err = run_stream(1, 64, Lr, Lc, "bf16", chunks=2)
    assert err <= BF16_ALARM, err


def test_more_pieces_than_the_contributor_mask():
    """One unit over ~630 KV tiles: at the default minimum piece it would be
    cut into ~148 pieces; the merger tracks contributors in a 64-bit mask, so
    the schedule raises the minimum piece until a unit has <= 65 pieces."""
    err = run_stream(1, 128, 80000, 130, "bf16", chunks=1)
    assert err <= BF16_ALARM, err


@pytest.mark.parametrize("vscale_log2", [15, -20])
def test_many_pieces_extreme_value_scales(vscale_log2):
    """Stream-K partials are fp16 rows with a per-row power-of-two scale (the
    row's max |O| lands in [2^14, 2^15)).  V scaled by 2^15 (unscaled fp16
    partials of the unnormalised O would overflow 65504) and by 2^-20 (they
    would underflow) still merge within the bf16 alarm; co-merged units
    (>= 3 pieces) and 13-partial merges both occur at Lr = 7000."""
    H, d, Lr, Lc = 2, 128, 7000, 300
    f = 2.0 ** vscale_log2
    si = syn.StreamInputs(H, d, Lr, Lc, "bf16", "D0", syn.SEED_BASE + 77)
    ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1)
    so = oracle.StreamOracle()
    _, k, v = si.chunk(0, 0, 0)
    ca.put_reference(0, 0, to_dev(k), to_dev(v) * f)          # power-of-two scale: exact in bf16
    so.put_reference(0, 0, k.f64, v.f64 * f)
    worst = 0.0
    for t in (1, 2):
        q, k, v = si.chunk(0, 0, t)
        o = torch.empty_like(to_dev(q))
        ca.attend(0, 0, t, to_dev(q), to_dev(k), to_dev(v) * f, o)
        ref = so.attend(0, 0, t, q.f64, k.f64, v.f64 * f)
        worst = max(worst, rel_err(from_dev(o), ref))
    ca.close()
    assert worst <= BF16_ALARM, worst


@pytest.mark.parametrize("dist", ["D1", "D2", "D3", "D6"])
def test_distributions_bf16(dist):
    err = run_stream(4, 128, 256, 640, "bf16", dist=dist, chunks=3)
    assert err <= BF16_ALARM, (dist, err)


@pytest.mark.parametrize("dist", ["D1", "D2", "D6"])
def test_distributions_fp32(dist):
    err = run_stream(2, 128, 200, 330, "fp32", dist=dist, chunks=3)
    assert err <= FP32_TOL, (dist, err)


def test_layers_and_steps_keep_separate_caches():
    """K/V cached per timestep per block -- 3 layers x 2 steps, 4 chunks."""
    err = run_stream(2, 128, 64, 192, "bf16", chunks=4, layers=3, steps=2)
    assert err <= BF16_ALARM, err


# ------------------------------------------------------------------ WAN-2.1 shapes

def test_wan512_single_layer_bf16_sampled():
    """BJ.configs[1]: 40 heads, d=128, Lr=1024 (one reference frame),
    Lc=3072 (3 latent frames): chunk 1 (Lk=4096) and chunk 2 (Lk=7168)."""
    rows = sample_rows(3072, k=40)
    err = run_stream(40, 128, 1024, 3072, "bf16", chunks=2, rows=rows)
    assert err <= BF16_ALARM, err


def test_wan720_bf16_sampled():
    """BJ.configs[4]: 720^2, 2025 tokens/frame: Lr=2025, Lc=6075 (ragged tiles)."""
    rows = sample_rows(6075, k=24)
    err = run_stream(40, 128, 2025, 6075, "bf16", chunks=2, rows=rows)
    assert err <= BF16_ALARM, err


def test_wan512_fp32_validation_sampled():
    rows = sample_rows(3072, k=12)
    err = run_stream(40, 128, 1024, 3072, "fp32", chunks=2, rows=rows)
    assert err <= FP32_TOL, err


def test_wan512_uniform_closed_form_all_rows():
    """S:42 closed form at full size, every row: q = 0 -> O = mean of the
    allowed V rows; segment-tagged V (D3) exposes a dropped/duplicated
    segment.  Expected value from numpy means of the bf16 inputs."""
    H, d, Lr, Lc = 40, 128, 1024, 3072
    si = syn.StreamInputs(H, d, Lr, Lc, "bf16", "D4", syn.seed_for(1, 4))
    ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1)
    _, kr, vr = si.chunk(0, 0, 0)
    ca.put_reference(0, 0, to_dev(kr), to_dev(vr))
    vals = [vr.f64]
    for t in (1, 2, 3):
        q, k, v = si.chunk(0, 0, t)
        o = torch.empty_like(to_dev(q))
        ca.attend(0, 0, t, to_dev(q), to_dev(k), to_dev(v), o)
        allowed = [vals[0]] + ([vals[-1]] if t >= 2 else []) + [v.f64]
        mean = np.concatenate(allowed).mean(axis=0)            # [H][d]
        got = from_dev(o)
        err = np.abs(got - mean[None]).max() / np.abs(mean).max()
        assert err <= BF16_TOL, (t, err)
        vals.append(v.f64)
    ca.close()


# ------------------------------------------------------------------ invariants

def test_deterministic_bitwise():
    """Q15 / S:68: fixed tile order, no atomics -> bitwise identical reruns."""
    H, d, Lr, Lc = 8, 128, 512, 1536
    si = syn.StreamInputs(H, d, Lr, Lc, "bf16", "D0", 5)
    outs = []
    for _ in range(2):
        ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1)
        _, kr, vr = si.chunk(0, 0, 0)
        ca.put_reference(0, 0, to_dev(kr), to_dev(vr))
        res = []
        for t in (1, 2, 3):
            q, k, v = si.chunk(0, 0, t)
            o = torch.empty_like(to_dev(q))
            ca.attend(0, 0, t, to_dev(q), to_dev(k), to_dev(v), o)
            res.append(o.view(torch.int16).cpu().numpy())
        outs.append(res)
        ca.close()
    for a, b in zip(*outs):
        assert (a == b).all()


def test_reference_immutable_and_constant_footprint():
    """reference bitwise unchanged after many chunks; the cache
    footprint is a closed form independent of stream length; chunk 200
    still matches the oracle."""
    H, d, Lr, Lc = 2, 128, 128, 256
    torch.manual_seed(syn.seed_for(9, 0))
    ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1)
    before = ca.cache_bytes
    kr = torch.randn(Lr, H, d, device="cuda").bfloat16()
    vr = torch.randn(Lr, H, d, device="cuda").bfloat16()
    ca.put_reference(0, 0, kr, vr)
    kp, vp = ca.ref_ptr(0, 0)
    snap = kr.clone()
    so = oracle.StreamOracle()
    so.put_reference(0, 0, from_dev(kr), from_dev(vr))
    for t in range(1, 201):
        q, k, v = (torch.randn(Lc, H, d, device="cuda").bfloat16() for _ in range(3))
        o = torch.empty_like(q)
        ca.attend(0, 0, t, q, k, v, o)
        ref = so.attend(0, 0, t, from_dev(q), from_dev(k), from_dev(v),
                        rows=[0, 77, 255] if t < 200 else None)
        got = from_dev(o)
        got = got if t == 200 else got[[0, 77, 255]]
        assert rel_err(got, ref) <= BF16_ALARM
    torch.cuda.synchronize()
    buf = torch.empty_like(kr)
    dev_copy(buf.data_ptr(), kp, kr.numel() * 2)
    assert torch.equal(buf.view(torch.int16), snap.view(torch.int16))
    assert tm.tm_kvcache_bytes(ca.cfg) == before
    ca.close()


def test_stream_order_errors_on_device():
    H, d = 2, 64
    ca = tm.ChunkAttention(H, d, 16, 32, 2, 2)
    q = torch.zeros(32, H, d, device="cuda", dtype=torch.bfloat16)
    o = torch.empty_like(q)
    r = torch.zeros(16, H, d, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(tm.TMError) as e:
        ca.attend(0, 0, 1, q, q, q, o)                      # cache miss
    assert e.value.status == 4
    ca.put_reference(0, -1, r, r)                           # all steps
    with pytest.raises(tm.TMError) as e:
        ca.attend(0, 1, 2, q, q, q, o)                      # skipped chunk 1
    assert e.value.status == 4
    ca.attend(0, 1, 1, q, q, q, o)
    ca.attend(0, 1, 1, q, q, q, o)                          # redo allowed
    with pytest.raises(tm.TMError) as e:
        ca.put_reference(0, 1, r, r)
    assert e.value.status == 5
    ca.put_reference(0, 0, r, r)                            # step 0 not started yet: allowed
    with pytest.raises(tm.TMError) as e:
        ca.attend(5, 0, 1, q, q, q, o)
    assert e.value.status == 1
    with pytest.raises(tm.TMError):
        ca.attend(0, 0, 0, q, q, q, o)                      # chunk 0 is the reference
    ca.reset()
    ca.put_reference(0, 1, r, r)                            # new stream
    ca.close()


def test_zero_copy_append_via_slot_ptr():
    """Writing K/V straight into tm_kvcache_slot_ptr skips the append copy
    and gives the same result."""
    H, d, Lr, Lc = 4, 128, 128, 384
    si = syn.StreamInputs(H, d, Lr, Lc, "bf16", "D0", 17)
    res = []
    for zero_copy in (False, True):
        ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1)
        _, kr, vr = si.chunk(0, 0, 0)
        ca.put_reference(0, 0, to_dev(kr), to_dev(vr))
        outs = []
        for t in (1, 2, 3):
            q, k, v = si.chunk(0, 0, t)
            kd, vd = to_dev(k), to_dev(v)
            if zero_copy:
                kp, vp = ca.slot_ptr(0, 0, t)
                dev_copy(kp, kd.data_ptr(), kd.numel() * 2)
                dev_copy(vp, vd.data_ptr(), vd.numel() * 2)
                kd_arg, vd_arg = kp, vp
            else:
                kd_arg, vd_arg = kd, vd
            o = torch.empty_like(kd)
            ca.attend(0, 0, t, to_dev(q), kd_arg, vd_arg, o)
            outs.append(o.view(torch.int16).cpu().numpy())
        res.append(outs)
        ca.close()
    for a, b in zip(*res):
        assert (a == b).all()


@pytest.mark.parametrize("what", ["prev_k", "ref_v"])
def test_corrupted_cache_is_detected(what):
    """Fault injection: corrupt one head of the cached c_{t-1}
    K (or the reference V) between chunks; the next chunk must then miss the
    oracle by far more than the bf16 alarm -- the parity check sees the cache,
    it does not just recompute from the inputs."""
    H, d, Lr, Lc = 4, 128, 128, 384
    si = syn.StreamInputs(H, d, Lr, Lc, "bf16", "D0", 23)
    ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1)
    so = oracle.StreamOracle()
    _, kr, vr = si.chunk(0, 0, 0)
    ca.put_reference(0, 0, to_dev(kr), to_dev(vr))
    so.put_reference(0, 0, kr.f64, vr.f64)
    q, k, v = si.chunk(0, 0, 1)
    o = torch.empty_like(to_dev(q))
    ca.attend(0, 0, 1, to_dev(q), to_dev(k), to_dev(v), o)
    assert rel_err(from_dev(o), so.attend(0, 0, 1, q.f64, k.f64, v.f64)) <= BF16_ALARM
    torch.cuda.synchronize()
    # overwrite head 1 of the cached tensor with large values
    if what == "prev_k":
        ptr, L = ca.slot_ptr(0, 0, 1)[0], Lc
    else:
        ptr, L = ca.ref_ptr(0, 0)[1], Lr
    garbage = torch.full((L, H, d), 8.0, device="cuda", dtype=torch.bfloat16)
    cur = torch.empty_like(garbage)
    dev_copy(cur.data_ptr(), ptr, cur.numel() * 2)
    cur[:, 1] = garbage[:, 1]
    dev_copy(ptr, cur.data_ptr(), cur.numel() * 2)
    q, k, v = si.chunk(0, 0, 2)
    ca.attend(0, 0, 2, to_dev(q), to_dev(k), to_dev(v), o)
    err = rel_err(from_dev(o), so.attend(0, 0, 2, q.f64, k.f64, v.f64))
    assert err > 20 * BF16_ALARM, err
    ca.close()


def test_launch_count_and_variant():
    ca = tm.ChunkAttention(2, 128, 128, 128, 1, 1)
    assert ca.variant == "sm100_tcgen05"
    x = torch.zeros(128, 2, 128, device="cuda", dtype=torch.bfloat16)
    ca.put_reference(0, 0, x, x)
    o = torch.empty_like(x)
    ca.attend(0, 0, 1, x, x, x, o)
    assert ca.launches == 1
    ca.close()
    cf = tm.ChunkAttention(2, 64, 16, 32, 1, 1, dtype=tm.TM_FP32)
    assert cf.variant == "fp32_simt"
    cf.close()


# ------------------------------------------------------------------ Euler (a7)

@pytest.mark.parametrize("v_dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("n", [1, 7, 8, 1000, 196_608, 388_800 + 3])
def test_euler_vs_oracle(v_dtype, n):
    """x <- x + dt*v: fp32 single-FMA vs the fp64 oracle,
    <= 1e-6 * max|x|."""
    x, v = syn.euler_inputs(n, syn.seed_for(7, 0), v_dtype)
    xd, vd = to_dev(x), to_dev(v)
    for dt in (1.0, 0.5, -0.125):
        ref = oracle.euler(from_dev(xd), v.f64, dt)
        tm.tm_flow_euler_step(None, xd, vd, DT[v_dtype], n, dt)
        torch.cuda.synchronize()
        got = from_dev(xd)
        assert np.abs(got - ref).max() <= 1e-6 * np.abs(ref).max()


def test_euler_constant_velocity_closed_form():
    """constant velocity c, N Euler steps of 1/N -> x0 + c."""
    n = 4096
    for N in (1, 2, 12, 24):
        x = torch.full((n,), 0.25, device="cuda")
        c = torch.full((n,), 3.0, device="cuda")
        for _ in range(N):
            tm.tm_flow_euler_step(None, x, c, tm.TM_FP32, n, 1.0 / N)
        torch.cuda.synchronize()
        assert torch.allclose(x, torch.full_like(x, 3.25), rtol=0, atol=1e-5 * N)


def test_euler_rectified_flow_identity():
    """Eqs 1-2: from x_t = t x1 + (1-t) x0 one step of dt along v = x1 - x0
    lands on x_{t+dt} (to fp32 rounding)."""
    n = 10_000
    rng = np.random.default_rng(3)
    x0, x1 = rng.standard_normal(n), rng.standard_normal(n)
    for t, dt in [(0.0, 1.0), (0.0, 0.5), (0.5, 0.5)]:
        xt = oracle.interpolate(x0, x1, t).astype(np.float32)
        v = oracle.velocity_target(x0, x1).astype(np.float32)
        xd, vd = torch.from_numpy(xt).cuda(), torch.from_numpy(v).cuda()
        tm.tm_flow_euler_step(None, xd, vd, tm.TM_FP32, n, dt)
        torch.cuda.synchronize()
        target = oracle.interpolate(x0, x1, t + dt)
        assert np.abs(xd.double().cpu().numpy() - target).max() < 1e-5


# ------------------------------------------------------------------ batch and exchange path

def test_batch_of_independent_streams():
    """B = 2 streams in one call ([B][L][H][d]); each equals its own oracle stream."""
    H, d, Lr, Lc, B = 3, 128, 100, 260, 2
    ins = [syn.StreamInputs(H, d, Lr, Lc, "bf16", "D0", syn.seed_for(8, 0, extra=b)) for b in range(B)]
    ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1, batch=B)
    sos = [oracle.StreamOracle() for _ in range(B)]
    refs = [si.chunk(0, 0, 0) for si in ins]
    kr = torch.stack([to_dev(r[1]) for r in refs])
    vr = torch.stack([to_dev(r[2]) for r in refs])
    ca.put_reference(0, 0, kr, vr)
    for so, r in zip(sos, refs):
        so.put_reference(0, 0, r[1].f64, r[2].f64)
    for t in (1, 2, 3):
        cs = [si.chunk(0, 0, t) for si in ins]
        q, k, v = (torch.stack([to_dev(c[i]) for c in cs]) for i in range(3))
        o = torch.empty_like(q)
        ca.attend(0, 0, t, q, k, v, o)
        for b in range(B):
            ref = sos[b].attend(0, 0, t, cs[b][0].f64, cs[b][1].f64, cs[b][2].f64)
            assert rel_err(from_dev(o[b]), ref) <= BF16_ALARM
    ca.close()


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_forced_ulysses_path_matches_direct(dtype, monkeypatch):
    """TM_FORCE_ULYSSES=1 runs the exchange path on one GPU (pack kernel,
    1-rank ncclAlltoAll, unpack into the cache slot, O back the same way):
    bitwise equal to the direct path, and within tolerance of the oracle."""
    H, d, Lr, Lc = 4, 128, 200, 333
    si = syn.StreamInputs(H, d, Lr, Lc, dtype, "D0", syn.seed_for(9, 1))
    outs = []
    for forced in (False, True):
        if forced:
            monkeypatch.setenv("TM_FORCE_ULYSSES", "1")
        ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1, dtype=DT[dtype])
        monkeypatch.delenv("TM_FORCE_ULYSSES", raising=False)
        _, kr, vr = si.chunk(0, 0, 0)
        ca.put_reference(0, 0, to_dev(kr), to_dev(vr))
        res = []
        so = oracle.StreamOracle()
        so.put_reference(0, 0, kr.f64, vr.f64)
        for t in (1, 2, 3):
            q, k, v = si.chunk(0, 0, t)
            o = torch.empty_like(to_dev(q))
            ca.attend(0, 0, t, to_dev(q), to_dev(k), to_dev(v), o)
            torch.cuda.synchronize()
            ref = so.attend(0, 0, t, q.f64, k.f64, v.f64)
            assert rel_err(from_dev(o), ref) <= (FP32_TOL if dtype == "fp32" else BF16_ALARM)
            res.append(o.view(torch.int16 if dtype == "bf16" else torch.int32).cpu().numpy())
        if forced:
            assert ca.launches >= 5          # pack x3, attention, pack, unpack (+ unpacks)
            ca.check()                       # the communicator reports no async error
        outs.append(res)
        ca.close()
    for a, b in zip(*outs):
        assert (a == b).all()


# ------------------------------------------------------------------ Table 1 variants

def test_table1_chunk7_bf16_sampled():
    """f3: chunk = 7 latent frames at 512^2 (Lc = 7168, Lk up to
    15360 at t >= 2), row-sampled against the oracle."""
    rows = sample_rows(7168, k=16)
    err = run_stream(40, 128, 1024, 7168, "bf16", chunks=2, rows=rows)
    assert err <= BF16_ALARM, err


def test_table1_four_steps_cache_slots():
    """f3: 4 denoising steps -> 4 cache step slots per layer;
    every (layer, step) keeps its own reference and previous chunk."""
    err = run_stream(4, 128, 128, 384, "bf16", chunks=3, layers=2, steps=4)
    assert err <= BF16_ALARM, err


# ------------------------------------------------------------------ chunk 0 generated

@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("Lr", [1, 300, 1024])
def test_reference_attention_mode(dtype, Lr):
    """tm_reference_attention: c_0's queries attend c_0 only -- the
    window oracle with one chunk -- and its K/V become the cached reference,
    so the following chunks match the streaming oracle fed the same K/V;
    step = -1 stores it for both steps."""
    H, d, Lc = 4, 128, 200
    rng = np.random.default_rng(syn.seed_for(15, 0, extra=Lr))
    q0, k0, v0 = syn.chunk_qkv(rng, Lr, H, d, dtype, "D0")
    ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 2, dtype=DT[dtype])
    o0 = torch.empty_like(to_dev(q0))
    ca.reference_attend(0, -1, to_dev(q0), to_dev(k0), to_dev(v0), o0)
    torch.cuda.synchronize()
    tol = FP32_TOL if dtype == "fp32" else BF16_ALARM
    ref0 = oracle.window_attention(q0.f64, k0.f64, v0.f64, [Lr])
    assert rel_err(from_dev(o0), ref0) <= tol
    si = syn.StreamInputs(H, d, Lr, Lc, dtype, "D0", syn.seed_for(15, 1, extra=Lr))
    so = oracle.StreamOracle()
    for st in range(2):
        so.put_reference(0, st, k0.f64, v0.f64)
    for t in (1, 2):
        for st in range(2):
            q, k, v = si.chunk(0, st, t)
            o = torch.empty_like(to_dev(q))
            ca.attend(0, st, t, to_dev(q), to_dev(k), to_dev(v), o)
            assert rel_err(from_dev(o), so.attend(0, st, t, q.f64, k.f64, v.f64)) <= tol
    with pytest.raises(tm.TMError) as e:              # immutable after chunk 1
        ca.reference_attend(0, 0, to_dev(q0), to_dev(k0), to_dev(v0), o0)
    assert e.value.status == 5
    ca.close()


# ------------------------------------------------------------------ full window

def _window_inputs(H, d, lens, dtype, dist, seed):
    rng = np.random.default_rng(seed)
    q, k, v = syn.chunk_qkv(rng, int(sum(lens)), H, d, dtype, dist)
    return q, k, v


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("lens", [[16, 32, 32], [130, 1, 257, 128, 5], [64] * 7, [300, 200, 100, 50]])
def test_window_attention_vs_oracle(dtype, lens):
    """f1: tm_window_attention (every chunk c attends {0, c-1, c}) vs the
    oracle's full-window form c1."""
    H, d = 3, 128
    q, k, v = _window_inputs(H, d, lens, dtype, "D0", syn.seed_for(10, 0, extra=len(lens)))
    ca = tm.ChunkAttention(H, d, 16, 16, 1, 1, dtype=DT[dtype])
    o = torch.empty_like(to_dev(q))
    ca.window(to_dev(q), to_dev(k), to_dev(v), o, lens)
    ref = oracle.window_attention(q.f64, k.f64, v.f64, lens)
    if dtype == "fp32":
        assert ca.launches == len(lens)              # validation mode: one launch per chunk
    else:
        assert 1 <= ca.launches <= len(lens)         # chunks batched (<= 8 blocks, 4 tail shapes)
    assert rel_err(from_dev(o), ref) <= (FP32_TOL if dtype == "fp32" else BF16_ALARM)
    with pytest.raises(tm.TMError) as e:
        ca.window(to_dev(q), to_dev(k), to_dev(v), o, lens[:-1] + [0, lens[-1]])
    assert e.value.status == 3                       # empty chunk: degenerate mask
    ca.close()


def test_window_wan512_21_frames_sampled():
    """f1 at WAN scale: the 21-latent-frame window = 7 chunks x 3 frames of
    1024 tokens, 21504 tokens, 40 heads; row-sampled in every chunk."""
    H, d, lens = 40, 128, [3072] * 7
    q, k, v = _window_inputs(H, d, lens, "bf16", "D0", syn.seed_for(10, 1))
    ca = tm.ChunkAttention(H, d, 16, 16, 1, 1)
    o = torch.empty_like(to_dev(q))
    ca.window(to_dev(q), to_dev(k), to_dev(v), o, lens)
    assert ca.launches == 1                          # all 7 query chunks in one launch
    rows = np.concatenate([c * 3072 + sample_rows(3072, k=3, seed=c) for c in range(7)])
    ref = oracle.window_attention(q.f64, k.f64, v.f64, lens, rows=rows)
    assert rel_err(from_dev(o)[rows], ref) <= BF16_ALARM
    ca.close()


def test_window_equals_streaming_bitwise():
    """S:303 on the GPU: the window form and the cache-streaming form run the
    same segment schedule, so each chunk's rows agree bit for bit."""
    H, d, Lr, Lc, n = 4, 128, 200, 384, 5
    lens = [Lr] + [Lc] * (n - 1)
    q, k, v = _window_inputs(H, d, lens, "bf16", "D0", syn.seed_for(10, 2))
    qd, kd, vd = to_dev(q), to_dev(k), to_dev(v)
    ca = tm.ChunkAttention(H, d, Lr, Lc, 1, 1)
    ow = torch.empty_like(qd)
    ca.window(qd, kd, vd, ow, lens)
    ca.put_reference(0, 0, kd[:Lr].contiguous(), vd[:Lr].contiguous())
    for t in range(1, n):
        sl = slice(Lr + (t - 1) * Lc, Lr + t * Lc)
        os_ = torch.empty_like(qd[sl])
        ca.attend(0, 0, t, qd[sl].contiguous(), kd[sl].contiguous(), vd[sl].contiguous(), os_)
        assert torch.equal(os_.view(torch.int16), ow[sl].view(torch.int16)), t
    ca.close()


# ------------------------------------------------------------------ sampler step

@pytest.mark.parametrize("v_dtype", ["fp32", "bf16"])
def test_sampler_step_with_given_noise_vs_oracle(v_dtype):
    """f2: x1_hat = x + (1 - t) v, Eq 1 re-noise with eps; the 2-NFE
    student schedule t = 0 -> 0.5 -> final (reading Q10), vs the oracle."""
    n = 196_608 + 5
    x, v = syn.euler_inputs(n, syn.seed_for(11, 0), v_dtype)
    eps = syn.euler_inputs(n, syn.seed_for(11, 1))[0]
    xd, vd, ed = to_dev(x), to_dev(v), to_dev(eps)
    xb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    ref = oracle.sampler_step(x.f64, v.f64, eps.f64, 0.0, 0.5)
    tm.tm_flow_sampler_step(None, xd, vd, DT[v_dtype], n, 0.0, 0.5, eps=ed, x_bf16_out=xb)
    torch.cuda.synchronize()
    assert np.abs(from_dev(xd) - ref).max() <= 1e-6 * np.abs(ref).max()
    assert torch.equal(xb, xd.to(torch.bfloat16))            # bf16 RNE of the new state
    ref2 = oracle.sampler_step(from_dev(xd), v.f64, None, 0.5, 1.0)
    tm.tm_flow_sampler_step(None, xd, vd, DT[v_dtype], n, 0.5, 1.0)
    torch.cuda.synchronize()
    assert np.abs(from_dev(xd) - ref2).max() <= 1e-6 * np.abs(ref2).max()


def test_sampler_in_kernel_philox_matches_oracle_generator():
    """f2 noise: with x = v = 0, t: 0 -> 0.5 the new state is eps / 2; the
    kernel's Philox4x32-10 + Box-Muller draws equal the oracle side's own
    implementation (KAT-pinned) to fp32 rounding; deterministic per seed."""
    n = 1_000_003
    for seed, offset in ((2506030990, 0), (7, 12345)):
        xd = torch.zeros(n, device="cuda")
        vd = torch.zeros(n, device="cuda")
        tm.tm_flow_sampler_step(None, xd, vd, tm.TM_FP32, n, 0.0, 0.5, seed=seed, offset=offset)
        torch.cuda.synchronize()
        z = 2.0 * xd.double().cpu().numpy()
        ref = oracle.philox_normal(n, seed, offset)
        assert np.abs(z - ref).max() < 2e-4
        x2 = torch.zeros(n, device="cuda")
        tm.tm_flow_sampler_step(None, x2, vd, tm.TM_FP32, n, 0.0, 0.5, seed=seed, offset=offset)
        torch.cuda.synchronize()
        assert torch.equal(x2, xd)
    with pytest.raises(tm.TMError):
        tm.tm_flow_sampler_step(None, xd, vd, tm.TM_FP32, n, 0.5, 0.5)     # t_next must exceed t



def test_sampler_uniform_rounding_to_one_is_finite():
    """f2 edge: Philox words in the top 128 values make the kernel's fp32
    uniform exactly 1 (ln u = 0, radius 0); the draw must stay finite.  The
    fp64 oracle keeps u < 1, radius sqrt(-2 ln u) <= 2.44e-4 there, which
    bounds the difference.  Counters from tests/golden/sampler_u_one.json
    (written by tests/golden/make_sampler_u_one.py from the oracle's Philox)."""
    import json
    with open(os.path.join(os.path.dirname(__file__), "golden", "sampler_u_one.json")) as f:
        g = json.load(f)
    assert {h["word"] for h in g["hits"]} == {0, 2}
    for h in g["hits"]:
        xd = torch.zeros(4, device="cuda")
        vd = torch.zeros(4, device="cuda")
        tm.tm_flow_sampler_step(None, xd, vd, tm.TM_FP32, 4, 0.0, 0.5, seed=g["seed"], offset=h["offset"])
        torch.cuda.synchronize()
        z = 2.0 * xd.double().cpu().numpy()
        assert np.isfinite(z).all(), z
        ref = oracle.philox_normal(4, g["seed"], h["offset"])
        pair = slice(h["word"], h["word"] + 2)         # the two draws sharing that radius
        assert np.abs(z[pair]).max() < 2.5e-4, z
        assert np.abs(z[pair] - ref[pair]).max() < 2.5e-4
        other = slice(2 - h["word"], 4 - h["word"])
        assert np.abs(z[other] - ref[other]).max() < 2e-4

# ------------------------------------------------------------------ audio cross-attention

def _audio_case(frames, T, A, H, d, n_face, dtype, seed, B=1):
    rng = np.random.default_rng(seed)
    q, _, _ = syn.chunk_qkv(rng, B * frames * T, H, d, dtype, "D0")
    k, v, _ = syn.chunk_qkv(rng, B * frames * A, H, d, dtype, "D0")
    face = np.sort(rng.choice(T, size=n_face, replace=False)).astype(np.int32)
    return q, k, v, face


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("frames,T,A,n_face", [(3, 64, 8, 20), (7, 40, 5, 40), (1, 33, 3, 1), (2, 50, 16, 7),
                                                  (7, 40, 48, 13), (4, 300, 40, 150)])
def test_audio_cross_attention_vs_oracle(dtype, frames, T, A, n_face):
    """f4: face rows attend the clamped 5-frame audio
    window; non-face rows are exactly zero."""
    H, d = 4, 128
    q, k, v, face = _audio_case(frames, T, A, H, d, n_face, dtype, syn.seed_for(12, frames, extra=T))
    ca = tm.ChunkAttention(H, d, 16, 16, 1, 1, dtype=DT[dtype])
    qd = to_dev(q).view(frames, T, H, d)
    kd, vd = to_dev(k).view(frames, A, H, d), to_dev(v).view(frames, A, H, d)
    o = torch.full_like(qd, 7.0)
    ca.audio(qd, kd, vd, o, torch.from_numpy(face).cuda())
    ref = oracle.audio_cross_attention(q.f64.reshape(frames, T, H, d), k.f64.reshape(frames, A, H, d),
                                       v.f64.reshape(frames, A, H, d), face)
    got = from_dev(o)
    non_face = np.setdiff1d(np.arange(T), face)
    assert (got[:, non_face] == 0).all()
    assert rel_err(got[:, face], ref[:, face]) <= (FP32_TOL if dtype == "fp32" else BF16_ALARM)
    ca.close()


def test_audio_cross_attention_wan512_chunk_batch2():
    """f4 at WAN-512 shape: a chunk of 3 latent frames of 32x32 tokens, a
    16x16 face region (256 tokens), 32 audio tokens per frame (synthetic), 40
    heads, batch of 2 streams."""
    frames, T, A, H, d, B = 3, 1024, 32, 40, 128, 2
    rng = np.random.default_rng(syn.seed_for(12, 99))
    qs, ks, vs = syn.chunk_qkv(rng, B * frames * T, H, d, "bf16", "D0")
    ka, va, _ = syn.chunk_qkv(rng, B * frames * A, H, d, "bf16", "D0")
    face = np.array([r * 32 + c for r in range(8, 24) for c in range(8, 24)], dtype=np.int32)
    ca = tm.ChunkAttention(H, d, 16, 16, 1, 1, batch=B)
    qd = to_dev(qs).view(B, frames, T, H, d)
    o = torch.empty_like(qd)
    ca.audio(qd, to_dev(ka).view(B, frames, A, H, d), to_dev(va).view(B, frames, A, H, d), o,
             torch.from_numpy(face).cuda())
    assert ca.launches == 2                          # prep (gather, face map) + one attention
    got = from_dev(o)
    non_face = np.setdiff1d(np.arange(T), face)
    assert (got[:, :, non_face] == 0).all()
    for b in range(B):
        ref = oracle.audio_cross_attention(qs.f64.reshape(B, frames, T, H, d)[b],
                                           ka.f64.reshape(B, frames, A, H, d)[b],
                                           va.f64.reshape(B, frames, A, H, d)[b], face)
        assert rel_err(got[b][:, face], ref[:, face]) <= BF16_ALARM
    ca.close()


def test_audio_cross_attention_more_frames_than_one_launch():
    """f4 with 20 frames: the bf16 path takes the frames 16 problems at a time,
    and a launch holds at most 8 schedule blocks, so the attention runs as
    three launches (8 + 8 + 4 frames); the first launch of each group zeroes
    that group's non-face rows.  Batch 2, d = 64, packed 8-row key boxes."""
    frames, T, A, H, d, B, n_face = 20, 48, 8, 3, 64, 2, 11
    rng = np.random.default_rng(syn.seed_for(12, 77))
    qs, _, _ = syn.chunk_qkv(rng, B * frames * T, H, d, "bf16", "D0")
    ka, va, _ = syn.chunk_qkv(rng, B * frames * A, H, d, "bf16", "D0")
    face = np.sort(rng.choice(T, size=n_face, replace=False)).astype(np.int32)
    ca = tm.ChunkAttention(H, d, 16, 16, 1, 1, batch=B)
    qd = to_dev(qs).view(B, frames, T, H, d)
    o = torch.full_like(qd, 7.0)
    ca.audio(qd, to_dev(ka).view(B, frames, A, H, d), to_dev(va).view(B, frames, A, H, d), o,
             torch.from_numpy(face).cuda())
    assert ca.launches == 4                          # prep + three attention launches
    got = from_dev(o)
    non_face = np.setdiff1d(np.arange(T), face)
    assert (got[:, :, non_face] == 0).all()
    for b in range(B):
        ref = oracle.audio_cross_attention(qs.f64.reshape(B, frames, T, H, d)[b],
                                           ka.f64.reshape(B, frames, A, H, d)[b],
                                           va.f64.reshape(B, frames, A, H, d)[b], face)
        assert rel_err(got[b][:, face], ref[:, face]) <= BF16_ALARM
    ca.close()


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("growth", [9.0, 5.0, 30.0, -9.0])
def test_running_max_moves_every_tile(dtype, growth):
    """Online-softmax rescale path: logits ramp along the keys so the row max
    grows (or, for growth < 0, shrinks) by `growth` log2 units per 128-key
    tile.  The kernel moves its running max only when a tile's max exceeds it
    by more than 8 (O and l rescaled then), so 9 and 30 rescale at every tile,
    5 skips (weights up to 2^8 are carried), -9 never moves after the first
    tile.  Exact after the final O / l either way: compared with the oracle."""
    H, d, L = 2, 128, 1000
    scale_log2 = np.log2(np.e) / np.sqrt(d)
    q_norm = 4.0
    slope = growth / (128 * q_norm * scale_log2)      # logit slope per key, log2 units
    rng = np.random.default_rng(syn.seed_for(11, 0, extra=int(growth) + 100))
    q, k, v = syn.ramp_qkv(rng, L, H, d, dtype, slope, q_norm)
    ca = tm.ChunkAttention(H, d, 16, 16, 1, 1, dtype=DT[dtype])
    o = torch.empty_like(to_dev(q))
    ca.window(to_dev(q), to_dev(k), to_dev(v), o, [L])
    ref = oracle.window_attention(q.f64, k.f64, v.f64, [L])
    assert rel_err(from_dev(o), ref) <= (FP32_TOL if dtype == "fp32" else BF16_ALARM)
    ca.close()


def test_fused_append_stress_small_head_counts():
    """Regression guard for the producer / append-warp parity ABA (DESIGN Sec 6,
    a3 store warp): fresh contexts at 10 and 20 heads (stream-K tails with
    merges, fused c_t append), a sync after every call; the broken protocol
    trapped within ~30 calls at 10 heads (this test caught it in 2 of 3 runs
    at 48 calls per context; now 96, twice at 10 heads).  Also checks the last
    output is finite."""
    H_list, d, Lr, Lc, NL = (10, 20, 10), 128, 1024, 3072, 8
    for H in H_list:
        g = torch.Generator(device="cuda").manual_seed(2506030990 + 3 * H)
        ca = tm.ChunkAttention(H, d, Lr, Lc, NL, 1)
        mk = lambda L: torch.randn(L, H, d, device="cuda", dtype=torch.bfloat16, generator=g)
        sets = [(mk(Lc), mk(Lc), mk(Lc)) for _ in range(3)]
        kr, vr = mk(Lr), mk(Lr)
        for layer in range(NL):
            ca.put_reference(layer, 0, kr, vr)
        o = torch.empty(Lc, H, d, device="cuda", dtype=torch.bfloat16)
        chunk = [0] * NL
        for i in range(96):
            layer = i % NL
            chunk[layer] += 1
            q, k, v = sets[i % 3]
            ca.attend(layer, 0, chunk[layer], q, k, v, o)
            torch.cuda.synchronize()
        assert torch.isfinite(o.float()).all()
        ca.close()
