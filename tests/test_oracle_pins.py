"""Pins of the fp64 oracle to things other than itself (CPU only).

Each test names what fixes the expected value: a cited example (golden
fixture), a closed form, an invariant, a textbook/library routine or an
independent brute force.  See DESIGN.md "Oracle pins" for the table.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from bruteforce import build_mask, dense_masked_attention

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------
# mask predicate
# --------------------------------------------------------------------------

def test_allowed_key_chunks_paper_examples():
    g = gold("mask_examples.json")["allowed_key_chunks"]
    for t, expect in g.items():
        assert oracle.allowed_key_chunks(int(t)) == expect


def test_allowed_key_chunks_negative_is_error():
    with pytest.raises(oracle.OracleError):
        oracle.allowed_key_chunks(-1)


def _attended_chunks(chunk_lens):
    """Read the window oracle's mask out of its OUTPUT: q = 0 (uniform
    weights over allowed keys) and V = one-hot of the key's chunk, so
    O[i] is the fraction of allowed keys per chunk; nonzero entries are the
    attended chunks."""
    n = len(chunk_lens)
    L = sum(chunk_lens)
    owner = np.repeat(np.arange(n), chunk_lens)
    q = np.zeros((L, 1, n))
    k = np.random.default_rng(1).standard_normal((L, 1, n))
    v = np.zeros((L, 1, n))
    v[np.arange(L), 0, owner] = 1.0
    o = oracle.window_attention(q, k, v, chunk_lens)
    return owner, o[:, 0, :]


@pytest.mark.parametrize("fpc,cpw", [(3, 7), (7, 3), (21, 1)])
def test_window_mask_bruteforce_21x21_frames(fpc, cpw):
    """S:615 acceptance 2: over all 21x21 latent-frame pairs the window
    oracle attends exactly the chunks the brute-force predicate allows."""
    frame_tokens = 2
    chunk_lens = [fpc * frame_tokens] * cpw
    owner, frac = _attended_chunks(chunk_lens)
    mask = build_mask(chunk_lens)          # independent predicate (tests/bruteforce.py)
    L = len(owner)
    for i in range(0, L, frame_tokens):    # one query token per frame
        for j in range(0, L, frame_tokens):
            attended = frac[i, owner[j]] > 0
            assert attended == mask[i][j], (i, j)


def test_window_7x3_density():
    """18 of 49 chunk pairs allowed for 7 chunks."""
    g = gold("mask_examples.json")
    owner, frac = _attended_chunks([1] * 7)
    assert int((frac > 0).sum()) == g["window_7x3_allowed_chunk_pairs"]
    assert frac.size == g["window_7x3_chunk_pairs"]


# --------------------------------------------------------------------------
# attention values (Eq 7)
# --------------------------------------------------------------------------

def test_hand_two_keys():
    g = gold("attention_hand.json")["two_keys"]
    q = np.array(g["q"]).reshape(1, 1, 1)
    k = np.array(g["k"]).reshape(2, 1, 1)
    v = np.array(g["v"]).reshape(2, 1, 1)
    # one chunk of 1 query token attending [ref | cur] = 2 keys via the stream form
    o = oracle.stream_attention(q, k[:1], v[:1], None, None, k[1:], v[1:], scale=1.0)
    assert abs(o[0, 0, 0] - g["o"]) < 1e-14


def test_hand_one_token_chunks():
    g = gold("attention_hand.json")["one_token_chunks_uniform"]
    L = 4
    q = np.zeros((L, 1, 1))
    k = np.random.default_rng(0).standard_normal((L, 1, 1))
    v = np.array(g["v"]).reshape(L, 1, 1)
    o = oracle.window_attention(q, k, v, [1, 1, 1, 1])
    np.testing.assert_allclose(o[:, 0, 0], g["o"], rtol=0, atol=1e-12)


def test_single_token_is_v_exactly():
    g = gold("attention_hand.json")["single_token"]
    q = np.array(g["q"]).reshape(1, 1, 2)
    k = np.array(g["k"]).reshape(1, 1, 2)
    v = np.array(g["v"]).reshape(1, 1, 2)
    o = oracle.window_attention(q, k, v, [1])
    assert (o.reshape(-1) == np.array(g["o"])).all()


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_window_vs_bruteforce(seed):
    """random q, k, v, random chunk layout vs the independent double
    loop (tests/bruteforce.py), max abs diff < 1e-10."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 5))
    chunk_lens = [int(x) for x in rng.integers(1, 4, size=n)]
    L = sum(chunk_lens)
    H, d = 2, int(rng.integers(1, 9))
    q, k, v = (rng.standard_normal((L, H, d)) * 2 for _ in range(3))
    scale = 1 / math.sqrt(d)
    o = oracle.window_attention(q, k, v, chunk_lens)
    bf = np.array(dense_masked_attention(q.tolist(), k.tolist(), v.tolist(),
                                         build_mask(chunk_lens), scale))
    assert np.abs(o - bf).max() < 1e-10


def test_stream_vs_bruteforce_with_ragged_segments():
    """Stream form (Lr, Lp, Lc of 1..5 tokens) vs the brute force on the
    concatenation with an all-true mask."""
    rng = np.random.default_rng(7)
    for Lr, Lp, Lc in [(1, 0, 1), (3, 2, 5), (5, 1, 2), (2, 5, 3)]:
        H, d = 2, 4
        parts = [rng.standard_normal((L, H, d)) for L in (Lr, Lp, Lc) for _ in range(2)]
        kr, vr, kp, vp, kc, vc = parts
        q = rng.standard_normal((Lc, H, d))
        o = oracle.stream_attention(q, kr, vr, kp if Lp else None, vp if Lp else None, kc, vc)
        K = np.concatenate([kr, kp, kc]) if Lp else np.concatenate([kr, kc])
        V = np.concatenate([vr, vp, vc]) if Lp else np.concatenate([vr, vc])
        # queries occupy the tail of a sequence whose keys are all allowed
        Lk = K.shape[0]
        qq = np.concatenate([np.zeros((Lk - Lc, H, d)), q])
        mask = [[True] * Lk for _ in range(Lk)]
        bf = np.array(dense_masked_attention(qq.tolist(), K.tolist(), V.tolist(), mask,
                                             1 / math.sqrt(d)))[Lk - Lc:]
        assert np.abs(o - bf).max() < 1e-10


def test_full_mask_equals_textbook_sdpa():
    """BJ.north_star / S:66: one chunk spanning the sequence -> all-true mask
    -> dense attention; compare with torch SDPA (fp64, CPU) and a numpy
    softmax, < 1e-12."""
    rng = np.random.default_rng(11)
    L, H, d = 37, 3, 16
    q, k, v = (rng.standard_normal((L, H, d)) for _ in range(3))
    o = oracle.window_attention(q, k, v, [L])
    t = lambda a: torch.from_numpy(a).permute(1, 0, 2)[None]  # [1][H][L][d]
    ref = torch.nn.functional.scaled_dot_product_attention(t(q), t(k), t(v))[0].permute(1, 0, 2).numpy()
    assert np.abs(o - ref).max() < 1e-12
    s = np.einsum("ihc,jhc->hij", q, k) / math.sqrt(d)
    p = np.exp(s - s.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    ref2 = np.einsum("hij,jhc->ihc", p, v)
    assert np.abs(o - ref2).max() < 1e-12


def test_rows_sum_to_one_and_convexity():
    """S:67 + BJ.north_star 'softmax rows summing to 1': V = ones -> O = 1
    within 1e-13; for random V every output coordinate lies within the
    [min, max] of the allowed V rows."""
    rng = np.random.default_rng(5)
    chunk_lens = [4, 6, 6, 6]
    L, H, d = sum(chunk_lens), 2, 8
    q, k = rng.standard_normal((L, H, d)) * 3, rng.standard_normal((L, H, d)) * 3
    o1 = oracle.window_attention(q, k, np.ones((L, H, d)), chunk_lens)
    assert np.abs(o1 - 1).max() <= 1e-13
    v = rng.standard_normal((L, H, d))
    o = oracle.window_attention(q, k, v, chunk_lens)
    mask = np.array(build_mask(chunk_lens))
    for i in range(L):
        sel = v[mask[i]]
        assert (o[i] >= sel.min(0) - 1e-15).all() and (o[i] <= sel.max(0) + 1e-15).all()


def test_large_magnitude_no_overflow():
    """D6-style logits of order 1e4: max subtraction keeps everything finite."""
    rng = np.random.default_rng(6)
    L, H, d = 12, 1, 8
    q, k = rng.standard_normal((L, H, d)) * 300, rng.standard_normal((L, H, d)) * 300
    v = rng.standard_normal((L, H, d))
    o = oracle.window_attention(q, k, v, [4, 4, 4])
    assert np.isfinite(o).all()
    assert np.abs(o).max() <= np.abs(v).max() + 1e-12


def test_uniform_closed_form_wan_size_segment_tagged():
    """S:42 + SURVEY Sec 8(c) pin: q = 0 -> O = mean of allowed V rows.  At
    the full WAN-512 shapes (H=40, d=128, Lr=1024, Lc=3072, t>=2) with
    segment-tagged V (V_ref = a, V_prev = b, V_cur = c) the closed form is
    (Lr a + Lc b + Lc c) / (Lr + 2 Lc); sampled rows."""
    H, d, Lr, Lc = 40, 128, 1024, 3072
    a, b, c = 1.0, -2.0, 0.5
    rng = np.random.default_rng(9)
    kr = rng.standard_normal((Lr, H, d)); kp = rng.standard_normal((Lc, H, d)); kc = rng.standard_normal((Lc, H, d))
    vr = np.full((Lr, H, d), a); vp = np.full((Lc, H, d), b); vc = np.full((Lc, H, d), c)
    q = np.zeros((Lc, H, d))
    rows = [0, 1777, Lc - 1]
    o = oracle.stream_attention(q, kr, vr, kp, vp, kc, vc, rows=rows)
    expect = (Lr * a + Lc * b + Lc * c) / (Lr + 2 * Lc)
    assert np.abs(o - expect).max() < 1e-12
    # t = 1: no previous segment
    o1 = oracle.stream_attention(q, kr, vr, None, None, kc, vc, rows=rows)
    assert np.abs(o1 - (Lr * a + Lc * c) / (Lr + Lc)).max() < 1e-12


def test_stream_equals_window():
    """S:303 / S:616: for each chunk t of a window, the streaming form with
    the oracle's own history equals the full-window rows, < 1e-9."""
    rng = np.random.default_rng(12)
    H, d, Lr, Lc, n = 2, 8, 5, 7, 5
    lens = [Lr] + [Lc] * (n - 1)
    L = sum(lens)
    q, k, v = (rng.standard_normal((L, H, d)) for _ in range(3))
    win = oracle.window_attention(q, k, v, lens)
    so = oracle.StreamOracle()
    so.put_reference(0, 0, k[:Lr], v[:Lr])
    for t in range(1, n):
        s = Lr + (t - 1) * Lc
        out = so.attend(0, 0, t, q[s:s + Lc], k[s:s + Lc], v[s:s + Lc])
        assert np.abs(out - win[s:s + Lc]).max() < 1e-9


def test_stream_order_errors():
    """S:287 (reference rewrite) and S:296 (cache miss / out of order)."""
    rng = np.random.default_rng(3)
    H, d = 1, 4
    kv = lambda L: (rng.standard_normal((L, H, d)), rng.standard_normal((L, H, d)))
    so = oracle.StreamOracle()
    with pytest.raises(oracle.OracleError):
        so.attend(0, 0, 1, *([rng.standard_normal((2, H, d))] * 3))   # no reference
    so.put_reference(0, 0, *kv(2))
    with pytest.raises(oracle.OracleError):
        so.attend(0, 0, 2, *([rng.standard_normal((2, H, d))] * 3))   # skipped chunk 1
    so.attend(0, 0, 1, rng.standard_normal((2, H, d)), *kv(2))
    with pytest.raises(oracle.OracleError):
        so.put_reference(0, 0, *kv(2))                                # rewrite after start


def test_dimension_errors():
    with pytest.raises(oracle.OracleError):
        oracle.window_attention(np.zeros((3, 1, 2)), np.zeros((3, 1, 2)), np.zeros((3, 1, 2)), [2])
    with pytest.raises(oracle.OracleError):
        oracle.stream_attention(np.zeros((3, 1, 2)), np.zeros((2, 1, 2)), np.zeros((2, 1, 3)),
                                None, None, np.zeros((3, 1, 2)), np.zeros((3, 1, 2)))


# --------------------------------------------------------------------------
# flow matching (Eqs 1-2) and the Euler step
# --------------------------------------------------------------------------

def test_flow_golden_examples():
    g = gold("flow_examples.json")
    for e in g["interpolate"]:
        assert oracle.interpolate([e["x0"]], [e["x1"]], e["t"])[0] == e["out"]
    for e in g["velocity_target"]:
        assert oracle.velocity_target([e["x0"]], [e["x1"]])[0] == e["out"]
    cv = g["constant_velocity"]
    for n in cv["steps"]:
        x = np.array([cv["x0"]])
        for _ in range(n):
            x = oracle.euler(x, np.array([cv["c"]]), 1.0 / n)
        assert abs(x[0] - cv["out"]) < 1e-13


def test_euler_lands_on_the_interpolant():
    """Eqs 1-2: x_ta + dt * (x1 - x0) == x_{ta+dt} (one Euler step along the
    exact rectified-flow velocity is exact), and d/dt interpolate ==
    velocity_target by central finite differences (< 1e-8)."""
    rng = np.random.default_rng(4)
    x0, x1 = rng.standard_normal(1000), rng.standard_normal(1000)
    v = oracle.velocity_target(x0, x1)
    for ta, dt in [(0.0, 1.0), (0.0, 0.5), (0.5, 0.5), (0.25, 0.125)]:
        xt = oracle.interpolate(x0, x1, ta)
        np.testing.assert_allclose(oracle.euler(xt, v, dt), oracle.interpolate(x0, x1, ta + dt),
                                   rtol=0, atol=1e-13)
    h = 1e-5
    fd = (oracle.interpolate(x0, x1, 0.3 + h) - oracle.interpolate(x0, x1, 0.3 - h)) / (2 * h)
    assert np.abs(fd - v).max() < 1e-8
    assert (oracle.interpolate(x0, x1, 0.0) == x0).all()
    assert (oracle.interpolate(x0, x1, 1.0) == x1).all()


# --------------------------------------------------------------------------
# f2: few-step sampler update and its noise generator
# --------------------------------------------------------------------------

def test_sampler_point_mass_recovers_x1():
    """a student exact for a point-mass dataset (u = (x1 - x_t)/(1 - t))
    returns x1; re-noising to t' lands on the Eq 1 interpolant of (eps, x1)."""
    rng = np.random.default_rng(21)
    x0, x1, eps = (rng.standard_normal(500) for _ in range(3))
    for t, t2 in [(0.0, 0.5), (0.25, 0.75), (0.5, 1.0)]:
        xt = oracle.interpolate(x0, x1, t)
        u = (x1 - xt) / (1.0 - t)
        out = oracle.sampler_step(xt, u, eps, t, t2)
        expect = x1 if t2 >= 1.0 else oracle.interpolate(eps, x1, t2)
        assert np.abs(out - expect).max() < 1e-12


def test_sampler_final_step_is_an_euler_step():
    """S:220 (reading Q10): the last schedule entry is one Euler step of
    dt = 1 - t (no re-noise)."""
    rng = np.random.default_rng(22)
    x, u = rng.standard_normal(300), rng.standard_normal(300)
    for t in (0.0, 0.5, 0.9):
        assert np.abs(oracle.sampler_step(x, u, None, t, 1.0) - oracle.euler(x, u, 1.0 - t)).max() == 0
    with pytest.raises(oracle.OracleError):
        oracle.sampler_step(x, u, None, 0.0, 0.5)       # re-noise needs eps


def test_philox_known_answers():
    g = gold("philox_kat.json")
    for vec in g["vectors"]:
        c = np.array([[int(w, 16) for w in vec["counter"]]], dtype=np.uint32)
        k = np.array([[int(w, 16) for w in vec["key"]]], dtype=np.uint32)
        out = oracle.philox4x32_10(c, k)[0]
        assert [int(w) for w in out] == [int(w, 16) for w in vec["out"]]


def test_philox_normal_moments():
    z = oracle.philox_normal(2_000_000, seed=2506030990, offset=3)
    assert abs(z.mean()) < 3e-3 and abs(z.var() - 1) < 4e-3
    assert abs(np.mean(z ** 4) - 3) < 0.03            # Gaussian kurtosis


def test_philox_normal_word_mapping_by_polar_identities():
    """Reading Q18: element i takes word i % 4 of the Philox
    block at counter (i // 4, 0, offset_lo, offset_hi), uniforms (w + 0.5)/2^32,
    Box-Muller pairs (w0, w1) and (w2, w3) with the radius from the first word
    and the angle from the second, cos on the even element.  Pinned through the
    polar decomposition of each output pair against the KAT-pinned Philox words:
    z_2j^2 + z_2j+1^2 = -2 ln u_2j and atan2(z_2j+1, z_2j) = 2 pi u_2j+1 (mod 2 pi),
    so a swapped sin/cos, another word pairing, a radius/angle word swap or a
    different counter layout fails."""
    seed, offset, n = 0x1234ABCD5678, (7 << 32) | 3, 4096
    z = oracle.philox_normal(n, seed, offset).reshape(-1, 4)
    blk = np.arange(n // 4, dtype=np.uint64)
    ctr = np.stack([(blk & np.uint64(0xFFFFFFFF)).astype(np.uint32), (blk >> np.uint64(32)).astype(np.uint32),
                    np.full(n // 4, 3, np.uint32), np.full(n // 4, 7, np.uint32)], axis=1)
    key = np.tile(np.array([[seed & 0xFFFFFFFF, seed >> 32]], dtype=np.uint32), (n // 4, 1))
    u = (oracle.philox4x32_10(ctr, key).astype(np.float64) + 0.5) / 2.0 ** 32
    for a, b in ((0, 1), (2, 3)):
        r2 = z[:, a] ** 2 + z[:, b] ** 2
        assert np.abs(r2 - (-2.0 * np.log(u[:, a]))).max() < 1e-9 * np.maximum(1.0, r2).max()
        ang = np.mod(np.arctan2(z[:, b], z[:, a]), 2 * np.pi)
        d = np.abs(ang - 2 * np.pi * u[:, b])
        assert np.minimum(d, 2 * np.pi - d).max() < 1e-9


# --------------------------------------------------------------------------
# f4: audio cross-attention with face-region query mask
# --------------------------------------------------------------------------

def test_audio_window_examples():
    for c in gold("audio_window.json")["cases"]:
        assert oracle.audio_window(c["frames"], c["frame_idx"], c["window"]) == c["window_frames"]


def _audio_inputs(frames=5, T=6, A=3, H=2, d=4, seed=30):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((frames, T, H, d)), rng.standard_normal((frames, A, H, d)),
            rng.standard_normal((frames, A, H, d)))


def test_audio_non_face_rows_untouched_and_bruteforce():
    """S:126 (non-face rows receive no update -> exactly 0 here) and the face
    rows vs the independent dense double loop over the clamped window."""
    q, k, v = _audio_inputs()
    frames, T, A = q.shape[0], q.shape[1], k.shape[1]
    face = [1, 4]
    out = oracle.audio_cross_attention(q, k, v, face)
    non_face = [t for t in range(T) if t not in face]
    assert (out[:, non_face] == 0).all()
    for f in range(frames):
        lo = [min(max(g, 0), frames - 1) for g in range(f - 2, f + 3)]   # restated rule
        K = np.concatenate([k[g] for g in lo])
        V = np.concatenate([v[g] for g in lo])
        Lk = K.shape[0]
        for t in face:
            qq = np.concatenate([np.zeros((Lk - 1,) + q.shape[2:]), q[f, t][None]])
            mask = [[True] * Lk for _ in range(Lk)]
            bf = np.array(dense_masked_attention(qq.tolist(), K.tolist(), V.tolist(), mask,
                                                 1 / math.sqrt(q.shape[-1])))[-1]
            assert np.abs(out[f, t] - bf).max() < 1e-10


def test_audio_single_face_single_token_is_v():
    """one face token, one audio token, window 1 -> O == V exactly."""
    q, k, v = _audio_inputs(frames=3, T=4, A=1)
    out = oracle.audio_cross_attention(q, k, v, [2], window=1)
    assert (out[:, 2] == v[:, 0]).all()


def test_audio_locality():
    """changing the audio of frame j changes frame i only if |i-j| <= 2."""
    q, k, v = _audio_inputs(frames=9, seed=31)
    base = oracle.audio_cross_attention(q, k, v, [0, 3, 5])
    k2 = k.copy()
    k2[4] += 1.0
    out = oracle.audio_cross_attention(q, k2, v, [0, 3, 5])
    changed = [f for f in range(9) if np.abs(out[f] - base[f]).max() > 0]
    assert changed == [2, 3, 4, 5, 6]


def test_audio_uniform_closed_form_with_edge_repetition():
    """q = 0: O = mean over the window's audio tokens, counting a repeated
    edge frame as often as it appears (frame 0 -> 3x frame 0 + frames 1, 2)."""
    q, k, v = _audio_inputs(frames=4, T=2, A=2, seed=32)
    out = oracle.audio_cross_attention(np.zeros_like(q), k, v, [0, 1])
    expect0 = (3 * v[0].sum(0) + v[1].sum(0) + v[2].sum(0)) / 10.0
    assert np.abs(out[0, 0] - expect0).max() < 1e-12


def test_audio_empty_face_mask_is_error():
    q, k, v = _audio_inputs()
    with pytest.raises(oracle.OracleError):
        oracle.audio_cross_attention(q, k, v, [])


def test_sampler_u_one_fixture_matches_oracle_philox():
    """tests/golden/sampler_u_one.json (GPU edge test of f2): each stored
    counter's word is the oracle Philox output and lies in the top 128 values."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "sampler_u_one.json")) as f:
        g = json.load(f)
    for h in g["hits"]:
        ctr = np.array([[0, 0, h["offset"] & 0xFFFFFFFF, h["offset"] >> 32]], dtype=np.uint32)
        key = np.array([[g["seed"] & 0xFFFFFFFF, g["seed"] >> 32]], dtype=np.uint32)
        w = int(oracle.philox4x32_10(ctr, key)[0, h["word"]])
        assert w == h["w"] and w >= 2**32 - 128


def test_philox_normal_pin_catches_mapping_mutants():
    """Pin strength for the word mapping: sin/cos swapped, pairs (w0, w2) /
    (w1, w3), radius and angle words swapped -- each breaks an identity of
    test_philox_normal_word_mapping_by_polar_identities."""
    n = 1024
    z = oracle.philox_normal(n, 99, 5).reshape(-1, 4)
    blk = np.arange(n // 4, dtype=np.uint32)
    ctr = np.stack([blk, np.zeros_like(blk), np.full_like(blk, 5), np.zeros_like(blk)], axis=1)
    key = np.tile(np.array([[99, 0]], dtype=np.uint32), (n // 4, 1))
    u = (oracle.philox4x32_10(ctr, key).astype(np.float64) + 0.5) / 2.0 ** 32

    def ok(zz):
        r2 = zz[:, 0] ** 2 + zz[:, 1] ** 2
        ang = np.mod(np.arctan2(zz[:, 1], zz[:, 0]), 2 * np.pi)
        d = np.abs(ang - 2 * np.pi * u[:, 1])
        return (np.abs(r2 + 2.0 * np.log(u[:, 0])).max() < 1e-9 and np.minimum(d, 2 * np.pi - d).max() < 1e-9)

    assert ok(z)
    r_a, r_b = np.sqrt(-2 * np.log(u[:, 0])), np.sqrt(-2 * np.log(u[:, 1]))
    mutants = {
        "sin_cos_swapped": np.stack([r_a * np.sin(2 * np.pi * u[:, 1]), r_a * np.cos(2 * np.pi * u[:, 1])], 1),
        "radius_angle_words_swapped": np.stack([r_b * np.cos(2 * np.pi * u[:, 0]),
                                                r_b * np.sin(2 * np.pi * u[:, 0])], 1),
        "pairing_w0_w2": np.stack([r_a * np.cos(2 * np.pi * u[:, 2]), r_a * np.sin(2 * np.pi * u[:, 2])], 1),
    }
    for name, zz in mutants.items():
        assert not ok(zz), name
