"""fp64 CPU oracle for the sparse-causal chunk-attention hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import this package.  The product
path (paper_2506_03099_b200) never imports it and shares no code with it.

The arithmetic lives in tm_oracle.c (plain fp64 C, OpenMP over rows x heads;
each function cites the PAPER.md passage it follows).  This module only
compiles it with gcc, marshals numpy arrays through ctypes, and keeps the
oracle's own stream history for the c_{t-1} replay (SURVEY.md Sec 8(c) c2:
"K_prev(t, layer, s) := K_cur(t-1, layer, s), replayed by the oracle from its
own history, not from the GPU cache").

Parity pins: tests/test_oracle_pins.py (all functions are pinned; see
DESIGN.md "Oracle pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

ERRORS = {0: "ok", -1: "dimension error", -2: "degenerate mask",
          -3: "negative chunk index", -4: "bad argument"}


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle error {code}: {ERRORS.get(code, '?')}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile tm_oracle.c -> liboracle.so (gcc -O2 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        path = os.environ.get("TM_ORACLE_LIB")   # mutation tests load a mutant here
        if not path:
            path = build()
        L = ctypes.CDLL(path)
        P = ctypes.POINTER
        d = ctypes.c_double
        i64 = ctypes.c_int64
        L.orc_allowed_key_chunks.argtypes = [i64, P(i64)]
        L.orc_window_attention.argtypes = [P(d), P(d), P(d), ctypes.c_int, ctypes.c_int,
                                           P(i64), ctypes.c_int, d, P(i64), i64, P(d)]
        L.orc_stream_attention.argtypes = [P(d), i64, ctypes.c_int, ctypes.c_int,
                                           P(d), P(d), i64, P(d), P(d), i64, P(d), P(d), d,
                                           P(i64), i64, P(d)]
        for f in ("orc_interpolate",):
            getattr(L, f).argtypes = [P(d), P(d), d, i64, P(d)]
        L.orc_velocity_target.argtypes = [P(d), P(d), i64, P(d)]
        L.orc_euler.argtypes = [P(d), P(d), i64, d, P(d)]
        L.orc_sampler_step.argtypes = [P(d), P(d), P(d), i64, d, d, P(d)]
        L.orc_audio_window.argtypes = [i64, i64, ctypes.c_int, P(i64)]
        L.orc_audio_cross_attention.argtypes = [P(d), P(d), P(d), i64, i64, i64, ctypes.c_int,
                                                ctypes.c_int, P(i64), i64, ctypes.c_int, d, P(d)]
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        L.orc_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def allowed_key_chunks(t: int) -> list[int]:
    out = (ctypes.c_int64 * 3)()
    n = lib().orc_allowed_key_chunks(int(t), out)
    if n < 0:
        raise OracleError(n)
    return [int(out[i]) for i in range(n)]


def _rows(rows, n):
    if rows is None:
        return None, n
    r = np.ascontiguousarray(rows, dtype=np.int64)
    return r, len(r)


def window_attention(q, k, v, chunk_lens, scale=None, rows=None):
    """c1: full-window sparse-causal attention (Eq 7 over mask {0, c-1, c}).

    q, k, v: [L][H][d] fp64 (token-major).  Returns [n_rows][H][d]."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    L, H, d = q.shape
    if k.shape != q.shape or v.shape != q.shape:
        raise OracleError(-1)
    cl = np.ascontiguousarray(chunk_lens, dtype=np.int64)
    if cl.sum() != L:
        raise OracleError(-1)
    scale = 1.0 / np.sqrt(d) if scale is None else float(scale)
    r, n = _rows(rows, L)
    out = np.empty((n, H, d), dtype=np.float64)
    rc = lib().orc_window_attention(_dp(q), _dp(k), _dp(v), H, d,
                                    cl.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(cl),
                                    scale,
                                    None if r is None else r.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                    n, _dp(out))
    if rc != 0:
        raise OracleError(rc)
    return out


def stream_attention(q, k_ref, v_ref, k_prev, v_prev, k_cur, v_cur, scale=None, rows=None):
    """c2: softmax over the concatenation [ref | prev | cur]; prev may be None (t = 1)."""
    q, k_ref, v_ref, k_cur, v_cur = map(_f64, (q, k_ref, v_ref, k_cur, v_cur))
    k_prev, v_prev = _f64(k_prev), _f64(v_prev)
    Lc, H, d = q.shape
    Lr = 0 if k_ref is None else k_ref.shape[0]
    Lp = 0 if k_prev is None else k_prev.shape[0]
    for a, L in ((k_ref, Lr), (v_ref, Lr), (k_prev, Lp), (v_prev, Lp), (k_cur, Lc), (v_cur, Lc)):
        if a is not None and a.shape != (L, H, d):
            raise OracleError(-1)
    scale = 1.0 / np.sqrt(d) if scale is None else float(scale)
    r, n = _rows(rows, Lc)
    out = np.empty((n, H, d), dtype=np.float64)
    rc = lib().orc_stream_attention(_dp(q), Lc, H, d, _dp(k_ref), _dp(v_ref), Lr,
                                    _dp(k_prev), _dp(v_prev), Lp, _dp(k_cur), _dp(v_cur), scale,
                                    None if r is None else r.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                    n, _dp(out))
    if rc != 0:
        raise OracleError(rc)
    return out


def interpolate(x0, x1, t):
    x0, x1 = _f64(x0), _f64(x1)
    if x0.shape != x1.shape:
        raise OracleError(-1)
    out = np.empty_like(x0)
    rc = lib().orc_interpolate(_dp(x0), _dp(x1), float(t), x0.size, _dp(out))
    if rc:
        raise OracleError(rc)
    return out


def velocity_target(x0, x1):
    x0, x1 = _f64(x0), _f64(x1)
    if x0.shape != x1.shape:
        raise OracleError(-1)
    out = np.empty_like(x0)
    rc = lib().orc_velocity_target(_dp(x0), _dp(x1), x0.size, _dp(out))
    if rc:
        raise OracleError(rc)
    return out


def euler(x, v, dt):
    x, v = _f64(x), _f64(v)
    if x.shape != v.shape:
        raise OracleError(-1)
    out = np.empty_like(x)
    rc = lib().orc_euler(_dp(x), _dp(v), x.size, float(dt), _dp(out))
    if rc:
        raise OracleError(rc)
    return out


def sampler_step(x, u, eps, t_cur, t_next):
    """S:224 few-step update: x1_hat = x + (1 - t_cur) u, then Eq 1 re-noise
    to t_next with eps (x1_hat itself when t_next >= 1)."""
    x, u = _f64(x), _f64(u)
    eps = _f64(eps)
    if x.shape != u.shape or (eps is not None and eps.shape != x.shape):
        raise OracleError(-1)
    out = np.empty_like(x)
    rc = lib().orc_sampler_step(_dp(x), _dp(u), _dp(eps), x.size, float(t_cur), float(t_next),
                                _dp(out))
    if rc:
        raise OracleError(rc)
    return out


def audio_window(frames, f, window=5):
    """P:125 window of latent frames around f, edges clamped by repetition."""
    out = (ctypes.c_int64 * window)()
    rc = lib().orc_audio_window(int(frames), int(f), int(window), out)
    if rc:
        raise OracleError(rc)
    return [int(out[i]) for i in range(window)]


def audio_cross_attention(q, k, v, face_ids, window=5, scale=None):
    """P:123-125 / S:120-129: q [frames][T][H][d], k/v [frames][A][H][d];
    face-token rows attend their frame's audio window; other rows are 0."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    frames, T, H, d = q.shape
    A = k.shape[1]
    if k.shape != (frames, A, H, d) or v.shape != k.shape:
        raise OracleError(-1)
    fid = np.ascontiguousarray(face_ids, dtype=np.int64)
    scale = 1.0 / np.sqrt(d) if scale is None else float(scale)
    out = np.empty_like(q)
    rc = lib().orc_audio_cross_attention(_dp(q), _dp(k), _dp(v), frames, T, A, H, d,
                                         fid.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                         len(fid), int(window), scale, _dp(out))
    if rc:
        raise OracleError(rc)
    return out


def philox4x32_10(counter, key):
    """Philox4x32-10 (Salmon et al., SC'11), numpy uint32 words: counter
    [..., 4], key [..., 2] -> [..., 4].  The oracle side's own implementation
    of the counter-based generator the sampler kernel uses."""
    M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
    c = [np.asarray(counter[..., i], dtype=np.uint32) for i in range(4)]
    k0 = np.asarray(key[..., 0], dtype=np.uint32)
    k1 = np.asarray(key[..., 1], dtype=np.uint32)
    for _ in range(10):
        p0 = c[0].astype(np.uint64) * M0
        p1 = c[2].astype(np.uint64) * M1
        hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), p0.astype(np.uint32)
        hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), p1.astype(np.uint32)
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = k0 + W0
        k1 = k1 + W1
    return np.stack(c, axis=-1)


def philox_normal(n, seed, offset):
    """N(0,1) draws of the sampler's generator, in fp64: element i uses word
    i % 4 of Philox(counter = (i // 4, 0, offset_lo, offset_hi), key = seed);
    uniforms (w + 0.5) / 2^32 and the Box-Muller pairs (w0, w1), (w2, w3)."""
    n4 = (n + 3) // 4
    ctr = np.zeros((n4, 4), dtype=np.uint32)
    idx = np.arange(n4, dtype=np.uint64)
    ctr[:, 0] = (idx & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    ctr[:, 1] = (idx >> np.uint64(32)).astype(np.uint32)
    ctr[:, 2] = np.uint32(offset & 0xFFFFFFFF)
    ctr[:, 3] = np.uint32((offset >> 32) & 0xFFFFFFFF)
    key = np.array([[seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF]], dtype=np.uint32)
    w = philox4x32_10(ctr, np.repeat(key, n4, axis=0)).astype(np.float64)
    uu = (w + 0.5) / 4294967296.0
    r0 = np.sqrt(-2.0 * np.log(uu[:, 0]))
    r1 = np.sqrt(-2.0 * np.log(uu[:, 2]))
    z = np.stack([r0 * np.cos(2 * np.pi * uu[:, 1]), r0 * np.sin(2 * np.pi * uu[:, 1]),
                  r1 * np.cos(2 * np.pi * uu[:, 3]), r1 * np.sin(2 * np.pi * uu[:, 3])], axis=1)
    return z.reshape(-1)[:n]


class StreamOracle:
    """The oracle's own KV history for streaming.

    put_reference(layer, step, k, v) once; attend(layer, step, t, q, k, v)
    for t = 1, 2, ... in order.  The previous chunk's K/V are replayed from
    this object's history, never from the GPU cache.  Enforces the same
    ordering contract as the C-ABI (cache miss -> error; reference
    rewrite after stream start -> error).
    """

    def __init__(self):
        self.ref = {}
        self.prev = {}         # (layer, step) -> K/V of the last chunk attended
        self.prev_used = {}    # (layer, step) -> the c_{t-1} K/V that chunk used (for a redo)
        self.last = {}

    def reset(self):
        self.__init__()

    def put_reference(self, layer, step, k, v):
        key = (layer, step)
        if self.last.get(key, 0) >= 1:
            raise OracleError(-4)      # reference rewrite after stream start
        self.ref[key] = (_f64(k), _f64(v))

    def attend(self, layer, step, t, q, k, v, rows=None):
        key = (layer, step)
        if key not in self.ref or t < 1:
            raise OracleError(-4)      # cache miss
        last = self.last.get(key, 0)
        if t == last + 1:
            prev = self.prev.get(key) if t >= 2 else None
        elif t == last:
            prev = self.prev_used[key]  # redo of the same chunk
        else:
            raise OracleError(-4)      # out-of-order chunk
        kr, vr = self.ref[key]
        kp, vp = (None, None) if prev is None else prev
        out = stream_attention(q, kr, vr, kp, vp, k, v, rows=rows)
        self.prev_used[key] = prev
        self.prev[key] = (_f64(k), _f64(v))
        self.last[key] = t
        return out
