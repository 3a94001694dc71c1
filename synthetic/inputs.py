"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no attention, no softmax, no
Euler update).  It only draws random numbers and rounds them to the storage
precision, so that both sides consume bit-identical inputs (SURVEY.md §8(c) c4:
"The oracle consumes the same rounded values, upcast exactly to fp64").

Workload recipe (SURVEY.md §8(d) value distributions):
  D0 iid N(0,1) for q, k, v                       (timing default)
  D1 peaky: q scaled by 6                         (sharp softmax)
  D2 reference-dominant: a shared unit direction u is added (x3) to q and to
     K_ref, so most attention mass sits on the cached reference segment
  D3 segment-tagged V: V_ref += 1, V_prev -= 1    (exposes a dropped segment)
  D4 q = 0 with D3's segment tags on V             (all logits equal -> closed form)
  D6 large magnitude: q, k scaled by 30           (max-subtraction guard)
Shapes come from BASELINE.json configs (SURVEY.md §8 notation): WAN-2.1 512^2
H=40, d=128, Lr=1024, Lc=3072; 720^2 Lr=2025, Lc=6075; tiny H=2, d=64, Lr=16,
Lc=32.

Seeds: base 2506030990; seed = base + 1000*config + 10*distribution + rank
(SURVEY.md §8(d) "Seeds").
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 2506030990

DISTRIBUTIONS = ("D0", "D1", "D2", "D3", "D4", "D6")


def seed_for(config: int, distribution: int = 0, rank: int = 0, extra: int = 0) -> int:
    return SEED_BASE + 1000 * config + 10 * distribution + rank + 100_000 * extra


def bf16_bits_rne(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bfloat16 (round-to-nearest-even); return uint16 bits.

    Storage conversion only (IEEE-754 bit manipulation); NaN is not produced by
    the generators so no NaN special-casing is needed here.
    """
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    bias = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + bias) >> 16).astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    """Exact upcast of bfloat16 bit patterns to float64."""
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


class Tensor:
    """A generated tensor in its storage form plus its exact fp64 upcast.

    `store` is uint16 (bf16 bits) or float32; `f64` is what the oracle reads.
    """

    def __init__(self, store: np.ndarray, dtype: str):
        self.store = np.ascontiguousarray(store)
        self.dtype = dtype
        if dtype == "bf16":
            self.f64 = bf16_bits_to_f64(self.store)
        elif dtype == "fp32":
            self.f64 = self.store.astype(np.float64)
        else:
            raise ValueError(dtype)

    @property
    def shape(self):
        return self.store.shape


def _finish(x: np.ndarray, dtype: str) -> Tensor:
    x = x.astype(np.float32)
    if dtype == "bf16":
        return Tensor(bf16_bits_rne(x), "bf16")
    return Tensor(x, "fp32")


def ramp_qkv(rng: np.random.Generator, L: int, H: int, d: int, dtype: str, slope: float,
             q_norm: float = 4.0):
    """Keys whose logits grow (slope > 0) or shrink (slope < 0) linearly along
    the sequence: q = q_norm * u_h + small noise, k_j = slope * j * u_h + noise,
    v ~ N(0, 1), with u_h a random unit direction per head.  The logit of key
    j is ~ q_norm * slope * j * <u, u> -- the running max moves on every KV
    tile (the online-softmax rescale path).  Input recipe only."""
    u = rng.standard_normal((H, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    q = q_norm * u[None] + 0.05 * rng.standard_normal((L, H, d))
    j = np.arange(L, dtype=np.float64)[:, None, None]
    k = slope * j * u[None] + 0.05 * rng.standard_normal((L, H, d))
    v = rng.standard_normal((L, H, d))
    return _finish(q, dtype), _finish(k, dtype), _finish(v, dtype)


def chunk_qkv(rng: np.random.Generator, L: int, H: int, d: int, dtype: str,
              dist: str = "D0", role: str = "cur", shared_dir=None):
    """Q, K, V for one block of L tokens, token-major [L][H][d].

    role in {"ref", "prev", "cur"} selects the D2/D3 modifications.
    """
    q = rng.standard_normal((L, H, d), dtype=np.float32)
    k = rng.standard_normal((L, H, d), dtype=np.float32)
    v = rng.standard_normal((L, H, d), dtype=np.float32)
    if dist == "D1":
        q *= 6.0
    elif dist == "D2":
        assert shared_dir is not None
        q += 3.0 * shared_dir[None, :, :]
        if role == "ref":
            k += 3.0 * shared_dir[None, :, :]
    elif dist in ("D3", "D4"):
        if role == "ref":
            v += 1.0
        elif role == "prev":
            v -= 1.0
        if dist == "D4":
            q[...] = 0.0
    elif dist == "D6":
        q *= 30.0
        k *= 30.0
    elif dist != "D0":
        raise ValueError(dist)
    return _finish(q, dtype), _finish(k, dtype), _finish(v, dtype)


def shared_direction(rng: np.random.Generator, H: int, d: int) -> np.ndarray:
    u = rng.standard_normal((H, d)).astype(np.float32)
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    return u * np.float32(np.sqrt(d) ** 0.5)


class StreamInputs:
    """Deterministic per-(layer, step, chunk) inputs of one stream.

    Chunk 0 is the reference (Lr tokens); chunks t>=1 have Lc tokens.  The
    K/V a chunk produces at (layer, step) is what the cache holds as
    "previous" for chunk t+1 (SURVEY.md §8(c) Q3 reading (a)).
    """

    def __init__(self, H, d, Lr, Lc, dtype="bf16", dist="D0", seed=SEED_BASE):
        self.H, self.d, self.Lr, self.Lc = H, d, Lr, Lc
        self.dtype, self.dist, self.seed = dtype, dist, seed
        rng = np.random.default_rng(seed)
        self.u = shared_direction(rng, H, d) if dist == "D2" else None

    def chunk(self, layer: int, step: int, t: int):
        """D3 in a stream: V_ref += 1, even chunks t>=2 get V -= 1, odd chunks
        are untagged, so within any call ref/prev/cur carry distinct tags."""
        rng = np.random.default_rng([self.seed, layer, step, t])
        L = self.Lr if t == 0 else self.Lc
        if t == 0:
            role = "ref"
        elif t % 2 == 0:
            role = "prev"
        else:
            role = "cur"
        return chunk_qkv(rng, L, self.H, self.d, self.dtype, self.dist, role, self.u)


def euler_inputs(n: int, seed: int, v_dtype: str = "fp32"):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n, dtype=np.float32)
    v = rng.standard_normal(n, dtype=np.float32)
    vt = _finish(v, v_dtype)
    return Tensor(x, "fp32"), vt
