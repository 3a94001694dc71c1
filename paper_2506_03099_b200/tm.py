"""Thin ctypes binding of libtm.so (include/tm.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  PyTorch is
used by callers for device memory, streams and process groups; this module
accepts torch tensors (or raw integer device pointers) and passes
data_ptr()s.  There is no CPU fallback: if libtm.so is missing or cannot be
loaded, import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# TM_LIB_PATH: A/B tuning of an alternative in-tree build (tools/); default libtm.so
LIB_PATH = os.environ.get("TM_LIB_PATH") or os.path.join(_PKG, "libtm.so")

TM_OK = 0
STATUS = {0: "TM_OK", 1: "TM_ERR_INVALID_ARG", 2: "TM_ERR_SHAPE", 3: "TM_ERR_DEGENERATE_MASK",
          4: "TM_ERR_STREAM_ORDER", 5: "TM_ERR_REF_IMMUTABLE", 6: "TM_ERR_NONFINITE",
          7: "TM_ERR_UNSUPPORTED", 8: "TM_ERR_CUDA", 9: "TM_ERR_NCCL"}
TM_BF16, TM_FP32 = 0, 1
TM_TRANSPORT_NCCL, TM_TRANSPORT_PEER = 0, 1
TM_PHASE_SEND, TM_PHASE_ATTEND, TM_PHASE_RECV, TM_PHASE_ALL = 1, 2, 4, 7
TM_PEER_HANDLE_BYTES = 72


class TMError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class tm_config(ctypes.Structure):
    _fields_ = [("heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("ref_tokens", ctypes.c_int32), ("chunk_tokens", ctypes.c_int32),
                ("num_layers", ctypes.c_int32), ("num_steps", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("softmax_scale", ctypes.c_float), ("world_size", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("device", ctypes.c_int32),
                ("transport", ctypes.c_int32), ("sched_heads", ctypes.c_int32)]


def make_config(heads, head_dim, ref_tokens, chunk_tokens, num_layers=1, num_steps=1, batch=1,
                dtype=TM_BF16, softmax_scale=0.0, world_size=1, rank=0, device=0,
                transport=TM_TRANSPORT_NCCL, sched_heads=0) -> tm_config:
    return tm_config(heads, head_dim, ref_tokens, chunk_tokens, num_layers, num_steps, batch,
                     dtype, softmax_scale, world_size, rank, device, transport, sched_heads)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtm.so not built at {LIB_PATH}; run `python -m "
                          f"paper_2506_03099_b200.build` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P, V, S = ctypes.POINTER, ctypes.c_void_p, ctypes.c_size_t
    i32, i64 = ctypes.c_int32, ctypes.c_int64
    cfgp = P(tm_config)
    sig = {
        "tm_version": ([], i32),
        "tm_last_error": ([], ctypes.c_char_p),
        "tm_kvcache_bytes": ([cfgp], S),
        "tm_workspace_bytes": ([cfgp], S),
        "tm_get_unique_id": ([ctypes.c_char_p], i32),
        "tm_attn_init": ([cfgp, ctypes.c_char_p, V, S, V, S, P(V)], i32),
        "tm_attn_destroy": ([V], i32),
        "tm_stream_reset": ([V], i32),
        "tm_kvcache_put_reference": ([V, i32, i32, V, V, V], i32),
        "tm_chunk_attention": ([V, i32, i32, i64, V, V, V, V, V], i32),
        "tm_chunk_attention_phases": ([V, i32, i32, i64, V, V, V, V, ctypes.c_uint32, V], i32),
        "tm_kvcache_put_reference_phases": ([V, i32, i32, V, V, ctypes.c_uint32, V], i32),
        "tm_peer_export": ([V, ctypes.c_char_p], i32),
        "tm_peer_connect": ([V, ctypes.c_char_p], i32),
        "tm_peer_connect_local": ([P(V), i32], i32),
        "tm_nccl_connect_local": ([P(V), i32], i32),
        "tm_peer_check": ([V], i32),
        "tm_peer_output_ptr": ([V, P(V)], i32),
        "tm_schedule_tail_host": ([i32, i32, i32, P(i32)], i32),
        "tm_peer_route_host": ([i32, V, V, i32, i64, i64, i64, i32, i32, i32, i32, i32], i32),
        "tm_kvcache_slot_ptr": ([V, i32, i32, i64, P(V), P(V)], i32),
        "tm_kvcache_ref_ptr": ([V, i32, i32, P(V), P(V)], i32),
        "tm_flow_euler_step": ([V, V, V, i32, i64, ctypes.c_float, V], i32),
        "tm_ulysses_shuffle_host": ([i32, V, V, i32, i64, i64, i32, i32, i32, i32], i32),
        "tm_window_attention": ([V, V, V, V, V, P(i64), i32, V], i32),
        "tm_reference_attention": ([V, i32, i32, V, V, V, V, V], i32),
        "tm_audio_scratch_bytes": ([V, i64, i64], S),
        "tm_audio_cross_attention": ([V, V, V, V, V, i64, i64, i64, V, i64, i32, V, S, V], i32),
        "tm_flow_sampler_step": ([V, V, V, i32, i64, ctypes.c_float, ctypes.c_float, V,
                                  ctypes.c_uint64, ctypes.c_uint64, V, V], i32),
        "tm_last_launch_count": ([V], i32),
        "tm_kernel_variant": ([V], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


lib = _load()

EXPORTED = ("tm_version", "tm_last_error", "tm_kvcache_bytes", "tm_workspace_bytes",
            "tm_get_unique_id", "tm_attn_init", "tm_attn_destroy", "tm_stream_reset",
            "tm_kvcache_put_reference", "tm_chunk_attention", "tm_kvcache_slot_ptr",
            "tm_kvcache_ref_ptr", "tm_flow_euler_step", "tm_ulysses_shuffle_host",
            "tm_window_attention", "tm_reference_attention", "tm_flow_sampler_step", "tm_audio_scratch_bytes",
            "tm_audio_cross_attention", "tm_chunk_attention_phases",
            "tm_kvcache_put_reference_phases", "tm_peer_export", "tm_peer_connect",
            "tm_peer_connect_local", "tm_nccl_connect_local", "tm_peer_check", "tm_peer_route_host", "tm_peer_output_ptr",
            "tm_schedule_tail_host",
            "tm_last_launch_count",
            "tm_kernel_variant")


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(s):
    """cudaStream_t of `s`; None means torch's CURRENT stream on the current
    device (not the legacy default stream, which torch's non-blocking side
    streams do not wait on)."""
    if s is None:
        import torch
        if not torch.cuda.is_available():     # host-only calls (argument errors, CPU tests)
            return None
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _check(status):
    if status != TM_OK:
        raise TMError(status, lib.tm_last_error().decode())


def tm_version() -> int:
    return lib.tm_version()


def tm_last_error() -> str:
    return lib.tm_last_error().decode()


def tm_kvcache_bytes(cfg: tm_config) -> int:
    return lib.tm_kvcache_bytes(ctypes.byref(cfg))


def tm_workspace_bytes(cfg: tm_config) -> int:
    return lib.tm_workspace_bytes(ctypes.byref(cfg))


def tm_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.tm_get_unique_id(buf))
    return buf.raw


def tm_attn_init(cfg: tm_config, nccl_id, cache, cache_bytes, workspace, ws_bytes):
    out = ctypes.c_void_p()
    _check(lib.tm_attn_init(ctypes.byref(cfg), nccl_id, _ptr(cache), cache_bytes,
                            _ptr(workspace), ws_bytes, ctypes.byref(out)))
    return out.value


def tm_attn_destroy(ctx) -> None:
    _check(lib.tm_attn_destroy(ctx))


def tm_stream_reset(ctx) -> None:
    _check(lib.tm_stream_reset(ctx))


def tm_kvcache_put_reference(ctx, layer, step, k, v, stream=None) -> None:
    _check(lib.tm_kvcache_put_reference(ctx, layer, step, _ptr(k), _ptr(v), _stream(stream)))


def tm_chunk_attention(ctx, layer, step, chunk, q, k, v, o, stream=None) -> None:
    _check(lib.tm_chunk_attention(ctx, layer, step, chunk, _ptr(q), _ptr(k), _ptr(v), _ptr(o),
                                  _stream(stream)))


def tm_chunk_attention_phases(ctx, layer, step, chunk, q, k, v, o, phases, stream=None) -> None:
    _check(lib.tm_chunk_attention_phases(ctx, layer, step, chunk, _ptr(q), _ptr(k), _ptr(v),
                                         _ptr(o), phases, _stream(stream)))


def tm_kvcache_put_reference_phases(ctx, layer, step, k, v, phases, stream=None) -> None:
    _check(lib.tm_kvcache_put_reference_phases(ctx, layer, step, _ptr(k), _ptr(v), phases,
                                               _stream(stream)))


def tm_peer_export(ctx) -> bytes:
    buf = ctypes.create_string_buffer(TM_PEER_HANDLE_BYTES)
    _check(lib.tm_peer_export(ctx, buf))
    return buf.raw


def tm_peer_connect(ctx, handles) -> None:
    """handles: the world_size exported handles, in rank order."""
    blob = b"".join(handles)
    _check(lib.tm_peer_connect(ctx, blob))


def tm_peer_connect_local(ctxs) -> None:
    arr = (ctypes.c_void_p * len(ctxs))(*ctxs)
    _check(lib.tm_peer_connect_local(arr, len(ctxs)))


def tm_nccl_connect_local(ctxs) -> None:
    arr = (ctypes.c_void_p * len(ctxs))(*ctxs)
    _check(lib.tm_nccl_connect_local(arr, len(ctxs)))


def tm_peer_output_ptr(ctx) -> int:
    o = ctypes.c_void_p()
    _check(lib.tm_peer_output_ptr(ctx, ctypes.byref(o)))
    return o.value


def tm_peer_check(ctx) -> None:
    _check(lib.tm_peer_check(ctx))


def tm_kvcache_slot_ptr(ctx, layer, step, chunk):
    k, v = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib.tm_kvcache_slot_ptr(ctx, layer, step, chunk, ctypes.byref(k), ctypes.byref(v)))
    return k.value, v.value


def tm_kvcache_ref_ptr(ctx, layer, step):
    k, v = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib.tm_kvcache_ref_ptr(ctx, layer, step, ctypes.byref(k), ctypes.byref(v)))
    return k.value, v.value


def tm_flow_euler_step(ctx, x, v, v_dtype, n, dt, stream=None) -> None:
    _check(lib.tm_flow_euler_step(ctx, _ptr(x), _ptr(v), v_dtype, n, dt, _stream(stream)))


def tm_flow_sampler_step(ctx, x, v, v_dtype, n, t_cur, t_next, eps=None, seed=0, offset=0,
                         x_bf16_out=None, stream=None) -> None:
    _check(lib.tm_flow_sampler_step(ctx, _ptr(x), _ptr(v), v_dtype, n, t_cur, t_next, _ptr(eps),
                                    seed, offset, _ptr(x_bf16_out), _stream(stream)))


def tm_audio_scratch_bytes(ctx, frames, n_face) -> int:
    return lib.tm_audio_scratch_bytes(ctx, frames, n_face)


def tm_audio_cross_attention(ctx, q, k_audio, v_audio, o, frames, tokens_per_frame,
                             audio_tokens_per_frame, face_ids, n_face, window, scratch,
                             scratch_bytes, stream=None) -> None:
    _check(lib.tm_audio_cross_attention(ctx, _ptr(q), _ptr(k_audio), _ptr(v_audio), _ptr(o), frames,
                                        tokens_per_frame, audio_tokens_per_frame, _ptr(face_ids),
                                        n_face, window, _ptr(scratch), scratch_bytes,
                                        _stream(stream)))


def tm_reference_attention(ctx, layer, step, q, k, v, o, stream=None) -> None:
    _check(lib.tm_reference_attention(ctx, layer, step, _ptr(q), _ptr(k), _ptr(v), _ptr(o),
                                      _stream(stream)))


def tm_window_attention(ctx, q, k, v, o, chunk_lens, stream=None) -> None:
    arr = (ctypes.c_int64 * len(chunk_lens))(*[int(x) for x in chunk_lens])
    _check(lib.tm_window_attention(ctx, _ptr(q), _ptr(k), _ptr(v), _ptr(o), arr, len(chunk_lens),
                                   _stream(stream)))


def tm_ulysses_shuffle_host(mode, src, dst, batch, shard_tokens, tokens, heads_per_rank,
                            world_size, head_dim, elem_bytes) -> None:
    """src/dst: contiguous numpy arrays (host memory)."""
    _check(lib.tm_ulysses_shuffle_host(mode, src.ctypes.data, dst.ctypes.data, batch, shard_tokens,
                                       tokens, heads_per_rank, world_size, head_dim, elem_bytes))


def tm_peer_route_host(mode, src, dst, batch, shard_tokens, tokens, window_tokens, heads_per_rank,
                       world_size, rank, head_dim, elem_bytes) -> None:
    """src/dst: contiguous numpy arrays (host memory)."""
    _check(lib.tm_peer_route_host(mode, src.ctypes.data, dst.ctypes.data, batch, shard_tokens,
                                  tokens, window_tokens, heads_per_rank, world_size, rank,
                                  head_dim, elem_bytes))


def tm_schedule_tail_host(units, tiles_per_unit, ctas):
    """The stream-K tail ranges (list of G+1 bounds) the kernel would use."""
    buf = (ctypes.c_int32 * (ctas + 1))()
    g = lib.tm_schedule_tail_host(units, tiles_per_unit, ctas, buf)
    if g < 0:
        raise TMError(1, lib.tm_last_error().decode())
    return list(buf[:g + 1])


def tm_last_launch_count(ctx) -> int:
    return lib.tm_last_launch_count(ctx)


def tm_kernel_variant(ctx) -> str:
    return lib.tm_kernel_variant(ctx).decode()


def _wrap_device_ptr(ptr, numel, dtype, device):
    """A torch tensor aliasing `numel` elements at device pointer `ptr` (no copy)."""
    import torch

    class _Holder:
        __cuda_array_interface__ = {
            "shape": (numel,), "typestr": "<i2", "data": (ptr, False), "version": 3}

    t = torch.as_tensor(_Holder(), device=torch.device("cuda", device))
    return t.view(dtype)


_cudart_lib = None


def _cudart():
    global _cudart_lib
    if _cudart_lib is None:
        _cudart_lib = ctypes.CDLL("libcudart.so.12")
        _cudart_lib.cudaMalloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t]
        _cudart_lib.cudaFree.argtypes = [ctypes.c_void_p]
        _cudart_lib.cudaMemset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t]
        _cudart_lib.cudaSetDevice.argtypes = [ctypes.c_int]
        _cudart_lib.cudaDeviceSynchronize.argtypes = []
    return _cudart_lib


def _cuda_malloc(nbytes, device):
    """Zeroed plain cudaMalloc block (IPC-exportable), or None if cudart is unavailable."""
    try:
        rt = _cudart()
    except OSError:
        return None
    rt.cudaSetDevice(device)
    p = ctypes.c_void_p()
    if rt.cudaMalloc(ctypes.byref(p), nbytes) != 0:
        raise TMError(8, f"cudaMalloc of {nbytes} bytes for the peer workspace failed")
    rt.cudaMemset(p, 0, nbytes)
    rt.cudaDeviceSynchronize()
    return p.value


def _cuda_free(ptr):
    try:
        _cudart().cudaFree(ptr)
    except OSError:
        pass


class ChunkAttention:
    """Owns a tm_ctx plus torch-allocated cache and workspace (plumbing only).

    Tensors passed to the methods are torch CUDA tensors in the layouts of
    include/tm.h: q/k/v/o [B][Lc(/P)][H][d], reference k/v [B][Lr(/P)][H][d].
    """

    def __init__(self, heads, head_dim, ref_tokens, chunk_tokens, num_layers=1, num_steps=1,
                 batch=1, dtype=TM_BF16, softmax_scale=0.0, world_size=1, rank=0, device=0,
                 nccl_id=None, transport=TM_TRANSPORT_NCCL, sched_heads=0):
        import torch
        self.cfg = make_config(heads, head_dim, ref_tokens, chunk_tokens, num_layers, num_steps,
                               batch, dtype, softmax_scale, world_size, rank, device, transport,
                               sched_heads)
        self.cache_bytes = tm_kvcache_bytes(self.cfg)
        self.ws_bytes = tm_workspace_bytes(self.cfg)
        if self.cache_bytes == 0 or self.ws_bytes == 0:
            raise TMError(2, f"invalid config: {tm_last_error()}")
        dev = torch.device("cuda", device)
        # torch's caching allocator returns >= 512-B aligned blocks; over-allocate
        # by 1 KiB and offset to honour the cache's 1024-B alignment.
        self._cache = torch.empty(self.cache_bytes + 1024, dtype=torch.uint8, device=dev)
        self._ws_raw = None
        if transport == TM_TRANSPORT_PEER and world_size > 1:
            # The peer window (in the workspace) is shared through CUDA IPC, which
            # needs a cudaMalloc allocation: a torch block may come from VMM
            # (expandable segments), which IPC cannot export.
            self._ws_raw = _cuda_malloc(self.ws_bytes + 1024, device)
        if self._ws_raw is None:
            self._ws = torch.zeros(self.ws_bytes + 1024, dtype=torch.uint8, device=dev)
            ws_base = self._ws.data_ptr()
        else:
            ws_base = self._ws_raw
        self.cache_ptr = (self._cache.data_ptr() + 1023) // 1024 * 1024
        self.ws_ptr = (ws_base + 1023) // 1024 * 1024
        self.ctx = tm_attn_init(self.cfg, nccl_id, self.cache_ptr, self.cache_bytes,
                                self.ws_ptr, self.ws_bytes)

    def close(self):
        if getattr(self, "ctx", None):
            tm_attn_destroy(self.ctx)
            self.ctx = None
        if getattr(self, "_ws_raw", None):
            _cuda_free(self._ws_raw)
            self._ws_raw = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self):
        tm_stream_reset(self.ctx)

    def put_reference(self, layer, step, k, v, stream=None):
        tm_kvcache_put_reference(self.ctx, layer, step, k, v, stream)

    def attend(self, layer, step, chunk, q, k, v, o, stream=None):
        tm_chunk_attention(self.ctx, layer, step, chunk, q, k, v, o, stream)
        return o

    def attend_phases(self, layer, step, chunk, q, k, v, o, phases, stream=None):
        tm_chunk_attention_phases(self.ctx, layer, step, chunk, q, k, v, o, phases, stream)
        return o

    def put_reference_phases(self, layer, step, k, v, phases, stream=None):
        tm_kvcache_put_reference_phases(self.ctx, layer, step, k, v, phases, stream)

    # -- peer transport group setup (TM_TRANSPORT_PEER)
    def export_handle(self) -> bytes:
        return tm_peer_export(self.ctx)

    def connect(self, handles):
        tm_peer_connect(self.ctx, handles)

    def connect_dist(self, group=None):
        """All-gather the window handles over torch.distributed and map the peers'."""
        import torch.distributed as dist
        mine = self.export_handle()
        allh = [None] * dist.get_world_size(group)
        dist.all_gather_object(allh, mine, group=group)
        self.connect(allh)

    @staticmethod
    def connect_local(cas):
        tm_peer_connect_local([c.ctx for c in cas])

    @staticmethod
    def nccl_connect_local(cas):
        """Loopback NCCL-transport group of contexts in this process (created
        with nccl_id=None): all-to-all as device copies (tm_nccl_connect_local)."""
        tm_nccl_connect_local([c.ctx for c in cas])

    def check(self):
        tm_peer_check(self.ctx)

    def output_window(self):
        """torch view of this rank's O window (zero-copy output, TM_TRANSPORT_PEER)."""
        import torch
        ptr = tm_peer_output_ptr(self.ctx)
        Ls = -(-self.cfg.chunk_tokens // self.cfg.world_size)
        shape = (self.cfg.batch, Ls, self.cfg.heads, self.cfg.head_dim)
        n = shape[0] * shape[1] * shape[2] * shape[3]
        # wrap the raw device pointer without copying (the ctx owns its lifetime)
        return _wrap_device_ptr(ptr, n, torch.bfloat16, self.cfg.device).view(shape)

    def slot_ptr(self, layer, step, chunk):
        return tm_kvcache_slot_ptr(self.ctx, layer, step, chunk)

    def ref_ptr(self, layer, step):
        return tm_kvcache_ref_ptr(self.ctx, layer, step)

    def reference_attend(self, layer, step, q, k, v, o, stream=None):
        """Chunk 0 generated by the model: o = attention over c_0, and k, v cached."""
        tm_reference_attention(self.ctx, layer, step, q, k, v, o, stream)
        return o

    def window(self, q, k, v, o, chunk_lens, stream=None):
        tm_window_attention(self.ctx, q, k, v, o, chunk_lens, stream)
        return o

    def audio(self, q, k_audio, v_audio, o, face_ids, window=5, stream=None):
        """q/o [B][frames][T][H][d], k/v [B][frames][A][H][d] (or without B for
        batch 1); face_ids: torch int32 CUDA tensor.  The scratch is allocated
        here once per launch stream and reused (calls on one stream are
        ordered, so a reuse never overlaps the previous call's kernels)."""
        import torch
        frames, T = q.shape[-4], q.shape[-3]
        A = k_audio.shape[-3]
        n = face_ids.numel()
        nb = tm_audio_scratch_bytes(self.ctx, frames, n)
        sh = _stream(stream)
        cache = self.__dict__.setdefault("_audio_scratch", {})
        scratch = cache.get(sh)
        if scratch is None or scratch.numel() < nb + 1024:
            if scratch is not None:
                # the previous block may still be read by queued kernels of `sh`
                scratch.record_stream(torch.cuda.ExternalStream(sh) if isinstance(sh, int)
                                      else torch.cuda.current_stream())
            scratch = torch.empty(nb + 1024, dtype=torch.uint8, device=q.device)
            if isinstance(sh, int) and sh != torch.cuda.current_stream().cuda_stream:
                # allocated on the current stream, used on `sh`
                scratch.record_stream(torch.cuda.ExternalStream(sh))
            cache[sh] = scratch
        ptr = (scratch.data_ptr() + 1023) // 1024 * 1024
        tm_audio_cross_attention(self.ctx, q, k_audio, v_audio, o, frames, T, A, face_ids, n,
                                 window, ptr, nb, sh)
        return o

    def euler(self, x, v, v_dtype, dt, stream=None):
        tm_flow_euler_step(self.ctx, x, v, v_dtype, x.numel(), dt, stream)

    @property
    def launches(self):
        return tm_last_launch_count(self.ctx)

    @property
    def variant(self):
        return tm_kernel_variant(self.ctx)
