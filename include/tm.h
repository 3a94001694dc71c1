/*
 * tm.h -- C ABI of the B200-native TalkingMachines sparse-causal chunk
 * attention library (arXiv 2506.03099).  libtm.so, built from
 * paper_2506_03099_b200/csrc for sm_100a.
 *
 * Citations: "P:n" = PAPER.md line n; "S:n" = SPEC.md line n.
 *
 * What the library computes (Sec 4.2, Eq 7): the queries of
 * latent-video chunk c_t attend bidirectionally to all tokens of c_t, to the
 * cached K/V of the previous chunk c_{t-1} and to the cached K/V of the
 * reference chunk c_0; "K and V include tokens from {c_0, c_{t-1}, c_t}
 * only".  The K/V of c_0 and c_{t-1} are cached "for each timestep,
 * over all transformer blocks", so they are reused across chunks and
 * across the denoising steps (2 NFE).  Plus the flow-matching Euler
 * update x <- x + dt*v (Eqs 1-2).
 *
 * Conventions
 *  - All tensors are dense, row-major, TOKEN-MAJOR: [B][L][H][d] (batch of
 *    independent streams, tokens, heads, head dim).  With world_size P > 1
 *    (Ulysses sequence parallelism) the caller passes its sequence
 *    shard [B][L/P][H][d]; the library exchanges to head shards internally.
 *    L/P is rounded up (shards padded) when P does not divide L.
 *  - dtype TM_BF16: q, k, v, o are bfloat16; cache bf16.  TM_FP32: fp32
 *    everywhere (validation mode).
 *  - Every device pointer is owned by the CALLER (allocated e.g. with torch)
 *    and must stay valid until the stream reaches the call.  The library
 *    owns only the opaque host tm_ctx (and, for P > 1, its NCCL
 *    communicator or its mappings of the peers' windows).  The library never
 *    allocates device memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Argument, shape and ordering errors are detected on the host before
 *    any launch; the call then has no side effects.  Device / NCCL errors
 *    return TM_ERR_CUDA / TM_ERR_NCCL.  tm_last_error() gives a message.
 *  - Thread-compatible, not thread-safe per ctx.  For P > 1 every call
 *    except tm_flow_euler_step is collective: all ranks call in the same
 *    order.
 *  - Environment (debug/test only): TM_DEBUG=1 synchronises after each call
 *    and checks outputs for NaN/Inf (TM_ERR_NONFINITE); TM_FORCE_ULYSSES=1
 *    makes a world_size == 1 context run the full exchange path (pack, a
 *    1-rank ncclAlltoAll, unpack) -- read by tm_workspace_bytes and
 *    tm_attn_init, so set it before both.
 */
#ifndef TM_H_
#define TM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TM_OK = 0,
    TM_ERR_INVALID_ARG = 1,     /* null pointer, bad enum, bad index            */
    TM_ERR_SHAPE = 2,           /* dimension error                        */
    TM_ERR_DEGENERATE_MASK = 3, /* an empty attend set                    */
    TM_ERR_STREAM_ORDER = 4,    /* cache miss / chunk out of order       */
    TM_ERR_REF_IMMUTABLE = 5,   /* reference rewrite after stream start  */
    TM_ERR_NONFINITE = 6,       /* NaN/Inf output, TM_DEBUG=1 only        */
    TM_ERR_UNSUPPORTED = 7,     /* valid but not implemented configuration       */
    TM_ERR_CUDA = 8,
    TM_ERR_NCCL = 9
} tm_status;

typedef enum { TM_BF16 = 0, TM_FP32 = 1 } tm_dtype;

/* How the Ulysses exchange moves data between the ranks.
 *  TM_TRANSPORT_NCCL: pack kernel -> ncclAlltoAll -> unpack kernel, each way.
 *  TM_TRANSPORT_PEER: no NCCL on the data path.  Every rank's workspace holds
 *    a window that all ranks map (CUDA IPC over NVLink, see tm_peer_export /
 *    tm_peer_connect).  The attention kernel itself pushes this rank's
 *    sequence shard of Q, K, V into the head owners' windows (NVLink stores),
 *    waits per Q tile / per K-V tile only for the source ranks that tile comes
 *    from (so the cached c_0 and c_{t-1} segments are attended while the
 *    current chunk is still in flight), and its epilogue stores each output
 *    row straight into the window of the rank that owns that token; a small
 *    receive kernel copies the finished O window to `o`.  bf16 only,
 *    world_size <= 8. */
typedef enum { TM_TRANSPORT_NCCL = 0, TM_TRANSPORT_PEER = 1 } tm_transport;

/* Phases of one collective call (tm_chunk_attention_phases,
 * tm_kvcache_put_reference_phases), TM_TRANSPORT_PEER only.  A call runs the
 * requested phases in order; the next call continues with the next phase of
 * the same operation.  Splitting lets ranks that share one device and one
 * process (tests) enqueue every rank's SEND before any rank's ATTEND.
 *   SEND    push this rank's shard into the owners' windows
 *   ATTEND  chunk: attention (waits for the pushes; O rows to their owners);
 *           reference: copy the received K/V window into the cache
 *   RECV    chunk: wait for every rank's O rows, copy them to o;
 *           reference: barrier (windows free again)
 * SEND|ATTEND in one call fuses the push into the attention kernel. */
#define TM_PHASE_SEND 1u
#define TM_PHASE_ATTEND 2u
#define TM_PHASE_RECV 4u
#define TM_PHASE_ALL 7u

/* Bytes of the handle tm_peer_export writes (CUDA IPC handle + offset). */
#define TM_PEER_HANDLE_BYTES 72

typedef struct {
    int32_t heads;         /* H, global number of attention heads (MHA; H_kv == H)   */
    int32_t head_dim;      /* d in {64, 128}                                          */
    int32_t ref_tokens;    /* Lr: tokens of the reference chunk c_0 (>= 1)            */
    int32_t chunk_tokens;  /* Lc: tokens per generated chunk (frames x tokens/frame)  */
    int32_t num_layers;    /* transformer blocks whose K/V are cached (40 for WAN)    */
    int32_t num_steps;     /* denoising steps (NFE) per chunk with a cache slot (2)   */
    int32_t batch;         /* B independent streams (>= 1)                            */
    int32_t dtype;         /* tm_dtype                                                */
    float softmax_scale;   /* 0 -> 1/sqrt(d), Eq 7                                    */
    int32_t world_size;    /* P, Ulysses group size; H % P == 0                       */
    int32_t rank;          /* this process's rank in [0, P)                           */
    int32_t device;        /* CUDA device ordinal used by this ctx                    */
    int32_t transport;     /* tm_transport (ignored when world_size == 1 and NCCL)    */
    int32_t sched_heads;   /* heads per SCHEDULE BLOCK of the attention kernel; 0 =
                            * all heads of the rank in one block (fastest).  k > 0
                            * (must divide heads / world_size): every k heads are
                            * scheduled as a block of their own -- which units are
                            * split for load balance, where, and the merge order are
                            * a function of the block's shape only -- so a head's
                            * output is BITWISE the same for every world size P
                            * with (heads / P) % k == 0 (e.g.
                            * k = 5 at H = 40 for P in {1, 2, 4, 8}).  The cost is
                            * measured in DESIGN.md Sec 7.                       */
} tm_config;

typedef struct tm_ctx tm_ctx;

/* Version of the ABI (major * 100 + minor). */
int32_t tm_version(void);   /* 102: tm_config.sched_heads, one-launch window / audio, loopback NCCL groups */

/* Thread-local message for the last non-OK status returned on this thread. */
const char* tm_last_error(void);

/* Bytes of the per-rank KV cache: for each (layer, step) the reference
 * K and V ([B][Lr][H/P][d]) and two rotating chunk slots of K and V
 * ([B][Lc][H/P][d] each), every region 1024-byte aligned.  A closed form of
 * the config, independent of stream length.  0 on invalid config. */
size_t tm_kvcache_bytes(const tm_config* cfg);

/* Bytes of device workspace: the split-unit partials and merge counters of
 * the attention schedule and a debug flag, plus the
 * Ulysses staging (NCCL transport, world_size > 1) or the peer window
 * (TM_TRANSPORT_PEER: counters and Q, K, V windows [B][max(Lc,Lr)][H/P][d],
 * O window [B][Lc/P][H][d]).  0 is never returned for a valid config. */
size_t tm_workspace_bytes(const tm_config* cfg);

/* NCCL unique id for world_size > 1 (rank 0 calls it; the harness
 * broadcasts the 128 bytes, e.g. with torch.distributed). */
tm_status tm_get_unique_id(uint8_t id[128]);

/* Create a context.  `cache` (device, >= tm_kvcache_bytes, 1024-B aligned)
 * and `workspace` (device, >= tm_workspace_bytes, 256-B aligned) are owned
 * by the caller and must outlive the ctx.  nccl_id: NULL when world_size==1
 * or with TM_TRANSPORT_PEER (which then needs tm_peer_connect before use);
 * NULL with TM_TRANSPORT_NCCL and world_size > 1 defers the communicator to a
 * loopback group (tm_nccl_connect_local).
 * Validates the config (TM_ERR_SHAPE for H % P != 0, d not in {64,128},
 * non-positive lengths).  Collective when world_size > 1. */
tm_status tm_attn_init(const tm_config* cfg, const uint8_t* nccl_id, void* cache,
                       size_t cache_bytes, void* workspace, size_t workspace_bytes,
                       tm_ctx** out);

tm_status tm_attn_destroy(tm_ctx* ctx);

/* Start a new stream: forget the chunk order and allow a new reference. */
tm_status tm_stream_reset(tm_ctx* ctx);

/* a1: store the reference chunk's K/V for (layer, step);
 * step = -1 stores it for every step.  k, v: device [B][Lr(/P)][H][d].
 * Once chunk 1 has been attended at a (layer, step), rewriting its reference
 * returns TM_ERR_REF_IMMUTABLE until tm_stream_reset. */
tm_status tm_kvcache_put_reference(tm_ctx* ctx, int32_t layer, int32_t step, const void* k,
                                   const void* v, void* stream);

/* a2-a6: attention of chunk `chunk` (>= 1) at (layer, step).
 * q, k, v: device [B][Lc(/P)][H][d], the chunk's post-projection queries,
 * keys and values; o: device output, same shape.  The chunk's K/V are
 * appended to cache slot chunk&1 (they become c_{t-1} for chunk+1); keys
 * and values attended are {c_0 (cache), c_{t-1} (cache, chunk >= 2), c_t}
 * (P:151).  Order per (layer, step): chunk == last + 1, or chunk == last
 * (a redo of the same chunk, which re-reads the same c_{t-1});
 * otherwise TM_ERR_STREAM_ORDER; chunk 1 without a reference ->
 * TM_ERR_STREAM_ORDER (cache miss).  k/v may alias the slot returned
 * by tm_kvcache_slot_ptr (zero-copy append).  With TM_TRANSPORT_PEER, o may be
 * the rank's O window (tm_peer_output_ptr: no receive copy); the call is then
 * an attention kernel (which also pushes this rank's shard) plus a receive
 * kernel, see tm_transport. */
tm_status tm_chunk_attention(tm_ctx* ctx, int32_t layer, int32_t step, int64_t chunk,
                             const void* q, const void* k, const void* v, void* o,
                             void* stream);

/* Chunk 0 generated by the model (SURVEY Sec 8(b) optional mode; P:141 c_0
 * "containing the ground truth image", "chunk 0 attends itself only"):
 * o = softmax(q k^T / sqrt(d)) v over the reference tokens only, and k, v are
 * stored as the reference of (layer, step) (step = -1: every step), as
 * tm_kvcache_put_reference would.  q, k, v, o: device [B][Lr][H][d].  Same
 * immutability rule as tm_kvcache_put_reference (TM_ERR_REF_IMMUTABLE after
 * chunk 1).  world_size 1 direct contexts only (else TM_ERR_UNSUPPORTED).
 * bf16: one launch (the attention kernel appends K/V into the cache as it
 * reads them). */
tm_status tm_reference_attention(tm_ctx* ctx, int32_t layer, int32_t step, const void* q,
                                 const void* k, const void* v, void* o, void* stream);

/* the full-window form (P:130-143 and Eq 7 over a whole
 * training window, e.g. 21 latent frames = 7 chunks x 3 frames, P:134-136;
 * the DMD student's teacher-forcing pattern): q, k, v, o are device
 * [B][L][H][d] over the window [c_0 | c_1 | ... | c_{n-1}] with chunk_len[c]
 * tokens in chunk c (host array, L = sum); every query of chunk c attends the
 * keys of chunks {0, c-1, c} as a set (chunk 0 attends itself only).
 * No cache is read or written; B, H, d, dtype and the scale come from ctx
 * (world_size must be 1, else TM_ERR_UNSUPPORTED).  An empty chunk returns
 * TM_ERR_DEGENERATE_MASK.  bf16: ONE attention launch for up to 16
 * chunks (each chunk's units scheduled exactly as a tm_chunk_attention call
 * over the same segments would schedule them, so chunk c's rows equal that
 * call's output bit for bit); fp32 mode: one launch per chunk. */
tm_status tm_window_attention(tm_ctx* ctx, const void* q, const void* k, const void* v, void* o,
                              const int64_t* chunk_len, int32_t n_chunks, void* stream);

/* audio cross-attention with a face-region query mask
 * (keys/values from audio tokens, cross-attended by the latent-frame
 * queries, "local attention masks that focus on facial regions"; P:125:
 * "each latent frame will attend only to the audio tokens within a window of
 * five latent frames centered around itself").
 *   q: device [B][frames][T][H][d]      latent tokens of `frames` latent frames
 *   k_audio, v_audio: device [B][frames][A][H][d]   projected audio tokens
 *   o: device [B][frames][T][H][d]      face rows: attention output; others 0
 *   face_ids: DEVICE int32 [n_face], token indices in [0, T) (the face region)
 *   window: odd, <= 5; frames outside [0, frames) are clamped by repeating the
 *   boundary frame (SPEC S:117 design decision; frame 0 -> {0,0,0,1,2}).
 *   scratch: device, >= tm_audio_scratch_bytes(ctx, frames, n_face), 1024-B
 *   aligned (gathered face rows of q; fp32 mode also of o; bf16 mode the
 *   inverse face map, 192 KiB).  Reused by the next call on the same stream.
 * n_face == 0 -> TM_ERR_DEGENERATE_MASK.  B, H, d, dtype, scale from
 * ctx (world_size 1).  bf16 launches: one prep kernel (gathers the face rows
 * of q, writes the inverse face map) and ONE attention launch for up to 16
 * frames whose epilogue writes each face row to o directly while its spare
 * warp zeroes the non-face rows; T <= 49152.
 * fp32 mode: gather, one attention per frame, zero, scatter. */
size_t tm_audio_scratch_bytes(const tm_ctx* ctx, int64_t frames, int64_t n_face);
tm_status tm_audio_cross_attention(tm_ctx* ctx, const void* q, const void* k_audio,
                                   const void* v_audio, void* o, int64_t frames,
                                   int64_t tokens_per_frame, int64_t audio_tokens_per_frame,
                                   const int32_t* face_ids, int64_t n_face, int32_t window,
                                   void* scratch, size_t scratch_bytes, void* stream);

/* Phased forms of tm_chunk_attention / tm_kvcache_put_reference for
 * TM_TRANSPORT_PEER (see TM_PHASE_*); `phases` = TM_PHASE_ALL is the plain
 * call.  Arguments are validated on the operation's first phase; the later
 * phases of the same operation must repeat them (TM_ERR_STREAM_ORDER
 * otherwise, or if a phase is skipped or a new operation starts before the
 * previous one finished its RECV phase).  NCCL contexts accept only ALL,
 * except loopback groups (tm_nccl_connect_local), where SEND packs the shard,
 * ATTEND exchanges, unpacks, attends and packs O, and RECV exchanges O and
 * unpacks it to o. */
tm_status tm_chunk_attention_phases(tm_ctx* ctx, int32_t layer, int32_t step, int64_t chunk,
                                    const void* q, const void* k, const void* v, void* o,
                                    uint32_t phases, void* stream);
tm_status tm_kvcache_put_reference_phases(tm_ctx* ctx, int32_t layer, int32_t step,
                                          const void* k, const void* v, uint32_t phases,
                                          void* stream);

/* TM_TRANSPORT_PEER group setup (collective; after tm_attn_init on every rank,
 * before any other call).  tm_peer_export writes this rank's window handle
 * (TM_PEER_HANDLE_BYTES: the CUDA IPC handle of the workspace allocation and
 * the window's offset in it); the harness all-gathers the handles (e.g.
 * torch.distributed) and every rank passes all of them, in rank order, to
 * tm_peer_connect, which maps the peers' windows (cudaIpcOpenMemHandle with
 * lazy peer access; closed by tm_attn_destroy).  The workspace must come from
 * cudaMalloc (torch's default caching allocator), not VMM.
 * tm_peer_connect_local connects `n` contexts of ONE process (virtual ranks,
 * e.g. several on one device for tests): ctxs[i] must have rank i. */
/* TM_TRANSPORT_NCCL loopback group (tests / single-process use): `n` >= 2
 * contexts of ONE process with world_size n, ctxs[i] of rank i, each created
 * with nccl_id = NULL (tm_attn_init then defers the communicator).  Their
 * all-to-alls become device copies between the contexts' workspaces (the same
 * block permutation ncclAlltoAll performs, so the pack / unpack kernels and
 * the head-sharded attention run exactly as with NCCL).  The contexts must be
 * driven on one stream with the phased calls, every rank's SEND before any
 * rank's ATTEND and every ATTEND before any RECV.  Until connected, their
 * exchanging calls return TM_ERR_STREAM_ORDER. */
tm_status tm_nccl_connect_local(tm_ctx* const* ctxs, int32_t n);

tm_status tm_peer_export(tm_ctx* ctx, uint8_t handle[TM_PEER_HANDLE_BYTES]);
tm_status tm_peer_connect(tm_ctx* ctx, const uint8_t* handles);
tm_status tm_peer_connect_local(tm_ctx* const* ctxs, int32_t n);

/* TM_TRANSPORT_PEER zero-copy output: the device pointer of this rank's O
 * window ([B][ceil(Lc/P)][H][d], bf16).  Passing it as `o` to
 * tm_chunk_attention(_phases) skips the receive copy: the RECV phase only
 * waits until every rank has stored its rows.  The window is rewritten by the
 * next call; rows past the end of the sequence (shard padding) are
 * unspecified (the copying RECV writes zeros there). */
tm_status tm_peer_output_ptr(tm_ctx* ctx, void** o);

/* Health check of a multi-rank context.  NCCL transport: the communicator's
 * asynchronous error state (ncclCommGetAsyncError -> TM_ERR_NCCL).  Peer
 * transport: synchronises the device and reports whether a device-side peer
 * wait timed out (10 s without the expected peer signal) since the last
 * check: TM_ERR_CUDA with a message, else TM_OK; clears the flag. */
tm_status tm_peer_check(tm_ctx* ctx);

/* Device pointers of the cache slot that chunk `chunk` at (layer, step) is
 * stored in ([B][Lc][H/P][d] each).  A caller may write the chunk's K/V
 * there before tm_chunk_attention to skip the append copy. */
tm_status tm_kvcache_slot_ptr(tm_ctx* ctx, int32_t layer, int32_t step, int64_t chunk,
                              void** k, void** v);

/* Device pointers of the reference region of (layer, step) ([B][Lr][H/P][d]). */
tm_status tm_kvcache_ref_ptr(tm_ctx* ctx, int32_t layer, int32_t step, void** k, void** v);

/* a7: x[i] <- x[i] + dt * v[i] for i < n, in place, one fp32
 * FMA per element (single rounding).  x: device fp32 [n]; v: device, dtype
 * v_dtype (TM_BF16 or TM_FP32) [n].  ctx may be NULL.  x and v must be
 * 16-byte aligned.  n == 0 is a no-op. */
tm_status tm_flow_euler_step(tm_ctx* ctx, float* x, const void* v, int32_t v_dtype, int64_t n,
                             float dt, void* stream);

/* one schedule entry of the few-step student (2 NFE,
 * P:153), fused: with the state x (device fp32 [n], in place)
 * at time t_cur (Eq 1 convention: 0 = noise, 1 = data) and the
 * predicted velocity v (TM_BF16 / TM_FP32 [n]):
 *     x1_hat = x + (1 - t_cur) * v
 *     x     <- t_next * x1_hat + (1 - t_next) * eps     (Eq 1 re-noise), or
 *     x     <- x1_hat                                     if t_next >= 1 (final)
 * eps: device fp32 [n], or NULL to draw N(0,1) in-kernel from Philox4x32-10
 * (counter = (i / 4, offset), key = seed; Box-Muller on word pairs) --
 * deterministic per (seed, offset, i).  x_bf16_out (nullable): bf16 copy of
 * the new x, the next NFE's model input.  Needs 0 <= t_cur < 1 and
 * t_next > t_cur.  x, v, eps 4-byte aligned. */
tm_status tm_flow_sampler_step(tm_ctx* ctx, float* x, const void* v, int32_t v_dtype, int64_t n,
                               float t_cur, float t_next, const float* eps, uint64_t seed,
                               uint64_t offset, void* x_bf16_out, void* stream);

/* Host reference of the Ulysses exchange layouts, the same index map
 * the device pack/unpack kernels use; for tests of the multi-rank host logic
 * without GPUs.  Buffers are host memory; rows of head_dim * elem_bytes bytes
 * (a multiple of 16).  Rank r holds tokens [r*Ls, r*Ls+Ls) of the sequence
 * (Ls = shard_tokens, tokens >= `tokens` are padding) and heads
 * [r*Hl, r*Hl+Hl) after the exchange (Hl = heads_per_rank, H = Hl*world_size).
 *   mode 0: [B][Ls][H][d]     -> [P][B][Ls][Hl][d]   (pack: block p goes to rank p)
 *   mode 1: [P][B][Ls][Hl][d] -> [B][L][Hl][d]       (unpack received blocks)
 *   mode 2: [B][L][Hl][d]     -> [P][B][Ls][Hl][d]   (pack outputs; pad rows zero)
 *   mode 3: [P][B][Ls][Hl][d] -> [B][Ls][H][d]       (unpack to the sequence shard) */
tm_status tm_ulysses_shuffle_host(int32_t mode, const void* src, void* dst, int32_t batch,
                                  int64_t shard_tokens, int64_t tokens, int32_t heads_per_rank,
                                  int32_t world_size, int32_t head_dim, int32_t elem_bytes);

/* Host reference of the peer transport's index maps (TM_TRANSPORT_PEER; the
 * same code the device push and attention epilogue use), for tests of the
 * multi-rank host logic without GPUs.  Host buffers; rows of head_dim *
 * elem_bytes bytes (a multiple of 16); Ls = shard_tokens, L = tokens,
 * Lw = window_tokens (>= L), Hl = heads_per_rank, H = Hl * world_size.
 *   mode 0 (push, row a2): src = rank's sequence shard [B][Ls][H][d];
 *          dst = the world_size windows [P][B][Lw][Hl][d]: head block p of
 *          token t goes to window p, row rank*Ls + t (padding tokens dropped).
 *   mode 1 (output, row a6): src = rank's head-shard output [B][L][Hl][d];
 *          dst = the world_size O windows [P][B][Ls][H][d]: row q goes to
 *          window q / Ls, row q % Ls, heads [rank*Hl, rank*Hl + Hl).
 * Words not routed are left untouched. */
tm_status tm_peer_route_host(int32_t mode, const void* src, void* dst, int32_t batch,
                             int64_t shard_tokens, int64_t tokens, int64_t window_tokens,
                             int32_t heads_per_rank, int32_t world_size, int32_t rank,
                             int32_t head_dim, int32_t elem_bytes);

/* Host reference of the attention kernel's tail schedule (stream-K; DESIGN
 * Sec 6), for tests without a GPU: the KV tiles of `units` tail units of
 * `tiles_per_unit` tiles each, flattened, are cut into G <= ctas contiguous
 * ranges [bounds[c], bounds[c+1]) (bounds: >= ctas + 1 ints), the minimum
 * piece raised until no unit is cut into more than 65 pieces (a split unit's
 * merger tracks its contributors in a 64-bit mask).  Returns G, or -1 on
 * invalid arguments (ctas <= 160). */
int32_t tm_schedule_tail_host(int32_t units, int32_t tiles_per_unit, int32_t ctas, int32_t* bounds);

/* Introspection for tests / bench: number of device kernels the last call
 * on this ctx launched (the TM_DEBUG finiteness check not counted), and the
 * attention kernel variant name ("sm100_tcgen05" or "fp32_simt"). */
int32_t tm_last_launch_count(const tm_ctx* ctx);
const char* tm_kernel_variant(const tm_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* TM_H_ */
