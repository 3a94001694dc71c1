// internal.h -- host-side declarations shared by the C-ABI (api.cpp) and the
// kernel launchers.  Not part of the public ABI (include/tm.h is).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <cuda_runtime.h>

namespace tmk {

constexpr int kMaxSegments = 5;   // {c_0, c_{t-1}, c_t}; f4 audio windows need up to 5
constexpr int kMaxPersistentCtas = 160;   // persistent grid cap (B200: 148 SMs)
constexpr int kMaxPeers = 8;      // peer transport: one NVSwitch node
constexpr int kMaxProblems = 16;  // problems per attention launch (f1 window chunks, f4 frames)
constexpr int kMaxBlocks = 8;     // schedule blocks per attention launch (see fmha_sm100.cu)
constexpr int kMaxSkClasses = 4;  // distinct stream-K tail shapes per launch
// Debug trace buffer (TM_TRACE build): 13 roles x 4096 clock64 events of CTA 0,
// then 8 words per CTA: globaltimer at entry, first S seen, second item start,
// exit, merge wait begin / end; tiles and items of the CTA.
constexpr int kTraceWords = 13 * 4096 + 8 * kMaxPersistentCtas;

// ---------------------------------------------------------------- peer transport
// The Ulysses exchange over NVLink peer memory instead of NCCL: each
// rank's workspace holds a WINDOW that every rank of the group maps (CUDA IPC,
// or plain pointers for ranks sharing a process).  Window layout:
//   PeerCounters (4 KiB) | Q [B][Lc][Hl][d] | K [B][Lw][Hl][d] | V [B][Lw][Hl][d] | O [B][Ls][H][d]
// (Lw = max(Lc, Lr); Ls = shard tokens).  Senders STORE into the owners'
// windows and bump the owners' monotone counters with release semantics;
// receivers acquire-poll their own counters against a host-tracked epoch.
struct PeerCounters {
    uint32_t arr[3][kMaxPeers];   // tensor T (0 Q, 1 K, 2 V) from source rank s: pushes landed
    uint32_t done[kMaxPeers];     // source rank s finished writing this rank's O rows / copy barrier
    uint32_t ticket[4];           // local last-CTA tickets (push T = 0..2, done = 3); zero between launches
    uint32_t err;                 // nonzero: a device-side wait timed out (see tm_peer_check)
};
static_assert(sizeof(PeerCounters) <= 4096, "counter block");

// One rank's push of up to three sequence-shard tensors to the head owners.
struct PeerPush {
    const void* src[3] = {nullptr, nullptr, nullptr};   // local [B][Ls][H][d]; null = not pushed
    void* dst[3][kMaxPeers] = {};                       // peer p's window of tensor T [B][Lw][Hl][d]
    PeerCounters* ctr[kMaxPeers] = {};                  // peer p's counters (ctr[rank] = own)
    PeerCounters* own = nullptr;                        // own counters (tickets, err)
    int B = 1, P = 1, rank = 0, W = 0;                  // W: 16-B words per (token, head block)
    int64_t Ls = 0, L = 0, Lw = 0;                      // shard tokens, valid tokens, window rows
};

// Peer side of one attention launch (row a5 between a2 and a6).
struct PeerAttnArgs {
    PeerCounters* own = nullptr;      // waits: Q (T=0) before each Q tile, K/V (T=1,2) before
    uint32_t epoch[3] = {0, 0, 0};    //   each tile of the window segment `wait_seg`
    int wait_seg = -1;
    int64_t src_rows = 0;             // window row r came from source rank r / src_rows
    bool push = false;                // fused: this kernel pushes `pp` before attending
    PeerPush pp;
    void* o_dst[kMaxPeers] = {};      // owner p's O window [B][Ls][H][d]
    int64_t o_rows = 0;               // output row q goes to owner q / o_rows, row q % o_rows
    int o_H = 0, o_h0 = 0;            // heads of a row in the O window; this rank's first head
    bool signal_done = false;         // bump every owner's done[rank] when all CTAs finished
    uint32_t wait_done = 0;           // nonzero: then wait for every rank's done (zero-copy receive)
    PeerCounters* done_ctr[kMaxPeers] = {};
    int P = 1, rank = 0;
};

// One contiguous K/V segment in token-major layout [B][len][H][d].
struct Segment {
    const void* k = nullptr;
    const void* v = nullptr;
    int64_t len = 0;               // tokens (0 = absent)
    int64_t bstride = 0;           // tokens between batch elements (0: = len)
};

// a4: the segment schedule of one chunk-attention call.
struct AttnProblem {
    const void* q = nullptr;       // [B][Lq][H][d]
    void* o = nullptr;             // [B][Lq][H][d]
    int64_t Lq = 0;
    int64_t q_bstride = 0;         // tokens between batch elements of q / o (0: = Lq)
    int B = 1, H = 1, d = 128;     // H = heads resident on this rank
    int nseg = 0;
    Segment seg[kMaxSegments];
    float scale = 0.f;             // softmax scale (1/sqrt(d), Eq 7)
    // a3 fused append (sm100 path): if set, the last segment's K/V tiles are also
    // written to these [B][len][H][d] buffers (the cache slot) by the kernel.
    void* store_k = nullptr;
    void* store_v = nullptr;
    const PeerAttnArgs* peer = nullptr;   // peer transport (sm100 path only)
    int max_ctas = 0;                     // persistent grid cap (0: one CTA per SM)
    int sched_heads = 0;                  // heads per schedule block (0: all; see tm_config)
};

// SM count of the CURRENT device, cached per device ordinal (a process may
// drive several GPUs through several contexts; each entry point selects its
// context's device first, see DeviceScope in api.cpp).
inline int current_sm_count() {
    constexpr int kMaxDev = 64;
    static int cache[kMaxDev] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
    if (dev >= kMaxDev) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 148;
    }
    int n = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
    if (n <= 0) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        __atomic_store_n(&cache[dev], n, __ATOMIC_RELAXED);
    }
    return n;
}

// Several attention problems in ONE launch over shared tensors (f1: the
// query chunks of a full window over their key chunks {0, c-1, c}, P:134-143;
// f4: the face rows of each latent frame over its clamped audio window,
// P:123-125).  Q [B][q_rows][H][d], K/V [B][kv_rows][H][d], O
// [B][o_rows][H][d] (batch strides in tokens, 0 = rows); problem i reads
// query rows [q_row0, q_row0 + Lq), its keys are nseg row ranges of K/V, and
// query q's output row is o_row0 + (o_row_map ? o_row_map[q] : q).
struct SubProblem {
    int64_t q_row0 = 0, Lq = 0, o_row0 = 0;
    int nseg = 0;
    int64_t seg_row0[kMaxSegments] = {};
    int64_t seg_len[kMaxSegments] = {};
};
struct MultiProblem {
    const void* q = nullptr;
    const void* k = nullptr;
    const void* v = nullptr;
    void* o = nullptr;
    int64_t q_rows = 0, q_bstride = 0, kv_rows = 0, kv_bstride = 0, o_rows = 0, o_bstride = 0;
    const int32_t* o_row_map = nullptr;   // device, nullable
    // f4: rows r of o ([B][o_rows] x H x d, o_rows = frames * zero_T) whose token
    // r % zero_T has zero_inv[token] < 0 are zeroed by the launch (device, nullable)
    const int32_t* zero_inv = nullptr;
    int64_t zero_T = 0, zero_row0 = 0, zero_rows = 0;   // rows [zero_row0, +zero_rows) of each batch
    int B = 1, H = 1, d = 128;
    float scale = 0.f;
    int nprob = 0;
    SubProblem prob[kMaxProblems];
    int max_ctas = 0;
    int sched_heads = 0;
    // keys of a problem = its segments concatenated without tile padding (when
    // every segment length is a multiple of 8; else padded as usual)
    bool pack_keys = false;
};

// Launch with programmatic dependent launch allowed (the kernel executes
// griddepcontrol.wait before touching global data, so its prologue overlaps the
// previous kernel's tail).  TM_PDL=0 disables the attribute (A/B).
bool pdl_enabled();
#ifdef __CUDACC__
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#endif

// Launchers; return cudaSuccess or the launch error.  `launches` is
// incremented by the number of kernels enqueued.
// `scratch` (fmha_sm100_scratch_bytes(d) bytes, zero-initialised once) holds
// the split-KV partials and merge counters; counters return to zero.
size_t fmha_sm100_scratch_bytes(int d);
// Host: the stream-K tail ranges of the attention schedule (fmha_sm100.cu):
// T tail units of n KV tiles each over at most C CTAs; writes G+1 bounds, returns G.
int tail_bounds(int T, int n, int C, int min_piece, int* bound);
// The same over runs of units of different sizes (run r: units[r] units of
// tiles[r] tiles each, flattened in order).
int tail_bounds_runs(int nruns, const int* units, const int* tiles, int C, int min_piece, int* bound);
// The kernel's schedule: tail_bounds with the minimum piece raised until no
// unit has more than kMaxUnitPieces pieces (64 contributors + the merger).
constexpr int kMaxUnitPieces = 65;
int tail_bounds_capped(int T, int n, int C, int* bound);
// `trace` (debug, may be null): 4 x 4096 uint64 clock64 timeline of CTA 0.
cudaError_t launch_fmha_sm100(const AttnProblem& p, void* scratch, cudaStream_t s, int* launches,
                              unsigned long long* trace = nullptr);
cudaError_t launch_fmha_sm100_multi(const MultiProblem& p, void* scratch, cudaStream_t s,
                                    int* launches, unsigned long long* trace = nullptr);
cudaError_t launch_fmha_fp32(const AttnProblem& p, cudaStream_t s, int* launches);
cudaError_t launch_euler(float* x, const void* v, int v_is_bf16, int64_t n, float dt,
                         cudaStream_t s, int* launches);
// f2: few-step sampler entry (see elementwise.cu); eps == nullptr -> Philox noise.
cudaError_t launch_sampler(float* x, const void* v, int v_is_bf16, const float* eps, int64_t n,
                           float t_cur, float t_next, uint64_t seed, uint64_t offset,
                           void* x_bf16, cudaStream_t s, int* launches);
// f4: gather (scatter = 0) / scatter (1) of face-token rows, ids device int32.
cudaError_t launch_face_rows(const void* src, void* dst, const int32_t* ids, int64_t BF, int64_t T,
                            int64_t nf, int row_bytes, int scatter, cudaStream_t s, int* launches);
// f4 (bf16): gather the face rows of q into qf and write the inverse face map
// inv[T] (token -> face slot or -1); the attention launch writes the face rows
// of o and zeroes the others (MultiProblem::zero_inv); T <= 49152.
cudaError_t launch_audio_prep(const void* q, void* qf, int32_t* inv, const int32_t* ids, int64_t BF,
                              int64_t T, int64_t nf, int row_bytes, cudaStream_t s, int* launches);
// Non-finite check: sets *flag (device int) to 1 if any element is NaN/Inf.
cudaError_t launch_nonfinite(const void* x, int is_bf16, int64_t n, int* flag, cudaStream_t s,
                             int* launches);

// Ulysses pack / unpack.  Token-major [B][L][H][d] <-> per-peer
// blocks; see ulysses.cu for the exact layouts.
cudaError_t launch_pack_seq_to_peers(const void* src, void* dst, int B, int64_t Ls, int H, int P,
                                     int d, int esize, cudaStream_t s, int* launches);
cudaError_t launch_unpack_peers_to_heads(const void* src, void* dst, int B, int64_t Ls,
                                         int64_t L, int Hl, int P, int d, int esize,
                                         cudaStream_t s, int* launches);
cudaError_t launch_pack_heads_to_peers(const void* src, void* dst, int B, int64_t Ls, int64_t L,
                                       int Hl, int P, int d, int esize, cudaStream_t s,
                                       int* launches);
cudaError_t launch_unpack_peers_to_seq(const void* src, void* dst, int B, int64_t Ls, int H,
                                       int P, int d, int esize, cudaStream_t s, int* launches);

// Peer transport kernels (peer.cu).
// push: every rank's shard tensors -> owners' windows, then arr[T][rank] += 1 at each owner.
// `ctas` = grid size (0: one CTA per SM).
cudaError_t launch_peer_push(const PeerPush& pp, cudaStream_t s, int* launches, int ctas = 0);
// recv_o: wait done[s] >= epoch for all s, then copy the O window [B][Ls][H][d] to o
// (rows of global token >= L zeroed: shard padding).
cudaError_t launch_peer_recv_o(PeerCounters* own, uint32_t epoch, int P, const void* owin, void* o,
                               int B, int64_t Ls, int64_t L, int rank, int row_bytes,
                               cudaStream_t s, int* launches);
// ref_store: wait arr[1..2][s] >= epoch for all s, copy K/V windows ([B][Lw][Hl][d], rows
// < Lr) into the cache reference region ([B][Lr][Hl][d]), then done[rank] += 1 at every peer.
cudaError_t launch_peer_ref_store(PeerCounters* const* ctr, PeerCounters* own, uint32_t epoch,
                                  int P, int rank, const void* kwin, const void* vwin, void* kref,
                                  void* vref, int B, int64_t Lw, int64_t Lr, int row_bytes,
                                  cudaStream_t s, int* launches);
// wait: done[s] >= epoch for all s (a barrier after ref_store).
cudaError_t launch_peer_wait_done(PeerCounters* own, uint32_t epoch, int P, cudaStream_t s,
                                  int* launches);

}  // namespace tmk
