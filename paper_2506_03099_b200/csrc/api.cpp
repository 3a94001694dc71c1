// api.cpp -- the C ABI of include/tm.h: config validation, the constant-
// memory KV cache (rows a1, a3), ordering state, the mask -> segment
// schedule (row a4), the Ulysses exchange (rows a2, a6) and dispatch to the
// sm_100a kernels (rows a5, a7).
//
// PAPER.md: P:137-151 (Sec 4.2 sparse causal attention, Eq 7), P:187 (KV
// cache of c_0 and c_{t-1} per timestep per block), P:171 (sequence
// parallelism), P:55-66 (flow matching, Eqs 1-2).  SPEC.md errors:
// S:39 (dimension / degenerate mask), S:287 (reference rewrite)
// (cache miss / order).
#include "../../include/tm.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "comm.h"
#include "internal.h"
#include "peer_map.h"
#include "ulysses_map.h"

using namespace tmk;

namespace {

thread_local std::string g_err;

// NVTX range around each public call (header-only NVTX v3: no cost without a
// profiler attached; ncu --nvtx / nsys show the tm_* calls on the timeline).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

tm_status fail(tm_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

constexpr size_t kAlign = 1024;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

tm_status validate(const tm_config* c) {
    if (!c) return fail(TM_ERR_INVALID_ARG, "null config");
    if (c->dtype != TM_BF16 && c->dtype != TM_FP32)
        return fail(TM_ERR_INVALID_ARG, "dtype %d not in {TM_BF16, TM_FP32}", c->dtype);
    if (c->heads <= 0 || c->ref_tokens <= 0 || c->chunk_tokens <= 0 || c->num_layers <= 0 ||
        c->num_steps <= 0 || c->batch <= 0)
        return fail(TM_ERR_SHAPE, "non-positive dimension (H=%d Lr=%d Lc=%d layers=%d steps=%d B=%d)",
                    c->heads, c->ref_tokens, c->chunk_tokens, c->num_layers, c->num_steps,
                    c->batch);
    if (c->head_dim != 64 && c->head_dim != 128)
        return fail(TM_ERR_SHAPE, "head_dim %d not in {64, 128}", c->head_dim);
    if (c->world_size <= 0 || c->rank < 0 || c->rank >= c->world_size)
        return fail(TM_ERR_INVALID_ARG, "rank %d / world_size %d", c->rank, c->world_size);
    if (c->heads % c->world_size)
        return fail(TM_ERR_SHAPE, "heads %d not divisible by world_size %d (Ulysses head sharding)",
                    c->heads, c->world_size);
    if (!(c->softmax_scale >= 0.f) || !std::isfinite(c->softmax_scale))
        return fail(TM_ERR_INVALID_ARG, "softmax_scale must be finite and >= 0");
    if (c->transport != TM_TRANSPORT_NCCL && c->transport != TM_TRANSPORT_PEER)
        return fail(TM_ERR_INVALID_ARG, "transport %d not in {TM_TRANSPORT_NCCL, TM_TRANSPORT_PEER}",
                    c->transport);
    if (c->sched_heads < 0 || (c->sched_heads > 0 && (c->heads / c->world_size) % c->sched_heads))
        return fail(TM_ERR_SHAPE, "sched_heads %d must be 0 or divide the %d heads per rank",
                    c->sched_heads, c->heads / c->world_size);
    if (c->transport == TM_TRANSPORT_PEER) {
        if (c->dtype != TM_BF16)
            return fail(TM_ERR_UNSUPPORTED, "TM_TRANSPORT_PEER is bf16 only (the fp32 validation "
                                            "mode uses the NCCL transport)");
        if (c->world_size > kMaxPeers)
            return fail(TM_ERR_UNSUPPORTED, "TM_TRANSPORT_PEER needs world_size <= %d", kMaxPeers);
    }
    return TM_OK;
}

// TM_FORCE_ULYSSES=1 (debug/test): a world_size == 1 context runs the full
// Ulysses exchange path (pack, 1-rank ncclAlltoAll, unpack) so the NCCL
// integration and the pack/unpack kernels can be checked on one GPU.
bool force_ulysses() {
    const char* e = getenv("TM_FORCE_ULYSSES");
    return e && *e && strcmp(e, "0") != 0;
}

struct Layout {
    bool exchange;                   // NCCL Ulysses path (P > 1, or forced)
    bool peer;                       // peer-memory Ulysses path (TM_TRANSPORT_PEER, any P)
    int64_t Lw;                      // peer window rows max(Lc, Lr)
    size_t win_off, win_bytes, win_tensor_bytes, win_o_bytes;
    int esize, Hl, P;
    int64_t Lr, Lc, Lr_s, Lc_s;     // full and per-rank shard token counts
    size_t ref_bytes, slot_bytes, region_bytes, cache_bytes;
    size_t flag_bytes, scratch_bytes, xfer_bytes, head_bytes, osend_bytes, ws_bytes;
};

Layout layout_of(const tm_config* c) {
    Layout L{};
    L.esize = c->dtype == TM_BF16 ? 2 : 4;
    L.P = c->world_size;
    L.Hl = c->heads / c->world_size;
    L.Lr = c->ref_tokens;
    L.Lc = c->chunk_tokens;
    L.Lr_s = ceil_div(L.Lr, L.P);
    L.Lc_s = ceil_div(L.Lc, L.P);
    const size_t row = size_t(L.Hl) * c->head_dim * L.esize;     // one token, local heads
    L.ref_bytes = align_up(size_t(c->batch) * L.Lr * row);
    L.slot_bytes = align_up(size_t(c->batch) * L.Lc * row);
    L.region_bytes = 2 * L.ref_bytes + 4 * L.slot_bytes;          // Kref Vref K0 V0 K1 V1
    L.cache_bytes = L.region_bytes * size_t(c->num_layers) * size_t(c->num_steps);
    L.flag_bytes = kAlign;
    L.scratch_bytes = c->dtype == TM_BF16 ? align_up(fmha_sm100_scratch_bytes(c->head_dim)) : 0;
    L.peer = c->transport == TM_TRANSPORT_PEER;
    L.exchange = !L.peer && (L.P > 1 || force_ulysses());
    if (L.peer) {
        L.Lw = std::max(L.Lc, L.Lr);
        L.win_tensor_bytes = align_up(size_t(c->batch) * L.Lw * row);
        L.win_o_bytes = align_up(size_t(c->batch) * L.Lc_s * size_t(c->heads) * c->head_dim * L.esize);
        L.win_off = L.flag_bytes + L.scratch_bytes;
        L.win_bytes = 4096 + 3 * L.win_tensor_bytes + L.win_o_bytes;
        L.ws_bytes = L.win_off + L.win_bytes;
    } else if (L.exchange) {
        const size_t full_row = size_t(c->heads) * c->head_dim * L.esize;
        const size_t qkv = 3 * align_up(size_t(c->batch) * L.Lc_s * full_row);
        const size_t kv = 2 * align_up(size_t(c->batch) * L.Lr_s * full_row);
        L.xfer_bytes = qkv > kv ? qkv : kv;
        L.head_bytes = L.slot_bytes;                               // Q or O, [B][Lc][Hl][d]
        // O's send blocks [P][B][Lc/P][Hl][d] have their own region: in a
        // loopback group (tm_nccl_connect_local) the other ranks may still read
        // this rank's Q/K/V send blocks after it has packed O.
        L.osend_bytes = align_up(size_t(c->batch) * L.Lc_s * full_row);
        L.ws_bytes = L.flag_bytes + L.scratch_bytes + 2 * L.xfer_bytes + 2 * L.head_bytes +
                     L.osend_bytes;
    } else {
        L.ws_bytes = L.flag_bytes + L.scratch_bytes;
    }
    return L;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Selects device `dev` for the scope of one public call and restores the
// caller's device on exit (a process may drive several GPUs through several
// contexts; the caller's current device is never changed by a tm_* call).
struct DeviceScope {
    int prev = -1;
    bool ok = true;
    explicit DeviceScope(int dev) {
        if (dev < 0) return;
        if (cudaGetDevice(&prev) != cudaSuccess) {
            prev = -1;
            ok = false;
            return;
        }
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
        else prev = -1;                  // nothing to restore
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

struct tm_ctx {
    tm_config cfg;
    Layout lay;
    uint8_t* cache;
    uint8_t* ws;
    float scale;
    std::vector<int64_t> last;        // [layer][step]: last chunk attended (0 = none)
    std::vector<uint8_t> ref_ok;      // [layer][step]: reference written
    void* comm = nullptr;
    bool lb_pending = false;           // NCCL transport, world > 1, no unique id: loopback group
    int launches = 0;
    bool debug = false;
    // peer transport
    bool connected = false;
    uint8_t* win[kMaxPeers] = {};      // every rank's window, mapped in this process
    std::vector<void*> ipc_opened;     // cudaIpcOpenMemHandle bases to close
    uint32_t e_arr[3] = {0, 0, 0};     // arrivals expected per source (Q, K, V)
    uint32_t e_done = 0;               // done signals expected per source
    // phased operation in flight: kind 0 none, 1 chunk, 2 reference
    int op_kind = 0;
    uint32_t op_done = 0;
    int op_layer = 0, op_step = 0;
    int64_t op_chunk = 0;
    const void* op_ptr[4] = {};
    unsigned long long* trace = nullptr;   // TM_TRACE=<file>: kernel timeline of CTA 0
    std::string trace_path;

    size_t idx(int layer, int step) const { return size_t(layer) * cfg.num_steps + step; }
    uint8_t* region(int layer, int step) const { return cache + idx(layer, step) * lay.region_bytes; }
    uint8_t* kref(int l, int s) const { return region(l, s); }
    uint8_t* vref(int l, int s) const { return region(l, s) + lay.ref_bytes; }
    uint8_t* kslot(int l, int s, int64_t t) const {
        return region(l, s) + 2 * lay.ref_bytes + (t & 1) * 2 * lay.slot_bytes;
    }
    uint8_t* vslot(int l, int s, int64_t t) const { return kslot(l, s, t) + lay.slot_bytes; }
    int* flag() const { return reinterpret_cast<int*>(ws); }
    uint8_t* scratch() const { return ws + lay.flag_bytes; }
    uint8_t* send() const { return scratch() + lay.scratch_bytes; }
    uint8_t* recv() const { return send() + lay.xfer_bytes; }
    uint8_t* qh() const { return recv() + lay.xfer_bytes; }
    uint8_t* oh() const { return qh() + lay.head_bytes; }
    uint8_t* osend() const { return oh() + lay.head_bytes; }
    // NCCL transport without a communicator: a loopback group of contexts in
    // one process (tm_nccl_connect_local), all-to-all = device copies.
    std::vector<tm_ctx*> lb_group;
    // peer window of rank r (own: r == cfg.rank)
    PeerCounters* ctr(int r) const { return reinterpret_cast<PeerCounters*>(win[r]); }
    uint8_t* wq(int r) const { return win[r] + 4096; }
    uint8_t* wk(int r) const { return wq(r) + lay.win_tensor_bytes; }
    uint8_t* wv(int r) const { return wk(r) + lay.win_tensor_bytes; }
    uint8_t* wo(int r) const { return wv(r) + lay.win_tensor_bytes; }
};

namespace {

tm_status cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return TM_OK;
    return fail(TM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

tm_status debug_check(tm_ctx* c, const void* x, int64_t n, int is_bf16, cudaStream_t s,
                      const char* what) {
    if (!c->debug) return TM_OK;
    tm_status st = cuda_check(cudaMemsetAsync(c->flag(), 0, sizeof(int), s), "debug memset");
    if (st) return st;
    st = cuda_check(launch_nonfinite(x, is_bf16, n, c->flag(), s, nullptr), "nonfinite check");
    if (st) return st;
    int h = 0;
    st = cuda_check(cudaMemcpyAsync(&h, c->flag(), sizeof(int), cudaMemcpyDeviceToHost, s),
                    "debug readback");
    if (st) return st;
    st = cuda_check(cudaStreamSynchronize(s), "debug sync");
    if (st) return st;
    if (h) return fail(TM_ERR_NONFINITE, "%s produced NaN/Inf (TM_DEBUG)", what);
    return TM_OK;
}

tm_status check_layer_step(const tm_ctx* c, int32_t layer, int32_t step, bool allow_all) {
    if (layer < 0 || layer >= c->cfg.num_layers)
        return fail(TM_ERR_INVALID_ARG, "layer %d outside [0, %d)", layer, c->cfg.num_layers);
    if (step == -1 && allow_all) return TM_OK;
    if (step < 0 || step >= c->cfg.num_steps)
        return fail(TM_ERR_INVALID_ARG, "step %d outside [0, %d)", step, c->cfg.num_steps);
    return TM_OK;
}

// The all-to-all of the NCCL transport: block p of `send` (bytes each) goes
// to rank p, block q of `recv` comes from rank q.  With a communicator:
// ncclAlltoAll.  In a loopback group (tm_nccl_connect_local; ranks of one
// process, e.g. virtual ranks on one device for tests) the same permutation
// is done with device copies from the other ranks' send regions: the group
// shares one stream and every rank's pack precedes any rank's exchange
// (the phased calls, TM_PHASE_*), so the copies see the packed blocks.
tm_status exchange_a2a(tm_ctx* c, const uint8_t* send, uint8_t* recv, size_t bytes, cudaStream_t s,
                       const char* what) {
    const int P = c->lay.P;
    if (c->comm) {
        const char* e = comm_alltoall(c->comm, send, recv, bytes, P, s);
        return e ? fail(TM_ERR_NCCL, "all-to-all (%s): %s", what, e) : TM_OK;
    }
    if (int(c->lb_group.size()) != P)
        return fail(TM_ERR_STREAM_ORDER, "NCCL transport without a communicator: connect the "
                                         "loopback group first (tm_nccl_connect_local)");
    const size_t off = size_t(send - c->ws);
    const int r = c->cfg.rank;
    for (int q = 0; q < P; ++q) {
        const uint8_t* src = c->lb_group[q]->ws + off + size_t(r) * bytes;
        tm_status st = cuda_check(cudaMemcpyAsync(recv + size_t(q) * bytes, src, bytes,
                                                  cudaMemcpyDeviceToDevice, s),
                                  "loopback all-to-all copy");
        if (st) return st;
    }
    return TM_OK;
}

// An NCCL-transport context can exchange: a communicator, or a connected
// loopback group.  Checked before any launch (host error, no side effects).
tm_status exchange_ready(const tm_ctx* c) {
    if (!c->lay.exchange || c->comm || int(c->lb_group.size()) == c->lay.P) return TM_OK;
    return fail(TM_ERR_STREAM_ORDER, "NCCL transport without a communicator: connect the loopback "
                                     "group first (tm_nccl_connect_local)");
}

// Ulysses seq -> head exchange of `ntensors` tensors of [B][Ls][H][d] each
// (P:171), in two halves: pack into the per-peer send blocks, then exchange
// and unpack the received blocks to dst[i] ([B][L][Hl][d]).
size_t xfer_block(const tm_ctx* c, int64_t Ls) {
    return align_up(size_t(c->cfg.batch) * Ls * c->cfg.heads * c->cfg.head_dim * c->lay.esize);
}

tm_status ulysses_pack_in(tm_ctx* c, int ntensors, const void* const* src, int64_t Ls,
                          cudaStream_t s) {
    const Layout& Ly = c->lay;
    const int d = c->cfg.head_dim, B = c->cfg.batch, H = c->cfg.heads;
    const size_t blk = xfer_block(c, Ls);
    for (int i = 0; i < ntensors; ++i) {
        tm_status st = cuda_check(launch_pack_seq_to_peers(src[i], c->send() + i * blk, B, Ls, H,
                                                           Ly.P, d, Ly.esize, s, &c->launches),
                                  "pack seq->peers");
        if (st) return st;
    }
    return TM_OK;
}

tm_status ulysses_exchange_in(tm_ctx* c, int ntensors, void* const* dst, int64_t Ls, int64_t L,
                              cudaStream_t s) {
    const Layout& Ly = c->lay;
    const int d = c->cfg.head_dim, B = c->cfg.batch;
    const size_t blk = xfer_block(c, Ls);
    const size_t per_peer = size_t(B) * Ls * Ly.Hl * d * Ly.esize;
    for (int i = 0; i < ntensors; ++i) {
        tm_status st = exchange_a2a(c, c->send() + i * blk, c->recv() + i * blk, per_peer, s,
                                    "seq->head");
        if (st) return st;
    }
    for (int i = 0; i < ntensors; ++i) {
        tm_status st = cuda_check(launch_unpack_peers_to_heads(c->recv() + i * blk, dst[i], B, Ls,
                                                               L, Ly.Hl, Ly.P, d, Ly.esize, s,
                                                               &c->launches),
                                  "unpack peers->heads");
        if (st) return st;
    }
    return TM_OK;
}

// ------------------------------------------------------------ peer transport

bool peer_separate_push() {   // A/B and debugging: push in its own kernel, not fused
    const char* e = getenv("TM_PEER_SEPARATE_PUSH");
    return e && *e && strcmp(e, "0") != 0;
}

// The push of this rank's sequence shard(s) [B][Ls][H][d] into the owners' windows.
PeerPush make_push(const tm_ctx* c, const void* q, const void* k, const void* v, int64_t Ls,
                   int64_t L) {
    const Layout& Ly = c->lay;
    PeerPush pp;
    pp.src[0] = q;
    pp.src[1] = k;
    pp.src[2] = v;
    for (int p = 0; p < Ly.P; ++p) {
        pp.dst[0][p] = c->wq(p);
        pp.dst[1][p] = c->wk(p);
        pp.dst[2][p] = c->wv(p);
        pp.ctr[p] = c->ctr(p);
    }
    pp.own = c->ctr(c->cfg.rank);
    pp.B = c->cfg.batch;
    pp.P = Ly.P;
    pp.rank = c->cfg.rank;
    pp.W = Ly.Hl * c->cfg.head_dim * Ly.esize / 16;
    pp.Ls = Ls;
    pp.L = L;
    pp.Lw = Ly.Lw;
    return pp;
}

// Phase bookkeeping of one collective operation (see TM_PHASE_* in tm.h).
tm_status begin_phases(tm_ctx* c, int kind, uint32_t phases, int layer, int step, int64_t chunk,
                       const void* a0, const void* a1, const void* a2, const void* a3, bool* first) {
    if (phases == 0 || phases > TM_PHASE_ALL || phases == (TM_PHASE_SEND | TM_PHASE_RECV))
        return fail(TM_ERR_INVALID_ARG, "phases 0x%x: a non-empty run of SEND, ATTEND, RECV", phases);
    if (!c->lay.peer && phases != TM_PHASE_ALL && !(c->lay.exchange && c->lb_pending))
        return fail(TM_ERR_UNSUPPORTED, "phased calls need TM_TRANSPORT_PEER or a loopback "
                                        "NCCL-transport group (tm_nccl_connect_local)");
    const uint32_t lowest = phases & (~phases + 1);
    if (c->op_kind == 0) {
        if (lowest != TM_PHASE_SEND)
            return fail(TM_ERR_STREAM_ORDER, "an operation starts with TM_PHASE_SEND");
        *first = true;
        return TM_OK;
    }
    const void* a[4] = {a0, a1, a2, a3};
    bool same = c->op_kind == kind && c->op_layer == layer && c->op_step == step &&
                c->op_chunk == chunk;
    for (int i = 0; i < 4; ++i) same = same && a[i] == c->op_ptr[i];
    if (!same)
        return fail(TM_ERR_STREAM_ORDER, "a phased operation is in flight: finish it (same "
                                         "arguments) before starting another");
    if (lowest != c->op_done + 1)
        return fail(TM_ERR_STREAM_ORDER, "phase 0x%x out of order (done 0x%x)", phases, c->op_done);
    *first = false;
    return TM_OK;
}

void note_phases(tm_ctx* c, int kind, uint32_t phases, int layer, int step, int64_t chunk,
                 const void* a0, const void* a1, const void* a2, const void* a3) {
    if (c->op_kind == 0) {
        c->op_kind = kind;
        c->op_layer = layer;
        c->op_step = step;
        c->op_chunk = chunk;
        c->op_ptr[0] = a0;
        c->op_ptr[1] = a1;
        c->op_ptr[2] = a2;
        c->op_ptr[3] = a3;
        c->op_done = 0;
    }
    c->op_done |= phases;
    if (c->op_done == TM_PHASE_ALL) {
        c->op_kind = 0;
        c->op_done = 0;
    }
}

using PFN_getAddressRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

PFN_getAddressRange address_range_fn() {
    static PFN_getAddressRange fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return PFN_getAddressRange(nullptr);
        return reinterpret_cast<PFN_getAddressRange>(f);
    }();
    return fn;
}

}  // namespace

extern "C" {

int32_t tm_version(void) { return 102; }

const char* tm_last_error(void) { return g_err.c_str(); }

size_t tm_kvcache_bytes(const tm_config* cfg) {
    if (validate(cfg) != TM_OK) return 0;
    return layout_of(cfg).cache_bytes;
}

size_t tm_workspace_bytes(const tm_config* cfg) {
    if (validate(cfg) != TM_OK) return 0;
    return layout_of(cfg).ws_bytes;
}

tm_status tm_get_unique_id(uint8_t id[128]) {
    if (!id) return fail(TM_ERR_INVALID_ARG, "null id");
    const char* e = comm_unique_id(id);
    return e ? fail(TM_ERR_NCCL, "%s", e) : TM_OK;
}

tm_status tm_attn_init(const tm_config* cfg, const uint8_t* nccl_id, void* cache,
                       size_t cache_bytes, void* workspace, size_t workspace_bytes, tm_ctx** out) {
    tm_status st = validate(cfg);
    if (st) return st;
    if (!out) return fail(TM_ERR_INVALID_ARG, "null out");
    *out = nullptr;
    const Layout L = layout_of(cfg);
    if (!cache || cache_bytes < L.cache_bytes)
        return fail(TM_ERR_INVALID_ARG, "cache buffer %zu bytes < required %zu", cache_bytes,
                    L.cache_bytes);
    if (reinterpret_cast<uintptr_t>(cache) % kAlign)
        return fail(TM_ERR_INVALID_ARG, "cache must be %zu-byte aligned", kAlign);
    if (!workspace || workspace_bytes < L.ws_bytes)
        return fail(TM_ERR_INVALID_ARG, "workspace %zu bytes < required %zu", workspace_bytes,
                    L.ws_bytes);
    if (reinterpret_cast<uintptr_t>(workspace) % 256)
        return fail(TM_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
    uint8_t local_id[128];
    if (L.exchange && cfg->world_size == 1 && !nccl_id) {   // forced 1-rank exchange
        const char* e = comm_unique_id(local_id);
        if (e) return fail(TM_ERR_NCCL, "%s", e);
        nccl_id = local_id;
    }
    // world_size > 1 without an id: a loopback group, connected later with
    // tm_nccl_connect_local (test / single-process use)
    const bool lb_pending = L.exchange && !nccl_id;
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return fail(TM_ERR_CUDA, "no CUDA device");
    DeviceScope dev_scope(cfg->device);  // restored on every return path
    if (!dev_scope.ok) return fail(TM_ERR_CUDA, "cannot select device %d", cfg->device);
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cfg->device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, cfg->device);
    if (major != 10 || minor != 0)
        return fail(TM_ERR_UNSUPPORTED, "device %d is sm_%d%d; libtm is built for sm_100a only",
                    cfg->device, major, minor);
    tm_ctx* c = new tm_ctx();
    c->cfg = *cfg;
    c->lay = L;
    c->cache = static_cast<uint8_t*>(cache);
    c->ws = static_cast<uint8_t*>(workspace);
    c->scale = cfg->softmax_scale > 0.f ? cfg->softmax_scale : 1.0f / std::sqrt(float(cfg->head_dim));
    c->last.assign(size_t(cfg->num_layers) * cfg->num_steps, 0);
    c->ref_ok.assign(size_t(cfg->num_layers) * cfg->num_steps, 0);
    // The split-KV scratch (merge counters) must start zeroed; kernels leave it zeroed.
    if (cudaMemset(c->ws, 0, L.ws_bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        delete c;
        return fail(TM_ERR_CUDA, "workspace initialisation failed");
    }
    const char* dbg = getenv("TM_DEBUG");
    c->debug = dbg && *dbg && strcmp(dbg, "0") != 0;
    if (const char* tp = getenv("TM_TRACE")) {
        if (*tp && cudaMalloc(&c->trace, kTraceWords * 8) == cudaSuccess) c->trace_path = tp;
    }
    if (L.peer) {
        c->win[cfg->rank] = c->ws + L.win_off;
        c->connected = L.P == 1;       // a one-rank group is its own peer
    }
    c->lb_pending = lb_pending;
    if (L.exchange && !lb_pending) {
        const char* e = comm_init(&c->comm, cfg->world_size, cfg->rank, nccl_id);
        if (e) {
            delete c;
            return fail(TM_ERR_NCCL, "ncclCommInitRank: %s", e);
        }
    }
    *out = c;
    return TM_OK;
}

tm_status tm_attn_destroy(tm_ctx* ctx) {
    if (!ctx) return fail(TM_ERR_INVALID_ARG, "null ctx");
    DeviceScope dev_scope(ctx->cfg.device);
    if (ctx->comm) comm_destroy(ctx->comm);
    for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
    if (ctx->trace) cudaFree(ctx->trace);
    delete ctx;
    return TM_OK;
}

tm_status tm_stream_reset(tm_ctx* ctx) {
    if (!ctx) return fail(TM_ERR_INVALID_ARG, "null ctx");
    std::fill(ctx->last.begin(), ctx->last.end(), 0);
    std::fill(ctx->ref_ok.begin(), ctx->ref_ok.end(), 0);
    return TM_OK;
}

tm_status tm_kvcache_ref_ptr(tm_ctx* ctx, int32_t layer, int32_t step, void** k, void** v) {
    if (!ctx || !k || !v) return fail(TM_ERR_INVALID_ARG, "null argument");
    tm_status st = check_layer_step(ctx, layer, step, false);
    if (st) return st;
    *k = ctx->kref(layer, step);
    *v = ctx->vref(layer, step);
    return TM_OK;
}

tm_status tm_kvcache_slot_ptr(tm_ctx* ctx, int32_t layer, int32_t step, int64_t chunk, void** k,
                              void** v) {
    if (!ctx || !k || !v) return fail(TM_ERR_INVALID_ARG, "null argument");
    tm_status st = check_layer_step(ctx, layer, step, false);
    if (st) return st;
    if (chunk < 1) return fail(TM_ERR_INVALID_ARG, "chunk %lld < 1", (long long)chunk);
    *k = ctx->kslot(layer, step, chunk);
    *v = ctx->vslot(layer, step, chunk);
    return TM_OK;
}

tm_status tm_kvcache_put_reference(tm_ctx* ctx, int32_t layer, int32_t step, const void* k,
                                   const void* v, void* stream) {
    return tm_kvcache_put_reference_phases(ctx, layer, step, k, v, TM_PHASE_ALL, stream);
}

tm_status tm_kvcache_put_reference_phases(tm_ctx* ctx, int32_t layer, int32_t step, const void* k,
                                          const void* v, uint32_t phases, void* stream) {
    NvtxRange nvtx_range("tm_kvcache_put_reference_phases");
    if (!ctx || !k || !v) return fail(TM_ERR_INVALID_ARG, "null argument");
    DeviceScope dev_scope(ctx->cfg.device);
    tm_status st = check_layer_step(ctx, layer, step, true);
    if (st) return st;
    st = exchange_ready(ctx);
    if (st) return st;
    bool first = false;
    st = begin_phases(ctx, 2, phases, layer, step, 0, k, v, nullptr, nullptr, &first);
    if (st) return st;
    const int s0 = step < 0 ? 0 : step, s1 = step < 0 ? ctx->cfg.num_steps : step + 1;
    if (first)
        for (int s = s0; s < s1; ++s)
            if (ctx->last[ctx->idx(layer, s)] >= 1)
                return fail(TM_ERR_REF_IMMUTABLE,
                            "reference of (layer %d, step %d) is immutable after chunk 1 until "
                            "tm_stream_reset (S:287)", layer, s);
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    const Layout& Ly = ctx->lay;
    ctx->launches = 0;
    if (Ly.peer) {
        // a1 over peer memory: push the reference shard into the owners' K/V
        // windows, copy the received window into the cache, then a barrier.
        if (!ctx->connected) return fail(TM_ERR_STREAM_ORDER, "peer group not connected (tm_peer_connect)");
        const int r = ctx->cfg.rank;
        const int row_bytes = Ly.Hl * ctx->cfg.head_dim * Ly.esize;
        if (phases & TM_PHASE_SEND) {
            const PeerPush pp = make_push(ctx, nullptr, k, v, Ly.Lr_s, Ly.Lr);
            st = cuda_check(launch_peer_push(pp, cs, &ctx->launches), "peer push (reference)");
            if (st) return st;
            ++ctx->e_arr[1];
            ++ctx->e_arr[2];
        }
        if (phases & TM_PHASE_ATTEND) {
            PeerCounters* ctrs[kMaxPeers];
            for (int p = 0; p < Ly.P; ++p) ctrs[p] = ctx->ctr(p);
            ++ctx->e_done;
            st = cuda_check(launch_peer_ref_store(ctrs, ctx->ctr(r), ctx->e_arr[1], Ly.P, r, ctx->wk(r),
                                                  ctx->wv(r), ctx->kref(layer, s0), ctx->vref(layer, s0),
                                                  ctx->cfg.batch, Ly.Lw, Ly.Lr, row_bytes, cs,
                                                  &ctx->launches),
                            "peer reference store");
            if (st) return st;
            for (int s = s0 + 1; s < s1; ++s) {
                st = cuda_check(cudaMemcpyAsync(ctx->kref(layer, s), ctx->kref(layer, s0),
                                                2 * Ly.ref_bytes, cudaMemcpyDeviceToDevice, cs),
                                "reference alias copy");
                if (st) return st;
            }
        }
        if (phases & TM_PHASE_RECV) {
            st = cuda_check(launch_peer_wait_done(ctx->ctr(r), ctx->e_done, Ly.P, cs, &ctx->launches),
                            "peer barrier");
            if (st) return st;
        }
        note_phases(ctx, 2, phases, layer, step, 0, k, v, nullptr, nullptr);
        if (phases & TM_PHASE_RECV)
            for (int s = s0; s < s1; ++s) ctx->ref_ok[ctx->idx(layer, s)] = 1;
        return TM_OK;
    }
    if (!Ly.exchange) {
        note_phases(ctx, 2, phases, layer, step, 0, k, v, nullptr, nullptr);
        const size_t bytes = size_t(ctx->cfg.batch) * Ly.Lr * Ly.Hl * ctx->cfg.head_dim * Ly.esize;
        for (int s = s0; s < s1; ++s) {
            st = cuda_check(cudaMemcpyAsync(ctx->kref(layer, s), k, bytes, cudaMemcpyDeviceToDevice, cs),
                            "reference K copy");
            if (!st) st = cuda_check(cudaMemcpyAsync(ctx->vref(layer, s), v, bytes,
                                                     cudaMemcpyDeviceToDevice, cs),
                                     "reference V copy");
            if (st) return st;
        }
    } else {
        // NCCL transport: SEND packs the shard, ATTEND exchanges and unpacks
        // into the cache's reference region (RECV has nothing left to do).
        if (phases & TM_PHASE_SEND) {
            const void* src[2] = {k, v};
            st = ulysses_pack_in(ctx, 2, src, Ly.Lr_s, cs);
            if (st) return st;
        }
        if (phases & TM_PHASE_ATTEND) {
            void* dst[2] = {ctx->kref(layer, s0), ctx->vref(layer, s0)};
            st = ulysses_exchange_in(ctx, 2, dst, Ly.Lr_s, Ly.Lr, cs);
            if (st) return st;
            for (int s = s0 + 1; s < s1; ++s) {
                st = cuda_check(cudaMemcpyAsync(ctx->kref(layer, s), ctx->kref(layer, s0),
                                                2 * Ly.ref_bytes, cudaMemcpyDeviceToDevice, cs),
                                "reference alias copy");
                if (st) return st;
            }
        }
        note_phases(ctx, 2, phases, layer, step, 0, k, v, nullptr, nullptr);
        if (!(phases & TM_PHASE_RECV)) return TM_OK;
    }
    for (int s = s0; s < s1; ++s) ctx->ref_ok[ctx->idx(layer, s)] = 1;
    return TM_OK;
}

// Debug builds (TM_TRACE=<file>): append the launch's trace words to the file
// (synchronises).  No-op otherwise.
static void dump_trace(tm_ctx* ctx, cudaStream_t cs) {
    if (!ctx->trace) return;
    std::vector<unsigned long long> h(kTraceWords);
    cudaMemcpyAsync(h.data(), ctx->trace, h.size() * 8, cudaMemcpyDeviceToHost, cs);
    cudaStreamSynchronize(cs);
    if (FILE* f = fopen(ctx->trace_path.c_str(), "ab")) {
        fwrite(h.data(), 8, h.size(), f);
        fclose(f);
    }
}

tm_status tm_chunk_attention(tm_ctx* ctx, int32_t layer, int32_t step, int64_t chunk,
                             const void* q, const void* k, const void* v, void* o, void* stream) {
    return tm_chunk_attention_phases(ctx, layer, step, chunk, q, k, v, o, TM_PHASE_ALL, stream);
}

tm_status tm_chunk_attention_phases(tm_ctx* ctx, int32_t layer, int32_t step, int64_t chunk,
                                    const void* q, const void* k, const void* v, void* o,
                                    uint32_t phases, void* stream) {
    NvtxRange nvtx_range("tm_chunk_attention_phases");
    if (!ctx || !q || !k || !v || !o) return fail(TM_ERR_INVALID_ARG, "null argument");
    DeviceScope dev_scope(ctx->cfg.device);
    tm_status st = check_layer_step(ctx, layer, step, false);
    if (st) return st;
    if (chunk < 1) return fail(TM_ERR_INVALID_ARG, "chunk %lld < 1 (the reference is chunk 0)",
                               (long long)chunk);
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
        return fail(TM_ERR_INVALID_ARG, "q, k, v, o must be 16-byte aligned");
    st = exchange_ready(ctx);
    if (st) return st;
    bool first = false;
    st = begin_phases(ctx, 1, phases, layer, step, chunk, q, k, v, o, &first);
    if (st) return st;
    const size_t li = ctx->idx(layer, step);
    if (first) {
        if (!ctx->ref_ok[li])
            return fail(TM_ERR_STREAM_ORDER, "cache miss: no reference for (layer %d, step %d) (S:296)",
                        layer, step);
        const int64_t last = ctx->last[li];
        if (chunk != last + 1 && chunk != last)
            return fail(TM_ERR_STREAM_ORDER,
                        "chunk %lld at (layer %d, step %d) out of order (last %lld; S:296)",
                        (long long)chunk, layer, step, (long long)last);
    }
    const tm_config& cf = ctx->cfg;
    const Layout& Ly = ctx->lay;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    ctx->launches = 0;
    if (Ly.peer) {
        if (!ctx->connected) return fail(TM_ERR_STREAM_ORDER, "peer group not connected (tm_peer_connect)");
        const int r = cf.rank;
        const bool fused = (phases & TM_PHASE_SEND) && (phases & TM_PHASE_ATTEND) && !peer_separate_push();
        const PeerPush pp = make_push(ctx, q, k, v, Ly.Lc_s, Ly.Lc);
        if (phases & TM_PHASE_SEND) {
            if (!fused) {
                st = cuda_check(launch_peer_push(pp, cs, &ctx->launches), "peer push");
                if (st) return st;
            }
            for (int T = 0; T < 3; ++T) ++ctx->e_arr[T];
        }
        if (phases & TM_PHASE_ATTEND) {
            // a2 + a3 + a4 + a5 + a6 in one kernel: Q and c_t's K/V come from this
            // rank's window (pushed by their sequence owners, fused when SEND is
            // part of this call), c_t is appended to slot chunk&1 from the smem
            // ring, and O rows are stored into their token owners' windows.
            AttnProblem pr;
            pr.q = ctx->wq(r);
            pr.q_bstride = Ly.Lw;
            pr.o = ctx->wo(r);
            pr.Lq = Ly.Lc;
            pr.B = cf.batch;
            pr.H = Ly.Hl;
            pr.d = cf.head_dim;
            pr.scale = ctx->scale;
            pr.sched_heads = ctx->cfg.sched_heads;
            pr.seg[pr.nseg++] = Segment{ctx->kref(layer, step), ctx->vref(layer, step), Ly.Lr};
            if (chunk >= 2)
                pr.seg[pr.nseg++] = Segment{ctx->kslot(layer, step, chunk - 1),
                                            ctx->vslot(layer, step, chunk - 1), Ly.Lc};
            pr.seg[pr.nseg++] = Segment{ctx->wk(r), ctx->wv(r), Ly.Lc, Ly.Lw};
            pr.store_k = ctx->kslot(layer, step, chunk);
            pr.store_v = ctx->vslot(layer, step, chunk);
            PeerAttnArgs pa;
            pa.own = ctx->ctr(r);
            for (int T = 0; T < 3; ++T) pa.epoch[T] = ctx->e_arr[T];
            pa.wait_seg = pr.nseg - 1;
            pa.src_rows = Ly.Lc_s;
            pa.push = fused;
            pa.pp = pp;
            for (int p = 0; p < Ly.P; ++p) {
                pa.o_dst[p] = ctx->wo(p);
                pa.done_ctr[p] = ctx->ctr(p);
            }
            pa.o_rows = Ly.Lc_s;
            pa.o_H = cf.heads;
            pa.o_h0 = r * Ly.Hl;
            pa.signal_done = true;
            pa.P = Ly.P;
            pa.rank = r;
            pr.peer = &pa;
            ++ctx->e_done;
            // zero-copy output with RECV in the same call: the kernel's last CTA
            // waits for every rank's rows itself; no receive kernel follows.
            if ((phases & TM_PHASE_RECV) && o == ctx->wo(r)) pa.wait_done = ctx->e_done;
            st = cuda_check(launch_fmha_sm100(pr, ctx->scratch(), cs, &ctx->launches),
                            "attention kernel launch (peer)");
            if (st) return st;
        }
        if ((phases & TM_PHASE_RECV) && (phases & TM_PHASE_ATTEND) && o == ctx->wo(r)) {
            // zero-copy output, waited for inside the attention kernel
        } else if ((phases & TM_PHASE_RECV) && o == ctx->wo(r)) {
            // zero-copy output (tm_peer_output_ptr): only wait for every rank's rows
            st = cuda_check(launch_peer_wait_done(ctx->ctr(r), ctx->e_done, Ly.P, cs, &ctx->launches),
                            "peer receive (zero-copy)");
            if (st) return st;
        } else if (phases & TM_PHASE_RECV) {
            st = cuda_check(launch_peer_recv_o(ctx->ctr(r), ctx->e_done, Ly.P, ctx->wo(r), o, cf.batch,
                                               Ly.Lc_s, Ly.Lc, r, cf.heads * cf.head_dim * Ly.esize,
                                               cs, &ctx->launches),
                            "peer receive");
            if (st) return st;
        }
        note_phases(ctx, 1, phases, layer, step, chunk, q, k, v, o);
        if (!(phases & TM_PHASE_RECV)) return TM_OK;
        ctx->last[li] = chunk;
        return debug_check(ctx, o, int64_t(cf.batch) * Ly.Lc_s * cf.heads * cf.head_dim, 1, cs,
                           "tm_chunk_attention");
    }
    note_phases(ctx, 1, phases, layer, step, chunk, q, k, v, o);

    void* kslot = ctx->kslot(layer, step, chunk);
    void* vslot = ctx->vslot(layer, step, chunk);
    const void* qattn = q;
    void* oattn = o;
    bool fused_append = false;
    if (!Ly.exchange) {
        // a3: append c_t's K/V into slot chunk&1 (skipped when the caller wrote them
        // there).  bf16: fused into the attention kernel (TMA store of the tiles it
        // loads); fp32 validation path: a device copy.
        if (cf.dtype == TM_BF16 && k != kslot && v != vslot) {
            fused_append = true;
        } else {
            const size_t bytes = size_t(cf.batch) * Ly.Lc * Ly.Hl * cf.head_dim * Ly.esize;
            if (k != kslot) {
                st = cuda_check(cudaMemcpyAsync(kslot, k, bytes, cudaMemcpyDeviceToDevice, cs), "K append");
                if (st) return st;
            }
            if (v != vslot) {
                st = cuda_check(cudaMemcpyAsync(vslot, v, bytes, cudaMemcpyDeviceToDevice, cs), "V append");
                if (st) return st;
            }
        }
    } else {
        // a2: seq -> head all-to-all; K/V land in the cache slot (a3), Q in
        // workspace.  Phases (loopback groups): SEND packs, ATTEND exchanges,
        // unpacks, attends and packs O, RECV exchanges O and unpacks it.
        if (phases & TM_PHASE_SEND) {
            const void* src[3] = {q, k, v};
            st = ulysses_pack_in(ctx, 3, src, Ly.Lc_s, cs);
            if (st) return st;
        }
        if (phases & TM_PHASE_ATTEND) {
            void* dst[3] = {ctx->qh(), kslot, vslot};
            st = ulysses_exchange_in(ctx, 3, dst, Ly.Lc_s, Ly.Lc, cs);
            if (st) return st;
        }
        qattn = ctx->qh();
        oattn = ctx->oh();
    }
    const bool attend = !Ly.exchange || (phases & TM_PHASE_ATTEND);

    // a4: mask {c_0, c_{t-1}, c_t} -> segment schedule.  c_{t-1} is
    // the other slot; at chunk 1 it coincides with c_0 and is not repeated
    // (set semantics).
    AttnProblem pr;
    pr.q = qattn;
    pr.o = oattn;
    pr.Lq = Ly.Lc;
    pr.B = cf.batch;
    pr.H = Ly.Hl;
    pr.d = cf.head_dim;
    pr.scale = ctx->scale;
    pr.sched_heads = ctx->cfg.sched_heads;
    pr.seg[pr.nseg++] = Segment{ctx->kref(layer, step), ctx->vref(layer, step), Ly.Lr};
    if (chunk >= 2)
        pr.seg[pr.nseg++] = Segment{ctx->kslot(layer, step, chunk - 1),
                                    ctx->vslot(layer, step, chunk - 1), Ly.Lc};
    if (fused_append) {
        pr.seg[pr.nseg++] = Segment{k, v, Ly.Lc};     // read c_t from the caller's buffers
        pr.store_k = kslot;                            // and append it to the cache slot
        pr.store_v = vslot;
    } else {
        pr.seg[pr.nseg++] = Segment{kslot, vslot, Ly.Lc};
    }

    if (attend) {
    if (ctx->trace) cudaMemsetAsync(ctx->trace, 0, kTraceWords * 8, cs);
    cudaError_t e = cf.dtype == TM_BF16 ? launch_fmha_sm100(pr, ctx->scratch(), cs, &ctx->launches, ctx->trace)
                                        : launch_fmha_fp32(pr, cs, &ctx->launches);
    st = cuda_check(e, "attention kernel launch");
    if (st) return st;
    }
    if (attend) dump_trace(ctx, cs);

    if (Ly.exchange) {
        // a6: head -> seq all-to-all of O (packed at the end of ATTEND into its
        // own send region, exchanged and unpacked in RECV).
        const size_t blk = size_t(cf.batch) * Ly.Lc_s * Ly.Hl * cf.head_dim * Ly.esize;
        if (phases & TM_PHASE_ATTEND) {
            st = cuda_check(launch_pack_heads_to_peers(ctx->oh(), ctx->osend(), cf.batch, Ly.Lc_s,
                                                       Ly.Lc, Ly.Hl, Ly.P, cf.head_dim, Ly.esize, cs,
                                                       &ctx->launches),
                            "pack heads->peers");
            if (st) return st;
        }
        if (!(phases & TM_PHASE_RECV)) return TM_OK;
        st = exchange_a2a(ctx, ctx->osend(), ctx->recv(), blk, cs, "head->seq");
        if (st) return st;
        st = cuda_check(launch_unpack_peers_to_seq(ctx->recv(), o, cf.batch, Ly.Lc_s, cf.heads, Ly.P,
                                                   cf.head_dim, Ly.esize, cs, &ctx->launches),
                        "unpack peers->seq");
        if (st) return st;
    }
    ctx->last[li] = chunk;
    const int64_t n_out = int64_t(cf.batch) * (Ly.exchange ? Ly.Lc_s : Ly.Lc) * cf.heads * cf.head_dim;
    return debug_check(ctx, o, n_out, cf.dtype == TM_BF16, cs, "tm_chunk_attention");
}

tm_status tm_reference_attention(tm_ctx* ctx, int32_t layer, int32_t step, const void* q,
                                 const void* k, const void* v, void* o, void* stream) {
    NvtxRange nvtx_range("tm_reference_attention");
    if (!ctx || !q || !k || !v || !o) return fail(TM_ERR_INVALID_ARG, "null argument");
    DeviceScope dev_scope(ctx->cfg.device);
    if (ctx->lay.exchange || ctx->lay.P > 1 || ctx->lay.peer)
        return fail(TM_ERR_UNSUPPORTED, "tm_reference_attention needs a world_size == 1 direct context");
    tm_status st = check_layer_step(ctx, layer, step, true);
    if (st) return st;
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
        return fail(TM_ERR_INVALID_ARG, "q, k, v, o must be 16-byte aligned");
    const int s0 = step < 0 ? 0 : step, s1 = step < 0 ? ctx->cfg.num_steps : step + 1;
    for (int s = s0; s < s1; ++s)
        if (ctx->last[ctx->idx(layer, s)] >= 1)
            return fail(TM_ERR_REF_IMMUTABLE,
                        "reference of (layer %d, step %d) is immutable after chunk 1 until "
                        "tm_stream_reset (S:287)", layer, s);
    const tm_config& cf = ctx->cfg;
    const Layout& Ly = ctx->lay;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    ctx->launches = 0;
    // c_0's queries attend c_0 only: one segment, and (bf16) the
    // kernel appends that segment's K/V into the reference region as it reads it.
    AttnProblem pr;
    pr.q = q;
    pr.o = o;
    pr.Lq = Ly.Lr;
    pr.B = cf.batch;
    pr.H = Ly.Hl;
    pr.d = cf.head_dim;
    pr.scale = ctx->scale;
    pr.sched_heads = ctx->cfg.sched_heads;
    pr.seg[pr.nseg++] = Segment{k, v, Ly.Lr};
    cudaError_t e;
    if (cf.dtype == TM_BF16) {
        pr.store_k = ctx->kref(layer, s0);
        pr.store_v = ctx->vref(layer, s0);
        e = launch_fmha_sm100(pr, ctx->scratch(), cs, &ctx->launches);
    } else {
        const size_t bytes = size_t(cf.batch) * Ly.Lr * Ly.Hl * cf.head_dim * Ly.esize;
        e = cudaMemcpyAsync(ctx->kref(layer, s0), k, bytes, cudaMemcpyDeviceToDevice, cs);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(ctx->vref(layer, s0), v, bytes, cudaMemcpyDeviceToDevice, cs);
        if (e == cudaSuccess) e = launch_fmha_fp32(pr, cs, &ctx->launches);
    }
    st = cuda_check(e, "reference attention launch");
    if (st) return st;
    for (int s = s0 + 1; s < s1; ++s) {
        st = cuda_check(cudaMemcpyAsync(ctx->kref(layer, s), ctx->kref(layer, s0), 2 * Ly.ref_bytes,
                                        cudaMemcpyDeviceToDevice, cs),
                        "reference alias copy");
        if (st) return st;
    }
    for (int s = s0; s < s1; ++s) ctx->ref_ok[ctx->idx(layer, s)] = 1;
    return debug_check(ctx, o, int64_t(cf.batch) * Ly.Lr * cf.heads * cf.head_dim,
                       cf.dtype == TM_BF16, cs, "tm_reference_attention");
}

tm_status tm_window_attention(tm_ctx* ctx, const void* q, const void* k, const void* v, void* o,
                              const int64_t* chunk_len, int32_t n_chunks, void* stream) {
    NvtxRange nvtx_range("tm_window_attention");
    if (!ctx || !q || !k || !v || !o || !chunk_len) return fail(TM_ERR_INVALID_ARG, "null argument");
    DeviceScope dev_scope(ctx->cfg.device);
    if (ctx->lay.exchange || ctx->lay.P > 1)
        return fail(TM_ERR_UNSUPPORTED, "tm_window_attention needs a world_size == 1 context");
    if (n_chunks <= 0) return fail(TM_ERR_SHAPE, "n_chunks = %d <= 0", n_chunks);
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
        return fail(TM_ERR_INVALID_ARG, "q, k, v, o must be 16-byte aligned");
    std::vector<int64_t> start(n_chunks + 1, 0);
    for (int c = 0; c < n_chunks; ++c) {
        if (chunk_len[c] <= 0)
            return fail(TM_ERR_DEGENERATE_MASK, "chunk %d is empty: its queries have no keys (S:39)", c);
        start[c + 1] = start[c] + chunk_len[c];
    }
    const tm_config& cf = ctx->cfg;
    const int64_t L = start[n_chunks];
    const size_t row = size_t(cf.heads) * cf.head_dim * ctx->lay.esize;     // one token
    const uint8_t* qb = static_cast<const uint8_t*>(q);
    const uint8_t* kb = static_cast<const uint8_t*>(k);
    const uint8_t* vb = static_cast<const uint8_t*>(v);
    uint8_t* ob = static_cast<uint8_t*>(o);
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    ctx->launches = 0;
    // a4 per query chunk c: key chunks {0, c-1, c} as a set (P:137-143, S:271:
    // chunk 0 attends itself only), each a token sub-range of the window.
    auto key_chunks = [](int c, int* kc) {
        int nk = 0;
        kc[nk++] = 0;
        if (c - 1 > 0) kc[nk++] = c - 1;
        if (c > 0) kc[nk++] = c;
        return nk;
    };
    if (cf.dtype == TM_BF16) {
        // bf16: the query chunks are problems of ONE launch (up to kMaxProblems
        // per launch; each chunk's units scheduled as in its own call).
        for (int c0 = 0; c0 < n_chunks; c0 += kMaxProblems) {
            MultiProblem mp;
            mp.q = q;
            mp.k = k;
            mp.v = v;
            mp.o = o;
            mp.q_rows = mp.kv_rows = mp.o_rows = L;
            mp.B = cf.batch;
            mp.H = cf.heads;
            mp.d = cf.head_dim;
            mp.scale = ctx->scale;
            mp.sched_heads = cf.sched_heads;
            mp.nprob = std::min<int>(kMaxProblems, n_chunks - c0);
            for (int i = 0; i < mp.nprob; ++i) {
                const int c = c0 + i;
                SubProblem& sp = mp.prob[i];
                sp.q_row0 = sp.o_row0 = start[c];
                sp.Lq = chunk_len[c];
                int kc[3];
                sp.nseg = key_chunks(c, kc);
                for (int j = 0; j < sp.nseg; ++j) {
                    sp.seg_row0[j] = start[kc[j]];
                    sp.seg_len[j] = chunk_len[kc[j]];
                }
            }
            tm_status st = cuda_check(launch_fmha_sm100_multi(mp, ctx->scratch(), cs, &ctx->launches, ctx->trace),
                                      "window attention launch");
            if (st) return st;
        }
        return debug_check(ctx, o, int64_t(cf.batch) * L * cf.heads * cf.head_dim, 1, cs,
                           "tm_window_attention");
    }
    for (int c = 0; c < n_chunks; ++c) {      // fp32 validation mode: one launch per chunk
        AttnProblem pr;
        pr.q = qb + start[c] * row;
        pr.o = ob + start[c] * row;
        pr.Lq = chunk_len[c];
        pr.q_bstride = L;
        pr.B = cf.batch;
        pr.H = cf.heads;
        pr.d = cf.head_dim;
        pr.scale = ctx->scale;
        int kc[3];
        const int nk = key_chunks(c, kc);
        for (int i = 0; i < nk; ++i)
            pr.seg[pr.nseg++] = Segment{kb + start[kc[i]] * row, vb + start[kc[i]] * row,
                                        chunk_len[kc[i]], L};
        const cudaError_t e = launch_fmha_fp32(pr, cs, &ctx->launches);
        tm_status st = cuda_check(e, "window attention launch");
        if (st) return st;
    }
    return debug_check(ctx, o, int64_t(cf.batch) * L * cf.heads * cf.head_dim, cf.dtype == TM_BF16,
                       cs, "tm_window_attention");
}

// Layout: the gathered face rows of q | O staging of the fp32 mode (the same
// size) | the inverse face map (bf16 mode; up to 49152 tokens per frame).
size_t tm_audio_scratch_bytes(const tm_ctx* ctx, int64_t frames, int64_t n_face) {
    if (!ctx || frames <= 0 || n_face <= 0) return 0;
    const size_t rows = size_t(ctx->cfg.batch) * frames * n_face;
    return 2 * align_up(rows * ctx->cfg.heads * ctx->cfg.head_dim * ctx->lay.esize) +
           align_up(size_t(49152) * 4);
}

tm_status tm_audio_cross_attention(tm_ctx* ctx, const void* q, const void* k_audio,
                                   const void* v_audio, void* o, int64_t frames,
                                   int64_t tokens_per_frame, int64_t audio_tokens_per_frame,
                                   const int32_t* face_ids, int64_t n_face, int32_t window,
                                   void* scratch, size_t scratch_bytes, void* stream) {
    NvtxRange nvtx_range("tm_audio_cross_attention");
    if (!ctx || !q || !k_audio || !v_audio || !o || !scratch)
        return fail(TM_ERR_INVALID_ARG, "null argument");
    DeviceScope dev_scope(ctx->cfg.device);
    if (ctx->lay.exchange || ctx->lay.P > 1)
        return fail(TM_ERR_UNSUPPORTED, "tm_audio_cross_attention needs a world_size == 1 context");
    if (frames <= 0 || tokens_per_frame <= 0 || audio_tokens_per_frame <= 0)
        return fail(TM_ERR_SHAPE, "non-positive frames / tokens");
    if (n_face <= 0 || !face_ids)
        return fail(TM_ERR_DEGENERATE_MASK, "empty face mask: no query attends the audio (S:124)");
    if (n_face > tokens_per_frame) return fail(TM_ERR_SHAPE, "more face tokens than frame tokens");
    if (ctx->cfg.dtype == TM_BF16 && tokens_per_frame > 49152)
        return fail(TM_ERR_UNSUPPORTED, "tokens_per_frame %lld > 49152 (face map in shared memory)",
                    (long long)tokens_per_frame);
    if (window <= 0 || window % 2 == 0) return fail(TM_ERR_INVALID_ARG, "window must be odd, got %d", window);
    if (window > kMaxSegments)
        return fail(TM_ERR_UNSUPPORTED, "window %d > %d: an edge window needs more segments",
                    window, kMaxSegments);
    if (scratch_bytes < tm_audio_scratch_bytes(ctx, frames, n_face))
        return fail(TM_ERR_INVALID_ARG, "scratch %zu bytes < tm_audio_scratch_bytes", scratch_bytes);
    if (!aligned16(q) || !aligned16(k_audio) || !aligned16(v_audio) || !aligned16(o) ||
        reinterpret_cast<uintptr_t>(scratch) % kAlign)
        return fail(TM_ERR_INVALID_ARG, "q, k, v, o 16-byte and scratch 1024-byte aligned required");
    const tm_config& cf = ctx->cfg;
    const int row = cf.heads * cf.head_dim * ctx->lay.esize;          // bytes per token
    const int64_t BF = int64_t(cf.batch) * frames;
    uint8_t* qf = static_cast<uint8_t*>(scratch);
    const size_t half = align_up(size_t(cf.batch) * frames * n_face * cf.heads * cf.head_dim * ctx->lay.esize);
    uint8_t* of = qf + half;                                          // 1024-B aligned
    int32_t* inv = reinterpret_cast<int32_t*>(qf + 2 * half);         // bf16: token -> face slot
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    ctx->launches = 0;
    const uint8_t* kb = static_cast<const uint8_t*>(k_audio);
    const uint8_t* vb = static_cast<const uint8_t*>(v_audio);
    // P:125 window of frame f, edges clamped by repetition, as runs
    // of consecutive frames = contiguous audio-token row ranges (<= W of them).
    auto window_runs = [&](int64_t f, int64_t* row0, int64_t* len) {
        int64_t win[kMaxSegments];
        for (int i = 0; i < window; ++i) {
            const int64_t g = f - window / 2 + i;
            win[i] = g < 0 ? 0 : (g > frames - 1 ? frames - 1 : g);
        }
        int n = 0, i = 0;
        while (i < window) {
            int j = i;
            while (j + 1 < window && win[j + 1] == win[j] + 1) ++j;
            row0[n] = win[i] * audio_tokens_per_frame;
            len[n] = (j - i + 1) * audio_tokens_per_frame;
            ++n;
            i = j + 1;
        }
        return n;
    };
    tm_status st;
    if (cf.dtype == TM_BF16) {
        // Two launches: (1) gather the face rows of q into scratch and write the
        // inverse face map; (2) every frame's face rows attend its audio window
        // as problems of ONE attention launch (up to kMaxProblems frames per
        // launch) whose epilogue writes each face row straight to its token row
        // of o, while its spare warp zeroes the non-face rows (they get no audio
        // update).
        static const int dbg_parts = [] {   // timing experiments only: 1 prep only, 2 attention only
            const char* e = getenv("TM_DBG_AUDIO_PART");
            return e ? atoi(e) : 0;
        }();
        if (dbg_parts != 2) {
            st = cuda_check(launch_audio_prep(q, qf, inv, face_ids, BF, tokens_per_frame, n_face, row, cs,
                                              &ctx->launches), "audio prep (face gather, face map)");
            if (st) return st;
        }
        for (int64_t f0 = 0; f0 < frames && dbg_parts != 1; f0 += kMaxProblems) {
            MultiProblem mp;
            mp.q = qf;
            mp.k = k_audio;
            mp.v = v_audio;
            mp.o = o;
            mp.q_rows = frames * n_face;
            mp.kv_rows = frames * audio_tokens_per_frame;
            mp.o_rows = frames * tokens_per_frame;
            mp.o_row_map = face_ids;
            mp.zero_inv = dbg_parts == 2 ? nullptr : inv;
            mp.pack_keys = !getenv("TM_AUDIO_NOPACK");   // A/B switch (timing only)
            mp.zero_T = tokens_per_frame;
            mp.zero_row0 = f0 * tokens_per_frame;
            mp.B = cf.batch;
            mp.H = cf.heads;
            mp.d = cf.head_dim;
            mp.scale = ctx->scale;
            mp.sched_heads = cf.sched_heads;
            mp.nprob = int(std::min<int64_t>(kMaxProblems, frames - f0));
            mp.zero_rows = mp.nprob * tokens_per_frame;
            for (int i = 0; i < mp.nprob; ++i) {
                const int64_t f = f0 + i;
                SubProblem& sp = mp.prob[i];
                sp.q_row0 = f * n_face;
                sp.Lq = n_face;
                sp.o_row0 = f * tokens_per_frame;
                sp.nseg = window_runs(f, sp.seg_row0, sp.seg_len);
            }
            if (ctx->trace) cudaMemsetAsync(ctx->trace, 0, kTraceWords * 8, cs);
            st = cuda_check(launch_fmha_sm100_multi(mp, ctx->scratch(), cs, &ctx->launches, ctx->trace),
                            "audio cross-attention launch");
            if (st) return st;
            dump_trace(ctx, cs);
        }
        return debug_check(ctx, o, BF * tokens_per_frame * cf.heads * cf.head_dim, 1, cs,
                           "tm_audio_cross_attention");
    }
    // fp32 validation mode: gather, one attention launch per frame, zero, scatter
    st = cuda_check(launch_face_rows(q, qf, face_ids, BF, tokens_per_frame, n_face, row, 0, cs,
                                     &ctx->launches), "face gather");
    if (st) return st;
    for (int64_t f = 0; f < frames; ++f) {
        AttnProblem pr;
        pr.q = qf + f * n_face * row;
        pr.o = of + f * n_face * row;
        pr.Lq = n_face;
        pr.q_bstride = frames * n_face;
        pr.B = cf.batch;
        pr.H = cf.heads;
        pr.d = cf.head_dim;
        pr.scale = ctx->scale;
        int64_t row0[kMaxSegments], len[kMaxSegments];
        const int nseg = window_runs(f, row0, len);
        for (int i = 0; i < nseg; ++i)
            pr.seg[pr.nseg++] = Segment{kb + row0[i] * row, vb + row0[i] * row, len[i],
                                        frames * audio_tokens_per_frame};
        st = cuda_check(launch_fmha_fp32(pr, cs, &ctx->launches), "audio cross-attention launch");
        if (st) return st;
    }
    st = cuda_check(cudaMemsetAsync(o, 0, size_t(BF) * tokens_per_frame * row, cs), "zero output");
    if (st) return st;
    st = cuda_check(launch_face_rows(of, o, face_ids, BF, tokens_per_frame, n_face, row, 1, cs,
                                     &ctx->launches), "face scatter");
    if (st) return st;
    return debug_check(ctx, o, BF * tokens_per_frame * cf.heads * cf.head_dim, cf.dtype == TM_BF16,
                       cs, "tm_audio_cross_attention");
}

tm_status tm_flow_euler_step(tm_ctx* ctx, float* x, const void* v, int32_t v_dtype, int64_t n,
                             float dt, void* stream) {
    NvtxRange nvtx_range("tm_flow_euler_step");
    DeviceScope dev_scope(ctx ? ctx->cfg.device : -1);
    if (n < 0) return fail(TM_ERR_SHAPE, "n = %lld < 0", (long long)n);
    if (n == 0) return TM_OK;
    if (!x || !v) return fail(TM_ERR_INVALID_ARG, "null argument");
    if (v_dtype != TM_BF16 && v_dtype != TM_FP32)
        return fail(TM_ERR_INVALID_ARG, "v_dtype %d not in {TM_BF16, TM_FP32}", v_dtype);
    if (!aligned16(x) || !aligned16(v)) return fail(TM_ERR_INVALID_ARG, "x and v must be 16-byte aligned");
    if (!std::isfinite(dt)) return fail(TM_ERR_INVALID_ARG, "dt must be finite");
    int dummy = 0;
    int* counter = ctx ? &ctx->launches : &dummy;
    if (ctx) ctx->launches = 0;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    tm_status st = cuda_check(launch_euler(x, v, v_dtype == TM_BF16, n, dt, cs, counter),
                              "euler launch");
    if (st || !ctx) return st;
    return debug_check(ctx, x, n, 0, cs, "tm_flow_euler_step");
}

tm_status tm_ulysses_shuffle_host(int32_t mode, const void* src, void* dst, int32_t batch,
                                  int64_t shard_tokens, int64_t tokens, int32_t heads_per_rank,
                                  int32_t world_size, int32_t head_dim, int32_t elem_bytes) {
    if (!src || !dst) return fail(TM_ERR_INVALID_ARG, "null buffer");
    if (mode < 0 || mode > 3) return fail(TM_ERR_INVALID_ARG, "mode %d not in [0, 3]", mode);
    if (batch <= 0 || shard_tokens <= 0 || tokens <= 0 || heads_per_rank <= 0 || world_size <= 0 ||
        head_dim <= 0 || elem_bytes <= 0 || (int64_t(head_dim) * elem_bytes) % 16 ||
        tokens > shard_tokens * world_size)
        return fail(TM_ERR_SHAPE, "invalid Ulysses shape");
    UlyssesShape s{batch, world_size, heads_per_rank, head_dim * elem_bytes / 16, shard_tokens, tokens};
    struct W16 { uint64_t a, b; };
    const W16* in = static_cast<const W16*>(src);
    W16* out = static_cast<W16*>(dst);
    const int64_t total = ulysses_words(s);
    for (int64_t idx = 0; idx < total; ++idx) {
        int64_t si, di;
        ulysses_map(s, mode, idx, si, di);
        if (di < 0) continue;
        out[di] = si == -2 ? W16{0, 0} : in[si];
    }
    return TM_OK;
}

int32_t tm_schedule_tail_host(int32_t units, int32_t tiles_per_unit, int32_t ctas, int32_t* bounds) {
    if (units <= 0 || tiles_per_unit <= 0 || ctas <= 0 || ctas > kMaxPersistentCtas || !bounds ||
        int64_t(units) * tiles_per_unit >= (int64_t(1) << 30)) {
        fail(TM_ERR_INVALID_ARG, "invalid schedule query");
        return -1;
    }
    return tail_bounds_capped(units, tiles_per_unit, ctas, bounds);
}

tm_status tm_peer_route_host(int32_t mode, const void* src, void* dst, int32_t batch,
                             int64_t shard_tokens, int64_t tokens, int64_t window_tokens,
                             int32_t heads_per_rank, int32_t world_size, int32_t rank,
                             int32_t head_dim, int32_t elem_bytes) {
    if (!src || !dst) return fail(TM_ERR_INVALID_ARG, "null buffer");
    if (mode != 0 && mode != 1) return fail(TM_ERR_INVALID_ARG, "mode %d not in {0, 1}", mode);
    if (batch <= 0 || shard_tokens <= 0 || tokens <= 0 || heads_per_rank <= 0 || world_size <= 0 ||
        rank < 0 || rank >= world_size || head_dim <= 0 || elem_bytes <= 0 ||
        (int64_t(head_dim) * elem_bytes) % 16 || tokens > shard_tokens * world_size ||
        window_tokens < tokens)
        return fail(TM_ERR_SHAPE, "invalid peer route shape");
    struct W16 { uint64_t a, b; };
    const W16* in = static_cast<const W16*>(src);
    W16* out = static_cast<W16*>(dst);
    const int dw = head_dim * elem_bytes / 16;                       // words per (token, head)
    const int H = heads_per_rank * world_size;
    if (mode == 0) {
        const uint32_t W = uint32_t(heads_per_rank * dw);
        const int64_t win = int64_t(batch) * window_tokens * W;       // words per window
        const uint64_t n = uint64_t(batch) * shard_tokens * world_size * W;
        if (n >= (uint64_t(1) << 31)) return fail(TM_ERR_SHAPE, "shard too large");
        for (uint32_t i = 0; i < uint32_t(n); ++i) {
            uint32_t p;
            int64_t off;
            if (peer_push_route(i, W, uint32_t(world_size), uint32_t(shard_tokens), tokens,
                                window_tokens, rank, p, off))
                out[p * win + off] = in[i];
        }
    } else {
        const int64_t owin = int64_t(batch) * shard_tokens * H * dw;  // words per O window
        for (int64_t b = 0; b < batch; ++b)
            for (int64_t q = 0; q < tokens; ++q)
                for (int h = 0; h < heads_per_rank; ++h) {
                    int owner = 0;
                    const int64_t row = peer_out_route(b, q, h, shard_tokens, shard_tokens, H,
                                                       rank * heads_per_rank, owner);
                    for (int w = 0; w < dw; ++w)
                        out[owner * owin + row * dw + w] =
                            in[((b * tokens + q) * heads_per_rank + h) * dw + w];
                }
    }
    return TM_OK;
}

tm_status tm_flow_sampler_step(tm_ctx* ctx, float* x, const void* v, int32_t v_dtype, int64_t n,
                               float t_cur, float t_next, const float* eps, uint64_t seed,
                               uint64_t offset, void* x_bf16_out, void* stream) {
    NvtxRange nvtx_range("tm_flow_sampler_step");
    DeviceScope dev_scope(ctx ? ctx->cfg.device : -1);
    if (n < 0) return fail(TM_ERR_SHAPE, "n = %lld < 0", (long long)n);
    if (n == 0) return TM_OK;
    if (!x || !v) return fail(TM_ERR_INVALID_ARG, "null argument");
    if (v_dtype != TM_BF16 && v_dtype != TM_FP32)
        return fail(TM_ERR_INVALID_ARG, "v_dtype %d not in {TM_BF16, TM_FP32}", v_dtype);
    if (!(t_cur >= 0.f && t_cur < 1.f) || !(t_next > t_cur) || !std::isfinite(t_next))
        return fail(TM_ERR_INVALID_ARG, "need 0 <= t_cur < 1 and t_next > t_cur (Eq 1 time)");
    int dummy = 0;
    int* counter = ctx ? &ctx->launches : &dummy;
    if (ctx) ctx->launches = 0;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    tm_status st = cuda_check(launch_sampler(x, v, v_dtype == TM_BF16, eps, n, t_cur, t_next, seed,
                                             offset, x_bf16_out, cs, counter),
                              "sampler launch");
    if (st || !ctx) return st;
    return debug_check(ctx, x, n, 0, cs, "tm_flow_sampler_step");
}

tm_status tm_peer_export(tm_ctx* ctx, uint8_t* handle) {
    if (!ctx || !handle) return fail(TM_ERR_INVALID_ARG, "null argument");
    DeviceScope dev_scope(ctx->cfg.device);
    if (!ctx->lay.peer) return fail(TM_ERR_INVALID_ARG, "not a TM_TRANSPORT_PEER context");
    auto range = address_range_fn();
    if (!range) return fail(TM_ERR_CUDA, "cuMemGetAddressRange unavailable");
    uint8_t* w = ctx->win[ctx->cfg.rank];
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(w)) != CUDA_SUCCESS)
        return fail(TM_ERR_CUDA, "cuMemGetAddressRange failed for the workspace");
    cudaIpcMemHandle_t h;
    tm_status st = cuda_check(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)),
                              "cudaIpcGetMemHandle (workspace must come from cudaMalloc)");
    if (st) return st;
    static_assert(sizeof(h) == 64, "IPC handle size");
    const uint64_t off = uint64_t(reinterpret_cast<uintptr_t>(w) - uintptr_t(base));
    memcpy(handle, &h, 64);
    memcpy(handle + 64, &off, 8);
    return TM_OK;
}

tm_status tm_peer_connect(tm_ctx* ctx, const uint8_t* handles) {
    if (!ctx || !handles) return fail(TM_ERR_INVALID_ARG, "null argument");
    DeviceScope dev_scope(ctx->cfg.device);
    if (!ctx->lay.peer) return fail(TM_ERR_INVALID_ARG, "not a TM_TRANSPORT_PEER context");
    if (ctx->connected) return fail(TM_ERR_STREAM_ORDER, "already connected");
    for (int p = 0; p < ctx->lay.P; ++p) {
        if (p == ctx->cfg.rank) continue;
        cudaIpcMemHandle_t h;
        uint64_t off = 0;
        memcpy(&h, handles + size_t(p) * TM_PEER_HANDLE_BYTES, 64);
        memcpy(&off, handles + size_t(p) * TM_PEER_HANDLE_BYTES + 64, 8);
        void* base = nullptr;
        tm_status st = cuda_check(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess),
                                  "cudaIpcOpenMemHandle (peer window)");
        if (st) {
            for (void* b : ctx->ipc_opened) cudaIpcCloseMemHandle(b);
            ctx->ipc_opened.clear();
            return st;
        }
        ctx->ipc_opened.push_back(base);
        ctx->win[p] = static_cast<uint8_t*>(base) + off;
    }
    ctx->connected = true;
    return TM_OK;
}

tm_status tm_peer_connect_local(tm_ctx* const* ctxs, int32_t n) {
    if (!ctxs || n <= 0 || n > kMaxPeers) return fail(TM_ERR_INVALID_ARG, "need 1..%d contexts", kMaxPeers);
    for (int i = 0; i < n; ++i) {
        const tm_ctx* c = ctxs[i];
        if (!c || !c->lay.peer || c->cfg.world_size != n || c->cfg.rank != i)
            return fail(TM_ERR_INVALID_ARG, "ctxs[%d] must be a TM_TRANSPORT_PEER context of rank %d "
                                            "in a group of %d", i, i, n);
        if (c->connected && n > 1) return fail(TM_ERR_STREAM_ORDER, "ctxs[%d] already connected", i);
    }
    for (int i = 0; i < n; ++i) {
        for (int p = 0; p < n; ++p) ctxs[i]->win[p] = ctxs[p]->win[p];
        ctxs[i]->connected = true;
    }
    return TM_OK;
}

tm_status tm_nccl_connect_local(tm_ctx* const* ctxs, int32_t n) {
    if (!ctxs || n <= 1 || n > 64) return fail(TM_ERR_INVALID_ARG, "need 2..64 contexts");
    for (int i = 0; i < n; ++i) {
        const tm_ctx* c = ctxs[i];
        if (!c || c->lay.peer || !c->lay.exchange || !c->lb_pending || c->cfg.world_size != n ||
            c->cfg.rank != i)
            return fail(TM_ERR_INVALID_ARG, "ctxs[%d] must be a TM_TRANSPORT_NCCL context of rank %d "
                                            "in a group of %d created without an NCCL unique id",
                        i, i, n);
        if (!c->lb_group.empty()) return fail(TM_ERR_STREAM_ORDER, "ctxs[%d] already connected", i);
        if (c->lay.ws_bytes != ctxs[0]->lay.ws_bytes)
            return fail(TM_ERR_INVALID_ARG, "ctxs[%d] has a different workspace layout", i);
    }
    for (int i = 0; i < n; ++i) ctxs[i]->lb_group.assign(ctxs, ctxs + n);
    return TM_OK;
}

tm_status tm_peer_output_ptr(tm_ctx* ctx, void** o) {
    if (!ctx || !o) return fail(TM_ERR_INVALID_ARG, "null argument");
    if (!ctx->lay.peer) return fail(TM_ERR_INVALID_ARG, "not a TM_TRANSPORT_PEER context");
    *o = ctx->wo(ctx->cfg.rank);
    return TM_OK;
}

tm_status tm_peer_check(tm_ctx* ctx) {
    if (!ctx) return fail(TM_ERR_INVALID_ARG, "null ctx");
    DeviceScope dev_scope(ctx->cfg.device);
    if (ctx->comm) {                       // NCCL transport: the communicator's async state
        const char* e = comm_async_error(ctx->comm);
        if (e) return fail(TM_ERR_NCCL, "NCCL asynchronous error: %s", e);
    }
    if (!ctx->lay.peer) return TM_OK;
    tm_status st = cuda_check(cudaDeviceSynchronize(), "synchronize");
    if (st) return st;
    uint32_t err = 0;
    uint32_t* e = &ctx->ctr(ctx->cfg.rank)->err;
    st = cuda_check(cudaMemcpy(&err, e, 4, cudaMemcpyDeviceToHost), "peer flag readback");
    if (st) return st;
    if (err) {
        cudaMemset(e, 0, 4);
        return fail(TM_ERR_CUDA, "a peer wait timed out (a rank did not send its part)");
    }
    return TM_OK;
}

int32_t tm_last_launch_count(const tm_ctx* ctx) { return ctx ? ctx->launches : -1; }

const char* tm_kernel_variant(const tm_ctx* ctx) {
    if (!ctx) return "";
    return ctx->cfg.dtype == TM_BF16 ? "sm100_tcgen05" : "fp32_simt";
}

}  // extern "C"
