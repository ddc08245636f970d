// capi.cu — the C ABI (include/sale_b200.h): argument validation with the
// reference's error classes, TMA tensor-map construction, work-unit tables,
// ctx-owned workspace, and the stage composition of run_pipeline
// (runner.hpp:63-80) on device buffers.
#include "sale_b200.h"

#include "common.cuh"
#include "internal.h"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

using namespace sale_b200;

struct sale_b200_ctx {
    int device = 0;
    std::string err;
    std::mutex mu;
    // workspace for sale_b200_select / sale_b200_prefill
    uint8_t *ws = nullptr;
    size_t ws_bytes = 0;
    double *d_taus = nullptr;
    int64_t taus_cap = 0;
    // estimator work-unit table, cached per token count
    EstUnit *d_units = nullptr;
    int64_t units_cap = 0;
    std::vector<int64_t> units_key; // tokens + geometry of the cached table
    int64_t n_units = 0;
    // host e2e buffers
    uint8_t *io = nullptr;
    size_t io_bytes = 0;
    cudaStream_t io_stream = nullptr;
    // chunked host pipeline (sale_b200_prefill_host): compute and D2H streams,
    // per-chunk estimator units grouped by chunk
    cudaStream_t comp_stream = nullptr, out_stream = nullptr, attn_stream = nullptr;
    EstUnit *d_cunits = nullptr;
    size_t cunits_bytes = 0;
    std::vector<int64_t> cunit_key;
    std::vector<int64_t> cunit_off;
    // optional per-stage event timing of sale_b200_prefill
    bool timing = false;
    cudaEvent_t ev[6] = {};
    // stream ordering of the ctx-owned workspace: the last call that used it
    // recorded ws_ev on ws_stream; a call on another stream waits for it
    cudaEvent_t ws_ev = nullptr;
    cudaStream_t ws_stream = nullptr;
    // empty-row check of block_sparse_attention with a caller mask: smallest
    // (b, h, row) index that attends nothing (device) and its pinned copy
    unsigned long long *d_empty = nullptr;
    unsigned long long *h_empty = nullptr;
};

namespace {

thread_local std::string g_create_error; // ctx-less calls (create, file formats)

int fail(sale_b200_ctx *ctx, int code, const std::string &msg) {
    if (ctx) ctx->err = msg;
    else g_create_error = msg;
    return code;
}

int cuda_fail(sale_b200_ctx *ctx, cudaError_t e, const char *where) {
    return fail(ctx, SALE_B200_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

#define SALE_CUDA(ctx, call)                                                                       \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);                                   \
    } while (0)

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Every ctx entry point runs on ctx's device and restores the caller's
// current device on return (a process may drive one ctx per GPU).
struct DeviceGuard {
    int prev = -1, dev;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int d) : dev(d) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
};
#define SALE_ENTER(ctx)                                                                            \
    if (!(ctx)) return SALE_B200_INVALID_ARGUMENT;                                                 \
    std::lock_guard<std::mutex> lk_((ctx)->mu);                                                    \
    DeviceGuard dg_((ctx)->device);                                                                \
    if (dg_.err != cudaSuccess) return cuda_fail(ctx, dg_.err, "cudaSetDevice")

// Workspace hand-off between streams (see the ctx fields).
int ws_begin(sale_b200_ctx *ctx, cudaStream_t stream) {
    if (ctx->ws_ev && ctx->ws_stream != stream)
        SALE_CUDA(ctx, cudaStreamWaitEvent(stream, ctx->ws_ev, 0));
    return SALE_B200_OK;
}
int ws_end(sale_b200_ctx *ctx, cudaStream_t stream) {
    if (!ctx->ws_ev) SALE_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ws_ev, cudaEventDisableTiming));
    SALE_CUDA(ctx, cudaEventRecord(ctx->ws_ev, stream));
    ctx->ws_stream = stream;
    return SALE_B200_OK;
}

// block_sparse_attention's domain_error (sparse_attention.hpp:88-90) for a
// caller-supplied mask: the kernel records the smallest empty (b, h, row)
// index; the call waits for it (the reference is synchronous) and reports it.
int empty_rows_begin(sale_b200_ctx *ctx, cudaStream_t stream) {
    if (!ctx->d_empty) {
        SALE_CUDA(ctx, cudaMalloc(&ctx->d_empty, sizeof(unsigned long long)));
        SALE_CUDA(ctx, cudaMallocHost(&ctx->h_empty, sizeof(unsigned long long)));
    }
    SALE_CUDA(ctx, cudaMemsetAsync(ctx->d_empty, 0xFF, sizeof(unsigned long long), stream));
    return SALE_B200_OK;
}
int empty_rows_end(sale_b200_ctx *ctx, cudaStream_t stream, int64_t batch, int64_t q_heads,
                   int64_t tokens) {
    SALE_CUDA(ctx, cudaMemcpyAsync(ctx->h_empty, ctx->d_empty, sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, stream));
    SALE_CUDA(ctx, cudaStreamSynchronize(stream));
    const unsigned long long x = *ctx->h_empty;
    if (x == ~0ull) return SALE_B200_OK;
    const int64_t row = static_cast<int64_t>(x % static_cast<unsigned long long>(tokens));
    const int64_t bh = static_cast<int64_t>(x / static_cast<unsigned long long>(tokens));
    std::string msg = "block_sparse_attention: query row " + std::to_string(row) + " attends no tokens";
    if (batch * q_heads > 1)
        msg += " (batch " + std::to_string(bh / q_heads) + ", head " + std::to_string(bh % q_heads) + ")";
    return fail(ctx, SALE_B200_DOMAIN_ERROR, msg);
}

// Stage boundaries: 0 start, 1 quantized, 2 base mask, 3 stats, 4 estimate, 5 attention.
void mark(sale_b200_ctx *ctx, int i, cudaStream_t stream) {
    if (ctx->timing) cudaEventRecord(ctx->ev[i], stream);
}

int check_shape(sale_b200_ctx *ctx, const sale_b200_shape *s) {
    if (!s) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "shape is NULL");
    if (s->batch < 1 || s->tokens < 1 || s->q_heads < 1 || s->kv_heads < 1)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "HeadInput: empty query");
    if (s->head_dim < 1) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "HeadInput: empty query");
    if (s->head_dim > kHeadDim)
        return fail(ctx, SALE_B200_UNSUPPORTED, "head_dim > 128 is not supported on the B200 path");
    if (s->q_heads % s->kv_heads != 0)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "q_heads must be a multiple of kv_heads");
    if (s->tokens > (1LL << 19))
        return fail(ctx, SALE_B200_UNSUPPORTED, "tokens > 524288 is not supported");
    if (s->batch * s->kv_heads > 65535)
        return fail(ctx, SALE_B200_UNSUPPORTED, "batch * kv_heads > 65535");
    return SALE_B200_OK;
}

// SelectionConfig::validate (selection.hpp:26-37), then the block sizes this
// path is built for (block_q 64, block_k 32: the tile shapes of every kernel).
// sink_tokens, local_tokens_min and segment_size may take any valid value.
int check_config(sale_b200_ctx *ctx, const sale_b200_selection_config *c) {
    sale_b200_selection_config d;
    sale_b200_default_config(&d);
    if (!c) c = &d;
    if (c->sink_tokens < 1)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "SelectionConfig: sink_tokens must be >= 1");
    if (c->block_q < 1 || c->block_k < 1)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "SelectionConfig: block sizes must be >= 1");
    if (c->local_tokens_min < c->block_k)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT,
                    "SelectionConfig: local_tokens_min must be >= block_k");
    if (c->segment_size < 1)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "SelectionConfig: segment_size must be >= 1");
    if (c->block_q != kBlockQ || c->block_k != kBlockK)
        return fail(ctx, SALE_B200_UNSUPPORTED,
                    "the B200 path implements block_q 64 and block_k 32 (any sink_tokens, "
                    "local_tokens_min and segment_size)");
    if (c->segment_size > (1 << 20) || c->local_tokens_min > (1LL << 40) || c->sink_tokens > (1LL << 40))
        return fail(ctx, SALE_B200_UNSUPPORTED, "SelectionConfig: value out of the supported range");
    return SALE_B200_OK;
}

// The block-level geometry of a (validated) config for `tokens` tokens
// (common.cuh Geom; selection.hpp:92-123, :199-202).
Geom geometry(const sale_b200_selection_config *c, int64_t tokens) {
    sale_b200_selection_config d;
    sale_b200_default_config(&d);
    if (!c) c = &d;
    Geom g;
    g.sb = static_cast<int>(cdiv(std::min<int64_t>(c->sink_tokens, tokens), kBlockK));
    g.nl = static_cast<int>(std::min<int64_t>(cdiv(c->local_tokens_min, kBlockK), 1 << 24));
    g.seg = static_cast<int>(c->segment_size);
    return g;
}

int check_taus(sale_b200_ctx *ctx, const double *taus, int64_t n) {
    if (!taus) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "taus is NULL");
    for (int64_t i = 0; i < n; ++i)
        if (!(taus[i] > 0.0 && taus[i] < 1.0))
            return fail(ctx, SALE_B200_INVALID_ARGUMENT, "SelectionConfig: tau must be in (0,1)");
    return SALE_B200_OK;
}

float inv_sqrt_dim(int64_t d) { return 1.0f / std::sqrt(static_cast<float>(d)); }

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 4-D map over [B][N][H][128] with a SWIZZLE_128B box of
// {box_inner elements, 1 head, box_rows tokens, 1 batch}.
// rows_limit (> 0): the map covers tokens [0, rows_limit) of each batch (the
// batch stride stays tokens rows); TMA zero-fills rows past it.
int make_map(sale_b200_ctx *ctx, CUtensorMap *map, const void *base, bool bf16, int64_t batch,
             int64_t tokens, int64_t heads, uint32_t box_inner, uint32_t box_rows,
             int64_t rows_limit = 0) {
    auto enc = tensor_map_encoder();
    if (!enc) return fail(ctx, SALE_B200_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    const uint64_t eb = bf16 ? 2 : 1;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(kHeadDim), static_cast<cuuint64_t>(heads),
                          static_cast<cuuint64_t>(rows_limit > 0 ? rows_limit : tokens),
                          static_cast<cuuint64_t>(batch)};
    cuuint64_t strides[3] = {kHeadDim * eb, static_cast<cuuint64_t>(heads) * kHeadDim * eb,
                             static_cast<cuuint64_t>(tokens * heads) * kHeadDim * eb};
    cuuint32_t box[4] = {box_inner, 1, box_rows, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 4,
                     const_cast<void *>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(ctx, SALE_B200_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return SALE_B200_OK;
}

// Estimator stages (128 keys = 4 key blocks each) of the 128-row tile m =
// query blocks 2m+1, 2m+2: enough for the larger of their E_i estimated
// blocks (default geometry: m - 1, one stage per segment).
int64_t tile_stages(int64_t m, int64_t nq, const Geom &g) {
    int64_t e = estimated_blocks(2 * m + 1, g);
    if (2 * m + 2 < nq) e = std::max(e, estimated_blocks(2 * m + 2, g));
    return (e + kSegment - 1) / kSegment;
}

// Work units of the estimator (estimate.cu): every 128-row tile with
// estimated blocks, split into chunks of 64 stages. Full chunks first (by
// chunk, then tile: concurrent CTAs share K-code chunks in L2), partial chunks
// last, largest first.
void append_units(std::vector<EstUnit> &units, int64_t m, int64_t nq, const Geom &g) {
    const int64_t f = tile_stages(m, nq, g);
    for (int64_t c = 0; c * kSegPerUnitHost < f; ++c)
        units.push_back({static_cast<int>(m), static_cast<int>(c),
                         static_cast<int>(std::min<int64_t>(kSegPerUnitHost, f - c * kSegPerUnitHost))});
}
void sort_units(std::vector<EstUnit> &units) {
    std::stable_sort(units.begin(), units.end(), [](const EstUnit &a, const EstUnit &b) {
        if (a.nseg != b.nseg) return a.nseg > b.nseg;
        if (a.c != b.c) return a.c < b.c;
        return a.m < b.m;
    });
}

int ensure_units(sale_b200_ctx *ctx, int64_t tokens, const Geom &geo, cudaStream_t stream) {
    const std::vector<int64_t> key = {tokens, geo.sb, geo.nl, geo.seg};
    if (ctx->units_key == key) return SALE_B200_OK;
    const int64_t nq = cdiv(tokens, kBlockQ);
    std::vector<EstUnit> units;
    for (int64_t m = 0; 2 * m + 1 < nq; ++m) append_units(units, m, nq, geo);
    sort_units(units);
    const int64_t n = static_cast<int64_t>(units.size());
    if (n > ctx->units_cap) {
        if (ctx->d_units) cudaFree(ctx->d_units);
        ctx->d_units = nullptr;
        SALE_CUDA(ctx, cudaMalloc(&ctx->d_units, sizeof(EstUnit) * std::max<int64_t>(n, 1)));
        ctx->units_cap = std::max<int64_t>(n, 1);
    }
    if (n)
        SALE_CUDA(ctx, cudaMemcpyAsync(ctx->d_units, units.data(), sizeof(EstUnit) * n,
                                       cudaMemcpyHostToDevice, stream));
    SALE_CUDA(ctx, cudaStreamSynchronize(stream));
    ctx->units_key = key;
    ctx->n_units = n;
    return SALE_B200_OK;
}

struct Workspace {
    int8_t *q_codes;
    int8_t *k_codes;
    float *q_scales;
    float *k_scales;
    float *thresh;
    uint32_t *mask;
};

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

int ensure_workspace(sale_b200_ctx *ctx, const sale_b200_shape &s, Workspace *w) {
    const int64_t B = s.batch, N = s.tokens, Hq = s.q_heads, Hkv = s.kv_heads;
    const int64_t nq = cdiv(N, kBlockQ), nk = cdiv(N, kBlockK), words = cdiv(nk, 32);
    const size_t sz[6] = {align256(B * N * Hq * kHeadDim), align256(B * N * Hkv * kHeadDim),
                          align256(sizeof(float) * B * Hq * N), align256(sizeof(float) * B * Hkv * nk),
                          align256(sizeof(float) * B * Hq * N),
                          align256(sizeof(uint32_t) * B * Hq * nq * words)};
    size_t total = 0;
    for (size_t x : sz) total += x;
    if (total > ctx->ws_bytes) {
        if (ctx->ws) cudaFree(ctx->ws);
        ctx->ws = nullptr;
        ctx->ws_bytes = 0;
        SALE_CUDA(ctx, cudaMalloc(&ctx->ws, total));
        ctx->ws_bytes = total;
    }
    uint8_t *p = ctx->ws;
    w->q_codes = reinterpret_cast<int8_t *>(p);
    p += sz[0];
    w->k_codes = reinterpret_cast<int8_t *>(p);
    p += sz[1];
    w->q_scales = reinterpret_cast<float *>(p);
    p += sz[2];
    w->k_scales = reinterpret_cast<float *>(p);
    p += sz[3];
    w->thresh = reinterpret_cast<float *>(p);
    p += sz[4];
    w->mask = reinterpret_cast<uint32_t *>(p);
    return SALE_B200_OK;
}

int upload_taus(sale_b200_ctx *ctx, const double *taus, int64_t n, cudaStream_t stream) {
    if (n > ctx->taus_cap) {
        if (ctx->d_taus) cudaFree(ctx->d_taus);
        ctx->d_taus = nullptr;
        SALE_CUDA(ctx, cudaMalloc(&ctx->d_taus, sizeof(double) * n));
        ctx->taus_cap = n;
    }
    SALE_CUDA(ctx, cudaMemcpyAsync(ctx->d_taus, taus, sizeof(double) * n, cudaMemcpyHostToDevice,
                                   stream));
    return SALE_B200_OK;
}

int select_impl(sale_b200_ctx *ctx, const void *q, const void *k, const int8_t *q_codes,
                const float *q_scales, const int8_t *k_codes, const float *k_scales,
                const sale_b200_shape &s, const double *taus, const Geom &geo, uint32_t *mask,
                float *thresh, const sale_b200_select_debug *dbg, cudaStream_t stream) {
    int st;
    if ((st = upload_taus(ctx, taus, s.q_heads, stream))) return st;
    if ((st = ensure_units(ctx, s.tokens, geo, stream))) return st;
    const float isd = inv_sqrt_dim(s.head_dim);
    SALE_CUDA(ctx, launch_base_mask(mask, s.batch, s.q_heads, s.tokens, geo, stream));
    mark(ctx, 2, stream);
    SALE_CUDA(ctx, launch_sink_local_stats(q, k, s.batch, s.tokens, s.q_heads, s.kv_heads, isd, geo,
                                           ctx->d_taus, thresh, dbg ? dbg->running_max : nullptr,
                                           dbg ? dbg->exp_sum : nullptr, dbg ? dbg->bound : nullptr,
                                           stream));
    mark(ctx, 3, stream);
    if (ctx->n_units == 0) {
        mark(ctx, 4, stream);
        return SALE_B200_OK;
    }
    CUtensorMap tm_qc, tm_kc;
    if ((st = make_map(ctx, &tm_qc, q_codes, false, s.batch, s.tokens, s.q_heads, 128, 128))) return st;
    if ((st = make_map(ctx, &tm_kc, k_codes, false, s.batch, s.tokens, s.kv_heads, 128, 128))) return st;
    SALE_CUDA(ctx, launch_estimate(tm_qc, tm_kc, ctx->d_units, ctx->n_units, q_scales, k_scales,
                                   thresh, mask, s.batch, s.tokens, static_cast<int>(s.q_heads),
                                   static_cast<int>(s.kv_heads), isd, geo,
                                   dbg ? dbg->block_max : nullptr, stream));
    SALE_CUDA(ctx, launch_segment_or(mask, s.batch, s.q_heads, s.tokens, geo, stream));
    mark(ctx, 4, stream);
    return SALE_B200_OK;
}

int attention_impl(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                   const sale_b200_shape &s, const uint32_t *mask, void *out, int32_t *coverage,
                   cudaStream_t stream, int64_t i_lo = 0, int64_t i_hi = -1,
                   unsigned long long *empty_rows = nullptr) {
    int st;
    CUtensorMap tk, tv;
    if ((st = make_map(ctx, &tk, k, true, s.batch, s.tokens, s.kv_heads, 64, 128))) return st;
    if ((st = make_map(ctx, &tv, v, true, s.batch, s.tokens, s.kv_heads, 64, 128))) return st;
    const float scale_log2 = inv_sqrt_dim(s.head_dim) * 1.4426950408889634f;
    SALE_CUDA(ctx, launch_sparse_attention(q, tk, tv, mask, out, coverage, s.batch, s.tokens,
                                           static_cast<int>(s.q_heads), static_cast<int>(s.kv_heads),
                                           scale_log2, stream, i_lo, i_hi, empty_rows));
    mark(ctx, 5, stream);
    return SALE_B200_OK;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Query-block boundaries of the chunked host pipeline: chunk c = query blocks
// [b_c, b_{c+1}); inner boundaries are odd so that every estimator tile
// (query blocks 2m+1, 2m+2) lies inside one chunk. Equal token spans.
std::vector<int64_t> chunk_bounds(int64_t nq, int chunks) {
    std::vector<int64_t> b(1, 0);
    for (int c = 1; c < chunks; ++c) {
        int64_t x = (nq * c) / chunks;
        x |= 1; // odd
        if (x > b.back() && x < nq) b.push_back(x);
    }
    b.push_back(nq);
    return b;
}

// Long sequences: 15 chunks, short at both ends (the first chunk's H2D and the
// last chunk's D2H are the exposed copies) and sized in between so that each
// chunk's H2D stays under the previous chunk's (causal, growing) compute.
std::vector<int64_t> chunk_bounds_long(int64_t nq) {
    static const double kFrac[] = {0.03, 0.07, 0.12, 0.18, 0.25, 0.33, 0.42, 0.52,
                                   0.62, 0.72, 0.82, 0.90, 0.95, 0.98};
    std::vector<int64_t> b(1, 0);
    for (double f : kFrac) {
        int64_t x = static_cast<int64_t>(f * static_cast<double>(nq));
        x |= 1; // odd
        if (x > b.back() && x < nq) b.push_back(x);
    }
    b.push_back(nq);
    return b;
}

// Estimator units grouped by chunk (tile m belongs to the chunk holding query
// block 2m+1), each group ordered like the global table.
int ensure_chunk_units(sale_b200_ctx *ctx, int64_t tokens, const Geom &geo,
                       const std::vector<int64_t> &bounds, cudaStream_t stream) {
    std::vector<int64_t> key(bounds);
    key.insert(key.end(), {tokens, geo.sb, geo.nl, geo.seg});
    if (key == ctx->cunit_key) return SALE_B200_OK;
    const int64_t nq = cdiv(tokens, kBlockQ);
    const size_t nch = bounds.size() - 1;
    std::vector<std::vector<EstUnit>> per(nch);
    for (int64_t m = 0; 2 * m + 1 < nq; ++m) {
        size_t c = 0;
        while (c + 1 < nch && bounds[c + 1] <= 2 * m + 1) ++c;
        append_units(per[c], m, nq, geo);
    }
    std::vector<EstUnit> flat;
    ctx->cunit_off.assign(1, 0);
    for (auto &v : per) {
        sort_units(v);
        flat.insert(flat.end(), v.begin(), v.end());
        ctx->cunit_off.push_back(static_cast<int64_t>(flat.size()));
    }
    const size_t bytes = sizeof(EstUnit) * std::max<size_t>(flat.size(), 1);
    if (bytes > ctx->cunits_bytes) {
        if (ctx->d_cunits) cudaFree(ctx->d_cunits);
        ctx->d_cunits = nullptr;
        ctx->cunits_bytes = 0;
        SALE_CUDA(ctx, cudaMalloc(&ctx->d_cunits, bytes));
        ctx->cunits_bytes = bytes;
    }
    if (!flat.empty())
        SALE_CUDA(ctx, cudaMemcpyAsync(ctx->d_cunits, flat.data(), sizeof(EstUnit) * flat.size(),
                                       cudaMemcpyHostToDevice, stream));
    SALE_CUDA(ctx, cudaStreamSynchronize(stream));
    ctx->cunit_key = key;
    return SALE_B200_OK;
}

} // namespace

namespace sale_b200 {
int set_error(sale_b200_ctx *ctx, int code, const std::string &msg) { return fail(ctx, code, msg); }
cudaError_t ensure_smem_attr(const void *func, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<int, const void *>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    for (const auto &x : done)
        if (x.first == dev && x.second == func) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e == cudaSuccess) done.emplace_back(dev, func);
    return e;
}
int ctx_device_of(const sale_b200_ctx *ctx) { return ctx->device; }
} // namespace sale_b200

extern "C" {

int sale_b200_version(void) { return 1; }

void sale_b200_default_config(sale_b200_selection_config *cfg) {
    cfg->sink_tokens = 32;
    cfg->local_tokens_min = 128;
    cfg->segment_size = 4;
    cfg->block_q = 64;
    cfg->block_k = 32;
}

int sale_b200_ctx_create(int device, sale_b200_ctx **out) {
    if (!out) return fail(nullptr, SALE_B200_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(nullptr, SALE_B200_CUDA_ERROR,
                    std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= n) return fail(nullptr, SALE_B200_INVALID_ARGUMENT, "bad device");
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess)
        return fail(nullptr, SALE_B200_CUDA_ERROR, cudaGetErrorString(e));
    if (prop.major != 10 || prop.minor != 0)
        return fail(nullptr, SALE_B200_UNSUPPORTED,
                    "sale_b200 is built for sm_100a (B200); device is sm_" +
                        std::to_string(prop.major) + std::to_string(prop.minor));
    if ((e = cudaSetDevice(device)) != cudaSuccess)
        return fail(nullptr, SALE_B200_CUDA_ERROR, cudaGetErrorString(e));
    auto *ctx = new sale_b200_ctx();
    ctx->device = device;
    *out = ctx;
    return SALE_B200_OK;
}

int sale_b200_device_alloc(sale_b200_ctx *ctx, uint64_t bytes, void **out) {
    if (!ctx || !out) return SALE_B200_INVALID_ARGUMENT;
    DeviceGuard dg_(ctx->device);
    if (dg_.err != cudaSuccess) return cuda_fail(ctx, dg_.err, "cudaSetDevice");
    SALE_CUDA(ctx, cudaMalloc(out, bytes ? bytes : 1));
    return SALE_B200_OK;
}

int sale_b200_device_free(sale_b200_ctx *ctx, void *ptr) {
    if (!ctx) return SALE_B200_INVALID_ARGUMENT;
    DeviceGuard dg_(ctx->device);
    if (dg_.err != cudaSuccess) return cuda_fail(ctx, dg_.err, "cudaSetDevice");
    if (ptr) SALE_CUDA(ctx, cudaFree(ptr));
    return SALE_B200_OK;
}

int sale_b200_copy_to_device(sale_b200_ctx *ctx, void *dst, const void *src, uint64_t bytes) {
    if (!ctx) return SALE_B200_INVALID_ARGUMENT;
    DeviceGuard dg_(ctx->device);
    if (dg_.err != cudaSuccess) return cuda_fail(ctx, dg_.err, "cudaSetDevice");
    SALE_CUDA(ctx, cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    return SALE_B200_OK;
}

int sale_b200_copy_to_host(sale_b200_ctx *ctx, void *dst, const void *src, uint64_t bytes) {
    if (!ctx) return SALE_B200_INVALID_ARGUMENT;
    DeviceGuard dg_(ctx->device);
    if (dg_.err != cudaSuccess) return cuda_fail(ctx, dg_.err, "cudaSetDevice");
    SALE_CUDA(ctx, cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    return SALE_B200_OK;
}

int sale_b200_memset(sale_b200_ctx *ctx, void *dst, int value, uint64_t bytes) {
    if (!ctx) return SALE_B200_INVALID_ARGUMENT;
    DeviceGuard dg_(ctx->device);
    if (dg_.err != cudaSuccess) return cuda_fail(ctx, dg_.err, "cudaSetDevice");
    SALE_CUDA(ctx, cudaMemset(dst, value, bytes));
    return SALE_B200_OK;
}

int sale_b200_synchronize(sale_b200_ctx *ctx) {
    if (!ctx) return SALE_B200_INVALID_ARGUMENT;
    DeviceGuard dg_(ctx->device);
    if (dg_.err != cudaSuccess) return cuda_fail(ctx, dg_.err, "cudaSetDevice");
    SALE_CUDA(ctx, cudaDeviceSynchronize());
    return SALE_B200_OK;
}

int sale_b200_estimator_profile(sale_b200_ctx *ctx, int enable, uint64_t *counters) {
    if (!ctx) return SALE_B200_INVALID_ARGUMENT;
    DeviceGuard dg_(ctx->device);
    if (dg_.err != cudaSuccess) return cuda_fail(ctx, dg_.err, "cudaSetDevice");
    SALE_CUDA(ctx, cudaDeviceSynchronize());
    SALE_CUDA(ctx, estimate_profile(enable, reinterpret_cast<unsigned long long *>(counters)));
    SALE_CUDA(ctx, stats_profile(enable, counters ? reinterpret_cast<unsigned long long *>(counters + 8)
                                                  : nullptr));
    return SALE_B200_OK;
}

int sale_b200_attention_profile(sale_b200_ctx *ctx, int enable, uint64_t *counters) {
    if (!ctx) return SALE_B200_INVALID_ARGUMENT;
    DeviceGuard dg_(ctx->device);
    if (dg_.err != cudaSuccess) return cuda_fail(ctx, dg_.err, "cudaSetDevice");
    SALE_CUDA(ctx, cudaDeviceSynchronize());
    SALE_CUDA(ctx, attention_profile(enable, reinterpret_cast<unsigned long long *>(counters)));
    return SALE_B200_OK;
}

int sale_b200_set_timing(sale_b200_ctx *ctx, int enable) {
    SALE_ENTER(ctx);
    if (enable && !ctx->ev[0])
        for (auto &e : ctx->ev) SALE_CUDA(ctx, cudaEventCreate(&e));
    ctx->timing = enable != 0;
    return SALE_B200_OK;
}

int sale_b200_stage_times(sale_b200_ctx *ctx, float *ms) {
    if (!ms) return SALE_B200_INVALID_ARGUMENT;
    SALE_ENTER(ctx);
    if (!ctx->ev[0]) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "timing was never enabled");
    SALE_CUDA(ctx, cudaEventSynchronize(ctx->ev[5]));
    for (int i = 0; i < 5; ++i) SALE_CUDA(ctx, cudaEventElapsedTime(&ms[i], ctx->ev[i], ctx->ev[i + 1]));
    return SALE_B200_OK;
}

void sale_b200_ctx_destroy(sale_b200_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->ws) cudaFree(ctx->ws);
    if (ctx->d_taus) cudaFree(ctx->d_taus);
    if (ctx->d_units) cudaFree(ctx->d_units);
    if (ctx->io) cudaFree(ctx->io);
    if (ctx->io_stream) cudaStreamDestroy(ctx->io_stream);
    if (ctx->comp_stream) cudaStreamDestroy(ctx->comp_stream);
    if (ctx->out_stream) cudaStreamDestroy(ctx->out_stream);
    if (ctx->attn_stream) cudaStreamDestroy(ctx->attn_stream);
    if (ctx->d_cunits) cudaFree(ctx->d_cunits);
    if (ctx->ws_ev) cudaEventDestroy(ctx->ws_ev);
    if (ctx->d_empty) cudaFree(ctx->d_empty);
    if (ctx->h_empty) cudaFreeHost(ctx->h_empty);
    delete ctx;
}

const char *sale_b200_last_error(const sale_b200_ctx *ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

int sale_b200_quantize(sale_b200_ctx *ctx, const void *x, int64_t batch, int64_t tokens,
                       int64_t heads, int64_t group_rows, int8_t *codes, float *scales,
                       void *stream) {
    SALE_ENTER(ctx);
    if (!x || !codes || !scales) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    if (batch < 1 || tokens < 1 || heads < 1)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "quantize: empty input");
    if (group_rows < 1) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "QuantizedMatrix: group_rows must be >= 1");
    if (group_rows != 1 && group_rows != kBlockK)
        return fail(ctx, SALE_B200_UNSUPPORTED, "group_rows must be 1 (per token) or 32 (per key block)");
    if (!aligned16(x) || !aligned16(codes))
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "buffers must be 16-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = group_rows == 1
                        ? launch_quantize_qk(x, nullptr, codes, scales, nullptr, nullptr, batch,
                                             tokens, heads, 1, s)
                        : launch_quantize_qk(nullptr, x, nullptr, nullptr, codes, scales, batch,
                                             tokens, 1, heads, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "quantize");
    return SALE_B200_OK;
}

int sale_b200_quantize_qk(sale_b200_ctx *ctx, const void *q, const void *k,
                          const sale_b200_shape *shape, int8_t *q_codes, float *q_scales,
                          int8_t *k_codes, float *k_scales, void *stream) {
    SALE_ENTER(ctx);
    int st;
    if ((st = check_shape(ctx, shape))) return st;
    if (!q || !k || !q_codes || !q_scales || !k_codes || !k_scales)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    SALE_CUDA(ctx, launch_quantize_qk(q, k, q_codes, q_scales, k_codes, k_scales, shape->batch,
                                      shape->tokens, shape->q_heads, shape->kv_heads,
                                      static_cast<cudaStream_t>(stream)));
    return SALE_B200_OK;
}

int sale_b200_select(sale_b200_ctx *ctx, const void *q, const void *k, const int8_t *q_codes,
                     const float *q_scales, const int8_t *k_codes, const float *k_scales,
                     const sale_b200_shape *shape, const double *taus,
                     const sale_b200_selection_config *cfg, uint32_t *mask_words,
                     const sale_b200_select_debug *dbg, void *stream) {
    SALE_ENTER(ctx);
    int st;
    if ((st = check_shape(ctx, shape))) return st;
    if ((st = check_config(ctx, cfg))) return st;
    if ((st = check_taus(ctx, taus, shape->q_heads))) return st;
    if (!q || !k || !q_codes || !q_scales || !k_codes || !k_scales || !mask_words)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    Workspace w;
    if ((st = ensure_workspace(ctx, *shape, &w))) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if ((st = ws_begin(ctx, s))) return st;
    if ((st = select_impl(ctx, q, k, q_codes, q_scales, k_codes, k_scales, *shape, taus,
                          geometry(cfg, shape->tokens), mask_words, w.thresh, dbg, s)))
        return st;
    return ws_end(ctx, s);
}

int sale_b200_sparse_attention(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                               const sale_b200_shape *shape, const uint32_t *mask_words,
                               void *out, int32_t *coverage, void *stream) {
    SALE_ENTER(ctx);
    int st;
    if ((st = check_shape(ctx, shape))) return st;
    if (!q || !k || !v || !out) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!mask_words) // all-true mask: every row attends its causal prefix
        return attention_impl(ctx, q, k, v, *shape, nullptr, out, coverage, s);
    if ((st = ws_begin(ctx, s)) || (st = empty_rows_begin(ctx, s))) return st;
    if ((st = attention_impl(ctx, q, k, v, *shape, mask_words, out, coverage, s, 0, -1, ctx->d_empty)))
        return st;
    if ((st = ws_end(ctx, s))) return st;
    return empty_rows_end(ctx, s, shape->batch, shape->q_heads, shape->tokens);
}

int sale_b200_flop_count(sale_b200_ctx *ctx, const uint32_t *mask_words, int64_t batch,
                         int64_t q_heads, int64_t tokens, int64_t *counts, void *stream) {
    SALE_ENTER(ctx);
    if (!mask_words || !counts) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    if (batch < 1 || q_heads < 1 || tokens < 1)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "flop_accounting: empty grid");
    SALE_CUDA(ctx, launch_flop_count(mask_words, batch, q_heads, tokens, counts,
                                     static_cast<cudaStream_t>(stream)));
    return SALE_B200_OK;
}

int sale_b200_prefill(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                      const sale_b200_shape *shape, const double *taus,
                      const sale_b200_selection_config *cfg, void *out, uint32_t *mask_out,
                      void *stream) {
    SALE_ENTER(ctx);
    int st;
    if ((st = check_shape(ctx, shape))) return st;
    if ((st = check_config(ctx, cfg))) return st;
    if ((st = check_taus(ctx, taus, shape->q_heads))) return st;
    if (!q || !k || !v || !out) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    Workspace w;
    if ((st = ensure_workspace(ctx, *shape, &w))) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t *mask = mask_out ? mask_out : w.mask;
    if ((st = ws_begin(ctx, s))) return st;
    mark(ctx, 0, s);
    SALE_CUDA(ctx, launch_quantize_qk(q, k, w.q_codes, w.q_scales, w.k_codes, w.k_scales,
                                      shape->batch, shape->tokens, shape->q_heads,
                                      shape->kv_heads, s));
    mark(ctx, 1, s);
    if ((st = select_impl(ctx, q, k, w.q_codes, w.q_scales, w.k_codes, w.k_scales, *shape, taus,
                          geometry(cfg, shape->tokens), mask, w.thresh, nullptr, s)))
        return st;
    // The Selection-Pass always keeps the sink block (selection.hpp:228-232),
    // which every row attends (token 0), so no row can be empty here.
    if ((st = attention_impl(ctx, q, k, v, *shape, mask, out, nullptr, s))) return st;
    return ws_end(ctx, s);
}

// A query-block range [i_lo, i_hi) of the prefill (one GPU's share when a
// (batch, KV group) is split across GPUs): K is quantized for
// every key the range attends ([0, t_hi)), Q only for the range's rows; the
// mask and output rows of the range are written, other rows are untouched.
// Boundaries are 0, nq or odd (estimator tiles pair query blocks 2m+1, 2m+2).
static int check_range(sale_b200_ctx *ctx, const sale_b200_shape *shape, int64_t i_lo, int64_t i_hi) {
    const int64_t nq = cdiv(shape->tokens, kBlockQ);
    if (i_lo < 0 || i_hi > nq || i_lo >= i_hi)
        return fail(ctx, SALE_B200_INVALID_ARGUMENT, "query-block range outside [0, nq)");
    if ((i_lo != 0 && (i_lo & 1) == 0) || (i_hi != nq && (i_hi & 1) == 0))
        return fail(ctx, SALE_B200_INVALID_ARGUMENT,
                    "query-block range boundaries must be 0, nq or odd");
    return SALE_B200_OK;
}

int sale_b200_prefill_range(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                            const sale_b200_shape *shape, const double *taus,
                            const sale_b200_selection_config *cfg, int64_t i_lo, int64_t i_hi,
                            void *out, uint32_t *mask_out, void *stream) {
    SALE_ENTER(ctx);
    int st;
    if ((st = check_shape(ctx, shape))) return st;
    if ((st = check_config(ctx, cfg))) return st;
    if ((st = check_taus(ctx, taus, shape->q_heads))) return st;
    if ((st = check_range(ctx, shape, i_lo, i_hi))) return st;
    if (!q || !k || !v || !out) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    const sale_b200_shape sh = *shape;
    const int64_t B = sh.batch, N = sh.tokens, Hq = sh.q_heads, Hkv = sh.kv_heads;
    const int64_t nq = cdiv(N, kBlockQ);
    Workspace w;
    if ((st = ensure_workspace(ctx, sh, &w))) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t *mask = mask_out ? mask_out : w.mask;
    std::vector<int64_t> bounds(1, 0);
    if (i_lo > 0) bounds.push_back(i_lo);
    if (i_hi < nq) bounds.push_back(i_hi);
    bounds.push_back(nq);
    const size_t grp = i_lo > 0 ? 1 : 0; // the unit group of [i_lo, i_hi)
    if ((st = ws_begin(ctx, s))) return st;
    if ((st = upload_taus(ctx, taus, Hq, s))) return st;
    const Geom geo = geometry(cfg, N);
    if ((st = ensure_chunk_units(ctx, N, geo, bounds, s))) return st;
    const int64_t t0 = i_lo * kBlockQ, t1 = std::min<int64_t>(i_hi * kBlockQ, N);
    mark(ctx, 0, s);
    SALE_CUDA(ctx, launch_quantize_qk(nullptr, k, nullptr, nullptr, w.k_codes, w.k_scales, B, N, Hq,
                                      Hkv, s, 0, t1));
    SALE_CUDA(ctx, launch_quantize_qk(q, nullptr, w.q_codes, w.q_scales, nullptr, nullptr, B, N, Hq,
                                      Hkv, s, t0, t1));
    mark(ctx, 1, s);
    const float isd = inv_sqrt_dim(sh.head_dim);
    SALE_CUDA(ctx, launch_base_mask(mask, B, Hq, N, geo, s, i_lo, i_hi));
    mark(ctx, 2, s);
    SALE_CUDA(ctx, launch_sink_local_stats(q, k, B, N, Hq, Hkv, isd, geo, ctx->d_taus, w.thresh, nullptr,
                                           nullptr, nullptr, s, i_lo, i_hi));
    mark(ctx, 3, s);
    const int64_t u0 = ctx->cunit_off[grp], u1 = ctx->cunit_off[grp + 1];
    if (u1 > u0) {
        CUtensorMap tm_qc, tm_kc;
        if ((st = make_map(ctx, &tm_qc, w.q_codes, false, B, N, Hq, 128, 128))) return st;
        if ((st = make_map(ctx, &tm_kc, w.k_codes, false, B, N, Hkv, 128, 128))) return st;
        SALE_CUDA(ctx, launch_estimate(tm_qc, tm_kc, ctx->d_cunits + u0, u1 - u0, w.q_scales,
                                       w.k_scales, w.thresh, mask, B, N, static_cast<int>(Hq),
                                       static_cast<int>(Hkv), isd, geo, nullptr, s));
        SALE_CUDA(ctx, launch_segment_or(mask, B, Hq, N, geo, s, i_lo, i_hi));
    }
    mark(ctx, 4, s);
    if ((st = attention_impl(ctx, q, k, v, sh, mask, out, nullptr, s, i_lo, i_hi))) return st;
    return ws_end(ctx, s);
}

int sale_b200_sparse_attention_range(sale_b200_ctx *ctx, const void *q, const void *k,
                                     const void *v, const sale_b200_shape *shape,
                                     const uint32_t *mask_words, int64_t i_lo, int64_t i_hi,
                                     void *out, int32_t *coverage, void *stream) {
    SALE_ENTER(ctx);
    int st;
    if ((st = check_shape(ctx, shape))) return st;
    if ((st = check_range(ctx, shape, i_lo, i_hi))) return st;
    if (!q || !k || !v || !out) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!mask_words) return attention_impl(ctx, q, k, v, *shape, nullptr, out, coverage, s, i_lo, i_hi);
    if ((st = ws_begin(ctx, s)) || (st = empty_rows_begin(ctx, s))) return st;
    if ((st = attention_impl(ctx, q, k, v, *shape, mask_words, out, coverage, s, i_lo, i_hi,
                             ctx->d_empty)))
        return st;
    if ((st = ws_end(ctx, s))) return st;
    return empty_rows_end(ctx, s, shape->batch, shape->q_heads, shape->tokens);
}

int sale_b200_prefill_host(sale_b200_ctx *ctx, const uint16_t *q, const uint16_t *k,
                           const uint16_t *v, const sale_b200_shape *shape, const double *taus,
                           const sale_b200_selection_config *cfg, uint16_t *out) {
    SALE_ENTER(ctx);
    int st;
    if ((st = check_shape(ctx, shape))) return st;
    if ((st = check_config(ctx, cfg))) return st;
    if ((st = check_taus(ctx, taus, shape->q_heads))) return st;
    if (!q || !k || !v || !out) return fail(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    const sale_b200_shape s = *shape;
    const int64_t B = s.batch, N = s.tokens, Hq = s.q_heads, Hkv = s.kv_heads;
    const size_t qbytes = 2 * B * N * Hq * kHeadDim, kbytes = 2 * B * N * Hkv * kHeadDim;
    const size_t need = 2 * align256(qbytes) + 2 * align256(kbytes);
    if (need > ctx->io_bytes) {
        if (ctx->io) cudaFree(ctx->io);
        ctx->io = nullptr;
        ctx->io_bytes = 0;
        SALE_CUDA(ctx, cudaMalloc(&ctx->io, need));
        ctx->io_bytes = need;
        SALE_CUDA(ctx, cudaMemset(ctx->io, 0, need));
    }
    for (cudaStream_t *p : {&ctx->io_stream, &ctx->comp_stream, &ctx->out_stream, &ctx->attn_stream})
        if (!*p) SALE_CUDA(ctx, cudaStreamCreateWithFlags(p, cudaStreamNonBlocking));
    uint8_t *dq = ctx->io, *dk = dq + align256(qbytes), *dv = dk + align256(kbytes),
            *dout = dv + align256(kbytes);
    cudaStream_t s_in = ctx->io_stream, s_comp = ctx->comp_stream, s_out = ctx->out_stream,
                 s_attn = ctx->attn_stream;
    // The prefill in token chunks on four streams: the H2D copies (s_in) run
    // ahead; the Selection-Pass of chunk c (K1, base mask, K2a, K2b: s_comp)
    // waits for chunk c's copy; the attention of chunk c (s_attn) waits for
    // its mask, so it overlaps the Selection-Pass of chunk c+1 (their CTAs
    // fill each other's tail waves); the D2H of chunk c (s_out) follows its
    // attention. Every stage reads
    // only data of its own and earlier chunks (causal): the attention's last
    // 128-key K / V tile may extend past the chunk end t1 (into rows the H2D of
    // chunk c+1 is still writing), so chunk c's K / V tensor maps end at t1 and
    // TMA fills those rows with zeros (their P is 0; stale data there could be
    // NaN, and 0 * NaN would poison the row). The result is bit-identical to the
    // one-shot sale_b200_prefill.
    const int64_t nq = cdiv(N, kBlockQ);
    const std::vector<int64_t> bounds =
        N >= 65536 ? chunk_bounds_long(nq) : chunk_bounds(nq, N >= 16384 ? 8 : (N >= 2048 ? 4 : 1));
    const size_t nch = bounds.size() - 1;
    Workspace w;
    if ((st = ensure_workspace(ctx, s, &w))) return st;
    if ((st = ws_begin(ctx, s_comp))) return st;
    if ((st = upload_taus(ctx, taus, Hq, s_comp))) return st;
    const Geom geo = geometry(cfg, N);
    if ((st = ensure_chunk_units(ctx, N, geo, bounds, s_comp))) return st;
    CUtensorMap tm_qc, tm_kc;
    if ((st = make_map(ctx, &tm_qc, w.q_codes, false, B, N, Hq, 128, 128))) return st;
    if ((st = make_map(ctx, &tm_kc, w.k_codes, false, B, N, Hkv, 128, 128))) return st;
    const float isd = inv_sqrt_dim(s.head_dim);
    const float scale_log2 = isd * 1.4426950408889634f;
    std::vector<cudaEvent_t> ev(3 * nch); // per chunk: copied in, selected, attended
    for (auto &e : ev) SALE_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct EvFree {
        std::vector<cudaEvent_t> &e;
        ~EvFree() {
            for (auto x : e) cudaEventDestroy(x);
        }
    } ev_free{ev};
    auto copy_rows = [&](void *dst, const void *src, int64_t heads, int64_t t0, int64_t t1,
                         cudaMemcpyKind kind, cudaStream_t st_) -> cudaError_t {
        const size_t row = static_cast<size_t>(heads) * kHeadDim * 2; // bytes per token
        const size_t off = static_cast<size_t>(t0) * row, pitch = static_cast<size_t>(N) * row;
        return cudaMemcpy2DAsync(static_cast<uint8_t *>(dst) + off, pitch,
                                 static_cast<const uint8_t *>(src) + off, pitch,
                                 static_cast<size_t>(t1 - t0) * row, static_cast<size_t>(B), kind, st_);
    };
    for (size_t c = 0; c < nch; ++c) {
        const int64_t i0 = bounds[c], i1 = bounds[c + 1];
        const int64_t t0 = i0 * kBlockQ, t1 = std::min<int64_t>(i1 * kBlockQ, N);
        SALE_CUDA(ctx, copy_rows(dq, q, Hq, t0, t1, cudaMemcpyHostToDevice, s_in));
        SALE_CUDA(ctx, copy_rows(dk, k, Hkv, t0, t1, cudaMemcpyHostToDevice, s_in));
        SALE_CUDA(ctx, copy_rows(dv, v, Hkv, t0, t1, cudaMemcpyHostToDevice, s_in));
        SALE_CUDA(ctx, cudaEventRecord(ev[3 * c], s_in));
        SALE_CUDA(ctx, cudaStreamWaitEvent(s_comp, ev[3 * c], 0));
        SALE_CUDA(ctx, launch_quantize_qk(dq, dk, w.q_codes, w.q_scales, w.k_codes, w.k_scales, B, N,
                                          Hq, Hkv, s_comp, t0, t1));
        SALE_CUDA(ctx, launch_base_mask(w.mask, B, Hq, N, geo, s_comp, i0, i1));
        SALE_CUDA(ctx, launch_sink_local_stats(dq, dk, B, N, Hq, Hkv, isd, geo, ctx->d_taus, w.thresh,
                                               nullptr, nullptr, nullptr, s_comp, i0, i1));
        const int64_t u0 = ctx->cunit_off[c], u1 = ctx->cunit_off[c + 1];
        if (u1 > u0)
            SALE_CUDA(ctx, launch_estimate(tm_qc, tm_kc, ctx->d_cunits + u0, u1 - u0, w.q_scales,
                                           w.k_scales, w.thresh, w.mask, B, N, static_cast<int>(Hq),
                                           static_cast<int>(Hkv), isd, geo, nullptr, s_comp));
        SALE_CUDA(ctx, launch_segment_or(w.mask, B, Hq, N, geo, s_comp, i0, i1));
        SALE_CUDA(ctx, cudaEventRecord(ev[3 * c + 1], s_comp));
        SALE_CUDA(ctx, cudaStreamWaitEvent(s_attn, ev[3 * c + 1], 0));
        CUtensorMap tk, tv; // K / V rows [0, t1) of the [B][N][Hkv][128] layout
        if ((st = make_map(ctx, &tk, dk, true, B, N, Hkv, 64, 128, t1))) return st;
        if ((st = make_map(ctx, &tv, dv, true, B, N, Hkv, 64, 128, t1))) return st;
        SALE_CUDA(ctx, launch_sparse_attention(dq, tk, tv, w.mask, dout, nullptr, B, N,
                                               static_cast<int>(Hq), static_cast<int>(Hkv),
                                               scale_log2, s_attn, i0, i1));
        SALE_CUDA(ctx, cudaEventRecord(ev[3 * c + 2], s_attn));
        SALE_CUDA(ctx, cudaStreamWaitEvent(s_out, ev[3 * c + 2], 0));
        SALE_CUDA(ctx, copy_rows(out, dout, Hq, t0, t1, cudaMemcpyDeviceToHost, s_out));
    }
    SALE_CUDA(ctx, cudaStreamSynchronize(s_out));
    SALE_CUDA(ctx, cudaStreamSynchronize(s_attn));
    SALE_CUDA(ctx, cudaStreamSynchronize(s_comp));
    return ws_end(ctx, s_comp);
}

} // extern "C"
