// pipeline.cu — the orchestration layer above the three stages, on device:
// run_pipeline (runner.hpp:37-108), sweep_thresholds (runner.hpp:119-165) and
// the calibration ladder calibrate_head / calibrate_model (calibrate.hpp:
// 121-175), with l1_error (calibrate.hpp:20-29) and the coverage statistics of
// a RunReport as device reductions. Every head of every batch runs in the same
// launches (per-head taus), so a calibration rung is one selection + one sparse
// pass for the whole model instead of a CPU loop over heads.
//
// The composition goes through the public C ABI (quantize / select / sparse
// attention / flop count), so these entry points add no second copy of the
// stage logic. Host file formats live in formats.cpp.
#include "sale_b200.h"

#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

namespace sale_b200 {

namespace {

constexpr int kL1Threads = 256;
constexpr int kL1Rows = 64; // rows per CTA; 4 threads per row, 32 channels each

// partial[bh][chunk] = sum over the chunk's rows of sum_{c < d} |ref - approx|,
// in double, reduced in a fixed order (deterministic).
__global__ void __launch_bounds__(kL1Threads)
l1_partial_kernel(const __nv_bfloat16 *__restrict__ ref, const __nv_bfloat16 *__restrict__ approx,
                  int64_t tokens, int64_t heads, int head_dim, int64_t nchunks,
                  double *__restrict__ partial) {
    const int64_t bh = blockIdx.y;
    const int64_t b = bh / heads, h = bh % heads;
    const int r = threadIdx.x >> 2, part = threadIdx.x & 3;
    const int64_t n = static_cast<int64_t>(blockIdx.x) * kL1Rows + r;
    double acc = 0.0;
    if (n < tokens) {
        const int64_t off = ((b * tokens + n) * heads + h) * kHeadDim + 32 * part;
#pragma unroll 4
        for (int c = 0; c < 32; ++c)
            if (32 * part + c < head_dim)
                acc += fabs(static_cast<double>(__bfloat162float(ref[off + c])) -
                            static_cast<double>(__bfloat162float(approx[off + c])));
    }
    __shared__ double red[kL1Threads];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kL1Threads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[bh * nchunks + blockIdx.x] = red[0];
}

__global__ void l1_final_kernel(const double *__restrict__ partial, int64_t nchunks, int64_t bhs,
                                int64_t tokens, double *__restrict__ out) {
    const int64_t bh = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (bh >= bhs) return;
    double s = 0.0;
    for (int64_t c = 0; c < nchunks; ++c) s += partial[bh * nchunks + c];
    out[bh] = s / static_cast<double>(tokens);
}

// out[bh] = {min, max, sum} of coverage[bh][0..N) (SparseAttentionOutput::coverage)
__global__ void __launch_bounds__(256)
coverage_stats_kernel(const int32_t *__restrict__ coverage, int64_t tokens, int64_t *__restrict__ out) {
    const int64_t bh = blockIdx.x;
    int64_t mn = INT64_MAX, mx = INT64_MIN, sum = 0;
    for (int64_t n = threadIdx.x; n < tokens; n += blockDim.x) {
        const int64_t v = coverage[bh * tokens + n];
        mn = v < mn ? v : mn;
        mx = v > mx ? v : mx;
        sum += v;
    }
    __shared__ int64_t smn[256], smx[256], ssum[256];
    smn[threadIdx.x] = mn, smx[threadIdx.x] = mx, ssum[threadIdx.x] = sum;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            smn[threadIdx.x] = min(smn[threadIdx.x], smn[threadIdx.x + s]);
            smx[threadIdx.x] = max(smx[threadIdx.x], smx[threadIdx.x + s]);
            ssum[threadIdx.x] += ssum[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[3 * bh] = smn[0];
        out[3 * bh + 1] = smx[0];
        out[3 * bh + 2] = ssum[0];
    }
}

int64_t cdiv64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Device buffers of one call, freed on scope exit.
struct Scratch {
    std::vector<void *> ptrs;
    ~Scratch() {
        for (void *p : ptrs) cudaFree(p);
    }
    template <class T> cudaError_t get(T **p, size_t bytes) {
        void *q = nullptr;
        cudaError_t e = cudaMalloc(&q, bytes < 256 ? 256 : bytes);
        if (e == cudaSuccess) ptrs.push_back(q);
        *p = static_cast<T *>(q);
        return e;
    }
};

#define PIPE_CUDA(ctx, call)                                                                       \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return set_error(ctx, SALE_B200_CUDA_ERROR, std::string(#call) + ": " +              \
                                                              cudaGetErrorString(e_));             \
    } while (0)
#define PIPE_OK(call)                                                                              \
    do {                                                                                           \
        int s_ = (call);                                                                           \
        if (s_ != SALE_B200_OK) return s_;                                                         \
    } while (0)

// Per-(batch, head) l1 errors of two bf16 outputs, to HOST out[B*Hq].
int l1_impl(sale_b200_ctx *ctx, const void *ref, const void *approx, const sale_b200_shape &s,
            double *host_out, cudaStream_t stream) {
    const int64_t bhs = s.batch * s.q_heads, nchunks = cdiv64(s.tokens, kL1Rows);
    Scratch sc;
    double *partial, *dev_out;
    PIPE_CUDA(ctx, sc.get(&partial, sizeof(double) * bhs * nchunks));
    PIPE_CUDA(ctx, sc.get(&dev_out, sizeof(double) * bhs));
    l1_partial_kernel<<<dim3(static_cast<unsigned>(nchunks), static_cast<unsigned>(bhs)), kL1Threads, 0,
                        stream>>>(static_cast<const __nv_bfloat16 *>(ref),
                                  static_cast<const __nv_bfloat16 *>(approx), s.tokens, s.q_heads,
                                  static_cast<int>(s.head_dim), nchunks, partial);
    PIPE_CUDA(ctx, cudaGetLastError());
    l1_final_kernel<<<static_cast<unsigned>(cdiv64(bhs, 128)), 128, 0, stream>>>(partial, nchunks, bhs,
                                                                                  s.tokens, dev_out);
    PIPE_CUDA(ctx, cudaGetLastError());
    PIPE_CUDA(ctx, cudaMemcpyAsync(host_out, dev_out, sizeof(double) * bhs, cudaMemcpyDeviceToHost, stream));
    PIPE_CUDA(ctx, cudaStreamSynchronize(stream));
    return SALE_B200_OK;
}

int check_common(sale_b200_ctx *ctx, const sale_b200_shape *shape, const void *q, const void *k,
                 const void *v) {
    if (!ctx) return SALE_B200_INVALID_ARGUMENT;
    if (!shape) return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "shape is NULL");
    if (!q || !k || !v) return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    return SALE_B200_OK;
}

// Quantized inputs + dense baseline of one sample (calibrate.hpp:84-96
// prepare_sample): tau-independent, computed once per sample.
struct Prepared {
    int8_t *qc = nullptr, *kc = nullptr;
    float *qs = nullptr, *ks = nullptr;
    void *dense = nullptr;
};

int prepare(sale_b200_ctx *ctx, Scratch &sc, const void *q, const void *k, const void *v,
            const sale_b200_shape &s, Prepared &p, cudaStream_t stream) {
    const int64_t nk = cdiv64(s.tokens, kBlockK);
    PIPE_CUDA(ctx, sc.get(&p.qc, s.batch * s.tokens * s.q_heads * kHeadDim));
    PIPE_CUDA(ctx, sc.get(&p.kc, s.batch * s.tokens * s.kv_heads * kHeadDim));
    PIPE_CUDA(ctx, sc.get(&p.qs, sizeof(float) * s.batch * s.q_heads * s.tokens));
    PIPE_CUDA(ctx, sc.get(&p.ks, sizeof(float) * s.batch * s.kv_heads * nk));
    PIPE_CUDA(ctx, sc.get(&p.dense, 2 * s.batch * s.tokens * s.q_heads * kHeadDim));
    PIPE_OK(sale_b200_quantize_qk(ctx, q, k, &s, p.qc, p.qs, p.kc, p.ks, stream));
    PIPE_OK(sale_b200_sparse_attention(ctx, q, k, v, &s, nullptr, p.dense, nullptr, stream));
    return SALE_B200_OK;
}

} // namespace
} // namespace sale_b200

using namespace sale_b200;

extern "C" {

int sale_b200_l1_error(sale_b200_ctx *ctx, const void *ref, const void *approx,
                       const sale_b200_shape *shape, double *out) {
    PIPE_OK(check_common(ctx, shape, ref, approx, ref));
    if (!out) return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    if (shape->batch < 1 || shape->tokens < 1 || shape->q_heads < 1 || shape->head_dim < 1 ||
        shape->head_dim > kHeadDim)
        return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "l1_error: shape mismatch");
    PIPE_CUDA(ctx, cudaSetDevice(ctx_device_of(ctx)));
    return l1_impl(ctx, ref, approx, *shape, out, nullptr);
}

int sale_b200_run_pipeline(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                           const sale_b200_shape *shape, const double *taus,
                           const sale_b200_selection_config *cfg, int dense_mask,
                           sale_b200_head_report *reports, sale_b200_stage_timing *timing) {
    PIPE_OK(check_common(ctx, shape, q, k, v));
    if (!taus || !reports) return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    PIPE_CUDA(ctx, cudaSetDevice(ctx_device_of(ctx)));
    const sale_b200_shape s = *shape;
    const int64_t bhs = s.batch * s.q_heads;
    const int64_t nq = cdiv64(s.tokens, kBlockQ), nk = cdiv64(s.tokens, kBlockK), words = cdiv64(nk, 32);
    cudaStream_t stream = nullptr;
    Scratch sc;
    Prepared p;
    uint32_t *mask;
    void *sparse;
    int32_t *coverage;
    int64_t *counts, *cov_stats;
    const int64_t nk_s = nk;
    (void)nk_s;
    PIPE_CUDA(ctx, sc.get(&p.qc, s.batch * s.tokens * s.q_heads * kHeadDim));
    PIPE_CUDA(ctx, sc.get(&p.kc, s.batch * s.tokens * s.kv_heads * kHeadDim));
    PIPE_CUDA(ctx, sc.get(&p.qs, sizeof(float) * bhs * s.tokens));
    PIPE_CUDA(ctx, sc.get(&p.ks, sizeof(float) * s.batch * s.kv_heads * nk));
    PIPE_CUDA(ctx, sc.get(&p.dense, 2 * s.batch * s.tokens * s.q_heads * kHeadDim));
    PIPE_CUDA(ctx, sc.get(&sparse, 2 * s.batch * s.tokens * s.q_heads * kHeadDim));
    PIPE_CUDA(ctx, sc.get(&mask, sizeof(uint32_t) * bhs * nq * words));
    PIPE_CUDA(ctx, sc.get(&coverage, sizeof(int32_t) * bhs * s.tokens));
    PIPE_CUDA(ctx, sc.get(&counts, sizeof(int64_t) * bhs * 3));
    PIPE_CUDA(ctx, sc.get(&cov_stats, sizeof(int64_t) * bhs * 3));
    cudaEvent_t ev[5];
    for (auto &e : ev) PIPE_CUDA(ctx, cudaEventCreate(&e));
    struct EvGuard {
        cudaEvent_t *e;
        ~EvGuard() {
            for (int i = 0; i < 5; ++i) cudaEventDestroy(e[i]);
        }
    } guard{ev};
    // the four timed stages of runner.hpp:63-85, each over every head at once
    PIPE_CUDA(ctx, cudaEventRecord(ev[0], stream));
    PIPE_OK(sale_b200_quantize_qk(ctx, q, k, &s, p.qc, p.qs, p.kc, p.ks, stream));
    PIPE_CUDA(ctx, cudaEventRecord(ev[1], stream));
    if (dense_mask) {
        PIPE_CUDA(ctx, cudaMemsetAsync(mask, 0xFF, sizeof(uint32_t) * bhs * nq * words, stream));
    } else {
        PIPE_OK(sale_b200_select(ctx, q, k, p.qc, p.qs, p.kc, p.ks, &s, taus, cfg, mask, nullptr, stream));
    }
    PIPE_CUDA(ctx, cudaEventRecord(ev[2], stream));
    PIPE_OK(sale_b200_sparse_attention(ctx, q, k, v, &s, mask, sparse, coverage, stream));
    PIPE_CUDA(ctx, cudaEventRecord(ev[3], stream));
    PIPE_OK(sale_b200_sparse_attention(ctx, q, k, v, &s, nullptr, p.dense, nullptr, stream));
    PIPE_CUDA(ctx, cudaEventRecord(ev[4], stream));
    PIPE_OK(sale_b200_flop_count(ctx, mask, s.batch, s.q_heads, s.tokens, counts, stream));
    coverage_stats_kernel<<<static_cast<unsigned>(bhs), 256, 0, stream>>>(coverage, s.tokens, cov_stats);
    PIPE_CUDA(ctx, cudaGetLastError());
    std::vector<double> err(bhs);
    PIPE_OK(l1_impl(ctx, p.dense, sparse, s, err.data(), stream));
    std::vector<int64_t> hc(bhs * 3), hs(bhs * 3);
    PIPE_CUDA(ctx, cudaMemcpy(hc.data(), counts, sizeof(int64_t) * bhs * 3, cudaMemcpyDeviceToHost));
    PIPE_CUDA(ctx, cudaMemcpy(hs.data(), cov_stats, sizeof(int64_t) * bhs * 3, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < bhs; ++i) {
        sale_b200_head_report &r = reports[i];
        r.head = i;
        r.tau = taus[i % s.q_heads];
        r.computed_blocks = hc[3 * i];
        r.skipped_blocks = hc[3 * i + 1];
        r.total_blocks = hc[3 * i + 2];
        // FlopCounts::sparsity (sparse_attention.hpp:26-29)
        r.sparsity = r.total_blocks ? static_cast<double>(r.skipped_blocks) / static_cast<double>(r.total_blocks) : 0.0;
        r.err = err[i];
        r.coverage_min = hs[3 * i];
        r.coverage_max = hs[3 * i + 1];
        r.coverage_mean = static_cast<double>(hs[3 * i + 2]) / static_cast<double>(s.tokens);
    }
    if (timing) {
        float ms[4];
        for (int i = 0; i < 4; ++i) PIPE_CUDA(ctx, cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
        timing->quantization_ms = ms[0];
        timing->selection_ms = ms[1];
        timing->computation_ms = ms[2];
        timing->dense_ms = ms[3];
    }
    return SALE_B200_OK;
}

int sale_b200_sweep_thresholds(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                               const sale_b200_shape *shape, const double *taus, int64_t n_taus,
                               const sale_b200_selection_config *cfg, sale_b200_sweep_row *rows) {
    PIPE_OK(check_common(ctx, shape, q, k, v));
    if (!taus || !rows) return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    if (n_taus < 1) return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "sweep_thresholds: empty grid");
    for (int64_t t = 0; t < n_taus; ++t)
        if (!(taus[t] > 0.0 && taus[t] < 1.0))
            return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "sweep_thresholds: tau outside (0,1)");
    PIPE_CUDA(ctx, cudaSetDevice(ctx_device_of(ctx)));
    const sale_b200_shape s = *shape;
    const int64_t bhs = s.batch * s.q_heads;
    const int64_t nq = cdiv64(s.tokens, kBlockQ), words = cdiv64(cdiv64(s.tokens, kBlockK), 32);
    cudaStream_t stream = nullptr;
    Scratch sc;
    Prepared p;
    PIPE_OK(prepare(ctx, sc, q, k, v, s, p, stream));
    uint32_t *mask;
    void *sparse;
    int64_t *counts;
    PIPE_CUDA(ctx, sc.get(&sparse, 2 * s.batch * s.tokens * s.q_heads * kHeadDim));
    PIPE_CUDA(ctx, sc.get(&mask, sizeof(uint32_t) * bhs * nq * words));
    PIPE_CUDA(ctx, sc.get(&counts, sizeof(int64_t) * bhs * 3));
    std::vector<double> tau_h(s.q_heads), err(bhs);
    std::vector<int64_t> hc(bhs * 3);
    for (int64_t t = 0; t < n_taus; ++t) {
        std::fill(tau_h.begin(), tau_h.end(), taus[t]);
        PIPE_OK(sale_b200_select(ctx, q, k, p.qc, p.qs, p.kc, p.ks, &s, tau_h.data(), cfg, mask, nullptr, stream));
        PIPE_OK(sale_b200_sparse_attention(ctx, q, k, v, &s, mask, sparse, nullptr, stream));
        PIPE_OK(sale_b200_flop_count(ctx, mask, s.batch, s.q_heads, s.tokens, counts, stream));
        PIPE_OK(l1_impl(ctx, p.dense, sparse, s, err.data(), stream));
        PIPE_CUDA(ctx, cudaMemcpy(hc.data(), counts, sizeof(int64_t) * bhs * 3, cudaMemcpyDeviceToHost));
        // runner.hpp:155-163: mean sparsity, max error over heads (head order)
        rows[t].tau = taus[t];
        rows[t].sparsity = 0.0;
        rows[t].err = 0.0;
        for (int64_t i = 0; i < bhs; ++i) {
            rows[t].sparsity += hc[3 * i + 2] ? static_cast<double>(hc[3 * i + 1]) / hc[3 * i + 2] : 0.0;
            rows[t].err = std::max(rows[t].err, err[i]);
        }
        rows[t].sparsity /= static_cast<double>(bhs);
    }
    return SALE_B200_OK;
}

int sale_b200_calibrate(sale_b200_ctx *ctx, const void *const *q_samples,
                        const void *const *k_samples, const void *const *v_samples,
                        int64_t n_samples, const sale_b200_shape *shape,
                        const sale_b200_calibration_settings *settings,
                        const sale_b200_selection_config *cfg, sale_b200_head_calibration *out) {
    if (!ctx) return SALE_B200_INVALID_ARGUMENT;
    if (!shape || !settings || !out) return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
    if (n_samples < 1 || !q_samples || !k_samples || !v_samples)
        return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "calibrate_model: no samples");
    // CalibrationSettings::validate (calibrate.hpp:61-67)
    if (!(settings->theta > 0.0))
        return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "CalibrationSettings: theta must be > 0");
    if (!(settings->tau0 > 0.0 && settings->tau0 < 1.0))
        return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "CalibrationSettings: tau0 must be in (0,1)");
    if (settings->max_halvings < 0)
        return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "CalibrationSettings: max_halvings must be >= 0");
    if (shape->batch != 1)
        return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "calibrate: samples carry batch 1 each");
    PIPE_CUDA(ctx, cudaSetDevice(ctx_device_of(ctx)));
    const sale_b200_shape s = *shape;
    const int64_t H = s.q_heads;
    const int64_t nq = cdiv64(s.tokens, kBlockQ), words = cdiv64(cdiv64(s.tokens, kBlockK), 32);
    cudaStream_t stream = nullptr;
    Scratch sc;
    std::vector<Prepared> prep(n_samples);
    for (int64_t i = 0; i < n_samples; ++i) {
        if (!q_samples[i] || !k_samples[i] || !v_samples[i])
            return set_error(ctx, SALE_B200_INVALID_ARGUMENT, "NULL buffer");
        PIPE_OK(prepare(ctx, sc, q_samples[i], k_samples[i], v_samples[i], s, prep[i], stream));
    }
    uint32_t *mask;
    void *sparse;
    PIPE_CUDA(ctx, sc.get(&sparse, 2 * s.tokens * H * kHeadDim));
    PIPE_CUDA(ctx, sc.get(&mask, sizeof(uint32_t) * H * nq * words));
    // the halving ladder, every head at its own tau (calibrate.hpp:134-144)
    std::vector<double> tau(H, settings->tau0), worst(H), err(H);
    std::vector<int> done(H, 0);
    for (int64_t h = 0; h < H; ++h) out[h] = {0, h, settings->tau0, 0, 0};
    for (int64_t rung = 0;; ++rung) {
        std::fill(worst.begin(), worst.end(), 0.0);
        for (int64_t i = 0; i < n_samples; ++i) {
            PIPE_OK(sale_b200_select(ctx, q_samples[i], k_samples[i], prep[i].qc, prep[i].qs, prep[i].kc,
                                     prep[i].ks, &s, tau.data(), cfg, mask, nullptr, stream));
            PIPE_OK(sale_b200_sparse_attention(ctx, q_samples[i], k_samples[i], v_samples[i], &s, mask,
                                               sparse, nullptr, stream));
            PIPE_OK(l1_impl(ctx, prep[i].dense, sparse, s, err.data(), stream));
            for (int64_t h = 0; h < H; ++h) worst[h] = std::max(worst[h], err[h]);
        }
        bool all = true;
        for (int64_t h = 0; h < H; ++h) {
            if (done[h]) continue;
            if (worst[h] <= settings->theta) {
                out[h] = {0, h, tau[h], 0, rung};
                done[h] = 1;
            } else if (rung == settings->max_halvings) {
                out[h] = {0, h, tau[h], 1, rung};
                done[h] = 1;
            } else {
                tau[h] *= 0.5; // converged heads keep their tau (their rows are unchanged)
                all = false;
            }
        }
        if (all) break;
    }
    return SALE_B200_OK;
}

} // extern "C"
