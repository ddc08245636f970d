// stats.cu — K2a: exact sink-local statistics and the per-row log-domain
// threshold, plus the base (always-computed) mask rows.
//
// Reproduces compute_sink_local_stats (selection.hpp:129-163) and
// threshold_bound (selection.hpp:168-173) bit-for-bit on bf16-valued inputs:
//   s_t   = fl32(dot_seq(q, k_t)) * inv_sqrt_d   — an FFMA chain over c = 0..d-1
//           (bf16 x bf16 products are exact in fp32, so FFMA == MUL+ADD)
//   m     = running max in double, in I_SL block order
//   sum_b = sequential double sum of exp(double(s_t) - m_b) over block b
//   l     = l * exp(m_old - m_new) + sum_b      — __dmul_rn/__dadd_rn, never fused
//   bound = m + log(max(tau * l, DBL_MIN))
// The only non-bit-exact element is CUDA's double exp/log (<= 1 ulp) vs glibc;
// see DESIGN.md "Parity" for why that cannot flip a mask bit in practice.
// K2b compares float estimates against fb = the smallest float >= bound, which
// is exactly equivalent to the reference's (double)est >= bound.
#include "common.cuh"

#include <cfloat>

namespace sale_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxSlBlocks = 7;                  // {0} U [2i-4, 2i+1]
constexpr int kMaxKeys = kMaxSlBlocks * kBlockK; // 224
constexpr int kKeyPitch = kMaxKeys;              // kT[c][t]
constexpr int kRows = kBlockQ;                   // 64

struct StatsSmem {
    union {
        struct {
            float qT[kHeadDim][kRows];     // 32 KB
            float kT[kHeadDim][kKeyPitch]; // 112 KB
        } in;
        double e[kRows][kMaxKeys];         // 112 KB (exp terms)
    } u;
    float logit[kRows][kMaxKeys];          // 56 KB
    double mblk[kRows][kMaxSlBlocks];      // running max after each block
    int blk_id[kMaxSlBlocks];
    int blk_len[kMaxSlBlocks];
};

__device__ __forceinline__ void bf16x8_to_f32(const uint4 &u, float *f) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

// grid: (nq - 3, heads, batch) — query blocks i >= 3 (non-empty middle).
__global__ void __launch_bounds__(kThreads, 1)
sink_local_stats_kernel(const __nv_bfloat16 *__restrict__ q, const __nv_bfloat16 *__restrict__ k,
                        int64_t tokens, int64_t hq, int64_t hkv, float inv_sqrt_d,
                        const double *__restrict__ taus, float *__restrict__ thresh,
                        double *__restrict__ dbg_m, double *__restrict__ dbg_l,
                        double *__restrict__ dbg_bound) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    StatsSmem &sm = *reinterpret_cast<StatsSmem *>(smem_raw);
    const int tid = threadIdx.x;
    const int64_t i = blockIdx.x + 3;
    const int64_t h = blockIdx.y;
    const int64_t b = blockIdx.z;
    const int64_t g = h / (hq / hkv);
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    const int64_t q0 = i * kBlockQ;
    const int64_t qrows = (q0 + kBlockQ <= tokens) ? kBlockQ : tokens - q0;
    const int64_t frontier = frontier_block(i, tokens, nk);

    // I_SL (selection.hpp:92-123) for the default geometry: {0} U [2i-4, frontier].
    const int nsl = static_cast<int>(1 + frontier - (2 * i - 4) + 1);
    if (tid < kMaxSlBlocks) {
        int id = -1, len = 0;
        if (tid < nsl) {
            id = tid == 0 ? 0 : static_cast<int>(2 * i - 4 + tid - 1);
            const int64_t kb = static_cast<int64_t>(id) * kBlockK;
            len = static_cast<int>((kb + kBlockK <= tokens) ? kBlockK : tokens - kb);
        }
        sm.blk_id[tid] = id;
        sm.blk_len[tid] = len;
    }

    // ---- stage Q (64 rows) and the <= 224 keys transposed into smem (fp32)
    for (int idx = tid; idx < kRows * (kHeadDim / 8); idx += kThreads) {
        const int r = idx % kRows, ch = idx / kRows;
        float f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (r < qrows) {
            const uint4 u = __ldg(reinterpret_cast<const uint4 *>(
                                      q + ((b * tokens + q0 + r) * hq + h) * kHeadDim) +
                                  ch);
            bf16x8_to_f32(u, f);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) sm.u.in.qT[ch * 8 + e][r] = f[e];
    }
    for (int idx = tid; idx < kMaxKeys * (kHeadDim / 8); idx += kThreads) {
        const int t = idx % kMaxKeys, ch = idx / kMaxKeys;
        const int slot = t / kBlockK, tt = t % kBlockK;
        float f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (slot < nsl) {
            const int64_t tok = (slot == 0 ? 0 : (2 * i - 4 + slot - 1) * kBlockK) + tt;
            if (tok < tokens) {
                const uint4 u = __ldg(reinterpret_cast<const uint4 *>(
                                          k + ((b * tokens + tok) * hkv + g) * kHeadDim) +
                                      ch);
                bf16x8_to_f32(u, f);
            }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) sm.u.in.kT[ch * 8 + e][t] = f[e];
    }
    __syncthreads();

    // ---- fp32 logits: thread = 4 rows x 14 keys, sequential over c.
    {
        const int rg = tid / 16, kg = tid % 16;
        float acc[4][14];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int j = 0; j < 14; ++j) acc[a][j] = 0.0f;
#pragma unroll 2
        for (int c = 0; c < kHeadDim; ++c) {
            const float4 qv = *reinterpret_cast<const float4 *>(&sm.u.in.qT[c][rg * 4]);
            float kv[14];
#pragma unroll
            for (int j = 0; j < 14; ++j) kv[j] = sm.u.in.kT[c][kg + 16 * j];
#pragma unroll
            for (int j = 0; j < 14; ++j) {
                acc[0][j] = __fmaf_rn(qv.x, kv[j], acc[0][j]);
                acc[1][j] = __fmaf_rn(qv.y, kv[j], acc[1][j]);
                acc[2][j] = __fmaf_rn(qv.z, kv[j], acc[2][j]);
                acc[3][j] = __fmaf_rn(qv.w, kv[j], acc[3][j]);
            }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int j = 0; j < 14; ++j)
                sm.logit[rg * 4 + a][kg + 16 * j] = __fmul_rn(acc[a][j], inv_sqrt_d);
    }
    __syncthreads();

    // ---- running max per (row, block) in I_SL order
    if (tid < kRows) {
        double m = -INFINITY;
        for (int s = 0; s < nsl; ++s) {
            double bm = -INFINITY;
            for (int t = 0; t < sm.blk_len[s]; ++t)
                bm = fmax(bm, static_cast<double>(sm.logit[tid][s * kBlockK + t]));
            m = fmax(m, bm);
            sm.mblk[tid][s] = m;
        }
    }
    __syncthreads();

    // ---- exp terms, all threads (the u.in staging area is dead now)
    for (int idx = tid; idx < kRows * kMaxKeys; idx += kThreads) {
        const int r = idx / kMaxKeys, t = idx % kMaxKeys;
        const int s = t / kBlockK;
        double e = 0.0;
        if (s < nsl && (t % kBlockK) < sm.blk_len[s])
            e = exp(static_cast<double>(sm.logit[r][t]) - sm.mblk[r][s]);
        sm.u.e[r][t] = e;
    }
    __syncthreads();

    // ---- sequential combination per row + bound
    if (tid < qrows) {
        const int r = tid;
        double l = 0.0, m_old = -INFINITY;
        for (int s = 0; s < nsl; ++s) {
            const double m_new = sm.mblk[r][s];
            double sum = 0.0;
            for (int t = 0; t < sm.blk_len[s]; ++t) sum = __dadd_rn(sum, sm.u.e[r][s * kBlockK + t]);
            l = __dadd_rn(__dmul_rn(l, exp(m_old - m_new)), sum);
            m_old = m_new;
        }
        const double tau = taus[h];
        double scaled = __dmul_rn(tau, l);
        if (scaled < DBL_MIN) scaled = DBL_MIN;
        const double bound = __dadd_rn(m_old, log(scaled));
        const int64_t o = (b * hq + h) * tokens + q0 + r;
        thresh[o] = __double2float_ru(bound);
        if (dbg_m) {
            dbg_m[o] = m_old;
            dbg_l[o] = l;
            dbg_bound[o] = bound;
        }
    }
}

// Base mask rows: I_SL U trailing partial run, i.e. {0} U [1 + 4 F_i, frontier]
// for i >= 3 and every causal block for i <= 2 (selection.hpp:228-245, :188).
// One thread per 32-bit word. Middle segments are OR-ed in by K2b.
__global__ void base_mask_kernel(uint32_t *__restrict__ mask, int64_t rows, int64_t nq,
                                 int64_t nk, int64_t words, int64_t tokens) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= rows * words) return;
    const int64_t w = idx % words;
    const int64_t i = (idx / words) % nq;
    const int64_t fr = frontier_block(i, tokens, nk);
    const int64_t lo = i >= 3 ? 1 + kSegment * full_segments(i) : 0;
    uint32_t bits = 0;
    for (int e = 0; e < 32; ++e) {
        const int64_t j = w * 32 + e;
        if (j == 0 || (j >= lo && j <= fr)) bits |= 1u << e;
    }
    mask[idx] = bits;
}

} // namespace

cudaError_t launch_sink_local_stats(const void *q, const void *k, int64_t batch, int64_t tokens,
                                    int64_t hq, int64_t hkv, float inv_sqrt_d, const double *taus,
                                    float *thresh, double *dbg_m, double *dbg_l, double *dbg_bound,
                                    cudaStream_t stream) {
    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    if (nq <= 3) return cudaSuccess;
    static bool configured = false;
    const size_t smem = sizeof(StatsSmem);
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(sink_local_stats_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid(static_cast<unsigned>(nq - 3), static_cast<unsigned>(hq),
              static_cast<unsigned>(batch));
    sink_local_stats_kernel<<<grid, kThreads, smem, stream>>>(
        static_cast<const __nv_bfloat16 *>(q), static_cast<const __nv_bfloat16 *>(k), tokens, hq,
        hkv, inv_sqrt_d, taus, thresh, dbg_m, dbg_l, dbg_bound);
    return cudaGetLastError();
}

cudaError_t launch_base_mask(uint32_t *mask, int64_t batch, int64_t hq, int64_t tokens,
                             cudaStream_t stream) {
    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    const int64_t words = (nk + 31) / 32;
    const int64_t total = batch * hq * nq * words;
    const int threads = 256;
    const int64_t blocks = (total + threads - 1) / threads;
    base_mask_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(mask, batch * hq * nq,
                                                                           nq, nk, words, tokens);
    return cudaGetLastError();
}

} // namespace sale_b200
