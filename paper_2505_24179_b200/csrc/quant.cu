// quant.cu — K1: fused 4-bit symmetric quantizer for Q (per token) and K (per
// 32-token key block) in ONE launch. Memory-bound: reads bf16 once, writes the
// int8 codes and fp32 scales once (3 B + scale per element).
//
// Bit-exact with the reference (quant.hpp:68-119):
//   peak  = max |x| over the group                          (exact)
//   scale = peak > 0 ? peak / 7.0f : 1.0f                     (__fdiv_rn, quant.hpp:99/114)
//   code  = clamp(lround((double)x / (double)scale), -7, 7)   (quant.hpp:83-86)
// The double division is replaced by an exact comparison: |x| rounds up to
// k+1 iff 2|x| >= (2k+1)*scale, evaluated as the sign of one fmaf (a single
// rounding of an exact value cannot change its sign). Because x and scale
// have <= 24-bit significands the true quotient is never within 2^-28 relative
// of a .5 tie unless it IS a tie, so lround(fl64(x/s)) equals this exact
// half-away-from-zero rounding.
#include "common.cuh"

namespace sale_b200 {

namespace {

__device__ __forceinline__ int8_t quantize_one(float x, float scale, float inv_scale) {
    const float a = fabsf(x);
    int k = static_cast<int>(a * inv_scale + 0.5f);
    k = k > 7 ? 7 : k;
    if (k > 0 && fmaf(static_cast<float>(2 * k - 1), scale, -2.0f * a) > 0.0f) {
        --k; // a < (k - 1/2) * scale
    } else if (k < 7 && fmaf(static_cast<float>(2 * k + 1), scale, -2.0f * a) <= 0.0f) {
        ++k; // a >= (k + 1/2) * scale: ties go away from zero
    }
    return static_cast<int8_t>(x < 0.0f ? -k : k);
}

__device__ __forceinline__ void unpack8(const uint4 &u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

__device__ __forceinline__ uint2 pack8(const int8_t (&c)[8]) {
    uint2 r;
    r.x = (uint32_t)(uint8_t)c[0] | ((uint32_t)(uint8_t)c[1] << 8) |
          ((uint32_t)(uint8_t)c[2] << 16) | ((uint32_t)(uint8_t)c[3] << 24);
    r.y = (uint32_t)(uint8_t)c[4] | ((uint32_t)(uint8_t)c[5] << 8) |
          ((uint32_t)(uint8_t)c[6] << 16) | ((uint32_t)(uint8_t)c[7] << 24);
    return r;
}

__device__ __forceinline__ float scale_of(float peak) {
    return peak > 0.0f ? __fdiv_rn(peak, 7.0f) : 1.0f;
}

constexpr int kThreads = 256;
constexpr int kRowsPerCta = 16;   // Q: 16 lanes x 8 elements per 128-wide row
constexpr int kLanesPerRow = 16;

// One CTA = 16 Q rows (consecutive (b, n, h) rows) or one K group
// (b, key block j, kv head h): 32 rows x 128, 16 elements per thread.
__global__ void __launch_bounds__(kThreads)
quantize_qk_kernel(const __nv_bfloat16 *__restrict__ q, const __nv_bfloat16 *__restrict__ k,
                   int8_t *__restrict__ q_codes, float *__restrict__ q_scales,
                   int8_t *__restrict__ k_codes, float *__restrict__ k_scales, int64_t batch,
                   int64_t tokens, int64_t hq, int64_t hkv, int64_t q_ctas) {
    const int tid = threadIdx.x;
    if (blockIdx.x < q_ctas) {
        const int64_t q_rows = batch * tokens * hq;
        const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + tid / kLanesPerRow;
        const int sub = tid % kLanesPerRow;
        float f[8];
        float peak = 0.0f;
        if (row < q_rows) {
            const uint4 u = __ldcs(reinterpret_cast<const uint4 *>(q + row * kHeadDim) + sub);
            unpack8(u, f);
#pragma unroll
            for (int i = 0; i < 8; ++i) peak = fmaxf(peak, fabsf(f[i]));
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) peak = fmaxf(peak, __shfl_xor_sync(0xffffffffu, peak, o));
        if (row >= q_rows) return;
        const float scale = scale_of(peak);
        const float inv = 1.0f / scale;
        int8_t c[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = quantize_one(f[i], scale, inv);
        __stcs(reinterpret_cast<uint2 *>(q_codes + row * kHeadDim) + sub, pack8(c));
        if (sub == 0) {
            // row = (b*N + n)*Hq + h  ->  scales[b][h][n]
            const int64_t h = row % hq;
            const int64_t bn = row / hq;
            const int64_t b = bn / tokens, n = bn % tokens;
            q_scales[(b * hq + h) * tokens + n] = scale;
        }
        return;
    }
    // ---- K group
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    const int64_t grp = static_cast<int64_t>(blockIdx.x) - q_ctas;
    const int64_t h = grp % hkv;
    const int64_t j = (grp / hkv) % nk;
    const int64_t b = grp / (hkv * nk);
    const int r = tid >> 3;         // token within the block (0..31)
    const int sub = (tid & 7) * 2;  // two 8-element chunks: 16 elements
    const int64_t tok = j * kBlockK + r;
    const bool valid = tok < tokens;
    const int64_t row = (b * tokens + tok) * hkv + h;
    float f0[8], f1[8];
    float peak = 0.0f;
    if (valid) {
        const uint4 *src = reinterpret_cast<const uint4 *>(k + row * kHeadDim) + sub;
        unpack8(__ldcs(src), f0);
        unpack8(__ldcs(src + 1), f1);
#pragma unroll
        for (int i = 0; i < 8; ++i) peak = fmaxf(peak, fmaxf(fabsf(f0[i]), fabsf(f1[i])));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) peak = fmaxf(peak, __shfl_xor_sync(0xffffffffu, peak, o));
    __shared__ float warp_peak[kThreads / 32];
    if ((tid & 31) == 0) warp_peak[tid >> 5] = peak;
    __syncthreads();
    peak = warp_peak[0];
#pragma unroll
    for (int w = 1; w < kThreads / 32; ++w) peak = fmaxf(peak, warp_peak[w]);
    const float scale = scale_of(peak);
    const float inv = 1.0f / scale;
    if (valid) {
        int8_t c0[8], c1[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            c0[i] = quantize_one(f0[i], scale, inv);
            c1[i] = quantize_one(f1[i], scale, inv);
        }
        uint2 *dst = reinterpret_cast<uint2 *>(k_codes + row * kHeadDim) + sub;
        __stcs(dst, pack8(c0));
        __stcs(dst + 1, pack8(c1));
    }
    if (tid == 0) k_scales[(b * hkv + h) * nk + j] = scale;
}

} // namespace

cudaError_t launch_quantize_qk(const void *q, const void *k, int8_t *q_codes, float *q_scales,
                               int8_t *k_codes, float *k_scales, int64_t batch, int64_t tokens,
                               int64_t hq, int64_t hkv, cudaStream_t stream) {
    const int64_t q_rows = q ? batch * tokens * hq : 0;
    const int64_t q_ctas = (q_rows + kRowsPerCta - 1) / kRowsPerCta;
    const int64_t k_ctas = k ? batch * ((tokens + kBlockK - 1) / kBlockK) * hkv : 0;
    const int64_t grid = q_ctas + k_ctas;
    if (grid == 0) return cudaSuccess;
    if (grid > 0x7FFFFFFF) return cudaErrorInvalidValue;
    quantize_qk_kernel<<<static_cast<unsigned>(grid), kThreads, 0, stream>>>(
        static_cast<const __nv_bfloat16 *>(q), static_cast<const __nv_bfloat16 *>(k), q_codes,
        q_scales, k_codes, k_scales, batch, tokens, hq, hkv, q_ctas);
    return cudaGetLastError();
}

} // namespace sale_b200
