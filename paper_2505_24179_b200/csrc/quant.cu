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

// Code of one element as a float in [-7, 7] (exact integer). All float
// arithmetic on the FMA / ALU pipes, no branches and no float<->int
// conversions (quarter-rate XU pipe). k0 = rint(a * inv) is within one of the
// exact code (inv is only approximately 1/scale); the two fmaf signs decide
// the exact half-away-from-zero rounding: a < (k0 - 1/2) scale -> k0 - 1,
// a >= (k0 + 1/2) scale -> k0 + 1 (a single rounding of an exact value cannot
// change its sign). k0 = 0 never steps down (the bound is negative) and k0 = 7
// never steps up (a <= peak < 7.5 scale), so no clamps are needed.
__device__ __forceinline__ float set_le0(float v) {
    float r;
    asm("set.le.f32.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ float set_gt0(float v) {
    float r;
    asm("set.gt.f32.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ float quantize_one(float x, float scale, float inv_scale) {
    constexpr float kMagic = 12582912.0f; // 1.5 * 2^23: x + kMagic rounds x to an integer
    const float a = fabsf(x);
    const float k0 = fmaf(a, inv_scale, kMagic) - kMagic;
    const float dn = set_gt0(fmaf(k0 - 0.5f, scale, -a)); // k0 -+ 1/2 are exact
    const float up = set_le0(fmaf(k0 + 0.5f, scale, -a));
    const float k = (k0 + up) - dn;
    return __uint_as_float(__float_as_uint(k) | (__float_as_uint(x) & 0x80000000u));
}

// Codes as floats -> eight int8 bytes: c + kMagic holds the two's complement
// integer in its low mantissa bits; PRMT gathers the low bytes.
__device__ __forceinline__ uint2 pack8f(const float (&c)[8]) {
    constexpr float kMagic = 12582912.0f;
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = __float_as_uint(c[i] + kMagic);
    uint2 r;
    r.x = __byte_perm(__byte_perm(w[0], w[1], 0x0040), __byte_perm(w[2], w[3], 0x0040), 0x5410);
    r.y = __byte_perm(__byte_perm(w[4], w[5], 0x0040), __byte_perm(w[6], w[7], 0x0040), 0x5410);
    return r;
}

__device__ __forceinline__ void unpack8(const uint4 &u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

__device__ __forceinline__ float scale_of(float peak) {
    return peak > 0.0f ? __fdiv_rn(peak, 7.0f) : 1.0f;
}
// An approximate 1/scale is enough (k0 only has to be within one); scales
// below 2^-100 are handled by exact power-of-two rescaling of a and scale.
__device__ __forceinline__ float rcp_approx(float v) {
    float r;
    asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}

constexpr int kThreads = 256;
constexpr int kLanesPerRow = 8;   // Q: 8 lanes x 16 elements per 128-wide row
constexpr int kQSlots = 2;        // Q rows per 8-lane group in flight (2 x 2 x 16 B loads per thread)
constexpr int kQRowsPerCta = kThreads / kLanesPerRow * kQSlots; // 64

// CTAs [0, q_ctas): 64 consecutive Q rows ((b, n, h) order), every thread
// loading its four 16-byte chunks before any math (memory-level parallelism);
// CTAs [q_ctas, ...): one K group (b, key block j, kv head h) = 32 rows x 128,
// 16 elements per thread. Scales need only 32-bit index math (rows < 2^31).
__global__ void __launch_bounds__(kThreads)
quantize_qk_kernel(const __nv_bfloat16 *__restrict__ q, const __nv_bfloat16 *__restrict__ k,
                   int8_t *__restrict__ q_codes, float *__restrict__ q_scales,
                   int8_t *__restrict__ k_codes, float *__restrict__ k_scales, int64_t batch,
                   int64_t tokens, int64_t hq, int64_t hkv, int64_t q_ctas, int64_t t_lo,
                   int64_t t_hi) {
    const int tid = threadIdx.x;
    if (blockIdx.x < q_ctas) {
        // local Q rows (b, n in [t_lo, t_hi), h) -> global rows (b*N + n)*Hq + h,
        // all in 32-bit arithmetic (batch * tokens * hq < 2^31 is checked at
        // launch); the whole-sequence case is the identity map.
        const uint32_t hq32 = static_cast<uint32_t>(hq), n32 = static_cast<uint32_t>(tokens);
        const uint32_t span = static_cast<uint32_t>((t_hi - t_lo) * hq);
        const uint32_t q_rows = static_cast<uint32_t>(batch) * span;
        const bool whole = t_lo == 0 && t_hi == tokens;
        const uint32_t lo_rows = static_cast<uint32_t>(t_lo) * hq32, n_rows = n32 * hq32;
        const int sub = tid % kLanesPerRow;
        const uint32_t loc0 = blockIdx.x * static_cast<uint32_t>(kQRowsPerCta) + tid / kLanesPerRow;
        uint32_t row[kQSlots];
        uint4 u[kQSlots][2];
#pragma unroll
        for (int sl = 0; sl < kQSlots; ++sl) {
            const uint32_t loc = loc0 + sl * (kThreads / kLanesPerRow);
            uint32_t rr = loc;
            if (!whole) {
                const uint32_t bb = loc / span;
                rr = bb * n_rows + lo_rows + (loc - bb * span);
            }
            row[sl] = loc < q_rows ? rr : 0xFFFFFFFFu;
            const uint4 *src = reinterpret_cast<const uint4 *>(q + static_cast<int64_t>(rr) * kHeadDim) + 2 * sub;
            u[sl][0] = loc < q_rows ? __ldcs(src) : make_uint4(0, 0, 0, 0);
            u[sl][1] = loc < q_rows ? __ldcs(src + 1) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int sl = 0; sl < kQSlots; ++sl) {
            float f0[8], f1[8];
            unpack8(u[sl][0], f0);
            unpack8(u[sl][1], f1);
            float peak = 0.0f;
#pragma unroll
            for (int i = 0; i < 8; ++i) peak = fmaxf(peak, fmaxf(fabsf(f0[i]), fabsf(f1[i])));
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) peak = fmaxf(peak, __shfl_xor_sync(0xffffffffu, peak, o));
            if (row[sl] == 0xFFFFFFFFu) continue;
            const float scale = scale_of(peak);
            float sc = scale;
            if (scale < 7.8886091e-31f) { // 2^-100: rescale exactly by 2^64
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    f0[i] *= 18446744073709551616.0f;
                    f1[i] *= 18446744073709551616.0f;
                }
                sc *= 18446744073709551616.0f;
            }
            const float inv = rcp_approx(sc);
            float c0[8], c1[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                c0[i] = quantize_one(f0[i], sc, inv);
                c1[i] = quantize_one(f1[i], sc, inv);
            }
            uint2 *dst = reinterpret_cast<uint2 *>(q_codes + static_cast<int64_t>(row[sl]) * kHeadDim) + 2 * sub;
            __stcs(dst, pack8f(c0));
            __stcs(dst + 1, pack8f(c1));
            if (sub == 0) {
                // row = (b*N + n)*Hq + h  ->  scales[b][h][n]
                const uint32_t h = row[sl] % hq32, bn = row[sl] / hq32;
                const uint32_t b = bn / n32, n = bn - b * n32;
                q_scales[(static_cast<int64_t>(b) * hq + h) * tokens + n] = scale;
            }
        }
        return;
    }
    // ---- K group
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    const int64_t j_lo = t_lo / kBlockK, nj = (t_hi + kBlockK - 1) / kBlockK - j_lo;
    const uint32_t grp = static_cast<uint32_t>(static_cast<int64_t>(blockIdx.x) - q_ctas);
    const uint32_t hkv32 = static_cast<uint32_t>(hkv), nj32 = static_cast<uint32_t>(nj);
    const int64_t h = grp % hkv32;
    const int64_t j = j_lo + (grp / hkv32) % nj32;
    const int64_t b = grp / (hkv32 * nj32);
    const int r = tid >> 3;         // token within the block (0..31)
    const int sub = (tid & 7) * 2;  // two 8-element chunks: 16 elements
    const int64_t tok = j * kBlockK + r;
    const bool valid = tok < tokens;
    const int64_t row = (b * tokens + tok) * hkv + h;
    float f0[8], f1[8];
    float peak = 0.0f;
    if (valid) {
        const uint4 *src = reinterpret_cast<const uint4 *>(k + row * kHeadDim) + sub;
        const uint4 u0 = __ldcs(src), u1 = __ldcs(src + 1);
        unpack8(u0, f0);
        unpack8(u1, f1);
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
    if (valid) {
        float sc = scale;
        if (scale < 7.8886091e-31f) { // 2^-100: rescale exactly by 2^64
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                f0[i] *= 18446744073709551616.0f;
                f1[i] *= 18446744073709551616.0f;
            }
            sc *= 18446744073709551616.0f;
        }
        const float inv = rcp_approx(sc);
        float c0[8], c1[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            c0[i] = quantize_one(f0[i], sc, inv);
            c1[i] = quantize_one(f1[i], sc, inv);
        }
        uint2 *dst = reinterpret_cast<uint2 *>(k_codes + row * kHeadDim) + sub;
        __stcs(dst, pack8f(c0));
        __stcs(dst + 1, pack8f(c1));
    }
    if (tid == 0) k_scales[(b * hkv + h) * nk + j] = scale;
}

} // namespace

cudaError_t launch_quantize_qk(const void *q, const void *k, int8_t *q_codes, float *q_scales,
                               int8_t *k_codes, float *k_scales, int64_t batch, int64_t tokens,
                               int64_t hq, int64_t hkv, cudaStream_t stream, int64_t t_lo,
                               int64_t t_hi) {
    if (t_hi < 0) t_hi = tokens;
    if (t_lo % kBlockK != 0 || t_lo < 0 || t_hi > tokens || t_lo >= t_hi) return cudaErrorInvalidValue;
    const int64_t q_rows = q ? batch * (t_hi - t_lo) * hq : 0;
    const int64_t q_ctas = (q_rows + kQRowsPerCta - 1) / kQRowsPerCta;
    if (batch * tokens * hq > 0x7FFFFFFF) return cudaErrorInvalidValue; // 32-bit scale index math
    const int64_t k_ctas = k ? batch * ((t_hi + kBlockK - 1) / kBlockK - t_lo / kBlockK) * hkv : 0;
    const int64_t grid = q_ctas + k_ctas;
    if (grid == 0) return cudaSuccess;
    if (grid > 0x7FFFFFFF) return cudaErrorInvalidValue;
    quantize_qk_kernel<<<static_cast<unsigned>(grid), kThreads, 0, stream>>>(
        static_cast<const __nv_bfloat16 *>(q), static_cast<const __nv_bfloat16 *>(k), q_codes,
        q_scales, k_codes, k_scales, batch, tokens, hq, hkv, q_ctas, t_lo, t_hi);
    return cudaGetLastError();
}

} // namespace sale_b200
