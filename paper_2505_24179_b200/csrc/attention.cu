// attention.cu — K3: block-sparse causal flash attention on tcgen05 (bf16 in,
// fp32 TMEM accumulators, fp32 online softmax) that visits only selected
// 64x32 blocks. With mask == nullptr it is the dense causal baseline (the
// all-ones-mask run of the same kernel).
//
// Replaces block_sparse_attention (sparse_attention.hpp:37-97) and, as the
// dense run, full_attention (attention.hpp:18-50). Semantics kept: a key token
// t contributes to row g iff t <= g and mask(qblock(g), kblock(t)) is set;
// fully-future mask bits are ignored; coverage[g] counts the attended tokens.
//
// CTA = one query block i (64 tokens) of TWO query heads of the same GQA group
// as one M=128 tile: both heads need exactly the same K/V and the same causal
// extent, and per-head masks of one query block overlap more than masks of
// adjacent query blocks (profiles/mask_stats.py). TMEM lane 32q + 16hh + t
// holds row 16q + t of head 2p + hh, so every lane quadrant (SMSP) has rows of
// both heads and a tile selected by one head only keeps one of the two softmax
// warps of every SMSP busy.
// Key tiles follow the segment grid of the Selection-Pass: tile 0 = the
// 32-key sink block, tile s+1 = keys [32+128s, 160+128s) = key blocks
// 1+4s..4+4s. A tile is visited iff any of its 8 (head, kblock) bits is set;
// inside a visited tile unselected 32-key sub-blocks and the causal diagonal
// are masked per row.
//
// TMEM (512 columns): O | l [0,144) | S0 [160,288) | S1 [288,416) | Q [416,480).
// Q sits in TMEM as the A operand of S = Q K^T (only K streams from shared
// memory; with A in SMEM an M=N=128 bf16 MMA needs the full 128 B/clk port),
// and P overwrites S in place as the A operand of O | l += P [V | 1]: the
// N = 144 PV MMA also produces the row sums l from a constant ones chunk.
//
// Pipeline (warp-specialised, one elected thread per role):
//   warp 0  TMA: K_j (released by S_j) and V_j (released by PV_j) into 3- / 2-
//           stage rings (SW128 tiles), K one tile ahead of V
//   warp 1  MMA: S_0, S_1, then per tile j: O | l += P_j [V_j | 1], S_{j+2} =
//           Q K^T into the buffer P_j came from
//   warp 2  TMEM allocator; warp 3 also builds the active tile list while the
//           others initialise barriers and the ones chunk
//   warps 3-10 softmax: warp (quadrant q, index w) owns TMEM lanes 32q + 16w +
//           [0, 16) (head 2p + w), two rows x 64 columns per thread through
//           16x256b loads; row max by two shuffles (no cross-warp barrier);
//           lazy-rescaled online softmax in the exp2 domain (O | l rescaled in
//           TMEM only when the running max grows by > 8); full tiles compute
//           P speculatively against the running references (redone in order
//           when a reference moves); P -> bf16 -> tcgen05.st over S.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace sale_b200 {

constexpr int kAttnThreads = 352;  // 3 control warps + 2 softmax warpgroups (warps 3-10)
constexpr int kMaxTiles = 4200;                // supports N <= 512K
constexpr int kKvStages = 3;                   // K ring
constexpr int kVStages = 2;                    // V ring (+ the constant ones chunk)
constexpr int kTileBytesHalf = 128 * 64 * 2;   // 128 rows x 64 bf16 = 16 KB
constexpr uint32_t kColO = 0, kColL = 128, kColS0 = 160, kColQ = 416;

struct AttnSmem {
    alignas(1024) uint8_t k[kKvStages][2][kTileBytesHalf];
    // V as the B operand of O|l += P [V | 1]: N = 144 = two 64-column chunks of
    // V and a chunk of ones (only 16 columns read) at stride kVStages x 16 KB
    alignas(1024) uint8_t v[3][kVStages][kTileBytesHalf];
    uint64_t q_ready, k_full[kKvStages], v_full[kVStages], k_empty[kKvStages], v_empty[kVStages];
    uint64_t s_full[2], p_full[2], pv_done[2];
    uint32_t tmem_base;
    int ntiles;
    int warp_tot[8];           // tile-list build: per-warp counts of a round
    long long prof_tp[4];      // profiling: MMA-side time P_j was observed (ring)
    uint32_t tiles[kMaxTiles]; // j | bits8 << 16
};

// Optional cycle instrumentation (sale_b200_attention_profile): [0] softmax
// loop total, [1] S-ready waits, [2] softmax_part time, [3] tiles (warp 3,
// lane 0, summed over CTAs); [4] MMA loop total, [5] K waits, [6] P waits,
// [7] V waits, [8] CTAs, [9] prologue (start -> tile list ready, thread 0),
// [10] epilogue (last tile -> end, warp 3 lane 0), [11] MMA-side P -> S chain,
// [12] tile-list warp start, [13] TMEM allocated, [14] tile list done,
// [15] barriers + ones chunk done.
bool g_attn_prof_host = false; // host: launch the kProf instance
__device__ unsigned long long g_attn_prof[16];

namespace {

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ unsigned long long pack_f2(float lo, float hi) {
    return (static_cast<unsigned long long>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}
// x = x * a + b on two packed fp32 lanes (FFMA2)
__device__ __forceinline__ void ffma2_f32(unsigned long long &x, unsigned long long a,
                                          unsigned long long b) {
    asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(a), "l"(b));
}
__device__ __forceinline__ void fadd2_f32(unsigned long long &x, unsigned long long a) {
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(a));
}

__device__ __forceinline__ void fsub2_f32(unsigned long long &x, unsigned long long a) {
    asm("sub.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(a));
}
// (t << 23) + p on the ALU pipe (SHF + IADD3) instead of an FMA-pipe IMAD
__device__ __forceinline__ uint32_t shl23_add(uint32_t t, uint32_t p) {
    uint32_t sh, r;
    asm("shf.l.wrap.b32 %0, %1, %2, 23;" : "=r"(sh) : "r"(0u), "r"(t)); // upper word of (t:0) << 23
    asm("add.u32 %0, %1, %2;" : "=r"(r) : "r"(sh), "r"(p));
    return r;
}

// 16-byte read-only load / 4-byte store with an L2 cache-policy hint
__device__ __forceinline__ uint4 ld_stream16(const uint4 *p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ void st_stream4(void *p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&p);
}

// O rows of this warp (16 TMEM lanes: thread rows T/4, T/4+8) *= alpha per
// row, once PV of every earlier tile has landed in O.
__device__ __forceinline__ void rescale_o16(uint32_t oAddr, float a0, float a1, uint64_t *pv_prev,
                                            uint32_t pv_parity) {
    mbar_wait(pv_prev, pv_parity);
    tc_fence_after();
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
        uint32_t o[32];
        tmem_ld16x256_x8(oAddr + 64 * cc, o);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * ((e & 2) ? a1 : a0));
        tmem_st16x256_x8(oAddr + 64 * cc, o);
    }
    uint32_t l4[4]; // the row sums l (O column kColL; columns kColL+8.. are not read)
    tmem_ld16x256_x1(oAddr + (kColL - kColO), l4);
    tmem_ld_wait();
#pragma unroll
    for (int e = 0; e < 4; ++e) l4[e] = __float_as_uint(__uint_as_float(l4[e]) * ((e & 2) ? a1 : a0));
    tmem_st16x256_x1(oAddr + (kColL - kColO), l4);
    tmem_st_wait();
}

struct SoftmaxState {
    float m[2] = {-INFINITY, -INFINITY}; // running max per row, exp2 domain (logit * scale_log2)
    int cov[2] = {0, 0};                 // attended tokens in this thread's columns
};

// One S tile for the 16 rows of this warp. Thread T owns rows T/4 and T/4+8
// of the warp's TMEM lanes and columns 8R + 2(T%4) + {0,1} (R < 16) of each:
// the row max is combined over the four threads of a row by two shuffles, so
// the two warps sharing a TMEM lane quadrant never synchronise with each other.
// nib: the row head's four 32-key sub-block bits of this tile; lim0/lim1:
// valid columns c <= lim per row (-1: none). S holds raw fp32 logits*sqrt(d);
// the bf16 P pairs go to columns [0, 64) of the same buffer (only this warp's
// lanes, whose S values are already in registers).
__device__ __forceinline__ void softmax_tile(uint32_t sAddr, uint32_t oAddr, uint32_t nib,
                                             int64_t lim0, int64_t lim1, int q4, float scale_log2,
                                             SoftmaxState &st, uint64_t *pv_prev, uint32_t pv_parity) {
    const bool any_valid = nib != 0u && (lim0 >= 0 || lim1 >= 0);
    uint32_t s[64];
    if (__all_sync(0xffffffffu, !any_valid)) {
        // nothing of this tile is attended by the warp's rows: P = 0, no exp work
#pragma unroll
        for (int e = 0; e < 32; ++e) s[e] = 0u;
        tmem_st16x128_x16(sAddr, s);
        tmem_st_wait();
        return;
    }
    const bool full = nib == 0xFu && lim0 >= 127 && lim1 >= 127;
    const unsigned long long sc2 = pack_f2(scale_log2, scale_log2);
    const bool spec = __all_sync(0xffffffffu, full && st.m[0] != -INFINITY && st.m[1] != -INFINITY);
    if (spec) {
        // S in two 64-column halves: the second half lands while the first
        // half's exps run
        tmem_ld16x256_x8(sAddr, s);
        tmem_ld_wait();
        tmem_ld16x256_x8(sAddr + 64, s + 32);
    } else {
        tmem_ld16x256_x16(sAddr, s);
        tmem_ld_wait();
    }
    if (spec) {
        // Speculative path (full tiles once both rows have a reference): P is
        // computed against the running references right away, interleaved
        // with the row max instead of after it; when no row max grows by > 8
        // (the usual case) the references stay and P is exactly what the
        // in-order path computes. Otherwise S is reloaded and the tile takes
        // the in-order path below.
        const unsigned long long nmf[2] = {pack_f2(-st.m[0], -st.m[0]), pack_f2(-st.m[1], -st.m[1])};
        float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int R = 0; R < 16; ++R)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (R == 8 && k == 0) tmem_ld_wait(); // the second half
                mx[2 * k + (R & 1)] =
                    fmax3(mx[2 * k + (R & 1)], __uint_as_float(s[4 * R + 2 * k]), __uint_as_float(s[4 * R + 2 * k + 1]));
                unsigned long long x =
                    (static_cast<unsigned long long>(s[4 * R + 2 * k + 1]) << 32) | s[4 * R + 2 * k];
                ffma2_f32(x, sc2, nmf[k]);
                float p0, p1;
                if ((R & 7) == 0 || (R & 7) == 3 || (R & 7) == 5) {
                    const unsigned long long xc =
                        pack_f2(fmaxf(__uint_as_float(static_cast<uint32_t>(x)), -125.0f),
                                fmaxf(__uint_as_float(static_cast<uint32_t>(x >> 32)), -125.0f));
                    unsigned long long t = xc;
                    fadd2_f32(t, pack_f2(12582912.0f, 12582912.0f));
                    unsigned long long r = t;
                    fadd2_f32(r, pack_f2(-12582912.0f, -12582912.0f));
                    unsigned long long f = xc;
                    fsub2_f32(f, r);
                    unsigned long long pp = pack_f2(0.05592204f, 0.05592204f);
                    ffma2_f32(pp, f, pack_f2(0.24264008f, 0.24264008f));
                    ffma2_f32(pp, f, pack_f2(0.69312102f, 0.69312102f));
                    ffma2_f32(pp, f, pack_f2(0.99992448f, 0.99992448f));
                    p0 = __uint_as_float(shl23_add(static_cast<uint32_t>(t), static_cast<uint32_t>(pp)));
                    p1 = __uint_as_float(shl23_add(static_cast<uint32_t>(t >> 32),
                                                   static_cast<uint32_t>(pp >> 32)));
                } else {
                    p0 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x)));
                    p1 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x >> 32)));
                }
                s[2 * R + k] = pack_bf16x2(p0, p1); // index 2R+k was already consumed
            }
        float u0 = fmaxf(mx[0], mx[1]), u1 = fmaxf(mx[2], mx[3]);
        u0 = fmaxf(u0, __shfl_xor_sync(0xffffffffu, u0, 1));
        u1 = fmaxf(u1, __shfl_xor_sync(0xffffffffu, u1, 1));
        u0 = fmaxf(u0, __shfl_xor_sync(0xffffffffu, u0, 2));
        u1 = fmaxf(u1, __shfl_xor_sync(0xffffffffu, u1, 2));
        const bool grow = fmaxf(st.m[0], u0 * scale_log2) > st.m[0] + 8.0f ||
                          fmaxf(st.m[1], u1 * scale_log2) > st.m[1] + 8.0f;
        if (!__any_sync(0xffffffffu, grow)) {
            st.cov[0] += 32;
            st.cov[1] += 32;
            tmem_st16x128_x16(sAddr, s);
            tmem_st_wait();
            return;
        }
        tmem_ld16x256_x16(sAddr, s); // a reference moves: redo in order
        tmem_ld_wait();
    }
    int nv0 = 64, nv1 = 64;
    if (!full) {
        nv0 = nv1 = 0;
#pragma unroll
        for (int R = 0; R < 16; ++R)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t c = 8 * R + 2 * q4 + e;
                const bool sub = (nib >> (R >> 2)) & 1u;
                const bool ok0 = sub && c <= lim0, ok1 = sub && c <= lim1;
                s[4 * R + e] = ok0 ? s[4 * R + e] : __float_as_uint(-INFINITY);
                s[4 * R + 2 + e] = ok1 ? s[4 * R + 2 + e] : __float_as_uint(-INFINITY);
                nv0 += ok0 ? 1 : 0;
                nv1 += ok1 ? 1 : 0;
            }
    } else {
        nv0 = nv1 = 32;
    }
    // row max: two chains per row, then the four threads of the row
    float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int R = 0; R < 16; R += 2) {
        mx[0] = fmax3(mx[0], __uint_as_float(s[4 * R]), __uint_as_float(s[4 * R + 1]));
        mx[1] = fmax3(mx[1], __uint_as_float(s[4 * R + 4]), __uint_as_float(s[4 * R + 5]));
        mx[2] = fmax3(mx[2], __uint_as_float(s[4 * R + 2]), __uint_as_float(s[4 * R + 3]));
        mx[3] = fmax3(mx[3], __uint_as_float(s[4 * R + 6]), __uint_as_float(s[4 * R + 7]));
    }
    float t0 = fmaxf(mx[0], mx[1]), t1 = fmaxf(mx[2], mx[3]);
    t0 = fmaxf(t0, __shfl_xor_sync(0xffffffffu, t0, 1));
    t1 = fmaxf(t1, __shfl_xor_sync(0xffffffffu, t1, 1));
    t0 = fmaxf(t0, __shfl_xor_sync(0xffffffffu, t0, 2));
    t1 = fmaxf(t1, __shfl_xor_sync(0xffffffffu, t1, 2));
    // lazy rescale: only when the running max grows by > 8 (exp2 domain); P is
    // computed against the new max, O is rescaled after P is stored (fewer
    // live registers), before p_full releases PV of this tile.
    float alpha[2];
    bool need_any = false;
    const float tm[2] = {t0, t1};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float m_new = fmaxf(st.m[k], tm[k] * scale_log2);
        const bool need = st.m[k] != -INFINITY && m_new > st.m[k] + 8.0f;
        alpha[k] = need ? ex2_approx(st.m[k] - m_new) : 1.0f;
        if (st.m[k] == -INFINITY || need) st.m[k] = m_new;
        need_any |= need;
    }
    const bool any_need = __any_sync(0xffffffffu, need_any);
    // p = exp2(s * scale_log2 - m); masked columns hold -inf -> p = 0. A row
    // with nothing valid yet keeps m = -inf: use 0 so -inf * scale - 0 = -inf.
    unsigned long long nm2[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float neg_m = st.m[k] == -INFINITY ? 0.0f : -st.m[k];
        nm2[k] = pack_f2(neg_m, neg_m);
    }
    if (__all_sync(0xffffffffu, full)) {
        // Full tiles: the pairs of R = 0, 3, 5 (mod 8) — 3/8 of them — take
        // exp2 on the FMA/ALU pipes (Cody-Waite split + degree-3 polynomial,
        // rel. err 1e-4 < bf16's 2^-8), the rest on MUFU (16 ex2/clk/SM).
        // Measured against 1/2, 1/4, 1/8 and other 3/8 placements on the bench
        // workload: dense 124-125 vs 129-133 ms, sparse 43.6 vs 45-46 ms
        // (profiles/README.md).
#pragma unroll
        for (int R = 0; R < 16; ++R)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                unsigned long long x =
                    (static_cast<unsigned long long>(s[4 * R + 2 * k + 1]) << 32) | s[4 * R + 2 * k];
                ffma2_f32(x, sc2, nm2[k]);
                float p0, p1;
                if ((R & 7) == 0 || (R & 7) == 3 || (R & 7) == 5) {
                    const unsigned long long xc =
                        pack_f2(fmaxf(__uint_as_float(static_cast<uint32_t>(x)), -125.0f),
                                fmaxf(__uint_as_float(static_cast<uint32_t>(x >> 32)), -125.0f));
                    unsigned long long t = xc;
                    fadd2_f32(t, pack_f2(12582912.0f, 12582912.0f));   // round to integer
                    unsigned long long r = t;
                    fadd2_f32(r, pack_f2(-12582912.0f, -12582912.0f)); // the integer, as float
                    unsigned long long f = xc;
                    fsub2_f32(f, r);                                   // f = x - r in [-.5, .5]
                    unsigned long long pp = pack_f2(0.05592204f, 0.05592204f);
                    ffma2_f32(pp, f, pack_f2(0.24264008f, 0.24264008f));
                    ffma2_f32(pp, f, pack_f2(0.69312102f, 0.69312102f));
                    ffma2_f32(pp, f, pack_f2(0.99992448f, 0.99992448f));
                    // 2^r * poly: integer r into the exponent field (ALU shift + add)
                    p0 = __uint_as_float(shl23_add(static_cast<uint32_t>(t), static_cast<uint32_t>(pp)));
                    p1 = __uint_as_float(shl23_add(static_cast<uint32_t>(t >> 32),
                                                   static_cast<uint32_t>(pp >> 32)));
                } else {
                    p0 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x)));
                    p1 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x >> 32)));
                }
                s[2 * R + k] = pack_bf16x2(p0, p1); // in place: index 2R+k was already consumed
            }
    } else {
#pragma unroll
        for (int R = 0; R < 16; ++R)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                unsigned long long x =
                    (static_cast<unsigned long long>(s[4 * R + 2 * k + 1]) << 32) | s[4 * R + 2 * k];
                ffma2_f32(x, sc2, nm2[k]); // x = x * scale + (-m), two lanes
                const float p0 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x)));
                const float p1 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x >> 32)));
                s[2 * R + k] = pack_bf16x2(p0, p1);
            }
    }
    st.cov[0] += nv0;
    st.cov[1] += nv1;
    tmem_st16x128_x16(sAddr, s);
    tmem_st_wait();
    if (any_need) rescale_o16(oAddr, alpha[0], alpha[1], pv_prev, pv_parity);
}

// kProf: the cycle-instrumented instance (sale_b200_attention_profile); the
// production instance carries no profiling code.
template <bool kProf>
__global__ void __launch_bounds__(kAttnThreads, 1)
sparse_attention_kernel(const __nv_bfloat16 *__restrict__ q, const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const uint32_t *__restrict__ mask,
                        __nv_bfloat16 *__restrict__ out, int32_t *__restrict__ coverage,
                        unsigned long long *__restrict__ empty_rows, int64_t tokens, int hq, int hkv,
                        float scale_log2, int64_t i_lo, int64_t ni, int wave_qb) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const long long t_kernel = clock64();
    AttnSmem &sm = *reinterpret_cast<AttnSmem *>(smem_raw + smem_pad_1k(smem_raw));
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int tid = threadIdx.x;

    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    const int64_t words = (nk + 31) / 32;
    // CTA order: (batch, KV head) major, then query blocks heaviest first, then
    // the head pairs of the GQA group — concurrently resident CTAs stream the
    // same K/V prefix, so the ~64 MB of K/V per KV head at 128K is read from
    // HBM about once and then served from L2.
    const int group = hq / hkv;
    const int npairs = (group + 1) / 2;
    // 32-bit index math (grid < 2^31; ni <= nq)
    const uint32_t bx = blockIdx.x, np32 = static_cast<uint32_t>(npairs), ni32 = static_cast<uint32_t>(ni);
    const uint32_t bq = bx / np32;
    const int p = static_cast<int>(bx - bq * np32);
    // query blocks [i_lo, i_lo + ni): a token-range slice (chunked host pipeline)
    const uint32_t bgq = bq / ni32;
    const int64_t i = i_lo + ni - 1 - static_cast<int64_t>(bq - bgq * ni32);
    const int bg = static_cast<int>(bgq);
    const int g = bg % hkv;
    const int b = bg / hkv;
    const int hA = g * group + 2 * p;
    const bool hasB = 2 * p + 1 < group;
    const int64_t q0 = i * kBlockQ;
    const int64_t qend = q0 + kBlockQ < tokens ? q0 + kBlockQ : tokens;

    if (tid == 0) {
        mbar_init(&sm.q_ready, 8);
        for (int s = 0; s < kKvStages; ++s) {
            mbar_init(&sm.k_full[s], 1);
            mbar_init(&sm.k_empty[s], 1);
        }
        for (int s = 0; s < kVStages; ++s) {
            mbar_init(&sm.v_full[s], 1);
            mbar_init(&sm.v_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.s_full[s], 1);
            mbar_init(&sm.p_full[s], 8);
            mbar_init(&sm.pv_done[s], 1);
        }
        fence_barrier_init();
    }
    // Q of the softmax warps' TMEM lanes: the global loads are issued before the
    // tile-list build (their latency overlaps it), the TMEM store follows the
    // CTA barrier (TMEM is allocated by then). Thread = TMEM lane 32 quad +
    // lane, column half wg.
    uint32_t qa[32];
    if (warp >= 3) {
        const uint64_t pol = policy_evict_first();
        const int wg = (warp - 3) >> 2, quad = warp & 3, hh = lane >> 4;
        const int64_t qrow = q0 + quad * 16 + (lane & 15);
        const bool q_ok = qrow < tokens && (hh == 0 || hasB);
        const uint4 *src = reinterpret_cast<const uint4 *>(
            q + ((static_cast<int64_t>(b) * tokens + (q_ok ? qrow : 0)) * hq + hA + hh) * kHeadDim + 64 * wg);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint4 w = q_ok ? ld_stream16(src + e, pol) : make_uint4(0, 0, 0, 0);
            qa[4 * e] = w.x, qa[4 * e + 1] = w.y, qa[4 * e + 2] = w.z, qa[4 * e + 3] = w.w;
        }
    }
    if (warp == 2) {
        tmem_alloc<512>(&sm.tmem_base);
        if (lane == 0 && kProf)
            atomicAdd(&g_attn_prof[13], static_cast<unsigned long long>(clock64() - t_kernel));
    } else if (warp >= 3) {
        // ---- active tile list (ascending), built by the 8 softmax warps while
        // the control warps set up: per round, warp w3 = warp - 3 takes pass
        // p = 8 round + w3 = segment-tile groups [32p, 32p + 32); lane t of a
        // pass owns the 8 tiles 8g+1 .. 8g+8 (g = 32p + t) = key blocks
        // 32g+1 .. 32g+32 (bits 1-31 of mask word g, bit 0 of word g+1); tile
        // 0 is the sink block. Prefix sums: ballots within a warp, the eight
        // warp totals through shared memory (one named barrier per round).
        const int w3 = warp - 3;
        const int64_t rowbase = (static_cast<int64_t>(b) * hq + hA) * nq + i;
        const uint32_t *rowA = mask ? mask + rowbase * words : nullptr;
        const uint32_t *rowB = (mask && hasB) ? mask + (rowbase + nq) * words : nullptr;
        const int total = qend > kBlockK ? 1 + static_cast<int>((qend - kBlockK + 127) / 128) : 1;
        const int64_t jmax = min(nk, (qend + kBlockK - 1) / kBlockK) - 1; // last causal key block
        const int groups = (total - 1 + 7) / 8;
        auto word = [&](const uint32_t *row, int64_t t) -> uint32_t {
            return !row ? 0xFFFFFFFFu : (t < words ? row[t] : 0u);
        };
        const uint32_t a0 = mask ? rowA[0] & 1u : 1u;
        const uint32_t b0 = !hasB ? 0u : (mask ? rowB[0] & 1u : 1u);
        const uint32_t sink = a0 | (b0 << 4);
        int carry = sink ? 1 : 0;
        if (tid == 96 && sink) sm.tiles[0] = sink << 16;
        const uint32_t lt = (1u << lane) - 1u;
        for (int base = 0; base < groups; base += 256) {
            const int t = base + 32 * w3 + lane; // this lane's group
            uint32_t xa = 0, xb = 0;
            if (t < groups) {
                const uint32_t wa = word(rowA, t), wa1 = word(rowA, t + 1);
                const uint32_t wb = hasB ? word(rowB, t) : 0u, wb1 = hasB ? word(rowB, t + 1) : 0u;
                const int64_t avail = jmax - 32LL * t; // blocks 32t+1 .. 32t+avail are causal
                const uint32_t cm = avail >= 32 ? 0xFFFFFFFFu : (avail <= 0 ? 0u : (1u << avail) - 1u);
                xa = ((wa >> 1) | (wa1 << 31)) & cm;
                xb = ((wb >> 1) | (wb1 << 31)) & cm;
            }
            uint32_t act = 0; // bit e: tile 8t+1+e active
#pragma unroll
            for (int e = 0; e < 8; ++e) act |= (((xa | xb) >> (4 * e)) & 0xFu) ? (1u << e) : 0u;
            const int c = __popc(act);
            int excl = 0, tot = 0;
#pragma unroll
            for (int bit = 0; bit < 4; ++bit) {
                const uint32_t m = __ballot_sync(0xffffffffu, (c >> bit) & 1);
                excl += __popc(m & lt) << bit;
                tot += __popc(m) << bit;
            }
            if (lane == 0) sm.warp_tot[w3] = tot;
            named_bar_sync(1, 256);
            int before = 0, all = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const int x = sm.warp_tot[w];
                before += w < w3 ? x : 0;
                all += x;
            }
            int pos = carry + before + excl;
            while (act) {
                const int e = __ffs(act) - 1;
                act &= act - 1;
                const uint32_t bits = ((xa >> (4 * e)) & 0xFu) | (((xb >> (4 * e)) & 0xFu) << 4);
                if (pos < kMaxTiles) sm.tiles[pos] = static_cast<uint32_t>(8 * t + 1 + e) | (bits << 16);
                ++pos;
            }
            carry += all;
            named_bar_sync(1, 256); // warp_tot is reused by the next round
        }
        if (tid == 96) sm.ntiles = carry < kMaxTiles ? carry : kMaxTiles;
        if (tid == 96 && kProf)
            atomicAdd(&g_attn_prof[14], static_cast<unsigned long long>(clock64() - t_kernel));
    } else {
        // the ones chunk of the PV B operand (bf16 1.0), read by the tensor core
        uint4 *ones = reinterpret_cast<uint4 *>(sm.v[2]);
        for (int e = tid; e < kVStages * kTileBytesHalf / 16; e += 64) // warps 0, 1
            ones[e] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (tid == 0 && kProf)
            atomicAdd(&g_attn_prof[15], static_cast<unsigned long long>(clock64() - t_kernel));
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0 && kProf)
        atomicAdd(&g_attn_prof[9], static_cast<unsigned long long>(clock64() - t_kernel));
    const uint32_t tmem = sm.tmem_base;
    const int ntiles = sm.ntiles;
    // Alternate groups of wave_qb query blocks (one wave of CTAs: SMs / head
    // pairs, counted from the heaviest block, the first to launch) walk their
    // key tiles in opposite directions, so a wave starts on the K / V tiles the
    // previous wave touched last (still in L2) instead of re-streaming the
    // head's K / V prefix from HBM. A function of i alone: range and chunked
    // launches compute every query block exactly as the one-shot launch.
    const bool rev = (((nq - 1 - i) / wave_qb) & 1) != 0;
    auto tile_at = [&](int jj) -> uint32_t { return sm.tiles[rev ? ntiles - 1 - jj : jj]; };

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA
        if (elect_one() && ntiles > 0) {
            tma_prefetch(&tm_k);
            tma_prefetch(&tm_v);
            // K / V of a KV head are re-read by every query block of its group:
            // keep them in L2 (Q and O stream through with evict_first)
            const uint64_t keep = policy_evict_last();
            // K_jj is released by S_jj, V_jj by PV_jj (one tile later): K runs
            // one tile ahead of V so a late PV never holds back the next K.
            auto key0_of = [&](int jj) {
                const int j = static_cast<int>(tile_at(jj) & 0xFFFFu);
                return j == 0 ? 0 : kBlockK + 128 * (j - 1);
            };
            for (int jj = 0; jj <= ntiles; ++jj) {
                if (jj < ntiles) {
                    const int st = jj % kKvStages;
                    const int key0 = key0_of(jj);
                    mbar_wait(&sm.k_empty[st], ((jj / kKvStages) & 1) ^ 1);
                    mbar_expect_tx(&sm.k_full[st], 2 * kTileBytesHalf);
                    tma_load_4d_hint(sm.k[st][0], &tm_k, &sm.k_full[st], 0, g, key0, b, keep);
                    tma_load_4d_hint(sm.k[st][1], &tm_k, &sm.k_full[st], 64, g, key0, b, keep);
                }
                if (jj > 0) {
                    const int vj = jj - 1;
                    const int st = vj % kVStages;
                    const int key0 = key0_of(vj);
                    mbar_wait(&sm.v_empty[st], ((vj / kVStages) & 1) ^ 1);
                    mbar_expect_tx(&sm.v_full[st], 2 * kTileBytesHalf);
                    tma_load_4d_hint(sm.v[0][st], &tm_v, &sm.v_full[st], 0, g, key0, b, keep);
                    tma_load_4d_hint(sm.v[1][st], &tm_v, &sm.v_full[st], 64, g, key0, b, keep);
                }
            }
            // drain: the last releases of every ring stage (S / PV commits) land
            // before the CTA exits, so no mbarrier phase completes unobserved
            for (int jj = ntiles > kKvStages ? ntiles - kKvStages : 0; jj < ntiles; ++jj)
                mbar_wait(&sm.k_empty[jj % kKvStages], (jj / kKvStages) & 1);
            for (int vj = ntiles > kVStages ? ntiles - kVStages : 0; vj < ntiles; ++vj)
                mbar_wait(&sm.v_empty[vj % kVStages], (vj / kVStages) & 1);
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA
        if (elect_one() && ntiles > 0) {
            constexpr uint32_t idesc_pv = idesc_bf16(128, 144, true); // O | l
            const bool prof = kProf;
            const long long t_start = clock64();
            long long w_k = 0, w_p = 0, w_v = 0, t0 = 0;
            mbar_wait(&sm.q_ready, 0);
            tc_fence_after();
            // Order on the tensor pipe: S_0, S_1, PV_0, S_2, PV_1, S_3, ...
            // S_{j+2} reuses S_j's buffer right behind PV_j (in-order pipe). The
            // K / V readiness checks come before the P wait, so once P_j is seen
            // PV_j and S_{j+2} issue with no further barrier latency.
            auto issue_s = [&](int jj) {
                const int st = jj % kKvStages;
                const int sb = jj & 1;
                const int j = static_cast<int>(tile_at(jj) & 0xFFFFu);
                const uint32_t idesc_s = j == 0 ? idesc_bf16(128, 32, false) : idesc_bf16(128, 128, false);
                const uint64_t kd0 = umma_desc_sw128(smem_u32(sm.k[st][0]), 16, 1024);
                const uint64_t kd1 = umma_desc_sw128(smem_u32(sm.k[st][1]), 16, 1024);
                const uint32_t dS = tmem + kColS0 + 128u * static_cast<uint32_t>(sb);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) { // K = 16 bf16 = 8 TMEM columns of Q
                    const uint64_t bd = (kk < 4 ? kd0 : kd1) + 2 * (kk & 3);
                    mma_bf16_ts(dS, tmem + kColQ + 8 * kk, bd, idesc_s, kk > 0);
                }
                tc_commit(&sm.s_full[sb]);
                tc_commit(&sm.k_empty[st]);
            };
            auto wait_k = [&](int jj) {
                if (prof) t0 = clock64();
                mbar_wait(&sm.k_full[jj % kKvStages], (jj / kKvStages) & 1);
                if (prof) w_k += clock64() - t0;
            };
            wait_k(0);
            tc_fence_after();
            issue_s(0);
            if (ntiles > 1) {
                wait_k(1);
                tc_fence_after();
                issue_s(1);
            }
            for (int pj = 0; pj < ntiles; ++pj) {
                const int nx = pj + 2;
                const int pst = pj % kVStages;
                const int psb = pj & 1;
                const int jp = static_cast<int>(tile_at(pj) & 0xFFFFu);
                const int steps = jp == 0 ? 2 : 8;
                if (nx < ntiles) wait_k(nx);
                if (prof) t0 = clock64();
                mbar_wait(&sm.v_full[pst], (pj / kVStages) & 1);
                if (prof) { w_v += clock64() - t0; t0 = clock64(); }
                mbar_wait(&sm.p_full[psb], (pj >> 1) & 1);
                if (prof) {
                    const long long tn = clock64();
                    w_p += tn - t0;
                    *reinterpret_cast<volatile long long *>(&sm.prof_tp[pj & 3]) = tn;
                }
                tc_fence_after();
                const uint64_t vd = umma_desc_sw128(smem_u32(sm.v[0][pst]), kVStages * kTileBytesHalf, 1024);
                const uint32_t aP = tmem + kColS0 + 128u * static_cast<uint32_t>(psb);
                for (int kk = 0; kk < steps; ++kk)
                    mma_bf16_ts(tmem + kColO, aP + 8 * kk, vd + 128 * kk, // +16 keys = 2 KB
                                idesc_pv, (pj > 0 || kk > 0) ? 1u : 0u);
                tc_commit(&sm.v_empty[pst]);
                tc_commit(&sm.pv_done[psb]);
                if (nx < ntiles) issue_s(nx);
            }
            if (prof) {
                atomicAdd(&g_attn_prof[4], static_cast<unsigned long long>(clock64() - t_start));
                atomicAdd(&g_attn_prof[5], static_cast<unsigned long long>(w_k));
                atomicAdd(&g_attn_prof[6], static_cast<unsigned long long>(w_p));
                atomicAdd(&g_attn_prof[7], static_cast<unsigned long long>(w_v));
                atomicAdd(&g_attn_prof[8], 1ull);
            }
        }
    } else if (warp >= 3) {
        // ------------------------------------------------------------ softmax
        // TMEM lane L = 32 quad + 16 hh + t holds row 16 quad + t of head hA + hh:
        // both heads have rows in every lane quadrant, so a tile selected by one
        // head only keeps one softmax warp busy on every SMSP.
        const int wg = (warp - 3) >> 2;          // second index of the warp in its quadrant
        const int quad = warp & 3;               // TMEM lane quadrant (warp id % 4)
        const uint64_t stream_pol = policy_evict_first();
        // Q staging: the rows loaded before the tile list, into TMEM
        {
            const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quad * 32) << 16);
            tmem_st32(lane_addr + kColQ + 32 * wg, qa);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.q_ready);
        }
        // softmax rows: warp (quad, wg) owns TMEM lanes 32 quad + 16 wg + [0, 16)
        // = rows 16 quad + [0, 16) of head hA + wg; thread rows rr0 = 16 quad +
        // lane/4 and rr1 = rr0 + 8
        const int half = wg;
        const int h = hA + half;
        const int q4 = lane & 3;
        const int rr0 = quad * 16 + (lane >> 2);
        const int64_t grow0 = q0 + rr0, grow1 = grow0 + 8;
        const bool ok0 = grow0 < tokens && (half == 0 || hasB);
        const bool ok1 = grow1 < tokens && (half == 0 || hasB);
        const uint32_t lane16 = tmem + (static_cast<uint32_t>(quad * 32 + 16 * wg) << 16);
        SoftmaxState st;
        const uint32_t oAddr = lane16 + kColO;
        const bool prof = warp == 3 && lane == 0 && kProf;
        const long long t_loop = clock64();
        long long w_s = 0, t_part = 0, t1 = 0, w_chain = 0, n_chain = 0;
        for (int jj = 0; jj < ntiles; ++jj) {
            const int sb = jj & 1;
            const uint32_t info = tile_at(jj);
            const int j = static_cast<int>(info & 0xFFFFu);
            const uint32_t nib = (info >> (16 + 4 * half)) & 0xFu;
            const int64_t key0 = j == 0 ? 0 : kBlockK + 128LL * (j - 1);
            if (prof) t1 = clock64();
            mbar_wait(&sm.s_full[sb], (jj >> 1) & 1);
            if (prof) {
                const long long t2 = clock64();
                w_s += t2 - t1;
                t1 = t2;
                if (jj >= 2) {
                    w_chain += t2 - *reinterpret_cast<volatile long long *>(&sm.prof_tp[(jj - 2) & 3]);
                    ++n_chain;
                }
            }
            tc_fence_after();
            const int pj = jj - 1;
            // The 32-key sink tile: columns >= 32 hold stale S data and are
            // masked like unselected sub-blocks.
            softmax_tile(lane16 + kColS0 + 128u * sb, oAddr, j == 0 ? (nib & 1u) : nib,
                         ok0 ? grow0 - key0 : -1, ok1 ? grow1 - key0 : -1, q4, scale_log2, st,
                         &sm.pv_done[pj & 1], (pj >> 1) & 1);
            if (prof) t_part += clock64() - t1;
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.p_full[sb]);
        }
        const long long t_epi = clock64();
        if (prof) {
            atomicAdd(&g_attn_prof[0], static_cast<unsigned long long>(t_epi - t_loop));
            atomicAdd(&g_attn_prof[1], static_cast<unsigned long long>(w_s));
            atomicAdd(&g_attn_prof[2], static_cast<unsigned long long>(t_part));
            atomicAdd(&g_attn_prof[3], static_cast<unsigned long long>(ntiles));
            atomicAdd(&g_attn_prof[11], static_cast<unsigned long long>(w_chain));
        }
        // ---- epilogue: coverage over the four threads of a row; l = the ones
        //      column of O | l; O / l -> bf16
        int ct[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            ct[k] = st.cov[k] + __shfl_xor_sync(0xffffffffu, st.cov[k], 1);
            ct[k] += __shfl_xor_sync(0xffffffffu, ct[k], 2);
        }
        float lt[2] = {0.0f, 0.0f};
        if (ntiles > 0) {
            const int last = ntiles - 1;
            mbar_wait(&sm.pv_done[last & 1], (last >> 1) & 1);
            tc_fence_after();
            uint32_t l4[4];
            tmem_ld16x256_x1(oAddr + (kColL - kColO), l4);
            tmem_ld_wait();
            lt[0] = __uint_as_float(l4[0]);
            lt[1] = __uint_as_float(l4[2]);
        }
        const float inv0 = lt[0] > 0.0f ? 1.0f / lt[0] : 0.0f;
        const float inv1 = lt[1] > 0.0f ? 1.0f / lt[1] : 0.0f;
        __nv_bfloat16 *dst0 = out + ((static_cast<int64_t>(b) * tokens + grow0) * hq + h) * kHeadDim;
        __nv_bfloat16 *dst1 = dst0 + 8LL * hq * kHeadDim;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            uint32_t o[32];
            if (ntiles > 0) {
                tmem_ld16x256_x8(oAddr + 64 * cc, o);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) o[e] = 0u;
            }
#pragma unroll
            for (int R = 0; R < 8; ++R) {
                const int col = 64 * cc + 8 * R + 2 * q4;
                if (ok0)
                    st_stream4(dst0 + col,
                               pack_bf16x2(__uint_as_float(o[4 * R]) * inv0, __uint_as_float(o[4 * R + 1]) * inv0),
                               stream_pol);
                if (ok1)
                    st_stream4(dst1 + col,
                               pack_bf16x2(__uint_as_float(o[4 * R + 2]) * inv1, __uint_as_float(o[4 * R + 3]) * inv1),
                               stream_pol);
            }
        }
        if (q4 == 0 && coverage) {
            int32_t *cv = coverage + (static_cast<int64_t>(b) * hq + h) * tokens;
            if (ok0) cv[grow0] = ct[0];
            if (ok1) cv[grow1] = ct[1];
        }
        // a row that attends no token: block_sparse_attention throws
        // std::domain_error for the first such row (sparse_attention.hpp:88-90);
        // the ABI reports the smallest (b, h, row) index
        if (q4 == 0 && empty_rows) {
            const unsigned long long base = (static_cast<unsigned long long>(b) * hq + h) * tokens;
            if (ok1 && ct[1] == 0) atomicMin(empty_rows, base + grow1);
            if (ok0 && ct[0] == 0) atomicMin(empty_rows, base + grow0);
        }
        if (prof) atomicAdd(&g_attn_prof[10], static_cast<unsigned long long>(clock64() - t_epi));
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

} // namespace

cudaError_t attention_profile(int enable, unsigned long long *out16) {
    if (out16) {
        cudaError_t e = cudaMemcpyFromSymbol(out16, g_attn_prof, sizeof(g_attn_prof));
        if (e != cudaSuccess) return e;
    }
    unsigned long long zero[16] = {};
    cudaError_t e = cudaMemcpyToSymbol(g_attn_prof, zero, sizeof(zero));
    if (e != cudaSuccess) return e;
    g_attn_prof_host = enable != 0;
    return cudaSuccess;
}

size_t attention_smem_bytes() { return sizeof(AttnSmem) + 1024; }

cudaError_t launch_sparse_attention(const void *q, const CUtensorMap &tm_k, const CUtensorMap &tm_v,
                                    const uint32_t *mask, void *out, int32_t *coverage,
                                    int64_t batch, int64_t tokens, int hq, int hkv, float scale_log2,
                                    cudaStream_t stream, int64_t i_lo, int64_t i_hi,
                                    unsigned long long *empty_rows) {
    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    if (nq / 2 + 3 > kMaxTiles) return cudaErrorInvalidValue;
    const size_t smem = attention_smem_bytes();
    const int npairs = (hq / hkv + 1) / 2;
    if (i_hi < 0 || i_hi > nq) i_hi = nq;
    if (i_hi <= i_lo) return cudaSuccess;
    const int64_t grid = batch * hkv * npairs * (i_hi - i_lo);
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int wave_qb = std::max(1, sms / npairs); // query blocks of one wave of CTAs
    // tests: SALE_B200_K3_WAVE_QB overrides the group size, so short sequences
    // also run the reversed-direction CTAs
    static const int wave_env = [] {
        const char *e = getenv("SALE_B200_K3_WAVE_QB");
        return e ? atoi(e) : 0;
    }();
    if (wave_env > 0) wave_qb = wave_env;
    auto kern = g_attn_prof_host ? sparse_attention_kernel<true> : sparse_attention_kernel<false>;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), smem);
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(grid), kAttnThreads, smem, stream>>>(
        static_cast<const __nv_bfloat16 *>(q), tm_k, tm_v, mask, static_cast<__nv_bfloat16 *>(out),
        coverage, empty_rows, tokens, hq, hkv, scale_log2, i_lo, i_hi - i_lo, wave_qb);
    return cudaGetLastError();
}

} // namespace sale_b200
