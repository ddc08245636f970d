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
// (rows 0-63 head 2p, rows 64-127 head 2p+1): both halves need exactly the same
// K/V and the same causal extent, and per-head masks of one query block
// overlap more than masks of adjacent query blocks (profiles/mask_stats.py).
// Key tiles follow the segment grid of the Selection-Pass: tile 0 = the
// 32-key sink block, tile s+1 = keys [32+128s, 160+128s) = key blocks
// 1+4s..4+4s. A tile is visited iff any of its 8 (head, kblock) bits is set;
// inside a visited tile unselected 32-key sub-blocks and the causal diagonal
// are masked per row.
//
// TMEM (512 columns): O [0,128) | S0 [128,256) | S1 [256,384) | Q [384,448).
// Q sits in TMEM as the A operand of S = Q K^T (only K streams from shared
// memory; with A in SMEM an M=N=128 bf16 MMA needs the full 128 B/clk port),
// and P overwrites S in place as the A operand of O += P V.
//
// Pipeline (warp-specialised, one elected thread per role):
//   warp 0  TMA: K_j, V_j into a 3-stage ring (SW128 tiles)
//   warp 1  MMA: S_j = Q K_j^T into TMEM buffer j%2 (8 x K=16), then
//           O += P_{j-1} V_{j-1}
//   warps 4-7  softmax, thread = row: Q row -> TMEM once; per tile tcgen05.ld S
//           row, mask, lazy-rescaled online softmax in the exp2 domain (O
//           rescaled in TMEM only when the running max grows by > 8),
//           P -> bf16 -> tcgen05.st over S.
#include "common.cuh"

namespace sale_b200 {

constexpr int kAttnThreads = 352;  // 3 control warps + 2 softmax warpgroups (warps 3-10)
constexpr int kMaxTiles = 4200;                // supports N <= 512K
constexpr int kKvStages = 3;
constexpr int kTileBytesHalf = 128 * 64 * 2;   // 128 rows x 64 bf16 = 16 KB
constexpr uint32_t kColO = 0, kColS0 = 128, kColQ = 384;

struct AttnSmem {
    alignas(1024) uint8_t k[kKvStages][2][kTileBytesHalf];
    alignas(1024) uint8_t v[kKvStages][2][kTileBytesHalf];
    uint64_t q_ready, k_full[kKvStages], v_full[kKvStages], kv_empty[kKvStages];
    uint64_t s_full[2], p_full[2], pv_done[2];
    uint32_t tmem_base;
    int ntiles;
    int warp_cnt[kAttnThreads / 32];
    float xch[2][2][128];   // [tile parity][column half][row]: partial row max
    float fin_l[128];       // end: column-half-1 partial l and coverage
    int fin_cov[128];
    uint32_t tiles[kMaxTiles]; // j | bits8 << 16
};

// Optional cycle instrumentation (sale_b200_attention_profile): [0] softmax
// loop total, [1] S-ready waits, [2] softmax_part time, [3] tiles (warp 3,
// lane 0, summed over CTAs); [4] MMA loop total, [5] K waits, [6] P waits,
// [7] V waits, [8] CTAs, [9] prologue (start -> tile list ready, thread 0),
// [10] epilogue (last tile -> end, warp 3 lane 0).
__device__ int g_attn_prof_on = 0;
__device__ unsigned long long g_attn_prof[16];

namespace {

__device__ __forceinline__ uint32_t mask_bits4(const uint32_t *row, int64_t words, int64_t j0) {
    // bits j0 .. j0+3 of a packed mask row
    const int64_t w = j0 >> 5;
    const int sh = static_cast<int>(j0 & 31);
    uint64_t v = row[w];
    if (w + 1 < words) v |= static_cast<uint64_t>(row[w + 1]) << 32;
    return static_cast<uint32_t>(v >> sh) & 0xFu;
}

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

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&p);
}

// O (this thread's 64-column half) *= alpha, once PV of every earlier tile has
// landed in O.
__device__ __forceinline__ void rescale_o(uint32_t oAddr, float alpha, uint64_t *pv_prev,
                                          uint32_t pv_parity) {
    mbar_wait(pv_prev, pv_parity);
    tc_fence_after();
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
        uint32_t o[32];
        tmem_ld32(oAddr + 32 * cc, o);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
        tmem_st32(oAddr + 32 * cc, o);
    }
    tmem_st_wait();
}

struct SoftmaxState {
    float m_run = -INFINITY; // running max, exp2 domain (logit * scale_log2)
    float l_run = 0.0f;      // running sum of p over this thread's column half
    int cov = 0;             // attended tokens in this thread's column half
};

// One S tile, one row, one column half (thread). The two softmax warpgroups
// split every tile's columns: warpgroup w owns tile columns [NC*w, NC*w + NC)
// (NC = 64 for segment tiles; the 32-key sink tile is all warpgroup 0's, NC = 32,
// and warpgroup 1 takes NC = 0). The row max is combined through shared memory
// (xch, one named barrier per lane quadrant = the two warps that own the same
// TMEM lanes); each half keeps its own partial l and coverage, summed at the
// end. Both halves therefore see the same running max and take the same lazy
// rescale decisions. S holds raw fp32 logits*sqrt(d); the bf16 P pairs of
// columns [c0, c0+NC) are written to TMEM columns [c0/2, c0/2 + NC/2) of the
// same buffer (written only after the barrier, i.e. after both halves have
// read their S columns).
template <int NC>
__device__ __forceinline__ void softmax_part(uint32_t sAddr, uint32_t pAddr, uint32_t oAddr,
                                             uint32_t nib, int64_t lim, float scale_log2,
                                             SoftmaxState &st, float *xch_mine,
                                             const float *xch_other, uint32_t bar_id,
                                             uint64_t *pv_prev, uint32_t pv_parity) {
    constexpr int NS = NC / 32 > 0 ? NC / 32 : 1; // 32-key sub-blocks in this half
    // nib: this half's sub-block bits; lim: valid columns c <= lim (half-relative)
    const bool any_valid = NC > 0 && nib != 0u && lim >= 0;
    const bool zero = __all_sync(0xffffffffu, !any_valid);
    uint32_t s[NC > 0 ? NC : 1];
    float mt = -INFINITY;
    int nvalid = 0;
    bool full = false;
    if constexpr (NC > 0) {
        if (!zero) {
#pragma unroll
            for (int c4 = 0; c4 < NC / 32; ++c4)
                tmem_ld32(sAddr + 32 * c4, *reinterpret_cast<uint32_t(*)[32]>(&s[32 * c4]));
            tmem_ld_wait();
            full = nib == ((1u << NS) - 1u) && lim >= NC - 1;
            nvalid = NC;
            if (!full) {
                nvalid = 0;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const bool ok = ((nib >> (c >> 5)) & 1u) && c <= lim;
                    s[c] = ok ? s[c] : __float_as_uint(-INFINITY);
                    nvalid += ok ? 1 : 0;
                }
            }
            // four independent max chains (latency), then combined
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int c = 0; c < NC; c += 8)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    mx[u] = fmax3(mx[u], __uint_as_float(s[c + 2 * u]), __uint_as_float(s[c + 2 * u + 1]));
            mt = fmax3(mx[0], mx[1], fmaxf(mx[2], mx[3]));
        }
    }
    // combine the row max with the other column half
    *xch_mine = mt;
    named_bar_sync(bar_id, 64);
    mt = fmaxf(mt, *xch_other);
    const float m_new = fmaxf(st.m_run, mt * scale_log2);
    // lazy rescale: only when the running max grows by > 8 (exp2 domain); P is
    // computed against the new max, O and l are rescaled after P is stored
    // (fewer live registers), before p_full releases PV of this tile.
    const bool need = st.m_run != -INFINITY && m_new > st.m_run + 8.0f;
    const float alpha = need ? ex2_approx(st.m_run - m_new) : 1.0f;
    if (st.m_run == -INFINITY || need) st.m_run = m_new;
    if (need) st.l_run *= alpha;
    const bool any_need = __any_sync(0xffffffffu, need);
    if constexpr (NC > 0) {
        if (zero) {
            // nothing of this half is attended by the warp's rows: P = 0, no exp work
            uint32_t z[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) z[e] = 0u;
            if constexpr (NC == 64) tmem_st32(pAddr, z);
            else tmem_st16(pAddr, *reinterpret_cast<uint32_t(*)[16]>(&z[0]));
            tmem_st_wait();
            if (any_need) rescale_o(oAddr, alpha, pv_prev, pv_parity);
            return;
        }
        // p = exp2(s * scale_log2 - m); masked columns hold -inf -> p = 0. A row
        // with nothing valid yet keeps m = -inf: use 0 so -inf * scale - 0 = -inf.
        const float neg_m = st.m_run == -INFINITY ? 0.0f : -st.m_run;
        const unsigned long long sc2 = pack_f2(scale_log2, scale_log2), nm2 = pack_f2(neg_m, neg_m);
        unsigned long long psum2 = 0ull;
        if (NC == 64 && __all_sync(0xffffffffu, full)) {
            // Full halves: every second pair takes exp2 on the FMA/ALU pipes
            // (Cody-Waite split + degree-3 polynomial, rel. err 1e-4 < bf16's
            // 2^-8), the rest on MUFU (16 ex2/clk/SM): per SMSP and tile the XU,
            // FMA and ALU pipes then carry about equal work.
#pragma unroll
            for (int c2 = 0; c2 < NC / 2; ++c2) {
                unsigned long long x = (static_cast<unsigned long long>(s[2 * c2 + 1]) << 32) | s[2 * c2];
                ffma2_f32(x, sc2, nm2);
                float p0, p1;
                if (c2 & 1) {
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
                fadd2_f32(psum2, pack_f2(p0, p1));
                s[c2] = pack_bf16x2(p0, p1);
            }
        } else {
#pragma unroll
            for (int c2 = 0; c2 < NC / 2; ++c2) {
                unsigned long long x = (static_cast<unsigned long long>(s[2 * c2 + 1]) << 32) | s[2 * c2];
                ffma2_f32(x, sc2, nm2); // x = x * scale + (-m), two lanes
                const float p0 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x)));
                const float p1 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x >> 32)));
                fadd2_f32(psum2, pack_f2(p0, p1));
                s[c2] = pack_bf16x2(p0, p1); // in place: s[c2] was consumed at step c2/2
            }
        }
        st.l_run += __uint_as_float(static_cast<uint32_t>(psum2)) +
                    __uint_as_float(static_cast<uint32_t>(psum2 >> 32));
        st.cov += nvalid;
        if constexpr (NC == 64) tmem_st32(pAddr, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        else tmem_st16(pAddr, *reinterpret_cast<uint32_t(*)[16]>(&s[0]));
        tmem_st_wait();
    }
    if (any_need) rescale_o(oAddr, alpha, pv_prev, pv_parity);
}

__global__ void __launch_bounds__(kAttnThreads, 1)
sparse_attention_kernel(const __nv_bfloat16 *__restrict__ q, const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const uint32_t *__restrict__ mask,
                        __nv_bfloat16 *__restrict__ out, int32_t *__restrict__ coverage,
                        int64_t tokens, int hq, int hkv, float scale_log2, int64_t i_lo,
                        int64_t ni) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
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
    const int p = static_cast<int>(blockIdx.x % npairs);
    // query blocks [i_lo, i_lo + ni): a token-range slice (chunked host pipeline)
    const int64_t i = i_lo + ni - 1 - static_cast<int64_t>((blockIdx.x / npairs) % ni);
    const int bg = static_cast<int>(blockIdx.x / (npairs * ni));
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
            mbar_init(&sm.v_full[s], 1);
            mbar_init(&sm.kv_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.s_full[s], 1);
            mbar_init(&sm.p_full[s], 8);
            mbar_init(&sm.pv_done[s], 1);
        }
        sm.ntiles = 0;
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(&sm.tmem_base);

    // ---- active tile list (block-wide stream compaction, ascending order)
    const int64_t rowbase = (static_cast<int64_t>(b) * hq + hA) * nq + i;
    const uint32_t *rowA = mask ? mask + rowbase * words : nullptr;
    const uint32_t *rowB = (mask && hasB) ? mask + (rowbase + nq) * words : nullptr;
    const int total = qend > kBlockK ? 1 + static_cast<int>((qend - kBlockK + 127) / 128) : 1;
    __syncthreads();
    for (int start = 0; start < total; start += kAttnThreads) {
        const int j = start + tid;
        uint32_t bits = 0;
        if (j < total) {
            const int64_t j0 = j == 0 ? 0 : 1 + 4LL * (j - 1);
            const int nsub = j == 0 ? 1 : 4;
            uint32_t causal = 0; // key blocks that exist and are not fully future
            for (int e = 0; e < nsub; ++e)
                if (j0 + e < nk && (j0 + e) * kBlockK < qend) causal |= 1u << e;
            const uint32_t nibA = mask ? mask_bits4(rowA, words, j0) : 0xFu;
            const uint32_t nibB = !hasB ? 0u : (mask ? mask_bits4(rowB, words, j0) : 0xFu);
            bits = (nibA & causal) | ((nibB & causal) << 4);
        }
        const bool active = bits != 0;
        const uint32_t ballot = __ballot_sync(0xffffffffu, active);
        if (lane == 0) sm.warp_cnt[warp] = __popc(ballot);
        __syncthreads();
        int base = sm.ntiles;
        for (int w = 0; w < warp; ++w) base += sm.warp_cnt[w];
        if (active) {
            const int pos = base + __popc(ballot & ((1u << lane) - 1u));
            if (pos < kMaxTiles) sm.tiles[pos] = static_cast<uint32_t>(j) | (bits << 16);
        }
        __syncthreads();
        if (tid == 0) {
            int s = sm.ntiles;
            for (int w = 0; w < kAttnThreads / 32; ++w) s += sm.warp_cnt[w];
            sm.ntiles = s < kMaxTiles ? s : kMaxTiles;
        }
        __syncthreads();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const int ntiles = sm.ntiles;

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA
        if (elect_one() && ntiles > 0) {
            tma_prefetch(&tm_k);
            tma_prefetch(&tm_v);
            for (int jj = 0; jj < ntiles; ++jj) {
                const int st = jj % kKvStages;
                const int j = static_cast<int>(sm.tiles[jj] & 0xFFFFu);
                const int key0 = j == 0 ? 0 : kBlockK + 128 * (j - 1);
                mbar_wait(&sm.kv_empty[st], ((jj / kKvStages) & 1) ^ 1);
                mbar_expect_tx(&sm.k_full[st], 2 * kTileBytesHalf);
                tma_load_4d(sm.k[st][0], &tm_k, &sm.k_full[st], 0, g, key0, b);
                tma_load_4d(sm.k[st][1], &tm_k, &sm.k_full[st], 64, g, key0, b);
                mbar_expect_tx(&sm.v_full[st], 2 * kTileBytesHalf);
                tma_load_4d(sm.v[st][0], &tm_v, &sm.v_full[st], 0, g, key0, b);
                tma_load_4d(sm.v[st][1], &tm_v, &sm.v_full[st], 64, g, key0, b);
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA
        if (elect_one() && ntiles > 0) {
            constexpr uint32_t idesc_pv = idesc_bf16(128, 128, true);
            const bool prof = g_attn_prof_on != 0;
            const long long t_start = clock64();
            long long w_k = 0, w_p = 0, w_v = 0, t0 = 0;
            mbar_wait(&sm.q_ready, 0);
            tc_fence_after();
            for (int jj = 0; jj <= ntiles; ++jj) {
                if (jj < ntiles) {
                    const int st = jj % kKvStages;
                    const int sb = jj & 1;
                    const int j = static_cast<int>(sm.tiles[jj] & 0xFFFFu);
                    const uint32_t idesc_s = j == 0 ? idesc_bf16(128, 32, false) : idesc_bf16(128, 128, false);
                    if (prof) t0 = clock64();
                    mbar_wait(&sm.k_full[st], (jj / kKvStages) & 1);
                    if (prof) w_k += clock64() - t0;
                    tc_fence_after();
                    const uint64_t kd0 = umma_desc_sw128(smem_u32(sm.k[st][0]), 16, 1024);
                    const uint64_t kd1 = umma_desc_sw128(smem_u32(sm.k[st][1]), 16, 1024);
                    const uint32_t dS = tmem + kColS0 + 128u * static_cast<uint32_t>(sb);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) { // K = 16 bf16 = 8 TMEM columns of Q
                        const uint64_t bd = (kk < 4 ? kd0 : kd1) + 2 * (kk & 3);
                        mma_bf16_ts(dS, tmem + kColQ + 8 * kk, bd, idesc_s, kk > 0);
                    }
                    tc_commit(&sm.s_full[sb]);
                }
                if (jj > 0) {
                    const int pj = jj - 1;
                    const int pst = pj % kKvStages;
                    const int psb = pj & 1;
                    const int jp = static_cast<int>(sm.tiles[pj] & 0xFFFFu);
                    const int steps = jp == 0 ? 2 : 8;
                    if (prof) t0 = clock64();
                    mbar_wait(&sm.p_full[psb], (pj >> 1) & 1);
                    if (prof) { w_p += clock64() - t0; t0 = clock64(); }
                    mbar_wait(&sm.v_full[pst], (pj / kKvStages) & 1);
                    if (prof) w_v += clock64() - t0;
                    tc_fence_after();
                    const uint64_t vd = umma_desc_sw128(smem_u32(sm.v[pst][0]), kTileBytesHalf, 1024);
                    const uint32_t aP = tmem + kColS0 + 128u * static_cast<uint32_t>(psb);
                    for (int kk = 0; kk < steps; ++kk)
                        mma_bf16_ts(tmem + kColO, aP + 8 * kk, vd + 128 * kk, // +16 keys = 2 KB
                                    idesc_pv, (pj > 0 || kk > 0) ? 1u : 0u);
                    tc_commit(&sm.kv_empty[pst]);
                    tc_commit(&sm.pv_done[psb]);
                }
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
        const int wg = (warp - 3) >> 2;          // column half of every tile
        const int quad = warp & 3;               // TMEM lane quadrant (warp id % 4)
        const int r = quad * 32 + lane;
        const int half = r >> 6;                 // 0: head hA, 1: head hA + 1
        const int h = hA + half;
        const int64_t grow = q0 + (r & 63);
        const bool row_ok = grow < tokens && (half == 0 || hasB);
        const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        const uint32_t bar_id = 1 + quad;
        // Q row half -> TMEM columns [kColQ + 32 wg, +32): the A operand of S = Q K^T
        {
            uint32_t a[32];
            const uint4 *src = reinterpret_cast<const uint4 *>(
                q + ((static_cast<int64_t>(b) * tokens + grow) * hq + h) * kHeadDim + 64 * wg);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint4 w = row_ok ? __ldg(src + e) : make_uint4(0, 0, 0, 0);
                a[4 * e] = w.x, a[4 * e + 1] = w.y, a[4 * e + 2] = w.z, a[4 * e + 3] = w.w;
            }
            tmem_st32(lane_addr + kColQ + 32 * wg, a);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.q_ready);
        }
        SoftmaxState st;
        const uint32_t oAddr = lane_addr + kColO + 64u * wg;
        const bool prof = warp == 3 && lane == 0 && g_attn_prof_on != 0;
        const long long t_loop = clock64();
        long long w_s = 0, t_part = 0, t1 = 0;
        for (int jj = 0; jj < ntiles; ++jj) {
            const int sb = jj & 1;
            const uint32_t info = sm.tiles[jj];
            const int j = static_cast<int>(info & 0xFFFFu);
            const uint32_t nib = (info >> (16 + 4 * half)) & 0xFu;
            const int64_t key0 = j == 0 ? 0 : kBlockK + 128LL * (j - 1);
            const uint32_t sBase = lane_addr + kColS0 + 128u * sb;
            float *xm = &sm.xch[sb][wg][r];
            const float *xo = &sm.xch[sb][wg ^ 1][r];
            if (prof) t1 = clock64();
            mbar_wait(&sm.s_full[sb], (jj >> 1) & 1);
            if (prof) { const long long t2 = clock64(); w_s += t2 - t1; t1 = t2; }
            tc_fence_after();
            const int pj = jj - 1;
            // The 32-key sink tile runs through the same 64-column code: its
            // columns >= 32 (stale S data) are masked like unselected sub-blocks,
            // so warpgroup 1 always takes the zero path there.
            const uint32_t nib_half = j == 0 ? (wg == 0 ? (nib & 1u) : 0u) : (nib >> (2 * wg)) & 3u;
            const int64_t lim = row_ok ? grow - key0 - 64 * wg : -1;
            softmax_part<64>(sBase + 64u * wg, sBase + 32u * wg, oAddr, nib_half, lim, scale_log2, st,
                             xm, xo, bar_id, &sm.pv_done[pj & 1], (pj >> 1) & 1);
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
        }
        // ---- epilogue: l = l_half0 + l_half1, O / l -> bf16 (each half its 64 columns)
        if (wg == 1) {
            sm.fin_l[r] = st.l_run;
            sm.fin_cov[r] = st.cov;
        }
        named_bar_sync(bar_id, 64);
        float l_tot = st.l_run;
        int cov_tot = st.cov;
        if (wg == 0) {
            l_tot += sm.fin_l[r];
            cov_tot += sm.fin_cov[r];
        }
        named_bar_sync(bar_id, 64);
        if (wg == 0) sm.fin_l[r] = l_tot; // one sum, used by both halves
        named_bar_sync(bar_id, 64);
        if (wg == 1) l_tot = sm.fin_l[r];
        if (ntiles > 0) {
            const int last = ntiles - 1;
            mbar_wait(&sm.pv_done[last & 1], (last >> 1) & 1);
            tc_fence_after();
        }
        const float inv_l = l_tot > 0.0f ? 1.0f / l_tot : 0.0f;
        __nv_bfloat16 *dst =
            out + ((static_cast<int64_t>(b) * tokens + grow) * hq + h) * kHeadDim + 64 * wg;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            uint32_t o[32];
            if (ntiles > 0) {
                tmem_ld32(oAddr + 32 * cc, o);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) o[e] = 0u;
            }
            if (row_ok) {
                uint4 w[4];
                uint32_t *wp = reinterpret_cast<uint32_t *>(w);
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    wp[e] = pack_bf16x2(__uint_as_float(o[2 * e]) * inv_l, __uint_as_float(o[2 * e + 1]) * inv_l);
                uint4 *d4 = reinterpret_cast<uint4 *>(dst + 32 * cc);
#pragma unroll
                for (int e = 0; e < 4; ++e) d4[e] = w[e];
            }
        }
        if (wg == 0 && row_ok && coverage)
            coverage[(static_cast<int64_t>(b) * hq + h) * tokens + grow] = cov_tot;
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
    return cudaMemcpyToSymbol(g_attn_prof_on, &enable, sizeof(int));
}

size_t attention_smem_bytes() { return sizeof(AttnSmem) + 1024; }

cudaError_t launch_sparse_attention(const void *q, const CUtensorMap &tm_k, const CUtensorMap &tm_v,
                                    const uint32_t *mask, void *out, int32_t *coverage,
                                    int64_t batch, int64_t tokens, int hq, int hkv, float scale_log2,
                                    cudaStream_t stream, int64_t i_lo, int64_t i_hi) {
    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    if (nq / 2 + 3 > kMaxTiles) return cudaErrorInvalidValue;
    static bool configured = false;
    const size_t smem = attention_smem_bytes();
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(sparse_attention_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int npairs = (hq / hkv + 1) / 2;
    if (i_hi < 0 || i_hi > nq) i_hi = nq;
    if (i_hi <= i_lo) return cudaSuccess;
    const int64_t grid = batch * hkv * npairs * (i_hi - i_lo);
    sparse_attention_kernel<<<static_cast<unsigned>(grid), kAttnThreads, smem, stream>>>(
        static_cast<const __nv_bfloat16 *>(q), tm_k, tm_v, mask, static_cast<__nv_bfloat16 *>(out),
        coverage, tokens, hq, hkv, scale_log2, i_lo, i_hi - i_lo);
    return cudaGetLastError();
}

} // namespace sale_b200
