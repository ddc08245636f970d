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
// adjacent query blocks (profiles/mask_stats.py). Row 16q + t of head 2p + hh
// is TMEM lane 32q + 16hh + t, so every lane quadrant (SMSP) has rows of both
// heads and a tile selected by one head only leaves the other head's warps
// with a zero-P store.
// Key tiles follow the segment grid of the Selection-Pass: tile 0 = the
// 32-key sink block, tile s+1 = keys [32+128s, 160+128s) = key blocks
// 1+4s..4+4s. A tile is visited iff any of its 8 (head, kblock) bits is set;
// inside a visited tile unselected 32-key sub-blocks and the causal diagonal
// are masked per row.
//
// TMEM (512 columns): O [0,128) | S0 [128,256) | S1 [256,384) | S2 [384,512):
// THREE S buffers, so the softmax of consecutive tiles overlaps — the MMA
// runs S_{j+3} while the softmax warps still work on S_{j+1} and S_{j+2}.
// Q is the A operand of S = Q K^T from shared memory (SS MMA; K streams
// through a 3-stage TMA ring, V through a 2-stage ring), P overwrites S in
// place as the A operand of O += P V (TS MMA). The row sums l are fp32 sums
// of P in the softmax warps' registers.
//
// Warps (20 = 5 warpgroups; setmaxnreg moves the control warpgroup's registers
// to the softmax warpgroups):
//   warp 0  TMEM allocator, then TMA: K_j (released by S_j) and V_j (released
//           by PV_j)
//   warp 1  MMA: S_0, S_1, S_2, then per tile j: O += P_j V_j, S_{j+3} into
//           the buffer P_j came from (in-order tensor pipe)
//   warps 4-19 softmax: warp (quad q, head hh, parity par) serves TMEM lanes
//           32q + 16hh + [0, 16) (16 rows of one head, two rows x 64 columns
//           per thread through 16x256b loads) for the tiles j = par (mod 2).
//           Two warps of each row set alternate over the tiles, so four warps
//           per SMSP work on two tiles at once; the running row reference
//           passes between them through shared memory right after each
//           tile's row max (m_xfer), before the exps. Lazy-rescaled online
//           softmax in the exp2 domain (O rescaled in TMEM only when the
//           reference grows by > 8); 3/8 of the full-tile exp2 pairs on an
//           FMA/ALU polynomial; P -> bf16 -> tcgen05.st over S.
#include "common.cuh"
#include "internal.h"

namespace sale_b200 {

constexpr int kCtlWarps = 4;                   // warpgroup 0: TMA (+ TMEM allocator), MMA, 2 idle
constexpr int kSmWarps = 8;                    // softmax: 2 per TMEM lane quadrant (tile parities)
constexpr int kAttnThreads = 32 * (kCtlWarps + kSmWarps);
constexpr int kCtlRegs = 56, kSmRegs = 224;    // setmaxnreg split of the CTA pool (384 x 168)
constexpr int kMaxTiles = 4200;                // supports N <= 512K
constexpr int kKvStages = 3;                   // K ring
constexpr int kVStages = 2;                    // V ring
constexpr int kSBufs = 3;                      // S / P buffers in TMEM
// s_full / p_full / pv_done per tile mod 6: a softmax warp serves every other
// tile, so with three buffers it would skip every other phase of a per-buffer
// barrier; per (tile mod 6) barriers are all observed by one parity's warps
constexpr int kTileBars = 2 * kSBufs;
constexpr int kTileBytesHalf = 128 * 64 * 2;   // 128 rows x 64 bf16 = 16 KB
constexpr uint32_t kColO = 0, kColS0 = 128;

struct AttnSmem {
    alignas(1024) uint8_t q[2][kTileBytesHalf];          // Q (A operand), two 64-column halves
    alignas(1024) uint8_t k[kKvStages][2][kTileBytesHalf];
    // V as the B operand of O += P V: N = 128 = two 64-column chunks at stride
    // kVStages x 16 KB
    alignas(1024) uint8_t v[2][kVStages][kTileBytesHalf];
    uint64_t q_ready, k_full[kKvStages], v_full[kVStages], k_empty[kKvStages], v_empty[kVStages];
    uint64_t s_full[kTileBars], p_full[kTileBars], pv_done[kTileBars];
    uint64_t m_xfer[8];        // [quad * 2 + receiving parity]
    float m_ref[128];          // [TMEM lane]: the last published row references
    float fin_m[2][128];       // epilogue: [parity][lane] last reference of l
    float fin_l[2][128];       //           and the partial row sum at that reference
    int fin_c[128];            //           coverage of the parity-1 warps
    uint32_t tmem_base;
    int ntiles;
    int warp_tot[kSmWarps];    // tile-list build: per-warp counts of a round
    uint32_t tiles[kMaxTiles]; // j | bits8 << 16
};

// Optional cycle instrumentation (sale_b200_attention_profile): [0] softmax
// loop total, [1] S-ready waits, [2] softmax_part time, [3] tiles (warp 4,
// lane 0, summed over CTAs; this warp serves every other tile); [4] MMA loop
// total, [5] K waits, [6] P waits, [7] V waits, [8] CTAs, [9] prologue (start
// -> tile list ready, thread 0), [10] epilogue (last tile -> end, warp 4 lane
// 0), [11] reference hand-off waits, [12] unused, [13] TMEM allocated, [14]
// tile list done, [15] barriers done.
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
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&p);
}
template <uint32_t kRegs> __device__ __forceinline__ void setmaxnreg_inc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs));
}
template <uint32_t kRegs> __device__ __forceinline__ void setmaxnreg_dec() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs));
}

// 32 lanes x 32 columns of 32-bit (thread t = lane t) into r[0..31]
__device__ __forceinline__ void tmem_ld32p(uint32_t taddr, uint32_t *r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : SALE_R16(r, 0), SALE_R16(r, 16)
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32p(uint32_t taddr, const uint32_t *r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
            taddr),
        SALE_W16(r, 0), SALE_W16(r, 16)
        : "memory");
}

// O row of this thread (its TMEM lane, 128 columns) *= alpha, once PV of
// every earlier tile has landed in O.
__device__ __forceinline__ void rescale_o_row(uint32_t oAddr, float alpha, uint64_t *pv_prev,
                                              uint32_t pv_parity) {
    mbar_wait(pv_prev, pv_parity);
    tc_fence_after();
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        uint32_t o[32];
        tmem_ld32p(oAddr + 32 * cc, o);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
        tmem_st32p(oAddr + 32 * cc, o);
    }
    tmem_st_wait();
}

struct SoftmaxState {
    float m = -INFINITY;        // reference (exp2 domain) of this thread's partial row sum
    unsigned long long l2 = 0;  // two fp32 partial sums of P (FADD2 lanes)
    int cov = 0;                // attended tokens of this row in this warp's tiles
};

// Phase A of one S tile: thread = one row (its TMEM lane), 128 columns in
// registers (four 32x32b loads), masked, and the row max in the thread. nib:
// the row head's four 32-key sub-block bits of this tile; lim: valid columns
// c <= lim (-1: none). Returns false (warp-uniform) when nothing of the tile
// is attended by the warp's rows; s is then untouched.
__device__ __forceinline__ bool softmax_load_max(uint32_t sAddr, uint32_t nib, int lim, uint32_t (&s)[128],
                                                 float &tmax, bool &full, SoftmaxState &st) {
    const bool any_valid = nib != 0u && lim >= 0;
    if (__all_sync(0xffffffffu, !any_valid)) {
        tmax = -INFINITY;
        return false;
    }
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) tmem_ld32p(sAddr + 32 * cc, s + 32 * cc);
    tmem_ld_wait();
    full = nib == 0xFu && lim >= 127;
    if (!__all_sync(0xffffffffu, full)) {
        int nv = 0;
#pragma unroll
        for (int c = 0; c < 128; ++c) {
            const bool ok = ((nib >> (c >> 5)) & 1u) && c <= lim;
            s[c] = ok ? s[c] : __float_as_uint(-INFINITY);
            nv += ok ? 1 : 0;
        }
        st.cov += nv;
    } else {
        st.cov += 128;
    }
    float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int c = 0; c < 128; c += 8) {
        mx[0] = fmax3(mx[0], __uint_as_float(s[c]), __uint_as_float(s[c + 1]));
        mx[1] = fmax3(mx[1], __uint_as_float(s[c + 2]), __uint_as_float(s[c + 3]));
        mx[2] = fmax3(mx[2], __uint_as_float(s[c + 4]), __uint_as_float(s[c + 5]));
        mx[3] = fmax3(mx[3], __uint_as_float(s[c + 6]), __uint_as_float(s[c + 7]));
    }
    tmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
    return true;
}

// Phase B: P = exp2(s * scale_log2 - m) against the row reference m (-inf while
// the row has attended nothing: masked columns hold -inf -> p = 0), the row
// sum added to st.l2, bf16 pairs to columns [0, 64) of the same S buffer.
__device__ __forceinline__ void softmax_exp_store(uint32_t sAddr, uint32_t (&s)[128], bool full, float m,
                                                  float scale_log2, SoftmaxState &st) {
    const unsigned long long sc2 = pack_f2(scale_log2, scale_log2);
    const float neg_m = m == -INFINITY ? 0.0f : -m;
    const unsigned long long nm2 = pack_f2(neg_m, neg_m);
    if (__all_sync(0xffffffffu, full)) {
        // Full tiles: 3/8 of the pairs (R = 0, 3, 5 mod 8) take exp2 on the
        // FMA/ALU pipes (Cody-Waite split + degree-3 polynomial, rel. err 1e-4
        // < bf16's 2^-8), the rest on MUFU (16 ex2/clk/SM).
#pragma unroll
        for (int R = 0; R < 64; ++R) {
            unsigned long long x = (static_cast<unsigned long long>(s[2 * R + 1]) << 32) | s[2 * R];
            ffma2_f32(x, sc2, nm2);
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
                p1 = __uint_as_float(shl23_add(static_cast<uint32_t>(t >> 32), static_cast<uint32_t>(pp >> 32)));
            } else {
                p0 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x)));
                p1 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x >> 32)));
            }
            fadd2_f32(st.l2, pack_f2(p0, p1));
            s[R] = pack_bf16x2(p0, p1); // in place: index R was already consumed
        }
    } else {
#pragma unroll
        for (int R = 0; R < 64; ++R) {
            unsigned long long x = (static_cast<unsigned long long>(s[2 * R + 1]) << 32) | s[2 * R];
            ffma2_f32(x, sc2, nm2); // x = x * scale + (-m), two lanes
            const float p0 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x)));
            const float p1 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x >> 32)));
            fadd2_f32(st.l2, pack_f2(p0, p1));
            s[R] = pack_bf16x2(p0, p1);
        }
    }
    tmem_st32p(sAddr, s);
    tmem_st32p(sAddr + 32, s + 32);
    tmem_st_wait();
}

// kProf: the cycle-instrumented instance (sale_b200_attention_profile); the
// production instance carries no profiling code.
template <bool kProf>
__global__ void __launch_bounds__(kAttnThreads, 1)
sparse_attention_kernel(const __nv_bfloat16 *__restrict__ q, const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const uint32_t *__restrict__ mask,
                        __nv_bfloat16 *__restrict__ out, int32_t *__restrict__ coverage,
                        unsigned long long *__restrict__ empty_rows, int64_t tokens, int hq, int hkv,
                        float scale_log2, int64_t i_lo, int64_t ni) {
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

    if (warp == 0) {
        tmem_alloc<512>(&sm.tmem_base);
        if (lane == 0 && kProf)
            atomicAdd(&g_attn_prof[13], static_cast<unsigned long long>(clock64() - t_kernel));
    } else if (tid == 32) {
        mbar_init(&sm.q_ready, kSmWarps);
        for (int s = 0; s < kKvStages; ++s) {
            mbar_init(&sm.k_full[s], 1);
            mbar_init(&sm.k_empty[s], 1);
        }
        for (int s = 0; s < kVStages; ++s) {
            mbar_init(&sm.v_full[s], 1);
            mbar_init(&sm.v_empty[s], 1);
        }
        for (int s = 0; s < kTileBars; ++s) {
            mbar_init(&sm.s_full[s], 1);
            mbar_init(&sm.p_full[s], kSmWarps / 2); // the warps of one tile parity
            mbar_init(&sm.pv_done[s], 1);
        }
        for (int s = 0; s < 8; ++s) mbar_init(&sm.m_xfer[s], 1);
        fence_barrier_init();
        if (kProf) atomicAdd(&g_attn_prof[15], static_cast<unsigned long long>(clock64() - t_kernel));
    } else if (warp >= kCtlWarps) {
        // ---- active tile list (ascending), built by the 16 softmax warps while
        // the control warps set up: per round, warp w = warp - 4 takes pass
        // p = 16 round + w = segment-tile groups [32p, 32p + 32); lane t of a
        // pass owns the 8 tiles 8g+1 .. 8g+8 (g = 32p + t) = key blocks
        // 32g+1 .. 32g+32 (bits 1-31 of mask word g, bit 0 of word g+1); tile
        // 0 is the sink block. Prefix sums: ballots within a warp, the sixteen
        // warp totals through shared memory (one named barrier per round).
        const int w3 = warp - kCtlWarps;
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
        if (w3 == 0 && lane == 0 && sink) sm.tiles[0] = sink << 16;
        const uint32_t lt = (1u << lane) - 1u;
        for (int base = 0; base < groups; base += 32 * kSmWarps) {
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
            named_bar_sync(1, 32 * kSmWarps);
            int before = 0, all = 0;
#pragma unroll
            for (int w = 0; w < kSmWarps; ++w) {
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
            named_bar_sync(1, 32 * kSmWarps); // warp_tot is reused by the next round
        }
        if (w3 == 0 && lane == 0) sm.ntiles = carry < kMaxTiles ? carry : kMaxTiles;
        if (w3 == 0 && lane == 0 && kProf)
            atomicAdd(&g_attn_prof[14], static_cast<unsigned long long>(clock64() - t_kernel));
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0 && kProf)
        atomicAdd(&g_attn_prof[9], static_cast<unsigned long long>(clock64() - t_kernel));
    const uint32_t tmem = sm.tmem_base;
    const int ntiles = sm.ntiles;

    if (warp < kCtlWarps) {
        setmaxnreg_dec<kCtlRegs>();
        if (warp == 0) {
            // ------------------------------------------------------------ TMA
            if (elect_one() && ntiles > 0) {
                tma_prefetch(&tm_k);
                tma_prefetch(&tm_v);
                // K_jj is released by S_jj, V_jj by PV_jj. The MMA issues S_{j+3}
                // right behind PV_j, so V trails K by two tiles here.
                auto key0_of = [&](int jj) {
                    const int j = static_cast<int>(sm.tiles[jj] & 0xFFFFu);
                    return j == 0 ? 0 : kBlockK + 128 * (j - 1);
                };
                auto load_v = [&](int vj) {
                    const int st = vj % kVStages;
                    const int key0 = key0_of(vj);
                    mbar_wait(&sm.v_empty[st], ((vj / kVStages) & 1) ^ 1);
                    mbar_expect_tx(&sm.v_full[st], 2 * kTileBytesHalf);
                    tma_load_4d(sm.v[0][st], &tm_v, &sm.v_full[st], 0, g, key0, b);
                    tma_load_4d(sm.v[1][st], &tm_v, &sm.v_full[st], 64, g, key0, b);
                };
                for (int jj = 0; jj < ntiles; ++jj) {
                    const int st = jj % kKvStages;
                    const int key0 = key0_of(jj);
                    mbar_wait(&sm.k_empty[st], ((jj / kKvStages) & 1) ^ 1);
                    mbar_expect_tx(&sm.k_full[st], 2 * kTileBytesHalf);
                    tma_load_4d(sm.k[st][0], &tm_k, &sm.k_full[st], 0, g, key0, b);
                    tma_load_4d(sm.k[st][1], &tm_k, &sm.k_full[st], 64, g, key0, b);
                    if (jj >= 2) load_v(jj - 2);
                }
                for (int vj = ntiles >= 2 ? ntiles - 2 : 0; vj < ntiles; ++vj) load_v(vj);
                // drain: the last releases of every ring stage (S / PV commits) land
                // before the CTA exits, so no mbarrier phase completes unobserved
                for (int jj = ntiles > kKvStages ? ntiles - kKvStages : 0; jj < ntiles; ++jj)
                    mbar_wait(&sm.k_empty[jj % kKvStages], (jj / kKvStages) & 1);
                for (int v2 = ntiles > kVStages ? ntiles - kVStages : 0; v2 < ntiles; ++v2)
                    mbar_wait(&sm.v_empty[v2 % kVStages], (v2 / kVStages) & 1);
            }
        } else if (warp == 1) {
            // ------------------------------------------------------------ MMA
            if (elect_one() && ntiles > 0) {
                constexpr uint32_t idesc_pv = idesc_bf16(128, 128, true);
                const bool prof = kProf;
                const long long t_start = clock64();
                long long w_k = 0, w_p = 0, w_v = 0, t0 = 0;
                mbar_wait(&sm.q_ready, 0);
                tc_fence_after();
                const uint64_t qd0 = umma_desc_sw128(smem_u32(sm.q[0]), 16, 1024);
                const uint64_t qd1 = umma_desc_sw128(smem_u32(sm.q[1]), 16, 1024);
                // Order on the tensor pipe: S_0, S_1, S_2, PV_0, S_3, PV_1, S_4, ...
                // S_{j+3} reuses S_j's buffer right behind PV_j (in-order pipe).
                auto issue_s = [&](int jj) {
                    const int st = jj % kKvStages;
                    const int sb = jj % kSBufs;
                    const int j = static_cast<int>(sm.tiles[jj] & 0xFFFFu);
                    const uint32_t idesc_s = j == 0 ? idesc_bf16(128, 32, false) : idesc_bf16(128, 128, false);
                    const uint64_t kd0 = umma_desc_sw128(smem_u32(sm.k[st][0]), 16, 1024);
                    const uint64_t kd1 = umma_desc_sw128(smem_u32(sm.k[st][1]), 16, 1024);
                    const uint32_t dS = tmem + kColS0 + 128u * static_cast<uint32_t>(sb);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) { // K = 16 bf16 = 32 B of a SW128 row
                        const uint64_t off = 2 * (kk & 3);
                        mma_bf16_ss(dS, (kk < 4 ? qd0 : qd1) + off, (kk < 4 ? kd0 : kd1) + off, idesc_s,
                                    kk > 0 ? 1u : 0u);
                    }
                    tc_commit(&sm.s_full[jj % kTileBars]);
                    tc_commit(&sm.k_empty[st]);
                };
                auto wait_k = [&](int jj) {
                    if (prof) t0 = clock64();
                    mbar_wait(&sm.k_full[jj % kKvStages], (jj / kKvStages) & 1);
                    if (prof) w_k += clock64() - t0;
                    tc_fence_after();
                };
                for (int jj = 0; jj < kSBufs && jj < ntiles; ++jj) {
                    wait_k(jj);
                    issue_s(jj);
                }
                for (int pj = 0; pj < ntiles; ++pj) {
                    const int nx = pj + kSBufs;
                    const int pst = pj % kVStages;
                    const int psb = pj % kSBufs;
                    const int jp = static_cast<int>(sm.tiles[pj] & 0xFFFFu);
                    const int steps = jp == 0 ? 2 : 8;
                    if (nx < ntiles) wait_k(nx);
                    if (prof) t0 = clock64();
                    mbar_wait(&sm.v_full[pst], (pj / kVStages) & 1);
                    if (prof) { w_v += clock64() - t0; t0 = clock64(); }
                    mbar_wait(&sm.p_full[pj % kTileBars], (pj / kTileBars) & 1);
                    if (prof) w_p += clock64() - t0;
                    tc_fence_after();
                    const uint64_t vd = umma_desc_sw128(smem_u32(sm.v[0][pst]), kVStages * kTileBytesHalf, 1024);
                    const uint32_t aP = tmem + kColS0 + 128u * static_cast<uint32_t>(psb);
                    for (int kk = 0; kk < steps; ++kk)
                        mma_bf16_ts(tmem + kColO, aP + 8 * kk, vd + 128 * kk, // +16 keys = 2 KB
                                    idesc_pv, (pj > 0 || kk > 0) ? 1u : 0u);
                    tc_commit(&sm.v_empty[pst]);
                    tc_commit(&sm.pv_done[pj % kTileBars]);
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
        }
    } else {
        setmaxnreg_inc<kSmRegs>();
        // ------------------------------------------------------------ softmax
        // warp (quad, par): thread = TMEM lane L = 32 quad + lane = row 16 quad +
        // lane % 16 of head hA + lane / 16; tiles j = par (mod 2)
        const int sw = warp - kCtlWarps;
        const int quad = warp & 3;
        const int par = sw >> 2;
        const int L = quad * 32 + lane;
        const int hh = lane >> 4;
        // Q staging: row L of the A operand, column half par, 16-byte chunks at
        // their SW128 positions
        {
            const int64_t qrow = q0 + quad * 16 + (lane & 15);
            const bool q_ok = qrow < tokens && (hh == 0 || hasB);
            const uint4 *src = reinterpret_cast<const uint4 *>(
                q + ((static_cast<int64_t>(b) * tokens + qrow) * hq + hA + hh) * kHeadDim + 64 * par);
            uint4 *dst = reinterpret_cast<uint4 *>(sm.q[par] + L * 128);
#pragma unroll
            for (int e = 0; e < 8; ++e) dst[e ^ (L & 7)] = q_ok ? __ldg(src + e) : make_uint4(0, 0, 0, 0);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.q_ready);
        }
        const int h = hA + hh;
        const int row = static_cast<int>(q0) + quad * 16 + (lane & 15); // token of this thread's row
        const bool ok = row < tokens && (hh == 0 || hasB);
        const uint32_t lane32 = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        const uint32_t oAddr = lane32 + kColO;
        uint64_t *xfer_in = &sm.m_xfer[quad * 2 + par];
        uint64_t *xfer_out = &sm.m_xfer[quad * 2 + (par ^ 1)];
        SoftmaxState st;
        const bool prof = sw == 0 && lane == 0 && kProf;
        const long long t_loop = clock64();
        long long w_s = 0, t_part = 0, t1 = 0, w_x = 0;
        for (int jj = par; jj < ntiles; jj += 2) {
            const int sb = jj % kSBufs;
            const uint32_t info = sm.tiles[jj];
            const int j = static_cast<int>(info & 0xFFFFu);
            uint32_t nib = (info >> (16 + 4 * hh)) & 0xFu;
            if (j == 0) nib &= 1u; // the 32-key sink tile: columns >= 32 hold stale S data
            // valid columns of this row (32-bit: tokens < 2^31), clamped
            const int key0 = j == 0 ? 0 : kBlockK + 128 * (j - 1);
            const int lim = ok ? min(row - key0, 1 << 20) : -1;
            const uint32_t sAddr = lane32 + kColS0 + 128u * static_cast<uint32_t>(sb);
            // the row reference after the previous tile (the other parity warp
            // publishes it right after its row max)
            float m = -INFINITY;
            if (jj > 0) {
                long long tx = 0;
                if (prof) tx = clock64();
                mbar_wait(xfer_in, ((jj - 1) >> 1) & 1);
                if (prof) w_x += clock64() - tx;
                m = sm.m_ref[L];
            }
            if (prof) t1 = clock64();
            mbar_wait(&sm.s_full[jj % kTileBars], (jj / kTileBars) & 1);
            if (prof) {
                const long long t2 = clock64();
                w_s += t2 - t1;
                t1 = t2;
            }
            tc_fence_after();
            uint32_t s[128];
            float tmax;
            bool full = false;
            const bool any = softmax_load_max(sAddr, nib, lim, s, tmax, full, st);
            // lazy rescale: the reference moves only when the row max grows by
            // > 8 (exp2 domain); O is rescaled after P is stored, before p_full
            // releases PV of this tile
            const float m_new = fmaxf(m, tmax * scale_log2);
            const bool need = m != -INFINITY && m_new > m + 8.0f;
            const float alpha = need ? ex2_approx(m - m_new) : 1.0f;
            if (m == -INFINITY || need) m = m_new;
            if (jj + 1 < ntiles) {
                sm.m_ref[L] = m;
                __syncwarp();
                if (lane == 0) mbar_arrive(xfer_out);
            }
            // this warp's partial row sum follows the reference
            if (m != st.m) {
                if (st.m != -INFINITY) {
                    const float a = ex2_approx(st.m - m);
                    st.l2 = pack_f2(__uint_as_float(static_cast<uint32_t>(st.l2)) * a,
                                    __uint_as_float(static_cast<uint32_t>(st.l2 >> 32)) * a);
                }
                st.m = m;
            }
            if (any) {
                softmax_exp_store(sAddr, s, full, m, scale_log2, st);
            } else {
                // nothing of this tile is attended by the warp's rows: P = 0
#pragma unroll
                for (int e = 0; e < 32; ++e) s[e] = 0u;
                tmem_st32p(sAddr, s);
                tmem_st32p(sAddr + 32, s);
                tmem_st_wait();
            }
            if (__any_sync(0xffffffffu, need)) {
                const int pj = jj - 1;
                rescale_o_row(oAddr, alpha, &sm.pv_done[pj % kTileBars], (pj / kTileBars) & 1);
            }
            if (prof) t_part += clock64() - t1;
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.p_full[jj % kTileBars]);
        }
        const long long t_epi = clock64();
        if (prof) {
            atomicAdd(&g_attn_prof[0], static_cast<unsigned long long>(t_epi - t_loop));
            atomicAdd(&g_attn_prof[1], static_cast<unsigned long long>(w_s));
            atomicAdd(&g_attn_prof[2], static_cast<unsigned long long>(t_part));
            atomicAdd(&g_attn_prof[3], static_cast<unsigned long long>(ntiles));
            atomicAdd(&g_attn_prof[11], static_cast<unsigned long long>(w_x));
        }
        // ---- epilogue: the row sums of the two parity warps at the larger (=
        //      final) reference, coverage likewise; O / l -> bf16, the parity-par
        //      warp writing columns [64 par, 64 par + 64) of its rows
        sm.fin_m[par][L] = st.m;
        sm.fin_l[par][L] = __uint_as_float(static_cast<uint32_t>(st.l2)) +
                           __uint_as_float(static_cast<uint32_t>(st.l2 >> 32));
        if (par == 1) sm.fin_c[L] = st.cov;
        named_bar_sync(2 + quad, 64); // the two parity warps of this quadrant
        const float m0 = sm.fin_m[0][L], m1 = sm.fin_m[1][L];
        const float mf = fmaxf(m0, m1);
        float lsum = 0.0f;
        if (m0 != -INFINITY) lsum += sm.fin_l[0][L] * ex2_approx(m0 - mf);
        if (m1 != -INFINITY) lsum += sm.fin_l[1][L] * ex2_approx(m1 - mf);
        const float inv = lsum > 0.0f ? 1.0f / lsum : 0.0f;
        const int ct = par == 0 ? st.cov + sm.fin_c[L] : 0;
        if (ntiles > 0) {
            const int last = ntiles - 1;
            mbar_wait(&sm.pv_done[last % kTileBars], (last / kTileBars) & 1);
            tc_fence_after();
        }
        {
            uint4 *dst = reinterpret_cast<uint4 *>(
                out + ((static_cast<int64_t>(b) * tokens + (ok ? row : 0)) * hq + h) * kHeadDim + 64 * par);
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                uint32_t o[32];
                if (ntiles > 0) { // warp-uniform: the tcgen05.ld is convergent
                    tmem_ld32p(oAddr + 64 * par + 32 * cc, o);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] = 0u;
                }
                if (ok) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        uint4 w;
                        w.x = pack_bf16x2(__uint_as_float(o[8 * e]) * inv, __uint_as_float(o[8 * e + 1]) * inv);
                        w.y = pack_bf16x2(__uint_as_float(o[8 * e + 2]) * inv, __uint_as_float(o[8 * e + 3]) * inv);
                        w.z = pack_bf16x2(__uint_as_float(o[8 * e + 4]) * inv, __uint_as_float(o[8 * e + 5]) * inv);
                        w.w = pack_bf16x2(__uint_as_float(o[8 * e + 6]) * inv, __uint_as_float(o[8 * e + 7]) * inv);
                        dst[4 * cc + e] = w;
                    }
                }
            }
        }
        if (par == 0 && ok && coverage) coverage[(static_cast<int64_t>(b) * hq + h) * tokens + row] = ct;
        // a row that attends no token: block_sparse_attention throws
        // std::domain_error for the first such row (sparse_attention.hpp:88-90);
        // the ABI reports the smallest (b, h, row) index
        if (par == 0 && ok && empty_rows && ct == 0)
            atomicMin(empty_rows, (static_cast<unsigned long long>(b) * hq + h) * tokens + row);
        if (prof) atomicAdd(&g_attn_prof[10], static_cast<unsigned long long>(clock64() - t_epi));
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
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
    auto kern = g_attn_prof_host ? sparse_attention_kernel<true> : sparse_attention_kernel<false>;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), smem);
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(grid), kAttnThreads, smem, stream>>>(
        static_cast<const __nv_bfloat16 *>(q), tm_k, tm_v, mask, static_cast<__nv_bfloat16 *>(out),
        coverage, empty_rows, tokens, hq, hkv, scale_log2, i_lo, i_hi - i_lo);
    return cudaGetLastError();
}

} // namespace sale_b200
