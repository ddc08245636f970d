// stats.cu — K2a: exact sink-local statistics and the per-row log-domain
// threshold, plus the base (always-computed) mask rows.
//
// Reproduces compute_sink_local_stats (selection.hpp:129-163) and
// threshold_bound (selection.hpp:168-173) bit-for-bit on bf16-valued inputs:
//   s_t   = fl32(dot_seq(q, k_t)) * inv_sqrt_d   — an FMA chain over c = 0..d-1
//           (bf16 x bf16 products are exact in fp32, so FMA == MUL+ADD); two
//           independent chains share one packed FFMA2 (fma.rn.f32x2)
//   m     = running max in double, in I_SL block order
//   sum_b = sequential double sum of exp(double(s_t) - m_b) over block b
//   l     = l * exp(m_old - m_new) + sum_b      — __dmul_rn/__dadd_rn, never fused
//   bound = m + log(max(tau * l, DBL_MIN))
// The only non-bit-exact element is CUDA's double exp/log (<= 1 ulp) vs glibc;
// see DESIGN.md "Parity" for why that cannot flip a mask bit in practice.
// K2b compares float estimates against fb = the smallest float >= bound, which
// is exactly equivalent to the reference's (double)est >= bound.
//
// CTA = one (batch, head, query block with a non-empty middle region): 64
// rows x the I_SL keys (<= 224 per chunk of 7 blocks) x d. Q and the keys are
// staged as bf16 with 16-byte cp.async into rows padded to 272 B (68 words: at
// most 2-way bank conflicts for the 16 key rows a warp reads), four channel
// quarters in flight at once; the FFMA2 chains convert with PRMT (ALU pipe).
// ~83 KB smem, two CTAs per SM. (Measured alternatives — fp32 operands staged
// once per quarter, and an 8-row x 14-key FFMA2 tile on 128 threads — moved
// the bound to shared-memory wavefronts / the non-dot phases and were slower:
// profiles/README.md.)
#include "common.cuh"
#include "exp_table.h"
#include "internal.h"

#include <cfloat>

namespace sale_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxSlBlocks = 7;                  // I_SL blocks per chunk: {0} U [2i-4, 2i+1] by default
constexpr int kMaxKeys = kMaxSlBlocks * kBlockK; // 224
constexpr int kRows = kBlockQ;                   // 64
constexpr int kPitch = 136;                      // bf16 per staged row (272 B, 16-B aligned)

struct StatsSmem {
    union {
        struct {
            __nv_bfloat16 q[kRows][kPitch];    // 16.5 KB
            __nv_bfloat16 k[kMaxKeys][kPitch]; // 57.75 KB
        } in;
        float logit[kRows][kMaxKeys + 1];      // 56 KB (after the dot phase), padded
    } u;
    double bmax[kRows][kMaxSlBlocks];          // block max, then running max
    double bsum[kRows][kMaxSlBlocks];          // per-block exp sums
    double escale[kRows][kMaxSlBlocks];        // exp(m_old - m_new) of each block's l update
    double carry[3][kRows];                    // per row across I_SL chunks: running max, m_old, l
    int blk_len[kMaxSlBlocks];
    double2 exp_tab[256];                      // {hi, lo} of 2^(j/256)
};

__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool valid) {
    const uint32_t d = smem_u32(dst);
    const int n = valid ? 16 : 0; // src-size 0 -> zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}

// exp(x) for x <= 0 (the sink-local sums: logit - running max), table driven:
// x = (256 e + j) ln2/256 + r, |r| <= ln2/512; exp(x) = 2^e 2^(j/256) e^r with
// 2^(j/256) as a double-double from the table and e^r - 1 by a degree-5
// polynomial; one final rounding (T_hi + fma(T_hi, q, T_lo)), i.e. within
// ~0.5 ulp like glibc's exp (selection.hpp:155-157 uses std::exp). 11 FP64
// operations against ~17 for the CUDA math library's exp. x < -700 returns 0
// instead of a value below 2^-1009: every block sum is added to l >= 1 (the
// running max element contributes exp(0) = 1), where such a term is lost in
// the rounding anyway, so l is unchanged.
__device__ __forceinline__ double exp_nonpos(double x, const double2 *tab) {
    const bool tiny = x < -700.0;
    x = tiny ? -700.0 : x;
    const double t = fma(x, 369.32993046757463, 6755399441055744.0); // 256/ln2, 1.5 * 2^52
    const int k = __double2loint(t);
    const double kd = t - 6755399441055744.0;
    double r = fma(kd, -2.7076061740622863e-03, x);  // ln2/256, hi
    r = fma(kd, -9.058776616587108e-20, r);          // ln2/256, lo
    double q = fma(r, 8.3333333333333332e-03, 4.1666666666666664e-02);
    q = fma(q, r, 1.6666666666666666e-01);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    q = q * r;                                       // e^r - 1
    const double2 tj = tab[k & 255];
    const double y = tj.x + fma(tj.x, q, tj.y);
    const double v = __hiloint2double(__double2hiint(y) + ((k >> 8) << 20), __double2loint(y));
    return tiny ? 0.0 : v;
}

__device__ __forceinline__ void ffma2(unsigned long long &acc, unsigned long long a,
                                      unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
// bf16 (low / high half of a 32-bit word) -> fp32 bits with a byte permute:
// ALU pipe, where a shift would compile to an FMA-pipe IMAD that competes with
// the dot products' FFMA2s.
__device__ __forceinline__ uint32_t bf16lo_f32(uint32_t w) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(r) : "r"(w));
    return r;
}
__device__ __forceinline__ uint32_t bf16hi_f32(uint32_t w) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0x3244;" : "=r"(r) : "r"(w));
    return r;
}
__device__ __forceinline__ unsigned long long pack2u(uint32_t lo, uint32_t hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
    return r;
}
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return (static_cast<unsigned long long>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}

} // namespace

// Optional phase timing (sale_b200_estimator_profile counters 8..15): cycles
// thread 0 spends in staging, dots, logit store, block max, running max, exp
// sums, final combine; summed over CTAs.
__device__ int g_stats_prof_on = 0;
__device__ unsigned long long g_stats_prof[8];

namespace {

// grid: (query blocks with a non-empty middle region, heads, batch). I_SL is
// processed in chunks of <= 7 blocks (one chunk for the default geometry):
// logits, block maxima, running max and exp sums per chunk, with the running
// max and the double exp-sum carried across chunks in I_SL order — the same
// sequence of operations as the reference's loop over the blocks.
__global__ void __launch_bounds__(kThreads, 2)
sink_local_stats_kernel(const __nv_bfloat16 *__restrict__ q, const __nv_bfloat16 *__restrict__ k,
                        int64_t tokens, int64_t hq, int64_t hkv, float inv_sqrt_d, Geom geo,
                        const double *__restrict__ taus, float *__restrict__ thresh,
                        double *__restrict__ dbg_m, double *__restrict__ dbg_l,
                        double *__restrict__ dbg_bound, int64_t i_first) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    StatsSmem &sm = *reinterpret_cast<StatsSmem *>(smem_raw);
    const int tid = threadIdx.x;
    const bool prof = tid == 0 && g_stats_prof_on != 0;
    long long tp[8];
    tp[0] = prof ? clock64() : 0;
#define SALE_PHASE(n) \
    if (prof) tp[n] = clock64();
    const int64_t i = blockIdx.x + i_first;
    const int64_t h = blockIdx.y;
    const int64_t b = blockIdx.z;
    const int64_t g = h / (hq / hkv);
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    const int64_t q0 = i * kBlockQ;
    const int qrows = static_cast<int>((q0 + kBlockQ <= tokens) ? kBlockQ : tokens - q0);
    const int64_t frontier = frontier_block(i, tokens, nk);
    // I_SL (selection.hpp:92-123) in ascending order: slots [0, sb) = the sink
    // blocks, slots sb.. = the local window lo .. frontier
    const int64_t lo = local_lo(i, geo);
    const int nsl = static_cast<int>(geo.sb + frontier - lo + 1);
    auto slot_token = [&](int slot) -> int64_t {
        return (slot < geo.sb ? slot : lo + slot - geo.sb) * kBlockK;
    };
    for (int e = tid; e < 256; e += kThreads)
        sm.exp_tab[e] = make_double2(c_exp2_256[2 * e], c_exp2_256[2 * e + 1]);
    // per-row state carried across I_SL chunks (row tid, owned by thread tid < 64;
    // in shared memory: registers are taken by the FFMA2 tile)
    if (tid < kRows) {
        sm.carry[0][tid] = -INFINITY;
        sm.carry[1][tid] = -INFINITY;
        sm.carry[2][tid] = 0.0;
    }

    for (int c0 = 0; c0 < nsl; c0 += kMaxSlBlocks) {
        const int cn = min(kMaxSlBlocks, nsl - c0); // blocks in this chunk
        if (tid < kMaxSlBlocks) {
            int len = 0;
            if (tid < cn) {
                const int64_t kb = slot_token(c0 + tid);
                len = static_cast<int>((kb + kBlockK <= tokens) ? kBlockK : tokens - kb);
            }
            sm.blk_len[tid] = len;
        }

        // ---- stage Q rows and I_SL keys (bf16) with cp.async, zero-filling rows
        //      past the sequence end, in four channel quarters (one commit group
        //      each): the dot chains run over c = 0..127 in order, so quarter qq's
        //      FMAs start as soon as it has landed while the later quarters stream.
        constexpr int kQCh = kHeadDim / 8 / 4; // 16-byte chunks per row and channel quarter
        static_assert(kRows * kQCh == kThreads, "one Q chunk per thread and quarter");
        // thread -> (Q row tid/4, chunk tid%4 of each quarter) and keys
        // t = tid/4 + 64 n (n < 4, t < 224), same chunk: row offsets computed once
        const int cq = tid & 3;
        const int rq = tid >> 2;
        const bool q_ok = rq < qrows;
        const __nv_bfloat16 *q_src = q + ((b * tokens + q0 + (q_ok ? rq : 0)) * hq + h) * kHeadDim + 8 * cq;
        const __nv_bfloat16 *k_src[4];
        bool k_ok[4];
#pragma unroll
        for (int n = 0; n < 4; ++n) {
            const int t = rq + 64 * n;
            const int slot = t / kBlockK;
            const int64_t tok = (t < kMaxKeys && slot < cn) ? slot_token(c0 + slot) + t % kBlockK : tokens;
            k_ok[n] = tok < tokens;
            k_src[n] = k + ((b * tokens + (k_ok[n] ? tok : 0)) * hkv + g) * kHeadDim + 8 * cq;
        }
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
            cp_async16(&sm.u.in.q[rq][8 * (qq * kQCh + cq)], q_src + 32 * qq, q_ok);
#pragma unroll
            for (int n = 0; n < 4; ++n) {
                const int t = rq + 64 * n;
                if (t < kMaxKeys) cp_async16(&sm.u.in.k[t][8 * (qq * kQCh + cq)], k_src[n] + 32 * qq, k_ok[n]);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        SALE_PHASE(1)

        // ---- fp32 logits: thread = 4 rows x 14 keys (kg + 16 j), sequential over c;
        //      key pairs (kg + 32p, kg + 32p + 16) share one FFMA2.
        {
            const int rg = tid / 16, kg = tid % 16;
            unsigned long long acc[4][7];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int p = 0; p < 7; ++p) acc[a][p] = 0ull;
            const uint32_t *qw[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) qw[a] = reinterpret_cast<const uint32_t *>(sm.u.in.q[rg * 4 + a]);
            const uint32_t *kw = reinterpret_cast<const uint32_t *>(sm.u.in.k[kg]);
            constexpr int kRowWords = kPitch / 2;
#pragma unroll 1
            for (int qq = 0; qq < 4; ++qq) {
                // quarter qq landed (this thread's copies), then everyone's
                if (qq == 0) asm volatile("cp.async.wait_group 3;" ::: "memory");
                else if (qq == 1) asm volatile("cp.async.wait_group 2;" ::: "memory");
                else if (qq == 2) asm volatile("cp.async.wait_group 1;" ::: "memory");
                else asm volatile("cp.async.wait_group 0;" ::: "memory");
                __syncthreads();
#pragma unroll 2
                for (int cw = 16 * qq; cw < 16 * qq + 16; ++cw) {
                    uint32_t qv[4], kv[14];
#pragma unroll
                    for (int a = 0; a < 4; ++a) qv[a] = qw[a][cw];
#pragma unroll
                    for (int j = 0; j < 14; ++j) kv[j] = kw[(16 * j) * kRowWords + cw];
                    // c = 2cw (low halves), then c = 2cw + 1 (high halves)
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        unsigned long long kp[7];
#pragma unroll
                        for (int p = 0; p < 7; ++p) {
                            const uint32_t x0 = half ? bf16hi_f32(kv[2 * p]) : bf16lo_f32(kv[2 * p]);
                            const uint32_t x1 = half ? bf16hi_f32(kv[2 * p + 1]) : bf16lo_f32(kv[2 * p + 1]);
                            kp[p] = pack2u(x0, x1);
                        }
#pragma unroll
                        for (int a = 0; a < 4; ++a) {
                            const uint32_t y = half ? bf16hi_f32(qv[a]) : bf16lo_f32(qv[a]);
                            const unsigned long long qq2 = pack2u(y, y);
#pragma unroll
                            for (int p = 0; p < 7; ++p) ffma2(acc[a][p], qq2, kp[p]);
                        }
                    }
                }
            }
            __syncthreads(); // staging area becomes the logit buffer
            SALE_PHASE(2)
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int p = 0; p < 7; ++p) {
                    const float lo = __uint_as_float(static_cast<uint32_t>(acc[a][p]));
                    const float hi = __uint_as_float(static_cast<uint32_t>(acc[a][p] >> 32));
                    sm.u.logit[rg * 4 + a][kg + 32 * p] = __fmul_rn(lo, inv_sqrt_d);
                    sm.u.logit[rg * 4 + a][kg + 32 * p + 16] = __fmul_rn(hi, inv_sqrt_d);
                }
        }
        __syncthreads();
        SALE_PHASE(3)

        // ---- (row, block) tasks: block max
        for (int task = tid; task < kRows * kMaxSlBlocks; task += kThreads) {
            const int r = task % kRows, sl = task / kRows; // lanes = rows: conflict-free
            // max of fp32 logits in fp32 (exact; the double of the max float equals
            // the reference's max over doubles), four chains, FP32 pipe not FP64
            float bm4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
            if (sl < cn) {
                const float *lg = &sm.u.logit[r][sl * kBlockK];
                if (sm.blk_len[sl] == kBlockK) {
#pragma unroll
                    for (int t = 0; t < kBlockK; ++t) bm4[t & 3] = fmaxf(bm4[t & 3], lg[t]);
                } else {
                    for (int t = 0; t < sm.blk_len[sl]; ++t) bm4[0] = fmaxf(bm4[0], lg[t]);
                }
            }
            sm.bmax[r][sl] = static_cast<double>(fmaxf(fmaxf(bm4[0], bm4[1]), fmaxf(bm4[2], bm4[3])));
        }
        __syncthreads();
        SALE_PHASE(4)
        if (tid < kRows) { // running max after each block, in I_SL order
            double m_run = sm.carry[0][tid];
            for (int sl = 0; sl < cn; ++sl) {
                m_run = fmax(m_run, sm.bmax[tid][sl]);
                sm.bmax[tid][sl] = m_run;
            }
            sm.carry[0][tid] = m_run;
        }
        __syncthreads();
        SALE_PHASE(5)
        // ---- (row, block) tasks: sequential double sum of exp(s_t - m_new)
        for (int task = tid; task < kRows * kMaxSlBlocks; task += kThreads) {
            const int r = task % kRows, sl = task / kRows;
            if (sl >= cn) continue;
            const double m_new = sm.bmax[r][sl];
            const float *lg = &sm.u.logit[r][sl * kBlockK];
            double sum = 0.0;
            if (sm.blk_len[sl] == kBlockK) {
                // independent exps first (ILP), then the reference's sequential sum
#pragma unroll
                for (int t0 = 0; t0 < kBlockK; t0 += 8) {
                    double e[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) e[t] = exp_nonpos(static_cast<double>(lg[t0 + t]) - m_new, sm.exp_tab);
#pragma unroll
                    for (int t = 0; t < 8; ++t) sum = __dadd_rn(sum, e[t]);
                }
            } else {
                for (int t = 0; t < sm.blk_len[sl]; ++t)
                    sum = __dadd_rn(sum, exp_nonpos(static_cast<double>(lg[t]) - m_new, sm.exp_tab));
            }
            sm.bsum[r][sl] = sum;
            // the rescale factor of this block's l update, exp(m_old - m_new)
            // (m_old = the running max before the block), computed here in
            // parallel instead of in the sequential per-row combine
            const double m_old = sl == 0 ? sm.carry[1][r] : sm.bmax[r][sl - 1];
            sm.escale[r][sl] = exp_nonpos(m_old - m_new, sm.exp_tab);
        }
        __syncthreads();
        SALE_PHASE(6)
        // ---- per row: l = l * exp(m_old - m_new) + sum_b, block by block
        if (tid < qrows) {
            double m_old = sm.carry[1][tid], l_run = sm.carry[2][tid];
            for (int sl = 0; sl < cn; ++sl) {
                l_run = __dadd_rn(__dmul_rn(l_run, sm.escale[tid][sl]), sm.bsum[tid][sl]);
                m_old = sm.bmax[tid][sl];
            }
            sm.carry[1][tid] = m_old;
            sm.carry[2][tid] = l_run;
        }
        if (c0 + kMaxSlBlocks < nsl) __syncthreads(); // the next chunk reuses the buffers
    }

    // ---- the bound (selection.hpp:168-173)
    if (tid < qrows) {
        const int r = tid;
        const double m_old = sm.carry[1][tid], l_run = sm.carry[2][tid];
        double scaled = __dmul_rn(taus[h], l_run);
        if (scaled < DBL_MIN) scaled = DBL_MIN;
        const double bound = __dadd_rn(m_old, log(scaled));
        const int64_t o = (b * hq + h) * tokens + q0 + r;
        thresh[o] = __double2float_ru(bound);
        if (dbg_m) {
            dbg_m[o] = m_old;
            dbg_l[o] = l_run;
            dbg_bound[o] = bound;
        }
    }
    if (prof) {
        tp[7] = clock64();
        for (int p = 0; p < 7; ++p)
            atomicAdd(&g_stats_prof[p], static_cast<unsigned long long>(tp[p + 1] - tp[p]));
        atomicAdd(&g_stats_prof[7], 1ull);
    }
#undef SALE_PHASE
}

// Base mask rows: I_SL U the trailing partial run, i.e. [0, sb) U
// [sb + E_i, frontier] with a non-empty middle and every causal block
// [0, frontier] otherwise (selection.hpp:228-245, :188). One thread per 32-bit
// word. Estimated middle segments are OR-ed in by K2b.
__global__ void base_mask_kernel(uint32_t *__restrict__ mask, int64_t rows, int64_t nq,
                                 int64_t nk, int64_t words, int64_t tokens, Geom geo, int64_t i_lo,
                                 int64_t ni) {
    // one thread per word; 32-bit index math (rows * ni * words < 2^31 is
    // checked at launch), the word's bits from the row's ranges by two shifts
    const uint32_t loc = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t w32 = static_cast<uint32_t>(words), ni32 = static_cast<uint32_t>(ni);
    if (loc >= static_cast<uint32_t>(rows) * ni32 * w32) return;
    const uint32_t rw = loc / w32;
    const int64_t w = loc - rw * w32;
    const uint32_t bh = rw / ni32;
    const int64_t i = i_lo + (rw - bh * ni32);
    const int64_t idx = (static_cast<int64_t>(bh) * nq + i) * words + w;
    const int64_t fr = frontier_block(i, tokens, nk);
    auto range_bits = [&](int64_t a, int64_t e) -> uint32_t { // blocks [a, e] in word w
        a = a > 32 * w ? a : 32 * w;
        e = e < 32 * w + 31 ? e : 32 * w + 31;
        if (a > e) return 0u;
        return (0xFFFFFFFFu >> (31 - static_cast<int>(e - 32 * w))) &
               (0xFFFFFFFFu << static_cast<int>(a - 32 * w));
    };
    uint32_t bits;
    if (has_middle(i, geo))
        bits = range_bits(0, geo.sb - 1) | range_bits(geo.sb + estimated_blocks(i, geo), fr);
    else
        bits = range_bits(0, fr);
    mask[idx] = bits;
}

} // namespace

cudaError_t launch_sink_local_stats(const void *q, const void *k, int64_t batch, int64_t tokens,
                                    int64_t hq, int64_t hkv, float inv_sqrt_d, const Geom &geo,
                                    const double *taus, float *thresh, double *dbg_m, double *dbg_l,
                                    double *dbg_bound, cudaStream_t stream, int64_t i_lo,
                                    int64_t i_hi) {
    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    if (i_hi < 0 || i_hi > nq) i_hi = nq;
    const int64_t fm = first_middle_block(geo);
    const int64_t i_first = i_lo > fm ? i_lo : fm; // blocks with a non-empty middle
    if (i_hi <= i_first) return cudaSuccess;
    const size_t smem = sizeof(StatsSmem);
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(sink_local_stats_kernel), smem);
    if (e != cudaSuccess) return e;
    dim3 grid(static_cast<unsigned>(i_hi - i_first), static_cast<unsigned>(hq),
              static_cast<unsigned>(batch));
    sink_local_stats_kernel<<<grid, kThreads, smem, stream>>>(
        static_cast<const __nv_bfloat16 *>(q), static_cast<const __nv_bfloat16 *>(k), tokens, hq,
        hkv, inv_sqrt_d, geo, taus, thresh, dbg_m, dbg_l, dbg_bound, i_first);
    return cudaGetLastError();
}

cudaError_t launch_base_mask(uint32_t *mask, int64_t batch, int64_t hq, int64_t tokens,
                             const Geom &geo, cudaStream_t stream, int64_t i_lo, int64_t i_hi) {
    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    const int64_t words = (nk + 31) / 32;
    if (i_hi < 0 || i_hi > nq) i_hi = nq;
    if (i_hi <= i_lo) return cudaSuccess;
    const int64_t total = batch * hq * (i_hi - i_lo) * words;
    if (total > 0x7FFFFFFF) return cudaErrorInvalidValue;
    const int threads = 256;
    const int64_t blocks = (total + threads - 1) / threads;
    base_mask_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
        mask, batch * hq, nq, nk, words, tokens, geo, i_lo, i_hi - i_lo);
    return cudaGetLastError();
}

} // namespace sale_b200

namespace sale_b200 {
cudaError_t stats_profile(int enable, unsigned long long *out8) {
    if (out8) {
        cudaError_t e = cudaMemcpyFromSymbol(out8, g_stats_prof, sizeof(g_stats_prof));
        if (e != cudaSuccess) return e;
    }
    unsigned long long zero[8] = {};
    cudaError_t e = cudaMemcpyToSymbol(g_stats_prof, zero, sizeof(zero));
    if (e != cudaSuccess) return e;
    return cudaMemcpyToSymbol(g_stats_prof_on, &enable, sizeof(int));
}
} // namespace sale_b200
