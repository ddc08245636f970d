// estimate.cu — K2b: the low-bit Q.K^T estimator of the Selection-Pass on the
// 5th-gen tensor cores (tcgen05.mma kind::i8, int32 accumulators in TMEM).
//
// Replaces the CPU hot loop approx_weight_block (quant.hpp:136-166) +
// max_then_dequantize (quant.hpp:170-179) + the relative-score decision and
// segment OR of selection_pass (selection.hpp:253-271).
//
// Work unit (one CTA, two CTAs resident per SM): one (batch, KV head, <=2
// query heads of that GQA group = kEstHeads) x one 128-row query tile x a
// chunk of up to kSegPerUnit (64) middle segments.
//   * The 128-row tile pairs query blocks (2m+1, 2m+2): both have the same
//     full-segment count F = m-1, so one key range
//     serves both. A = 2 heads x [128 rows x 128 int8 codes] (32 KB) is loaded
//     once by TMA.
//   * One stage = one segment = 128 keys of K codes (16 KB) through a
//     kEstStages (4) deep TMA ring. Every tcgen05.mma has M = N = 128, K = 32
//     (profiles/r1_mma_microbench.txt: an MMA instruction costs >= 46 cycles
//     whatever its N, so N = 32/64 tiles waste the tensor core; at N >= 128 i8
//     runs at 8192 MAC/clk/SM).
//   * TMEM: one 128-column int32 accumulator per head (256 columns per CTA,
//     512 per SM with both CTAs); a stage is 2 heads x 4 K-steps, head h into
//     buffer h. The two resident CTAs' MMAs interleave on the tensor pipe and
//     hide each other's issue -> commit -> drain -> release round trip.
//   * Epilogue (kEpiWarps = 8 warps = 4 lane quadrants x 2 pairs of key
//     blocks, thread = row): tcgen05.ld .pack::16b (|products| <= 128*49 fits
//     int16), buffer released right after the load, 16-bit SIMD max per
//     32-key block, est = ((q_scale * k_scale) * inv_sqrt_d) * (float)max,
//     est >= fb_row — the reference's float arithmetic. A warp vote ORs rows,
//     shared-memory atomicOr ORs the rows of the two query blocks, and one
//     atomicOr per selected segment writes the packed mask.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace sale_b200 {

constexpr int kSegPerUnit = 64;            // segments per work unit (8192 keys)
constexpr int kSegWords = kSegPerUnit / 32;
constexpr int kEstHeads = 2;               // query heads per CTA (two CTAs per SM)
constexpr int kEstStages = 4;              // TMA ring depth
constexpr int kStageKeys = kSegment * kBlockK;       // 128 keys = one segment
constexpr int kATileBytes = 128 * kHeadDim;          // 16 KB per head
constexpr int kBStageBytes = kStageKeys * kHeadDim;  // 16 KB
constexpr int kEpiWarps = 8;               // (lane quadrant, pair of key blocks) per warp
constexpr int kEstThreads = 128 + 32 * kEpiWarps; // warps 0-3 control, 4-19 epilogue

static_assert(kSegPerUnit == kSegPerUnitHost, "unit size mismatch");

struct EstSmem {
    alignas(1024) uint8_t a[kEstHeads][kATileBytes];
    alignas(1024) uint8_t bst[kEstStages][kBStageBytes];
    uint64_t full[kEstStages];
    uint64_t empty[kEstStages];
    uint64_t a_full;
    uint64_t tmem_full[kEstHeads];
    uint64_t tmem_empty[kEstHeads];
    uint32_t tmem_base;
    uint32_t seg_bits[kEstHeads][2][kSegWords];
    uint32_t blk_bits[kEstHeads][2][kSegment * kSegWords]; // general geometry: per middle block
    float ks[kSegment * kSegPerUnit];
};

// Optional wait-time instrumentation (sale_b200_est_profile): cycles the MMA
// issuer spends blocked on K stages / accumulator buffers, and the epilogue on
// accumulators. Off unless enabled; one global flag read per CTA.
__device__ int g_est_prof_on = 0;
static int g_est_mode_host = 0; // host copy: which kernel instance launches
__device__ unsigned long long g_est_prof[8];

namespace {

// kMode: 0 production, 1 parity debug (block maxima out), 2 cycle profiling,
// 3 profiling with the epilogue work skipped. The epilogue's per-head path is
// latency-critical (every extra instruction there costs issue slack; see
// profiles/README.md), so the diagnostics are separate instances.
// kGen: any selection geometry (Geom): the unit's stages start at key block
// sb, a query block estimates its own E_i blocks, and the epilogue ORs raw
// per-block decisions into the mask; segment_or_kernel then widens them to
// segments (segment_aggregate). !kGen: the default geometry, where one stage
// is exactly one segment and the epilogue writes aggregated segments.
template <int kMode, bool kGen>
__global__ void __launch_bounds__(kEstThreads, 2)
estimate_kernel(const __grid_constant__ CUtensorMap tm_qc, const __grid_constant__ CUtensorMap tm_kc,
                const EstUnit *__restrict__ units, const float *__restrict__ q_scales,
                const float *__restrict__ k_scales, const float *__restrict__ thresh,
                uint32_t *__restrict__ mask, int64_t tokens, int hq, int hkv, int nsub,
                float inv_sqrt_d, Geom geo, int32_t *__restrict__ dbg_max) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // dynamic smem base is only 16-B aligned by contract: round up to 1 KB
    EstSmem &sm = *reinterpret_cast<EstSmem *>(smem_raw + smem_pad_1k(smem_raw));
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    const EstUnit u = units[blockIdx.x];
    const int y = blockIdx.y;
    const int sub = y % nsub;
    const int g = (y / nsub) % hkv;
    const int b = y / (nsub * hkv);
    const int group = hq / hkv;
    const int h0 = g * group + sub * kEstHeads;
    const int nh = min(kEstHeads, group - sub * kEstHeads);
    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    const int64_t words = (nk + 31) / 32;
    const int nstages = u.nseg;
    const int row0 = 128 * u.m + 64;
    const int key_base = kBlockK * geo.sb + kStageKeys * kSegPerUnit * u.c; // first key of the unit

    if (threadIdx.x == 0) {
        for (int s = 0; s < kEstStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        mbar_init(&sm.a_full, 1);
        for (int s = 0; s < kEstHeads; ++s) {
            mbar_init(&sm.tmem_full[s], 1);
            mbar_init(&sm.tmem_empty[s], kEpiWarps); // all epilogue warps drain every group
        }
        for (int hh = 0; hh < kEstHeads; ++hh)
            for (int x = 0; x < 2; ++x) {
                for (int w = 0; w < kSegWords; ++w) sm.seg_bits[hh][x][w] = 0;
                for (int w = 0; w < kSegment * kSegWords; ++w) sm.blk_bits[hh][x][w] = 0;
            }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<kEstHeads * 128>(&sm.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        // ---------------------------------------------------------- TMA producer
        if (elect_one()) {
            tma_prefetch(&tm_qc);
            tma_prefetch(&tm_kc);
            mbar_expect_tx(&sm.a_full, static_cast<uint32_t>(nh * kATileBytes));
            for (int hh = 0; hh < nh; ++hh)
                tma_load_4d(sm.a[hh], &tm_qc, &sm.a_full, 0, h0 + hh, row0, b);
            for (int k = 0; k < nstages; ++k) {
                const int st = k % kEstStages;
                mbar_wait(&sm.empty[st], ((k / kEstStages) & 1) ^ 1);
                mbar_expect_tx(&sm.full[st], kBStageBytes);
                tma_load_4d(sm.bst[st], &tm_kc, &sm.full[st], 0, g, key_base + kStageKeys * k, b);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (elect_one()) {
            constexpr uint32_t idesc = idesc_i8(128, kStageKeys);
            uint64_t adesc[kEstHeads];
            for (int hh = 0; hh < kEstHeads; ++hh)
                adesc[hh] = umma_desc_sw128(smem_u32(sm.a[hh]), 16, 1024);
            constexpr bool prof = kMode >= 2;
            long long t_start = clock64(), w_full = 0, w_empty = 0;
            mbar_wait(&sm.a_full, 0);
            const long long w_a = clock64() - t_start;
            tc_fence_after();
            for (int k = 0; k < nstages; ++k) {
                const int st = k % kEstStages;
                long long t0 = prof ? clock64() : 0;
                mbar_wait(&sm.full[st], (k / kEstStages) & 1);
                if (prof) w_full += clock64() - t0;
                const uint64_t bdesc = umma_desc_sw128(smem_u32(sm.bst[st]), 16, 1024);
#pragma unroll
                for (int hh = 0; hh < kEstHeads; ++hh) {
                    if (hh >= nh) break;
                    // head hh owns TMEM columns [128 hh, 128 hh + 128): its
                    // epilogue of stage k-1 had three other heads' MMAs to finish.
                    // (The issue latency of this thread is on the critical path:
                    // the tensor pipe queues only a few MMAs, so nothing else here.)
                    if constexpr (prof) {
                        const long long te = clock64();
                        mbar_wait(&sm.tmem_empty[hh], (k & 1) ^ 1);
                        w_empty += clock64() - te;
                    } else {
                        mbar_wait(&sm.tmem_empty[hh], (k & 1) ^ 1);
                    }
                    tc_fence_after();
                    const uint32_t d = tmem + 128 * hh;
#pragma unroll
                    for (int kk = 0; kk < kHeadDim / 32; ++kk)
                        mma_i8_ss(d, adesc[hh] + 2 * kk, bdesc + 2 * kk, idesc, kk > 0);
                    tc_commit(&sm.tmem_full[hh]);
                }
                tc_commit(&sm.empty[st]);
            }
            if (prof) {
                atomicAdd(&g_est_prof[0], static_cast<unsigned long long>(clock64() - t_start));
                atomicAdd(&g_est_prof[1], static_cast<unsigned long long>(w_a));
                atomicAdd(&g_est_prof[2], static_cast<unsigned long long>(w_full));
                atomicAdd(&g_est_prof[3], static_cast<unsigned long long>(w_empty));
                atomicAdd(&g_est_prof[4], static_cast<unsigned long long>(nstages));
            }
        }
    } else if (warp >= 4) {
        // -------------------------------------------------------------- epilogue
        const int ew = warp - 4;
        const int quad = warp & 3;            // TMEM lane quadrant this warp may access
        const int r = quad * 32 + lane;       // row within the 128-row tile
        const int64_t tok = row0 + r;
        const bool row_ok = tok < tokens;
        // Every head's buffer is drained by all 8 warps: warp = (quadrant, key
        // blocks chunk, chunk + 1 of the segment = 64 accumulator columns).
        const int chunk = 2 * (ew >> 2);
        float qs[kEstHeads], fb[kEstHeads];
#pragma unroll
        for (int hh = 0; hh < kEstHeads; ++hh) {
            qs[hh] = 0.0f;
            fb[hh] = INFINITY;
            if (hh < nh && row_ok) {
                const int64_t o = (static_cast<int64_t>(b) * hq + h0 + hh) * tokens + tok;
                qs[hh] = q_scales[o];
                fb[hh] = thresh[o];
            }
        }
        const float *ks_row = k_scales + (static_cast<int64_t>(b) * hkv + g) * nk;
        const int64_t jb_base = key_base / kBlockK;
        // the unit's key-block scales, staged once (no global load per stage)
        for (int x = threadIdx.x - 128; x < kSegment * nstages; x += 32 * kEpiWarps)
            sm.ks[x] = jb_base + x < nk ? ks_row[jb_base + x] : 1.0f;
        // general geometry: this row's estimated blocks, counted from the
        // unit's first block (blocks past it are not decided here)
        const int64_t qi_row = 2 * static_cast<int64_t>(u.m) + 1 + (quad >> 1);
        const int e_row = kGen ? static_cast<int>(estimated_blocks(qi_row, geo) -
                                                  static_cast<int64_t>(kSegment) * kSegPerUnit * u.c)
                               : 0;
        named_bar_sync(1, 32 * kEpiWarps);
        const bool dbg = kMode == 1 && row_ok;
        constexpr bool epi_skip = kMode == 3;
        const uint32_t acc = tmem + (static_cast<uint32_t>(quad * 32) << 16) + 32 * chunk;
        const bool prof = kMode >= 2 && ew == 0;
        long long w_epi = 0;
        const long long t_epi = clock64();
        // per-row selection flags: bit k of flags[hh][k >> 5] = some column of
        // this row's key block in segment k passed; OR-reduced over rows once
        // (general geometry: bits 2k, 2k + 1 of gflags[hh][k >> 4] = blocks
        // 4k + chunk, 4k + chunk + 1 of the unit)
        uint32_t flags[kEstHeads][kSegWords];
        uint32_t gflags[kEstHeads][kGen ? 2 * kSegWords : 1];
#pragma unroll
        for (int hh = 0; hh < kEstHeads; ++hh) {
#pragma unroll
            for (int w = 0; w < kSegWords; ++w) flags[hh][w] = 0u;
#pragma unroll
            for (int w = 0; w < (kGen ? 2 * kSegWords : 1); ++w) gflags[hh][w] = 0u;
        }
        for (int k = 0; k < nstages; ++k) {
            const float ks = sm.ks[4 * k + chunk], ks1 = sm.ks[4 * k + chunk + 1];
            const uint32_t kbit = 1u << (k & 31);
            const uint32_t kb0 = (k >> 5) == 0 ? kbit : 0u, kb1 = kbit ^ kb0;
            static_assert(kSegWords == 2, "flag words");
            // one head at a time: its buffer is released as soon as the values
            // are in registers (the issuer then has the other three heads' MMAs
            // of slack), the reduction runs while the next head's MMAs execute
#pragma unroll
            for (int hh = 0; hh < kEstHeads; ++hh) {
                if (hh >= nh) break; // warp-uniform
                long long t0 = 0;
                if constexpr (kMode >= 2) t0 = prof ? clock64() : 0;
                mbar_wait(&sm.tmem_full[hh], k & 1);
                if constexpr (kMode >= 2)
                    if (prof) w_epi += clock64() - t0;
                tc_fence_after();
                if constexpr (epi_skip) { // diagnostic (profile mode 2): MMA side alone
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.tmem_empty[hh]);
                    continue;
                }
                uint32_t v[32];
                tmem_ld64_pack16(acc + 128 * hh, v);
                tmem_ld_wait(); // warp-collective: every lane's values are in registers
                tc_fence_before();
                if (lane == 0) mbar_arrive(&sm.tmem_empty[hh]);
                // int16 pairs: v[0..15] key block chunk, v[16..31] chunk + 1
#pragma unroll
                for (int s = 8; s > 0; s >>= 1)
#pragma unroll
                    for (int e = 0; e < s; ++e) {
                        v[e] = __vmaxs2(v[e], v[e + s]);
                        v[16 + e] = __vmaxs2(v[16 + e], v[16 + e + s]);
                    }
                const int mx0 = max(static_cast<int>(static_cast<int16_t>(v[0] & 0xFFFFu)),
                                    static_cast<int>(static_cast<int16_t>(v[0] >> 16)));
                const int mx1 = max(static_cast<int>(static_cast<int16_t>(v[16] & 0xFFFFu)),
                                    static_cast<int>(static_cast<int16_t>(v[16] >> 16)));
                const float est0 = __fmul_rn(__fmul_rn(__fmul_rn(qs[hh], ks), inv_sqrt_d), static_cast<float>(mx0));
                const float est1 = __fmul_rn(__fmul_rn(__fmul_rn(qs[hh], ks1), inv_sqrt_d), static_cast<float>(mx1));
                if constexpr (kGen) {
                    const int jb = 4 * k + chunk; // the unit's block of est0
                    const uint32_t bits = ((est0 >= fb[hh] && jb < e_row) ? 1u : 0u) |
                                          ((est1 >= fb[hh] && jb + 1 < e_row) ? 2u : 0u);
                    const uint32_t sh = static_cast<uint32_t>(2 * (k & 15));
#pragma unroll
                    for (int w = 0; w < 2 * kSegWords; ++w) gflags[hh][w] |= (k >> 4) == w ? bits << sh : 0u;
                } else {
                    const bool pass = est0 >= fb[hh] || est1 >= fb[hh];
                    flags[hh][0] |= pass ? kb0 : 0u;
                    flags[hh][1] |= pass ? kb1 : 0u;
                }
                if constexpr (kMode == 1)
                    if (dbg) {
                        const int64_t jb = jb_base + 4 * k + chunk;
                        int32_t *dm = dbg_max + ((static_cast<int64_t>(b) * hq + h0 + hh) * tokens + tok) * nk + jb;
                        if (jb < nk) dm[0] = mx0;
                        if (jb + 1 < nk) dm[1] = mx1;
                    }
            }
        }
        // OR over the warp's 32 rows; the two query blocks of the tile are the
        // lane quadrants {0,1} and {2,3}
        if constexpr (kGen) {
            // spread the 2-bit stage groups to nibbles (bits chunk, chunk + 1)
#pragma unroll
            for (int hh = 0; hh < kEstHeads; ++hh)
#pragma unroll
                for (int w = 0; w < 2 * kSegWords; ++w) {
                    const uint32_t any = __reduce_or_sync(0xffffffffu, gflags[hh][w]);
                    if (lane == 0 && any && hh < nh)
#pragma unroll
                        for (int half16 = 0; half16 < 2; ++half16) {
                            uint32_t y = (any >> (16 * half16)) & 0xFFFFu;
                            y = (y | (y << 8)) & 0x00FF00FFu;
                            y = (y | (y << 4)) & 0x0F0F0F0Fu;
                            y = (y | (y << 2)) & 0x33333333u;
                            if (y) atomicOr(&sm.blk_bits[hh][quad >> 1][2 * w + half16], y << chunk);
                        }
                }
        } else {
#pragma unroll
            for (int hh = 0; hh < kEstHeads; ++hh)
#pragma unroll
                for (int w = 0; w < kSegWords; ++w) {
                    const uint32_t any = __reduce_or_sync(0xffffffffu, flags[hh][w]);
                    if (lane == 0 && any && hh < nh) atomicOr(&sm.seg_bits[hh][quad >> 1][w], any);
                }
        }
        if (prof && lane == 0) {
            atomicAdd(&g_est_prof[5], static_cast<unsigned long long>(clock64() - t_epi));
            atomicAdd(&g_est_prof[6], static_cast<unsigned long long>(w_epi));
        }
        named_bar_sync(1, 32 * kEpiWarps);
        if (ew == 0 && lane < 2 * kEstHeads) {
            const int h = lane >> 1, half = lane & 1;
            const int64_t qi = 2 * static_cast<int64_t>(u.m) + 1 + half;
            if (kGen && h < nh && qi < nq) {
                // raw block decisions at blocks sb + 256 c + x (segment_or_kernel widens them)
                uint32_t *row = mask + ((static_cast<int64_t>(b) * hq + h0 + h) * nq + qi) * words;
                const int64_t j0 = geo.sb + static_cast<int64_t>(kSegment) * kSegPerUnit * u.c;
                for (int bw = 0; bw < kSegment * kSegWords; ++bw) {
                    const uint32_t bits = sm.blk_bits[h][half][bw];
                    if (!bits) continue;
                    const int64_t j = j0 + 32 * bw;
                    const uint32_t w0 = static_cast<uint32_t>(j >> 5), sh = j & 31;
                    atomicOr(row + w0, bits << sh);
                    if (sh) atomicOr(row + w0 + 1, bits >> (32 - sh));
                }
            } else if (h < nh && qi < nq) {
                uint32_t *row = mask + ((static_cast<int64_t>(b) * hq + h0 + h) * nq + qi) * words;
                for (int sw = 0; sw < kSegWords; ++sw) {
                    uint32_t bits = sm.seg_bits[h][half][sw];
                    while (bits) {
                        const int s = 32 * sw + __ffs(bits) - 1;
                        bits &= bits - 1;
                        const int64_t sg = static_cast<int64_t>(kSegPerUnit) * u.c + s;
                        const int64_t j0 = 1 + kSegment * sg; // blocks j0 .. j0+3
                        const uint32_t w0 = static_cast<uint32_t>(j0 >> 5), sh = j0 & 31;
                        atomicOr(row + w0, 0xFu << sh);
                        if (sh > 28) atomicOr(row + w0 + 1, 0xFu >> (32 - sh));
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kEstHeads * 128>(tmem);
    }
}

// ---------------------------------------------------------------------------
// Production instance for the default geometry: stages of TWO segments (256
// keys), tcgen05.mma M = 128, N = 256, K = 32 — half the MMA instructions of
// the one-segment kernel above for the same work, and 96 instead of 128 B/clk
// of shared-memory operand reads per MMA (A 4 KB + B 8 KB per 128 cycles).
// One CTA per SM: TMEM = 2 heads x 256 int32 columns; the accumulator of head
// 0 is drained while head 1's MMAs run (512 cycles) and vice versa. A stage is
// 2 x 16 KB of K codes (two 128-key TMA boxes back to back: the SW128 layout
// of 256 rows); an odd last segment runs as an N = 128 stage. Epilogue warp
// (lane quadrant q, c2) drains the 128 columns of segment 2k + c2: two
// .pack::16b loads, release, then the same int16 max / float estimate /
// threshold test as above.
constexpr int kWideStages = 3;
constexpr int kWideStageBytes = 2 * kBStageBytes; // 32 KB

struct EstWideSmem {
    alignas(1024) uint8_t a[kEstHeads][kATileBytes];
    alignas(1024) uint8_t bst[kWideStages][kWideStageBytes];
    uint64_t full[kWideStages];
    uint64_t empty[kWideStages];
    uint64_t a_full;
    uint64_t tmem_full[kEstHeads];
    uint64_t tmem_empty[kEstHeads];
    uint32_t tmem_base;
    uint32_t seg_bits[kEstHeads][2][kSegWords];
    float ks[kSegment * kSegPerUnit];
};

__global__ void __launch_bounds__(kEstThreads, 1)
estimate_wide_kernel(const __grid_constant__ CUtensorMap tm_qc, const __grid_constant__ CUtensorMap tm_kc,
                     const EstUnit *__restrict__ units, const float *__restrict__ q_scales,
                     const float *__restrict__ k_scales, const float *__restrict__ thresh,
                     uint32_t *__restrict__ mask, int64_t tokens, int hq, int hkv, int nsub,
                     float inv_sqrt_d) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    EstWideSmem &sm = *reinterpret_cast<EstWideSmem *>(smem_raw + smem_pad_1k(smem_raw));
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    const EstUnit u = units[blockIdx.x];
    const int y = blockIdx.y;
    const int sub = y % nsub;
    const int g = (y / nsub) % hkv;
    const int b = y / (nsub * hkv);
    const int group = hq / hkv;
    const int h0 = g * group + sub * kEstHeads;
    const int nh = min(kEstHeads, group - sub * kEstHeads);
    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    const int64_t words = (nk + 31) / 32;
    const int nseg = u.nseg;
    const int nstages = (nseg + 1) / 2;
    const int row0 = 128 * u.m + 64;
    const int key_base = kBlockK + kStageKeys * kSegPerUnit * u.c; // default geometry: sb = 1

    if (threadIdx.x == 0) {
        for (int s = 0; s < kWideStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        mbar_init(&sm.a_full, 1);
        for (int s = 0; s < kEstHeads; ++s) {
            mbar_init(&sm.tmem_full[s], 1);
            mbar_init(&sm.tmem_empty[s], kEpiWarps);
        }
        for (int hh = 0; hh < kEstHeads; ++hh)
            for (int x = 0; x < 2; ++x)
                for (int w = 0; w < kSegWords; ++w) sm.seg_bits[hh][x][w] = 0;
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<kEstHeads * 256>(&sm.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        // ---------------------------------------------------------- TMA producer
        if (elect_one()) {
            tma_prefetch(&tm_qc);
            tma_prefetch(&tm_kc);
            mbar_expect_tx(&sm.a_full, static_cast<uint32_t>(nh * kATileBytes));
            for (int hh = 0; hh < nh; ++hh)
                tma_load_4d(sm.a[hh], &tm_qc, &sm.a_full, 0, h0 + hh, row0, b);
            for (int k = 0; k < nstages; ++k) {
                const int st = k % kWideStages;
                const int segs = min(2, nseg - 2 * k);
                mbar_wait(&sm.empty[st], ((k / kWideStages) & 1) ^ 1);
                mbar_expect_tx(&sm.full[st], static_cast<uint32_t>(segs * kBStageBytes));
                for (int x = 0; x < segs; ++x)
                    tma_load_4d(sm.bst[st] + x * kBStageBytes, &tm_kc, &sm.full[st], 0, g,
                                key_base + kStageKeys * (2 * k + x), b);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (elect_one()) {
            uint64_t adesc[kEstHeads];
            for (int hh = 0; hh < kEstHeads; ++hh)
                adesc[hh] = umma_desc_sw128(smem_u32(sm.a[hh]), 16, 1024);
            mbar_wait(&sm.a_full, 0);
            tc_fence_after();
            for (int k = 0; k < nstages; ++k) {
                const int st = k % kWideStages;
                const uint32_t idesc = 2 * k + 1 < nseg ? idesc_i8(128, 256) : idesc_i8(128, 128);
                mbar_wait(&sm.full[st], (k / kWideStages) & 1);
                const uint64_t bdesc = umma_desc_sw128(smem_u32(sm.bst[st]), 16, 1024);
#pragma unroll
                for (int hh = 0; hh < kEstHeads; ++hh) {
                    if (hh >= nh) break;
                    mbar_wait(&sm.tmem_empty[hh], (k & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem + 256 * hh;
#pragma unroll
                    for (int kk = 0; kk < kHeadDim / 32; ++kk)
                        mma_i8_ss(d, adesc[hh] + 2 * kk, bdesc + 2 * kk, idesc, kk > 0);
                    tc_commit(&sm.tmem_full[hh]);
                }
                tc_commit(&sm.empty[st]);
            }
        }
    } else if (warp >= 4) {
        // -------------------------------------------------------------- epilogue
        const int ew = warp - 4;
        const int quad = warp & 3;            // TMEM lane quadrant this warp may access
        const int c2 = ew >> 2;               // which segment of a two-segment stage
        const int r = quad * 32 + lane;       // row within the 128-row tile
        const int64_t tok = row0 + r;
        const bool row_ok = tok < tokens;
        float qs[kEstHeads], fb[kEstHeads];
#pragma unroll
        for (int hh = 0; hh < kEstHeads; ++hh) {
            qs[hh] = 0.0f;
            fb[hh] = INFINITY;
            if (hh < nh && row_ok) {
                const int64_t o = (static_cast<int64_t>(b) * hq + h0 + hh) * tokens + tok;
                qs[hh] = q_scales[o];
                fb[hh] = thresh[o];
            }
        }
        const float *ks_row = k_scales + (static_cast<int64_t>(b) * hkv + g) * nk;
        const int64_t jb_base = key_base / kBlockK;
        for (int x = threadIdx.x - 128; x < kSegment * nseg; x += 32 * kEpiWarps)
            sm.ks[x] = jb_base + x < nk ? ks_row[jb_base + x] : 1.0f;
        named_bar_sync(1, 32 * kEpiWarps);
        const uint32_t acc = tmem + (static_cast<uint32_t>(quad * 32) << 16) + 128 * c2;
        uint32_t flags[kEstHeads][kSegWords];
#pragma unroll
        for (int hh = 0; hh < kEstHeads; ++hh)
#pragma unroll
            for (int w = 0; w < kSegWords; ++w) flags[hh][w] = 0u;
        for (int k = 0; k < nstages; ++k) {
            const int sg = 2 * k + c2;              // this warp's segment of the unit
            const bool live = sg < nseg;            // warp-uniform (odd last stage)
            const int sgc = live ? sg : 2 * k;
            const float ksa = sm.ks[4 * sgc], ksb = sm.ks[4 * sgc + 1];
            const float ksc = sm.ks[4 * sgc + 2], ksd = sm.ks[4 * sgc + 3];
            const uint32_t sbit = 1u << (sg & 31);
            const uint32_t sb0 = (sg >> 5) == 0 ? sbit : 0u, sb1 = sbit ^ sb0;
#pragma unroll
            for (int hh = 0; hh < kEstHeads; ++hh) {
                if (hh >= nh) break; // warp-uniform
                mbar_wait(&sm.tmem_full[hh], k & 1);
                tc_fence_after();
                uint32_t v[32], w2[32];
                if (live) {
                    tmem_ld64_pack16(acc + 256 * hh, v);
                    tmem_ld64_pack16(acc + 256 * hh + 64, w2);
                    tmem_ld_wait();
                }
                tc_fence_before();
                if (lane == 0) mbar_arrive(&sm.tmem_empty[hh]);
                if (!live) continue;
#pragma unroll
                for (int s = 8; s > 0; s >>= 1)
#pragma unroll
                    for (int e = 0; e < s; ++e) {
                        v[e] = __vmaxs2(v[e], v[e + s]);
                        v[16 + e] = __vmaxs2(v[16 + e], v[16 + e + s]);
                        w2[e] = __vmaxs2(w2[e], w2[e + s]);
                        w2[16 + e] = __vmaxs2(w2[16 + e], w2[16 + e + s]);
                    }
                auto mx = [](uint32_t x) {
                    return max(static_cast<int>(static_cast<int16_t>(x & 0xFFFFu)),
                               static_cast<int>(static_cast<int16_t>(x >> 16)));
                };
                const float e0 = __fmul_rn(__fmul_rn(__fmul_rn(qs[hh], ksa), inv_sqrt_d), static_cast<float>(mx(v[0])));
                const float e1 = __fmul_rn(__fmul_rn(__fmul_rn(qs[hh], ksb), inv_sqrt_d), static_cast<float>(mx(v[16])));
                const float e2 = __fmul_rn(__fmul_rn(__fmul_rn(qs[hh], ksc), inv_sqrt_d), static_cast<float>(mx(w2[0])));
                const float e3 = __fmul_rn(__fmul_rn(__fmul_rn(qs[hh], ksd), inv_sqrt_d), static_cast<float>(mx(w2[16])));
                const bool pass = e0 >= fb[hh] || e1 >= fb[hh] || e2 >= fb[hh] || e3 >= fb[hh];
                flags[hh][0] |= pass ? sb0 : 0u;
                flags[hh][1] |= pass ? sb1 : 0u;
            }
        }
#pragma unroll
        for (int hh = 0; hh < kEstHeads; ++hh)
#pragma unroll
            for (int w = 0; w < kSegWords; ++w) {
                const uint32_t any = __reduce_or_sync(0xffffffffu, flags[hh][w]);
                if (lane == 0 && any && hh < nh) atomicOr(&sm.seg_bits[hh][quad >> 1][w], any);
            }
        named_bar_sync(1, 32 * kEpiWarps);
        if (ew == 0 && lane < 2 * kEstHeads) {
            const int h = lane >> 1, half = lane & 1;
            const int64_t qi = 2 * static_cast<int64_t>(u.m) + 1 + half;
            if (h < nh && qi < nq) {
                uint32_t *row = mask + ((static_cast<int64_t>(b) * hq + h0 + h) * nq + qi) * words;
                for (int sw = 0; sw < kSegWords; ++sw) {
                    uint32_t bits = sm.seg_bits[h][half][sw];
                    while (bits) {
                        const int s = 32 * sw + __ffs(bits) - 1;
                        bits &= bits - 1;
                        const int64_t sgl = static_cast<int64_t>(kSegPerUnit) * u.c + s;
                        const int64_t j0 = 1 + kSegment * sgl; // blocks j0 .. j0+3
                        const uint32_t w0 = static_cast<uint32_t>(j0 >> 5), sh = j0 & 31;
                        atomicOr(row + w0, 0xFu << sh);
                        if (sh > 28) atomicOr(row + w0 + 1, 0xFu >> (32 - sh));
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kEstHeads * 256>(tmem);
    }
}

} // namespace

size_t estimate_smem_bytes() { return sizeof(EstSmem) + 1024; }

cudaError_t estimate_profile(int enable, unsigned long long *out8) {
    if (out8) {
        cudaError_t e = cudaMemcpyFromSymbol(out8, g_est_prof, sizeof(g_est_prof));
        if (e != cudaSuccess) return e;
    }
    unsigned long long zero[8] = {};
    cudaError_t e = cudaMemcpyToSymbol(g_est_prof, zero, sizeof(zero));
    if (e != cudaSuccess) return e;
    g_est_mode_host = enable;
    return cudaMemcpyToSymbol(g_est_prof_on, &enable, sizeof(int));
}

cudaError_t launch_estimate(const CUtensorMap &tm_qc, const CUtensorMap &tm_kc, const EstUnit *units,
                            int64_t n_units, const float *q_scales, const float *k_scales,
                            const float *thresh, uint32_t *mask, int64_t batch, int64_t tokens,
                            int hq, int hkv, float inv_sqrt_d, const Geom &geo, int32_t *dbg_max,
                            cudaStream_t stream) {
    if (n_units == 0) return cudaSuccess;
    const size_t smem = estimate_smem_bytes();
    const int mode = dbg_max ? 1 : (g_est_mode_host == 0 ? 0 : (g_est_mode_host == 2 ? 3 : 2));
    using Kern = decltype(&estimate_kernel<0, false>);
    Kern kern;
    if (is_default_geom(geo))
        kern = mode == 0 ? estimate_kernel<0, false> : mode == 1 ? estimate_kernel<1, false>
             : mode == 2 ? estimate_kernel<2, false> : estimate_kernel<3, false>;
    else
        kern = mode == 1 ? estimate_kernel<1, true> : estimate_kernel<0, true>;
    const int group = hq / hkv;
    const int nsub = (group + kEstHeads - 1) / kEstHeads;
    dim3 grid(static_cast<unsigned>(n_units), static_cast<unsigned>(batch * hkv * nsub));
    static const bool narrow = getenv("SALE_B200_EST_NARROW") != nullptr; // A/B switch
    if (mode == 0 && is_default_geom(geo) && !narrow) {
        const size_t wsmem = sizeof(EstWideSmem) + 1024;
        cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(estimate_wide_kernel), wsmem);
        if (e != cudaSuccess) return e;
        estimate_wide_kernel<<<grid, kEstThreads, wsmem, stream>>>(tm_qc, tm_kc, units, q_scales, k_scales,
                                                                  thresh, mask, tokens, hq, hkv, nsub,
                                                                  inv_sqrt_d);
        return cudaGetLastError();
    }
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kEstThreads, smem, stream>>>(tm_qc, tm_kc, units, q_scales, k_scales, thresh, mask,
                                              tokens, hq, hkv, nsub, inv_sqrt_d, geo, dbg_max);
    return cudaGetLastError();
}

namespace {
// segment_aggregate (selection.hpp:182-195) over the raw per-block decisions
// the general-geometry estimator wrote: full segment s of query block i
// (blocks [sb + seg s, sb + seg (s + 1)), s < F_i) is selected iff any of its
// blocks is, so a selected segment only gains bits — OR-ing its full range
// touches no other segment's bits, and lanes can work on segments
// independently. One warp per mask row.
__global__ void __launch_bounds__(256)
segment_or_kernel(uint32_t *__restrict__ mask, int64_t rows, int64_t nq, int64_t words, Geom geo,
                  int64_t i_lo, int64_t ni) {
    const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= rows * ni) return;
    const int64_t bh = wid / ni, i = i_lo + wid % ni;
    const int64_t F = full_segments(i, geo);
    uint32_t *row = mask + (bh * nq + i) * words;
    for (int64_t s = lane; s < F; s += 32) {
        const int64_t a = geo.sb + static_cast<int64_t>(geo.seg) * s, e = a + geo.seg; // [a, e)
        bool any = false;
        for (int64_t w = a >> 5; w <= (e - 1) >> 5 && !any; ++w) {
            const int64_t lo = w * 32 > a ? w * 32 : a, hi = (w + 1) * 32 < e ? (w + 1) * 32 : e;
            const uint32_t m = (0xFFFFFFFFu >> (32 - (hi - lo))) << (lo - w * 32);
            any = (row[w] & m) != 0u;
        }
        if (!any) continue;
        for (int64_t w = a >> 5; w <= (e - 1) >> 5; ++w) {
            const int64_t lo = w * 32 > a ? w * 32 : a, hi = (w + 1) * 32 < e ? (w + 1) * 32 : e;
            atomicOr(row + w, (0xFFFFFFFFu >> (32 - (hi - lo))) << (lo - w * 32));
        }
    }
}
} // namespace

cudaError_t launch_segment_or(uint32_t *mask, int64_t batch, int64_t hq, int64_t tokens,
                              const Geom &geo, cudaStream_t stream, int64_t i_lo, int64_t i_hi) {
    if (is_default_geom(geo)) return cudaSuccess; // the estimator wrote whole segments
    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    if (i_hi < 0 || i_hi > nq) i_hi = nq;
    if (i_hi <= i_lo) return cudaSuccess;
    const int64_t warps = batch * hq * (i_hi - i_lo);
    segment_or_kernel<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, stream>>>(
        mask, batch * hq, nq, (nk + 31) / 32, geo, i_lo, i_hi - i_lo);
    return cudaGetLastError();
}

} // namespace sale_b200
