// common.cuh — sm_100a building blocks shared by the SALE kernels:
// mbarriers, TMA (cp.async.bulk.tensor), tcgen05 (TMEM alloc / MMA / ld / st)
// and the UMMA shared-memory + instruction descriptors. Inline PTX only; no
// CUTLASS. Layout conventions used by every kernel:
//   * activations  bf16 [B][N][H][128]   (token-major, heads interleaved)
//   * 4-bit codes  int8 [B][N][H][128]   (same layout, values in [-7, 7])
//   * q scales     f32  [B][Hq][N]       (one per token, quant.hpp:95-104)
//   * k scales     f32  [B][Hkv][Nk]     (one per 32-token key block, quant.hpp:107-119)
//   * masks        u32  [B][Hq][Nq][W]   (W = ceil(Nk/32); bit j%32 of word j/32 = block (i, j))
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda.h>
#include <cuda_runtime.h>

// A wait on an mbarrier longer than this traps (turns a protocol bug into a
// launch error instead of a hung GPU). The compute-sanitizer build raises it:
// instrumented kernels run orders of magnitude slower.
#ifndef SALE_B200_WAIT_TIMEOUT_NS
#define SALE_B200_WAIT_TIMEOUT_NS 4000000000ull
#endif

namespace sale_b200 {

constexpr int kHeadDim = 128;   // storage pitch of every row (elements)
constexpr int kBlockQ = 64;     // SelectionConfig::block_q default (selection.hpp:22)
constexpr int kBlockK = 32;     // SelectionConfig::block_k default (selection.hpp:23)
constexpr int kSegment = 4;     // SelectionConfig::segment_size default (selection.hpp:21)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Bytes to add to the dynamic shared memory base to reach 1 KB alignment
// (SW128 tiles). Indexing smem_raw with it keeps the compiler's knowledge that
// the struct lives in shared memory (LDS/STS, not generic LD/ST), which a
// round trip through uintptr_t would lose.
__device__ __forceinline__ uint32_t smem_pad_1k(const void *base) {
    return (1024u - (smem_u32(base) & 1023u)) & 1023u;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n .reg .pred p;\n .reg .b32 r;\n"
        " elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(pred));
    return pred != 0;
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ uint64_t global_timer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Spin on mbarrier.test_wait (non-blocking) instead of try_wait: reacts to the
// phase flip without try_wait's suspend/wake-up latency; for short, hot
// hand-offs where the waiting warp has nothing else to do.
__device__ __forceinline__ bool mbar_test_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_spin(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t spins = 0;
    uint64_t t0 = 0;
    while (!mbar_test_wait(a, parity)) {
        if ((++spins & 4095u) == 0) {
            if (t0 == 0) t0 = global_timer_ns();
            else if (global_timer_ns() - t0 > SALE_B200_WAIT_TIMEOUT_NS) __trap();
        }
    }
}

// Waits for the phase with the given parity. A wait that exceeds ~4 s traps
// (turns a protocol bug into a launch error instead of a hung GPU).
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    if (mbar_try_wait(a, parity)) return;
    const uint64_t t0 = global_timer_ns();
    uint32_t spins = 0;
    while (!mbar_try_wait(a, parity)) {
        if ((++spins & 1023u) == 0 && global_timer_ns() - t0 > SALE_B200_WAIT_TIMEOUT_NS) {
#ifdef SALE_B200_DEBUG_WAIT
            printf("mbar_wait timeout: block %d thread %d bar smem+%u parity %u\n", blockIdx.x, threadIdx.x,
                   a & 0xFFFFFu, parity);
#endif
            __trap();
        }
    }
}

// ------------------------------------------------------------------ clusters
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// Full cluster barrier (every thread of every CTA of the cluster).
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Shared::cluster address of the same shared-memory object in CTA `rank`.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// Arrive on an mbarrier of CTA `rank` (possibly this CTA). Default (CTA-scope
// release) semantics: the .release.cluster form adds a MEMBAR.GPU per arrive.
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t rank) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(smem_u32(bar), rank))
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}

// ----------------------------------------------------------------------- TMA
// Cluster-scope wait (the barrier receives arrivals from other CTAs).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    if (mbar_try_wait_cluster(a, parity)) return;
    const uint64_t t0 = global_timer_ns();
    uint32_t spins = 0;
    while (!mbar_try_wait_cluster(a, parity)) {
        if ((++spins & 1023u) == 0 && global_timer_ns() - t0 > SALE_B200_WAIT_TIMEOUT_NS) {
#ifdef SALE_B200_DEBUG_WAIT
            printf("mbar_wait timeout: block %d thread %d bar smem+%u parity %u\n", blockIdx.x, threadIdx.x,
                   a & 0xFFFFFu, parity);
#endif
            __trap();
        }
    }
}

__device__ __forceinline__ void tma_prefetch(const void *tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *smem_dst, const void *tmap, uint64_t *bar, int c0,
                                            int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
// Same box into the same shared-memory offset of every CTA in cta_mask; each
// destination CTA's mbarrier (same offset) receives complete_tx for its copy.
__device__ __forceinline__ void tma_load_4d_mc(void *smem_dst, const void *tmap, uint64_t *bar,
                                               int c0, int c1, int c2, int c3, uint16_t cta_mask) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "h"(cta_mask)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d_hint(void *smem_dst, const void *tmap, uint64_t *bar,
                                                 int c0, int c1, int c2, int c3, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ------------------------------------------------------------------- tcgen05
template <uint32_t kCols> __device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols> __device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Arrives on an mbarrier once every tcgen05.mma issued so far by this thread
// has completed (implies fence::before_thread_sync).
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
// As tc_commit, arriving on the barrier at the same offset in every CTA of cta_mask.
__device__ __forceinline__ void tc_commit_mc(uint64_t *bar, uint16_t cta_mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(cta_mask)
        : "memory");
}
// ---- CTA pairs (cta_group::2, a cluster of two CTAs on one TPC)
// TMA into this CTA's shared memory, completing bytes on the LEADER CTA's
// mbarrier at the same offset (peer bit cleared).
__device__ __forceinline__ void tma_load_4d_2sm(void *smem_dst, const void *tmap, uint64_t *bar,
                                                int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(tmap), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
template <uint32_t kCols> __device__ __forceinline__ void tmem_alloc_2sm(uint32_t *dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols> __device__ __forceinline__ void tmem_dealloc_2sm(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}
// Pair MMA (issued by the leader CTA): M = 256 rows, A rows 0-127 from the
// leader's shared memory and 128-255 from the peer's (same descriptor), B split
// along N between the two CTAs; D rows 0-127 in the leader's TMEM, 128-255 in
// the peer's (same column address).
__device__ __forceinline__ void mma_i8_ss_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on the barrier at this offset in every CTA of cta_mask once the pair
// MMAs issued so far have completed.
__device__ __forceinline__ void tc_commit_2sm_mc(uint64_t *bar, uint16_t cta_mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(cta_mask)
        : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, int8 x int8 -> int32
__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Warp-uniform issue: the whole warp executes the call (so descriptors and
// loop state stay in uniform registers) and elect.sync picks the one lane that
// issues. elect.sync with a full mask always picks the same lane, so a later
// tc_commit_elect tracks exactly these MMAs.
__device__ __forceinline__ void mma_i8_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p, e;\n .reg .b32 r;\n setp.ne.b32 p, %4, 0;\n"
        " elect.sync r|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t *bar) {
    asm volatile(
        "{\n .reg .pred e;\n .reg .b32 r;\n elect.sync r|e, 0xffffffff;\n"
        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
            smem_u32(bar))
        : "memory");
}
// D[tmem] (+)= A[smem] * B[smem], bf16 x bf16 -> f32
__device__ __forceinline__ void mma_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T, int8 x int8 -> int32 (A resident in TMEM:
// only B streams from shared memory)
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem], bf16 x bf16 -> f32 (A = P kept in TMEM)
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

#define SALE_R16(p, o)                                                                            \
    "=r"(p[o + 0]), "=r"(p[o + 1]), "=r"(p[o + 2]), "=r"(p[o + 3]), "=r"(p[o + 4]),               \
        "=r"(p[o + 5]), "=r"(p[o + 6]), "=r"(p[o + 7]), "=r"(p[o + 8]), "=r"(p[o + 9]),           \
        "=r"(p[o + 10]), "=r"(p[o + 11]), "=r"(p[o + 12]), "=r"(p[o + 13]), "=r"(p[o + 14]),      \
        "=r"(p[o + 15])
#define SALE_W16(p, o)                                                                            \
    "r"(p[o + 0]), "r"(p[o + 1]), "r"(p[o + 2]), "r"(p[o + 3]), "r"(p[o + 4]), "r"(p[o + 5]),     \
        "r"(p[o + 6]), "r"(p[o + 7]), "r"(p[o + 8]), "r"(p[o + 9]), "r"(p[o + 10]),               \
        "r"(p[o + 11]), "r"(p[o + 12]), "r"(p[o + 13]), "r"(p[o + 14]), "r"(p[o + 15])

// 32 lanes x 32 columns of 32-bit -> 32 regs per thread (thread t = lane t).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : SALE_R16(r, 0), SALE_R16(r, 16)
        : "r"(taddr));
}
// 32 lanes x 32 columns, keeping the low 16 bits of each column, packed in
// pairs (even column in the low half) -> 16 regs.
__device__ __forceinline__ void tmem_ld32_pack16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,"
        "%11,%12,%13,%14,%15}, [%16];"
        : SALE_R16(r, 0)
        : "r"(taddr));
}
// 32 lanes x 64 columns, low 16 bits of each column packed in pairs -> 32 regs.
__device__ __forceinline__ void tmem_ld64_pack16(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : SALE_R16(r, 0), SALE_R16(r, 16)
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
            taddr),
        SALE_W16(r, 0), SALE_W16(r, 16)
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16};" ::"r"(taddr),
        SALE_W16(r, 0)
        : "memory");
}

// 16-lane shapes (a warp may address lanes [0,16) or [16,32) of its quadrant).
// 16x256b.x8: 16 lanes x 64 columns; thread T holds lanes T/4 and T/4+8 at
// columns 8R + 2(T%4) + e: r[4R + 2*(second lane) + e], R < 8, e < 2.
__device__ __forceinline__ void tmem_ld16x256_x8(uint32_t taddr, uint32_t *r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : SALE_R16(r, 0), SALE_R16(r, 16)
        : "r"(taddr));
}
// 16x256b.x16: 16 lanes x 128 columns, r[4R + 2*(second lane) + e], R < 16.
__device__ __forceinline__ void tmem_ld16x256_x16(uint32_t taddr, uint32_t *r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,"
        "%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,"
        "%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : SALE_R16(r, 0), SALE_R16(r, 16), SALE_R16(r, 32), SALE_R16(r, 48)
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16x256_x8(uint32_t taddr, const uint32_t *r) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
            taddr),
        SALE_W16(r, 0), SALE_W16(r, 16)
        : "memory");
}
// 16x128b.x16: 16 lanes x 64 columns; thread T holds lanes T/4 and T/4+8 at
// column 4R + T%4: r[2R + (second lane)], R < 16.
__device__ __forceinline__ void tmem_st16x128_x16(uint32_t taddr, const uint32_t *r) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x128b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
            taddr),
        SALE_W16(r, 0), SALE_W16(r, 16)
        : "memory");
}

// 16x128b.x8: 16 lanes x 32 columns; thread T: lanes T/4, T/4+8 at column
// 4R + T%4: r[2R + (second lane)], R < 8.
__device__ __forceinline__ void tmem_st16x128_x8(uint32_t taddr, const uint32_t *r) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16};" ::"r"(taddr),
        SALE_W16(r, 0)
        : "memory");
}

// 16x256b.x1: 16 lanes x 8 columns, thread T: lanes T/4, T/4+8 at columns
// 2(T%4) + e: r[2 * (second lane) + e].
__device__ __forceinline__ void tmem_ld16x256_x1(uint32_t taddr, uint32_t *r) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16x256_x1(uint32_t taddr, const uint32_t *r) {
    asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
                 : "memory");
}

// ------------------------------------------------------------- descriptors
// UMMA shared-memory descriptor, SWIZZLE_128B (cute::UMMA::SmemDescriptor,
// version 1 for sm_100). lbo/sbo in bytes.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}
// Instruction descriptors (cute::UMMA::InstrDescriptor bit layout).
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, bool b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(b_mn_major) << 16) |
           (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Selection geometry with block_q = 64, block_k = 32 (selection.hpp:18-38,
// :92-123, :199-202, :236-245; SURVEY.md Appendix C for the defaults):
//   sb  = ceil(min(sink_tokens, N) / 32)  sink blocks = the middle's start
//   nl  = ceil(local_tokens_min / 32)     fully-past blocks of the local window
//   seg = segment_size
// Query block i: local window [lo_i, frontier_i], lo_i = max(0, 2i - nl);
// I_SL = [0, sb) U [lo_i, frontier_i]; middle = [sb, lo_i) when lo_i > sb;
// full segments F_i = (lo_i - sb) / seg, i.e. E_i = seg * F_i estimated
// blocks [sb, sb + E_i); the trailing partial run [sb + E_i, lo_i) is forced.
// Defaults (sb 1, nl 4, seg 4): I_SL = {0} U [2i-4, frontier], F_i =
// floor((2i-5)/4), middle non-empty from i = 3.
struct Geom {
    int sb;  // sink blocks
    int nl;  // local fully-past blocks
    int seg; // segment size (blocks)
};

__host__ __device__ __forceinline__ int64_t frontier_block(int64_t i, int64_t n, int64_t nk) {
    const int64_t qend = (i + 1) * kBlockQ < n ? (i + 1) * kBlockQ : n;
    const int64_t f = (qend - 1) / kBlockK;
    return f < nk - 1 ? f : nk - 1;
}
__host__ __device__ __forceinline__ int64_t local_lo(int64_t i, const Geom &g) {
    const int64_t lo = 2 * i - g.nl;
    return lo > 0 ? lo : 0;
}
__host__ __device__ __forceinline__ bool has_middle(int64_t i, const Geom &g) {
    return local_lo(i, g) > g.sb;
}
// First query block with a non-empty middle region: 2i - nl > sb.
__host__ __device__ __forceinline__ int64_t first_middle_block(const Geom &g) {
    return (g.nl + g.sb) / 2 + 1;
}
__host__ __device__ __forceinline__ int64_t full_segments(int64_t i, const Geom &g) {
    return has_middle(i, g) ? (local_lo(i, g) - g.sb) / g.seg : 0;
}
// Estimated middle blocks of query block i (E_i = seg * F_i).
__host__ __device__ __forceinline__ int64_t estimated_blocks(int64_t i, const Geom &g) {
    return static_cast<int64_t>(g.seg) * full_segments(i, g);
}
__host__ __device__ __forceinline__ bool is_default_geom(const Geom &g) {
    return g.sb == 1 && g.nl == 4 && g.seg == kSegment;
}

} // namespace sale_b200
