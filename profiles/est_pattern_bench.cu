// est_pattern_bench.cu — the K2b estimator's MMA issue pattern in isolation:
// 4 query heads (A tiles, 16 KB each, SMEM) x 128-key K stages (B, 16 KB) ->
// 4 TMEM accumulators of M=128 x N=128 int32, 4 x K=32 tcgen05.mma.kind::i8 per
// head per stage, tcgen05.commit per head, an epilogue that drains every
// accumulator with 16 warps. Variants switch the B stream (static vs. TMA
// from HBM/L2) and the epilogue TMEM loads on/off, to separate the MMA rate,
// the commit round trip, SMEM contention and the drain. Cycles per stage from
// the issuing thread, averaged over 148 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_24179_b200/csrc \
//        profiles/est_pattern_bench.cu -o profiles/est_pattern_bench -lcuda
#include "common.cuh"

#include <cstdio>

using namespace sale_b200;

constexpr int kStages = 6, kHeads = 4, kEpiWarps = 16;

struct Smem {
    alignas(1024) uint8_t a[kHeads][16384];
    alignas(1024) uint8_t b[kStages][16384];
    uint64_t full[kStages], empty[kStages], tfull[kHeads], tempty[kHeads];
    uint32_t tbase;
};

__device__ int g_random_data = 0;
__device__ int g_ring = kStages, g_plain = 0, g_nowait = 0, g_real_epi = 0;

template <bool TMA, bool LOADS, int NACC>
__global__ void __launch_bounds__(128 + 32 * kEpiWarps, 1)
bench(const __grid_constant__ CUtensorMap tm, int nstages, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    Smem &sm = *reinterpret_cast<Smem *>(raw + smem_pad_1k(raw));
    const int warp = threadIdx.x >> 5;
    const bool rnd = g_random_data != 0;
    auto code4 = [](uint32_t x) { // four int8 codes in [-7, 7] from a hash
        x *= 0x9E3779B1u; x ^= x >> 15; x *= 0x85EBCA77u; x ^= x >> 13;
        uint32_t r = 0;
        for (int e = 0; e < 4; ++e) r |= (static_cast<uint32_t>(static_cast<int>((x >> (8 * e)) % 15u) - 7) & 0xFFu) << (8 * e);
        return r;
    };
    for (int i = threadIdx.x; i < (int)sizeof(sm.a) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(sm.a)[i] = rnd ? code4(i * 7 + blockIdx.x) : 0x01010101u * (i & 3);
    for (int i = threadIdx.x; i < (int)sizeof(sm.b) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(sm.b)[i] = rnd ? code4(i * 13 + 5) : 0x01010101u * (i & 5);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&sm.full[s], 1), mbar_init(&sm.empty[s], 1);
        for (int h = 0; h < kHeads; ++h) mbar_init(&sm.tfull[h], 1), mbar_init(&sm.tempty[h], kEpiWarps);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(&sm.tbase);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tbase;
    if (warp == 0) {
        if (TMA && elect_one()) {
            for (int k = 0; k < nstages; ++k) {
                const int st = k % g_ring;
                mbar_wait(&sm.empty[st], ((k / g_ring) & 1) ^ 1);
                if (g_plain) { mbar_arrive(&sm.full[st]); continue; }
                mbar_expect_tx(&sm.full[st], 16384);
                tma_load_4d(sm.b[st], &tm, &sm.full[st], 0, 0, (blockIdx.x * 997 + k) % 4096 * 128, 0);
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            constexpr uint32_t idesc = idesc_i8(128, 128);
            const long long t0 = clock64();
            long long wacc = 0;
            for (int k = 0; k < nstages; ++k) {
                const int st = k % g_ring;
                if (TMA) mbar_wait(&sm.full[st], (k / g_ring) & 1);
                tc_fence_after();
                const uint64_t bd = umma_desc_sw128(smem_u32(sm.b[st]), 16, 1024);
                for (int hh = 0; hh < kHeads; ++hh) {
                    const int acc = (k * kHeads + hh) % NACC;
                    const int use = (k * kHeads + hh) / NACC;
                    const long long tw = clock64();
                    if (!g_nowait) mbar_wait(&sm.tempty[acc], (use & 1) ^ 1);
                    wacc += clock64() - tw;
                    tc_fence_after();
                    const uint64_t ad = umma_desc_sw128(smem_u32(sm.a[hh]), 16, 1024);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_i8_ss(tmem + 128 * acc, ad + 2 * kk, bd + 2 * kk, idesc, kk > 0);
                    tc_commit(&sm.tfull[acc]);
                }
                if (TMA) tc_commit(&sm.empty[st]);
            }
            const long long t1 = clock64();
            atomicAdd(&out[0], static_cast<unsigned long long>(t1 - t0));
            atomicAdd(&out[1], static_cast<unsigned long long>(wacc));
        }
    } else if (warp >= 4 && !g_nowait) {
        const int ew = warp - 4, quad = warp & 3, chunk = ew >> 2;
        const uint32_t base = tmem + (static_cast<uint32_t>(quad * 32) << 16) + 32 * chunk;
        uint32_t sink = 0;
        const float lane_f = static_cast<float>(threadIdx.x & 31) * 0.01f;
        const bool real_epi = g_real_epi != 0;
        for (int i = 0; i < nstages * kHeads; ++i) {
            const int acc = i % NACC, use = i / NACC;
            mbar_wait(&sm.tfull[acc], use & 1);
            tc_fence_after();
            if (LOADS) {
                uint32_t v[16];
                tmem_ld32_pack16(base + 128 * acc, v);
                tmem_ld_wait();
                if (real_epi) {
                    tc_fence_before();
                    __syncwarp();
                    if ((threadIdx.x & 31) == 0) mbar_arrive(&sm.tempty[acc]);
#pragma unroll
                    for (int s = 8; s > 0; s >>= 1)
#pragma unroll
                        for (int e = 0; e < s; ++e) v[e] = __vmaxs2(v[e], v[e + s]);
                    const int lo = static_cast<int16_t>(v[0] & 0xFFFFu);
                    const int hi = static_cast<int16_t>(v[0] >> 16);
                    const int mx = lo > hi ? lo : hi;
                    const float rs = __fmul_rn(__fmul_rn(1.0f + lane_f, 0.5f), 0.088f);
                    const float est = __fmul_rn(rs, static_cast<float>(mx));
                    sink |= est >= 3.0f ? (1u << (i & 31)) : 0u;
                    continue;
                }
#pragma unroll
                for (int e = 0; e < 16; ++e) sink ^= v[e];
            }
            tc_fence_before();
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&sm.tempty[acc]);
        }
        if (sink == 0x12345678u) out[7] = sink;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <bool TMA, bool LOADS, int NACC>
void run(const char *name, const CUtensorMap &tm, unsigned long long *d, int nst = 512, int waves = 1) {
    const size_t smem = sizeof(Smem) + 1024;
    cudaFuncSetAttribute(bench<TMA, LOADS, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 64);
        bench<TMA, LOADS, NACC><<<148 * waves, 128 + 32 * kEpiWarps, smem>>>(tm, nst, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    }
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-44s %6.0f cyc/stage (ideal 1024), accumulator wait %5.0f cyc/stage\n", name,
           (double)h[0] / 148 / waves / nst, (double)h[1] / 148 / waves / nst);
}

int main() {
    const size_t rows = 4096 * 128;
    uint8_t *g;
    cudaMalloc(&g, rows * 128);
    cudaMemset(g, 1, rows * 128);
    CUtensorMap tm;
    cuuint64_t dims[4] = {128, 1, rows, 1};
    cuuint64_t strides[3] = {128, 128, rows * 128};
    cuuint32_t box[4] = {128, 1, 128, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, g, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("tmap %d\n", (int)r); return 1; }
    unsigned long long *d;
    cudaMalloc(&d, 64);
    run<false, false, 4>("static B, no epilogue loads, 4 acc", tm, d);
    run<false, true, 4>("static B, epilogue loads, 4 acc", tm, d);
    run<true, false, 4>("TMA B, no epilogue loads, 4 acc", tm, d);
    run<true, true, 4>("TMA B, epilogue loads, 4 acc", tm, d);
    run<true, true, 4>("TMA B, loads, 4 acc, 64-stage units x8", tm, d, 64, 8);
    run<true, true, 4>("TMA B, loads, 4 acc, 16-stage units x32", tm, d, 16, 32);
    int one = 1;
    cudaMemcpyToSymbol(g_random_data, &one, sizeof(int));
    run<false, false, 4>("RANDOM codes: static B, no loads, 4 acc", tm, d);
    run<false, true, 4>("RANDOM codes: static B, loads, 4 acc", tm, d);
    run<false, true, 4>("RANDOM codes: static B, loads, 4 acc, LONG (~40 ms)", tm, d, 1024, 64);
    run<true, true, 4>("RANDOM codes: TMA B, loads, 4 acc, LONG (~40 ms)", tm, d, 1024, 64);
    int v;
    v = 1; cudaMemcpyToSymbol(g_real_epi, &v, 4);
    run<true, true, 4>("TMA B, REAL epilogue compute, 4 acc", tm, d);
    run<false, true, 4>("static B, REAL epilogue compute, 4 acc", tm, d);
    v = 0; cudaMemcpyToSymbol(g_real_epi, &v, 4);
    v = 4; cudaMemcpyToSymbol(g_ring, &v, 4);
    v = 1; cudaMemcpyToSymbol(g_plain, &v, 4);
    run<true, false, 4>("ring 4, plain producer, handoff", tm, d);
    v = 1; cudaMemcpyToSymbol(g_nowait, &v, 4);
    run<true, false, 4>("ring 4, plain producer, NO handoff (real mode 7)", tm, d);
    v = 6; cudaMemcpyToSymbol(g_ring, &v, 4);
    run<true, false, 4>("ring 6, plain producer, NO handoff", tm, d);
    v = 0; cudaMemcpyToSymbol(g_plain, &v, 4);
    run<true, false, 4>("ring 6, TMA producer, NO handoff", tm, d);
    v = 0; cudaMemcpyToSymbol(g_nowait, &v, 4);
    run<false, false, 2>("static B, no epilogue loads, 2 acc", tm, d);
    run<false, false, 3>("static B, no epilogue loads, 3 acc", tm, d);
    return 0;
}
