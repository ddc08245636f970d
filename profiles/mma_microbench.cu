// mma_microbench.cu — measures tcgen05.mma issue/throughput on this B200 for
// the shapes the SALE kernels use (one CTA per SM, one elected thread issuing
// back-to-back MMAs; operands are dummy data). Prints cycles per MMA and the
// implied per-SM MAC rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2505_24179_b200/csrc profiles/mma_microbench.cu -o profiles/mma_microbench
#include "common.cuh"

#include <cstdio>

using namespace sale_b200;

template <int KIND, int N, bool A_TMEM>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, unsigned long long *cycles) {
    __shared__ __align__(1024) uint8_t bsm[256 * 128];
    uint8_t *a = bsm; // operand values are irrelevant: A aliases B
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 256 * 128 / 4; i += 128) reinterpret_cast<uint32_t *>(bsm)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    if (threadIdx.x == 0) {
        // KIND 0: i8 (K=32 bytes per MMA), KIND 1: bf16 (K=16 elements = 32 bytes)
        const uint32_t idesc = KIND == 0 ? idesc_i8(128, N) : idesc_bf16(128, N, false);
        const uint64_t ad = umma_desc_sw128(smem_u32(a), 16, 1024);
        const uint64_t bd = umma_desc_sw128(smem_u32(bsm), 16, 1024);
        const uint32_t dcol = A_TMEM ? 256 : 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = tmem + dcol + ((it & 1) ? 0 : 0);
            if (KIND == 0) {
                if (A_TMEM) mma_i8_ts(d, tmem + 8 * (it & 3), bd + 2 * (it & 3), idesc, it > 0);
                else mma_i8_ss(d, ad + 2 * (it & 3), bd + 2 * (it & 3), idesc, it > 0);
            } else {
                if (A_TMEM) mma_bf16_ts(d, tmem + 8 * (it & 3), bd + 2 * (it & 3), idesc, it > 0);
                else mma_bf16_ss(d, ad + 2 * (it & 3), bd + 2 * (it & 3), idesc, it > 0);
            }
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        const long long t1 = clock64();
        atomicAdd(cycles, static_cast<unsigned long long>(t1 - t0));
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int KIND, int N, bool A_TMEM> void run(const char *name) {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    const int iters = 4096, ctas = 148;
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 8);
        mma_bench<KIND, N, A_TMEM><<<ctas, 128>>>(iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: %s\n", name, cudaGetErrorString(e));
            return;
        }
    }
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = static_cast<double>(c) / ctas / iters;
    const double macs = 128.0 * N * 32.0 / (KIND == 0 ? 1 : 2);
    printf("%-28s %7.1f cycles/MMA  %8.0f MAC/clk/SM\n", name, cyc, macs / cyc);
    cudaFree(d);
}

// Distinct A (16 KB) and B (16 KB) regions: SMEM must deliver both operands.
template <int KIND>
__global__ void __launch_bounds__(128, 1) mma_bench_distinct(int iters, unsigned long long *cycles) {
    __shared__ __align__(1024) uint8_t a[128 * 128];
    __shared__ __align__(1024) uint8_t bsm[128 * 128];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 128 * 128 / 4; i += 128) {
        reinterpret_cast<uint32_t *>(a)[i] = 0x01010101u * (i & 3);
        reinterpret_cast<uint32_t *>(bsm)[i] = 0x01010101u * (i & 5);
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    if (threadIdx.x == 0) {
        const uint32_t idesc = KIND == 0 ? idesc_i8(128, 128) : idesc_bf16(128, 128, false);
        const uint64_t ad = umma_desc_sw128(smem_u32(a), 16, 1024);
        const uint64_t bd = umma_desc_sw128(smem_u32(bsm), 16, 1024);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = tmem + 128 * (it & 3);
            if (KIND == 0) mma_i8_ss(d, ad + 2 * (it & 3), bd + 2 * (it & 3), idesc, it > 3);
            else mma_bf16_ss(d, ad + 2 * (it & 3), bd + 2 * (it & 3), idesc, it > 3);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        const long long t1 = clock64();
        atomicAdd(cycles, static_cast<unsigned long long>(t1 - t0));
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int KIND> void run_distinct(const char *name) {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    const int iters = 4096, ctas = 148;
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 8);
        mma_bench_distinct<KIND><<<ctas, 128>>>(iters, d);
        cudaDeviceSynchronize();
    }
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = static_cast<double>(c) / ctas / iters;
    const double macs = 128.0 * 128 * 32.0 / (KIND == 0 ? 1 : 2);
    printf("%-28s %7.1f cycles/MMA  %8.0f MAC/clk/SM\n", name, cyc, macs / cyc);
    cudaFree(d);
}

// Warp-uniform issue: the whole warp runs the loop (descriptors stay in
// uniform registers) and elect.sync picks the lane that issues each MMA.
__device__ __forceinline__ void mma_i8_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p, e;\n .reg .b32 r;\n setp.ne.b32 p, %4, 0;\n"
        " elect.sync r|e, 0xffffffff;\n"
        " @e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

template <int N>
__global__ void __launch_bounds__(128, 1) mma_bench_warp(int iters, unsigned long long *cycles) {
    __shared__ __align__(1024) uint8_t bsm[256 * 128];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 256 * 128 / 4; i += 128) reinterpret_cast<uint32_t *>(bsm)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    if (threadIdx.x < 32) {
        const uint32_t idesc = idesc_i8(128, N);
        const uint64_t ad = umma_desc_sw128(smem_u32(bsm), 16, 1024);
        const uint64_t bd = umma_desc_sw128(smem_u32(bsm) + 16384, 16, 1024);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
            mma_i8_ss_elect(tmem + 128 * (it & 3), ad + 2 * (it & 3), bd + 2 * (it & 3), idesc, it > 3);
        if (elect_one()) tc_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        const long long t1 = clock64();
        if (threadIdx.x == 0) atomicAdd(cycles, static_cast<unsigned long long>(t1 - t0));
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int N> void run_warp(const char *name) {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    const int iters = 4096, ctas = 148;
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 8);
        mma_bench_warp<N><<<ctas, 128>>>(iters, d);
        cudaDeviceSynchronize();
    }
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = static_cast<double>(c) / ctas / iters;
    printf("%-28s %7.1f cycles/MMA  %8.0f MAC/clk/SM\n", name, cyc, 128.0 * N * 32 / cyc);
    cudaFree(d);
}

// The estimator's issue pattern: per group of 4 MMAs one mbarrier wait (on a
// barrier this thread has just completed itself, i.e. never blocking), a
// fence, and one tcgen05.commit — measures the bookkeeping cost per MMA.
__global__ void __launch_bounds__(128, 1) mma_bench_sync(int iters, unsigned long long *cycles) {
    __shared__ __align__(1024) uint8_t bsm[256 * 128];
    __shared__ uint64_t bar, bar2, bar3;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 256 * 128 / 4; i += 128) reinterpret_cast<uint32_t *>(bsm)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1);
        mbar_init(&bar3, 1);
        fence_barrier_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_i8(128, 128);
        const uint64_t ad = umma_desc_sw128(smem_u32(bsm), 16, 1024);
        const uint64_t bd = umma_desc_sw128(smem_u32(bsm) + 16384, 16, 1024);
        const long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters / 4; ++it) {
            mbar_arrive(&bar2);
            mbar_wait(&bar2, ph);
            ph ^= 1;
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                mma_i8_ss(tmem + 128 * (it & 3), ad + 2 * kk, bd + 2 * kk, idesc, kk > 0);
            tc_commit(&bar3);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        const long long t1 = clock64();
        atomicAdd(cycles, static_cast<unsigned long long>(t1 - t0));
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

void run_sync(const char *name) {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    const int iters = 4096, ctas = 148;
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 8);
        mma_bench_sync<<<ctas, 128>>>(iters, d);
        cudaDeviceSynchronize();
    }
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = static_cast<double>(c) / ctas / iters;
    printf("%-28s %7.1f cycles/MMA  %8.0f MAC/clk/SM\n", name, cyc, 128.0 * 128 * 32 / cyc);
    cudaFree(d);
}

int main() {
    run_sync("i8 N128 + wait/fence/commit per 4");
    run_warp<32>("i8 N32  warp-uniform issue");
    run_warp<64>("i8 N64  warp-uniform issue");
    run_warp<128>("i8 N128 warp-uniform issue");
    run_distinct<0>("i8  M128 N128 SS distinct");
    run_distinct<1>("bf16 M128 N128 SS distinct");
    run<0, 32, true>("i8  M128 N32  A=TMEM");
    run<0, 64, true>("i8  M128 N64  A=TMEM");
    run<0, 128, true>("i8  M128 N128 A=TMEM");
    run<0, 256, true>("i8  M128 N256 A=TMEM");
    run<0, 32, false>("i8  M128 N32  A=SMEM");
    run<0, 64, false>("i8  M128 N64  A=SMEM");
    run<0, 128, false>("i8  M128 N128 A=SMEM");
    run<0, 256, false>("i8  M128 N256 A=SMEM");
    run<1, 32, true>("bf16 M128 N32  A=TMEM");
    run<1, 64, true>("bf16 M128 N64  A=TMEM");
    run<1, 128, true>("bf16 M128 N128 A=TMEM");
    run<1, 256, true>("bf16 M128 N256 A=TMEM");
    run<1, 128, false>("bf16 M128 N128 A=SMEM");
    run<1, 256, false>("bf16 M128 N256 A=SMEM");
    return 0;
}
