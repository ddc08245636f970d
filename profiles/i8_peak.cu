// i8_peak.cu — the measured tcgen05 kind::i8 (and, for comparison, kind::f16
// bf16) tensor rate of this B200, the denominator of K2b's roofline
// (bench.py measured_i8_peak). One CTA per SM, one elected thread issuing
// back-to-back M=128, N=256, K=32 MMAs from two distinct 32 KB shared-memory
// operands holding random codes in [-7, 7] (the estimator's value range, so
// the datapath toggles like the real kernel), into two alternating 256-column
// TMEM accumulators. "burst" = a ~50 ms launch after warm-up, "sustained" =
// back-to-back launches for ~4 s (the clock then settles under the power cap,
// as it does inside a 128K prefill). Clocks are sampled by the driver script
// (i8_peak.sh) with nvidia-smi during the run.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2505_24179_b200/csrc profiles/i8_peak.cu -o profiles/i8_peak
#include "common.cuh"

#include <chrono>
#include <cstdio>
#include <cstdlib>

using namespace sale_b200;

template <int KIND>
__global__ void __launch_bounds__(128, 1) peak_kernel(long long iters, unsigned seed) {
    extern __shared__ __align__(1024) uint8_t dyn[];
    uint8_t *a = dyn + smem_pad_1k(dyn);  // A: 128 rows x 128 B (16 KB)
    uint8_t *b = a + 128 * 128;           // B: 256 rows x 128 B (32 KB)
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    unsigned x = seed ^ (blockIdx.x * 2654435761u);
    for (int i = threadIdx.x; i < 256 * 128; i += 128) {
        x = x * 1664525u + 1013904223u;
        const int v = static_cast<int>((x >> 16) % 15u) - 7;
        // i8: codes; bf16: the code's bf16 bit pattern low/high byte pairs
        if (i < 128 * 128) a[i] = static_cast<uint8_t>(KIND == 0 ? v : ((i & 1) ? 0x40 + (v & 7) : 0));
        x = x * 1664525u + 1013904223u;
        const int w = static_cast<int>((x >> 16) % 15u) - 7;
        b[i] = static_cast<uint8_t>(KIND == 0 ? w : ((i & 1) ? 0x40 + (w & 7) : 0));
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
        const uint32_t idesc = KIND == 0 ? idesc_i8(128, 256) : idesc_bf16(128, 256, false);
        const uint64_t ad = umma_desc_sw128(smem_u32(a), 16, 1024);
        const uint64_t bd = umma_desc_sw128(smem_u32(b), 16, 1024);
        for (long long it = 0; it < iters; ++it) {
            const uint32_t d = tmem + 256 * static_cast<uint32_t>((it >> 2) & 1);
            const int kk = static_cast<int>(it & 3);
            if (KIND == 0) mma_i8_ss(d, ad + 2 * kk, bd + 2 * kk, idesc, kk > 0);
            else mma_bf16_ss(d, ad + 2 * kk, bd + 2 * kk, idesc, kk > 0);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int KIND> double rate(long long iters, int launches, double *ms_out) {
    const int sms = 148;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int smem = 128 * 128 + 256 * 128 + 1024;
    cudaFuncSetAttribute(peak_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    peak_kernel<KIND><<<sms, 128, smem>>>(iters / 8, 1u); // warm-up
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int l = 0; l < launches; ++l) peak_kernel<KIND><<<sms, 128, smem>>>(iters, 7u + l);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    if (err != cudaSuccess) {
        fprintf(stderr, "kernel failed: %s\n", cudaGetErrorString(err));
        exit(1);
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *ms_out = ms;
    // MACs per MMA = 128 * 256 * K, K = 32 (i8) or 16 (bf16); 2 ops per MAC
    const double ops = 2.0 * 128 * 256 * (KIND == 0 ? 32 : 16) * static_cast<double>(iters) * sms * launches;
    return ops / (ms * 1e-3) / 1e12;
}

int main() {
    double ms_b = 0, ms_s = 0, ms_fb = 0, ms_fs = 0;
    // ~128 cycles per N=256 MMA: 400k MMAs ~ 27 ms at 1.9 GHz
    const double burst = rate<0>(400000, 2, &ms_b);
    const double sus = rate<0>(400000, 120, &ms_s);
    const double fburst = rate<1>(400000, 2, &ms_fb);
    const double fsus = rate<1>(400000, 120, &ms_fs);
    printf("{\"burst_tops\": %.1f, \"sustained_tops\": %.1f, \"burst_ms\": %.1f, \"sustained_ms\": %.1f, "
           "\"bf16_burst_tflops\": %.1f, \"bf16_sustained_tflops\": %.1f, "
           "\"shape\": \"tcgen05.mma.cta_group::1 kind::i8 M128 N256 K32, SMEM A/B, 148 CTAs x 1 issuer\"}\n",
           burst, sus, ms_b, ms_s, fburst, fsus);
    return 0;
}
