// ex2_microbench.cu — MUFU.EX2 element throughput on this B200 by operand
// type: ex2.approx.f32 (1 element per lane) vs ex2.approx.ftz.bf16x2 and
// ex2.approx.f16x2 (2 elements per lane). 148 CTAs x 256 threads, 8
// independent chains per thread; prints elements / cycle / SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 profiles/ex2_microbench.cu -o profiles/ex2_microbench
#include <cstdio>
#include <cstdint>

template <int KIND>
__global__ void __launch_bounds__(256) bench(uint32_t *out, int iters, long long *cyc) {
    uint32_t v[8];
    for (int e = 0; e < 8; ++e) v[e] = 0xBF00BF00u ^ (threadIdx.x * 8 + e); // ~ -0.5 in both halves
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(v[e]));
            if (KIND == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[e]));
            if (KIND == 2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[e]));
        }
    }
    const long long t1 = clock64();
    uint32_t x = 0;
    for (int e = 0; e < 8; ++e) x ^= v[e];
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long *>(cyc), (unsigned long long)(t1 - t0));
}

template <int KIND> void run(const char *name) {
    uint32_t *out;
    long long *cyc;
    cudaMalloc(&out, 148 * 256 * 4 * 4);
    cudaMalloc(&cyc, 8);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(cyc, 0, 8);
        bench<KIND><<<148 * 2, 256>>>(out, iters, cyc);
        cudaDeviceSynchronize();
    }
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double cycles = double(c) / (148 * 2);          // per CTA
    const double elems = double(iters) * 8 * 256 * (KIND == 0 ? 1 : 2) * 2; // per SM (2 CTAs)
    printf("%-24s %6.2f elements/clk/SM (%.0f cycles per CTA)\n", name, elems / cycles, cycles);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<0>("ex2.approx.ftz.f32");
    run<1>("ex2.approx.ftz.bf16x2");
    run<2>("ex2.approx.f16x2");
    return 0;
}
