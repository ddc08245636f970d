// tmem_microbench.cu — tcgen05.ld throughput on this B200: W warps per CTA
// (one CTA per SM) repeatedly load TMEM columns; prints bytes of TMEM cells
// read per clock per SM for the load shapes the SALE epilogues use.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2505_24179_b200/csrc profiles/tmem_microbench.cu -o profiles/tmem_microbench
#include "common.cuh"

#include <cstdio>

using namespace sale_b200;

template <int MODE>
__global__ void tmem_bench(int iters, unsigned long long *cycles, unsigned *sink) {
    __shared__ uint32_t tbase;
    if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase + (static_cast<uint32_t>((threadIdx.x / 32) % 4 * 32) << 16);
    const int w = threadIdx.x / 32;
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t col = ((it * 4 + w / 4) * 32) & 511;
        if (MODE == 0) { // 32 cols, pack::16b -> 16 regs
            uint32_t v[16];
            tmem_ld32_pack16(tmem + col, v);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) acc ^= v[e];
        } else { // 32 cols, 32-bit -> 32 regs
            uint32_t v[32];
            tmem_ld32(tmem + col, v);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) acc ^= v[e];
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(cycles, static_cast<unsigned long long>(t1 - t0));
    if (acc == 0x12345678u) sink[0] = acc;
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tbase);
    }
}

template <int MODE> void run(const char *name, int warps) {
    unsigned long long *d;
    unsigned *s;
    cudaMalloc(&d, 8);
    cudaMalloc(&s, 4);
    const int iters = 2048, ctas = 148;
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 8);
        tmem_bench<MODE><<<ctas, 32 * warps>>>(iters, d, s);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    }
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = static_cast<double>(c) / ctas;
    const double bytes = static_cast<double>(iters) * warps * 32 * 32 * 4; // cells read
    printf("%-34s warps=%2d  %7.1f B/clk/SM (cells)  %6.1f cyc per warp-load\n", name, warps,
           bytes / cyc, cyc / iters);
    cudaFree(d);
    cudaFree(s);
}

int main() {
    for (int w : {4, 8, 16, 32}) run<0>("ld.32x32b.x16.pack::16b (32 cols)", w);
    for (int w : {4, 8, 16, 32}) run<1>("ld.32x32b.x32 (32 cols)", w);
    return 0;
}
