// pipe_microbench.cu — issue cost of the softmax instruction mix on one SM:
// warp-instructions per cycle per SMSP for FFMA, FFMA2, FADD2, MUFU.EX2,
// FMNMX, FMNMX3, F2FP (bf16x2 pack), LEA.HI, with 1/2/4 warps per SMSP, 8
// independent chains per thread. nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

constexpr int kIters = 4096;

template <int OP>
__global__ void bench(float *out, long long *cyc, float a0) {
    float v[16];
    unsigned long long w[8];
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = a0 + threadIdx.x * 1e-3f + e;
#pragma unroll
    for (int e = 0; e < 8; ++e) w[e] = (static_cast<unsigned long long>(__float_as_uint(v[2 * e + 1])) << 32) | __float_as_uint(v[2 * e]);
    const unsigned long long m2 = (static_cast<unsigned long long>(__float_as_uint(0.999f)) << 32) | __float_as_uint(0.999f);
    const unsigned long long c2 = (static_cast<unsigned long long>(__float_as_uint(1e-7f)) << 32) | __float_as_uint(1e-7f);
    uint32_t u[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) u[e] = __float_as_uint(v[e]);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (OP == 0) v[e] = fmaf(v[e], 0.999f, 1e-7f);
            if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(w[e]) : "l"(m2), "l"(c2));
            if (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[e]) : "l"(c2));
            if (OP == 3) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[e]));
            if (OP == 4) asm volatile("max.f32 %0, %0, %1;" : "+f"(v[e]) : "f"(v[e + 8]));
            if (OP == 5) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(v[e]) : "f"(v[e + 8]), "f"(v[15 - e]));
            if (OP == 6) { __nv_bfloat162 p = __floats2bfloat162_rn(v[e], v[e + 8]); u[e] ^= *reinterpret_cast<uint32_t *>(&p); v[e] += 1e-9f * 0; asm volatile("" : "+r"(u[e])); }
            if (OP == 7) asm volatile("{.reg .b32 s; shf.l.wrap.b32 s, 0, %0, 23; add.u32 %0, s, %1;}" : "+r"(u[e]) : "r"(u[7 - e]));
            if (OP == 8) asm volatile("mul.f32 %0, %0, 0f3F7FBE77;" : "+f"(v[e]));
            if (OP == 9) asm volatile("{.reg .f32 t; mul.f32 t, %0, 0fBF000000; ex2.approx.ftz.f32 %0, t;}" : "+f"(v[e]));
            if (OP == 10) asm volatile("mul.f32 %0, %0, 0fBF000000;" : "+f"(v[e]));
            if (OP == 12) { // FFMA2 -> two MUFU on the halves -> repack
                unsigned long long x = w[e];
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(m2), "l"(c2));
                float a = __uint_as_float(static_cast<uint32_t>(x)), b = __uint_as_float(static_cast<uint32_t>(x >> 32));
                asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
                asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
                w[e] = (static_cast<unsigned long long>(__float_as_uint(b) & 0x3fffffffu) << 32) | (__float_as_uint(a) & 0x3fffffffu);
            }
            if (OP == 13) { // scalar FFMA -> MUFU
                float a = fmaf(v[e], -0.5f, 0.1f);
                asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
                v[e] = a;
            }
            if (OP == 11) asm volatile("{.reg .f32 t; mul.f32 t, %0, 0fBF000000; ex2.approx.f32 %0, t;}" : "+f"(v[e]));
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) s += v[e];
#pragma unroll
    for (int e = 0; e < 8; ++e) s += __uint_as_float(static_cast<uint32_t>(w[e])) + __uint_as_float(u[e]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP> void run(const char *name, float *out, long long *cyc) {
    for (int wps : {1, 2, 4}) {
        const int threads = 128 * wps; // wps warps per SMSP
        bench<OP><<<1, threads>>>(out, cyc, 1.0f);
        bench<OP><<<1, threads>>>(out, cyc, 1.0f);
        long long c;
        cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
        const double instr = static_cast<double>(kIters) * 8 * wps; // per SMSP
        printf("%-8s warps/SMSP=%d  %.2f cycles per warp-instruction per SMSP\n", name, wps, c / instr);
    }
}

int main() {
    float *out;
    long long *cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 1024);
    run<0>("FFMA", out, cyc);
    run<8>("FMUL", out, cyc);
    run<1>("FFMA2", out, cyc);
    run<2>("FADD2", out, cyc);
    run<3>("MUFU.EX2", out, cyc);
    run<4>("FMNMX", out, cyc);
    run<5>("FMNMX3", out, cyc);
    run<6>("F2FP+LOP", out, cyc);
    run<7>("LEA.HI", out, cyc);
    run<9>("FMUL+EX2(normal inputs)", out, cyc);
    run<10>("FMUL(ref)", out, cyc);
    run<11>("FMUL+EX2 noftz", out, cyc);
    run<12>("FFMA2+2xEX2 (per pair)", out, cyc);
    run<13>("FFMA+EX2", out, cyc);
    return 0;
}
