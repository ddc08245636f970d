// softmax_microbench.cu — cycles per 64-column softmax half-tile (the K3 exp
// loop: scale, exp2 via MUFU or the FMA/ALU polynomial, row sum, bf16 pack)
// on registers only, 1 or 2 warps per SMSP, for several polynomial fractions.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__device__ __forceinline__ unsigned long long pack_f2(float lo, float hi) {
    return (static_cast<unsigned long long>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ void ffma2_f32(unsigned long long &x, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(a), "l"(b));
}
__device__ __forceinline__ void fadd2_f32(unsigned long long &x, unsigned long long a) {
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(a));
}
__device__ __forceinline__ void fsub2_f32(unsigned long long &x, unsigned long long a) {
    asm("sub.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(a));
}
__device__ __forceinline__ uint32_t shl23_add(uint32_t t, uint32_t p) {
    uint32_t sh, r;
    asm("shf.l.wrap.b32 %0, %1, %2, 23;" : "=r"(sh) : "r"(0u), "r"(t));
    asm("add.u32 %0, %1, %2;" : "=r"(r) : "r"(sh), "r"(p));
    return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&p);
}

template <int POLY_OF_8, int VAR = 0>
__global__ void bench(uint32_t *io, long long *cyc, int iters) {
    uint32_t s[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) s[c] = __float_as_uint(-0.01f * c - threadIdx.x * 1e-4f);
    const float scale = 1.4426950f * 0.0883883f;
    float l = 0.0f, neg_m = 0.25f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const unsigned long long sc2 = pack_f2(scale, scale), nm2 = pack_f2(neg_m, neg_m);
        unsigned long long psum2 = 0ull;
#pragma unroll
        for (int c2 = 0; c2 < 32; ++c2) {
            unsigned long long x = (static_cast<unsigned long long>(s[2 * c2 + 1]) << 32) | s[2 * c2];
            ffma2_f32(x, sc2, nm2);
            float p0, p1;
            if ((c2 & 7) < POLY_OF_8) {
                const unsigned long long xc = pack_f2(fmaxf(__uint_as_float(static_cast<uint32_t>(x)), -125.0f),
                                                      fmaxf(__uint_as_float(static_cast<uint32_t>(x >> 32)), -125.0f));
                unsigned long long t = xc;
                fadd2_f32(t, pack_f2(12582912.0f, 12582912.0f));
                unsigned long long r = t;
                fadd2_f32(r, pack_f2(-12582912.0f, -12582912.0f));
                unsigned long long f = xc;
                fsub2_f32(f, r);
                unsigned long long pp = pack_f2(0.05592204f, 0.05592204f);
                ffma2_f32(pp, f, pack_f2(0.24264008f, 0.24264008f));
                ffma2_f32(pp, f, pack_f2(0.69312102f, 0.69312102f));
                ffma2_f32(pp, f, pack_f2(0.99992448f, 0.99992448f));
                p0 = __uint_as_float(shl23_add(static_cast<uint32_t>(t), static_cast<uint32_t>(pp)));
                p1 = __uint_as_float(shl23_add(static_cast<uint32_t>(t >> 32), static_cast<uint32_t>(pp >> 32)));
            } else {
                p0 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x)));
                p1 = ex2_approx(__uint_as_float(static_cast<uint32_t>(x >> 32)));
            }
            if (VAR != 1) fadd2_f32(psum2, pack_f2(p0, p1));
            else psum2 ^= static_cast<unsigned long long>(__float_as_uint(p0) ^ __float_as_uint(p1));
            if (VAR != 2) s[32 + (c2 & 31)] ^= pack_bf16x2(p0, p1) & 1u; // keep the pack live
            else s[32 + (c2 & 31)] ^= (__float_as_uint(p0) + __float_as_uint(p1)) & 1u;
        }
        l += __uint_as_float(static_cast<uint32_t>(psum2)) + __uint_as_float(static_cast<uint32_t>(psum2 >> 32));
        neg_m = neg_m * 0.999f;
    }
    const long long t1 = clock64();
    uint32_t acc = __float_as_uint(l);
#pragma unroll
    for (int c = 0; c < 64; ++c) acc ^= s[c];
    io[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int P, int V = 0> void run(uint32_t *io, long long *cyc) {
    for (int wps : {1, 2, 4}) {
        const int iters = 256;
        bench<P, V><<<1, 128 * wps>>>(io, cyc, iters);
        bench<P, V><<<1, 128 * wps>>>(io, cyc, iters);
        long long c;
        cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
        printf("variant %d poly %d/8, warps/SMSP=%d: %.0f cycles per 64-column half-tile per SMSP (all warps)\n", V, P, wps,
               static_cast<double>(c) / iters);
    }
}

int main() {
    uint32_t *io;
    long long *cyc;
    cudaMalloc(&io, 1 << 20);
    cudaMalloc(&cyc, 64);
    run<0>(io, cyc);
    run<0, 1>(io, cyc);
    run<0, 2>(io, cyc);
    run<2>(io, cyc);
    run<3>(io, cyc);
    run<4>(io, cyc);
    run<5>(io, cyc);
    return 0;
}
