// m64_probe.cu — tcgen05.mma with M = 64 (cta_group::1, kind::f16): (1) which
// TMEM lanes hold the 64 rows of D (and whether a lane offset of 16 in the D /
// A address moves them to the other half of each lane quadrant), (2) its cost
// per instruction against M = 128. Decides whether K3 can run the MMAs of a key
// tile selected by only one head of its pair at half size.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2505_24179_b200/csrc profiles/m64_probe.cu -o profiles/m64_probe
#include "common.cuh"

#include <cstdio>

using namespace sale_b200;

__device__ __forceinline__ void st_bf16(uint8_t *tile, int row, int col, float v) {
    // K-major SW128: row r at r * 128 B, 16-byte chunk c at (c ^ (r & 7))
    const int chunk = col / 8, within = col % 8;
    __nv_bfloat16 *p = reinterpret_cast<__nv_bfloat16 *>(tile + row * 128 + ((chunk ^ (row & 7)) * 16) + within * 2);
    *p = __float2bfloat16(v);
}

// layout: D = A B^T, A[r][0] = r + 1, B[n][0] = 1 -> D[r][n] = r + 1. lane_off
// is added to the D (and A for TS) TMEM lane field. out[lane] = D column 0.
__global__ void __launch_bounds__(128, 1) layout_probe(int m, int lane_off, int ts, float *out) {
    __shared__ __align__(1024) uint8_t a[128 * 128];
    __shared__ __align__(1024) uint8_t bm[128 * 128];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 128 * 128 / 4; i += 128) {
        reinterpret_cast<uint32_t *>(a)[i] = 0;
        reinterpret_cast<uint32_t *>(bm)[i] = 0;
    }
    __syncthreads();
    if (threadIdx.x < 128) {
        st_bf16(a, threadIdx.x, 0, threadIdx.x < m ? static_cast<float>(threadIdx.x + 1) : 0.0f);
        st_bf16(bm, threadIdx.x, 0, 1.0f);
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
    // clear D columns [0, 32) of every lane, and stage A into TMEM columns
    // [256, 264) for the TS form (thread = lane = row, bf16 pairs)
    {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        uint32_t z[32];
        for (int e = 0; e < 32; ++e) z[e] = 0u;
        tmem_st32(tmem + (static_cast<uint32_t>(warp * 32) << 16), z);
        const int r = warp * 32 + lane; // A row r lives in lane r (M = 128 layout)
        uint32_t av[32];
        for (int e = 0; e < 32; ++e) av[e] = 0u;
        // the TS operand for M = 64 at lane_off: rows 0..63 in the lanes the
        // D layout uses; stage row value (lane index based) so the probe shows
        // which lane feeds which output row
        av[0] = __float_as_uint(0.0f);
        const float v = static_cast<float>(r + 1);
        __nv_bfloat162 p = __floats2bfloat162_rn(v, 0.0f);
        av[0] = *reinterpret_cast<uint32_t *>(&p);
        tmem_st32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 256, av);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16(m, 128, false);
        const uint64_t ad = umma_desc_sw128(smem_u32(a), 16, 1024);
        const uint64_t bd = umma_desc_sw128(smem_u32(bm), 16, 1024);
        const uint32_t d = tmem + (static_cast<uint32_t>(lane_off) << 16);
        if (ts) mma_bf16_ts(d, tmem + (static_cast<uint32_t>(lane_off) << 16) + 256, bd, idesc, 0u);
        else mma_bf16_ss(d, ad, bd, idesc, 0u);
        tc_commit(&bar);
        mbar_wait(&bar, 0);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    {
        const int warp = threadIdx.x >> 5;
        uint32_t r[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16), r);
        tmem_ld_wait();
        out[threadIdx.x] = __uint_as_float(r[0]);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int M, int N, bool TS>
__global__ void __launch_bounds__(128, 1) cost_probe(int iters, unsigned long long *cycles) {
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
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16(M, N, false);
        const uint64_t bd = umma_desc_sw128(smem_u32(bsm), 16, 1024);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (TS) mma_bf16_ts(tmem, tmem + 256 + 8 * (it & 3), bd + 2 * (it & 3), idesc, it > 0);
            else mma_bf16_ss(tmem, bd + 2 * (it & 3), bd + 2 * (it & 3), idesc, it > 0);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        atomicAdd(cycles, static_cast<unsigned long long>(clock64() - t0));
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int M, int N, bool TS> void cost(const char *name) {
    unsigned long long *d, h = 0;
    cudaMalloc(&d, 8);
    cudaMemset(d, 0, 8);
    const int iters = 4096;
    cost_probe<M, N, TS><<<148, 128>>>(iters, d);
    cudaMemset(d, 0, 8);
    cost_probe<M, N, TS><<<148, 128>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %s  %.1f cycles/MMA\n", name, cudaGetErrorString(e), double(h) / 148 / iters);
    cudaFree(d);
}

int main() {
    float *d, h[128];
    cudaMalloc(&d, 128 * 4);
    for (int ts = 0; ts < 2; ++ts)
        for (int m : {128, 64})
            for (int off : {0, 16}) {
                if (m == 128 && off) continue;
                cudaMemset(d, 0, 128 * 4);
                layout_probe<<<1, 128>>>(m, off, ts, d);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(h, d, 128 * 4, cudaMemcpyDeviceToHost);
                printf("layout %s M=%d lane_off=%d: %s\n  lane:value ", ts ? "TS" : "SS", m, off, cudaGetErrorString(e));
                for (int l = 0; l < 128; ++l)
                    if (h[l] != 0.0f) printf("%d:%g ", l, h[l]);
                printf("\n");
                if (e != cudaSuccess) return 1;
            }
    cost<128, 128, true>("bf16 M128 N128 TS");
    cost<64, 128, true>("bf16 M64  N128 TS");
    cost<128, 144, true>("bf16 M128 N144 TS");
    cost<64, 144, true>("bf16 M64  N144 TS");
    cost<128, 128, false>("bf16 M128 N128 SS");
    cost<64, 128, false>("bf16 M64  N128 SS");
    cost<64, 256, true>("bf16 M64  N256 TS");
    return 0;
}
