// accounting.cu — flop_accounting (sparse_attention.hpp:101-118) over packed
// masks: per (batch, head) the number of computed / skipped / total causal
// blocks. Fully-future bits are outside the accounting (:108-110).
#include "common.cuh"

namespace sale_b200 {

namespace {

// one thread per mask row (b, h, i); counts [B*Hq][3]
__global__ void flop_count_kernel(const uint32_t *__restrict__ mask, int64_t rows, int64_t nq,
                                  int64_t nk, int64_t words, int64_t tokens,
                                  unsigned long long *__restrict__ counts) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= rows) return;
    const int64_t i = idx % nq;
    const int64_t bh = idx / nq;
    const int64_t fr = frontier_block(i, tokens, nk); // causal blocks: 0..fr
    const uint32_t *row = mask + idx * words;
    unsigned long long computed = 0;
    for (int64_t w = 0; w * 32 <= fr; ++w) {
        uint32_t v = row[w];
        const int64_t hi = fr - w * 32; // last valid bit index in this word
        if (hi < 31) v &= (2u << hi) - 1u;
        computed += __popc(v);
    }
    const unsigned long long total = static_cast<unsigned long long>(fr + 1);
    atomicAdd(&counts[bh * 3 + 0], computed);
    atomicAdd(&counts[bh * 3 + 1], total - computed);
    atomicAdd(&counts[bh * 3 + 2], total);
}

} // namespace

cudaError_t launch_flop_count(const uint32_t *mask, int64_t batch, int64_t hq, int64_t tokens,
                              int64_t *counts, cudaStream_t stream) {
    const int64_t nq = (tokens + kBlockQ - 1) / kBlockQ;
    const int64_t nk = (tokens + kBlockK - 1) / kBlockK;
    const int64_t words = (nk + 31) / 32;
    const int64_t rows = batch * hq * nq;
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int64_t) * 3 * batch * hq, stream);
    if (e != cudaSuccess) return e;
    const int threads = 256;
    flop_count_kernel<<<static_cast<unsigned>((rows + threads - 1) / threads), threads, 0, stream>>>(
        mask, rows, nq, nk, words, tokens, reinterpret_cast<unsigned long long *>(counts));
    return cudaGetLastError();
}

} // namespace sale_b200
