// internal.h — launcher declarations shared between the kernels and the C ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

struct sale_b200_ctx;

namespace sale_b200 {

struct Geom; // common.cuh: the selection geometry (sink blocks, local blocks, segment)

// capi.cu: record an error on ctx (or the calling thread's ctx-less slot when
// ctx is NULL) and return code; ctx's device.
int set_error(sale_b200_ctx *ctx, int code, const std::string &msg);
int ctx_device_of(const sale_b200_ctx *ctx);

// cudaFuncAttributeMaxDynamicSharedMemorySize for `func` on the CURRENT
// device, set once per (device, function): the attribute is per device, so a
// process driving contexts on several GPUs configures each of them.
cudaError_t ensure_smem_attr(const void *func, size_t bytes);

struct EstUnit {
    int m;    // 128-row query tile: rows [128m+64, 128m+192) = query blocks 2m+1, 2m+2
    int c;    // chunk of kSegPerUnit middle segments
    int nseg; // segments in this unit
};
constexpr int kSegPerUnitHost = 64;

cudaError_t launch_quantize_qk(const void *q, const void *k, int8_t *q_codes, float *q_scales,
                               int8_t *k_codes, float *k_scales, int64_t batch, int64_t tokens,
                               int64_t hq, int64_t hkv, cudaStream_t stream, int64_t t_lo = 0,
                               int64_t t_hi = -1);

cudaError_t launch_sink_local_stats(const void *q, const void *k, int64_t batch, int64_t tokens,
                                    int64_t hq, int64_t hkv, float inv_sqrt_d, const Geom &geo,
                                    const double *taus, float *thresh, double *dbg_m, double *dbg_l,
                                    double *dbg_bound, cudaStream_t stream, int64_t i_lo = 0,
                                    int64_t i_hi = -1);

cudaError_t launch_base_mask(uint32_t *mask, int64_t batch, int64_t hq, int64_t tokens,
                             const Geom &geo, cudaStream_t stream, int64_t i_lo = 0,
                             int64_t i_hi = -1);

// general geometry only (no-op for the default): segment_aggregate over the
// estimator's raw block decisions of query blocks [i_lo, i_hi)
cudaError_t launch_segment_or(uint32_t *mask, int64_t batch, int64_t hq, int64_t tokens,
                              const Geom &geo, cudaStream_t stream, int64_t i_lo = 0,
                              int64_t i_hi = -1);

size_t estimate_smem_bytes();
cudaError_t estimate_profile(int enable, unsigned long long *out8);
cudaError_t stats_profile(int enable, unsigned long long *out8);
cudaError_t launch_estimate(const CUtensorMap &tm_qc, const CUtensorMap &tm_kc, const EstUnit *units,
                            int64_t n_units, const float *q_scales, const float *k_scales,
                            const float *thresh, uint32_t *mask, int64_t batch, int64_t tokens,
                            int hq, int hkv, float inv_sqrt_d, const Geom &geo, int32_t *dbg_max,
                            cudaStream_t stream);

size_t attention_smem_bytes();
cudaError_t attention_profile(int enable, unsigned long long *out16);
cudaError_t launch_sparse_attention(const void *q, const CUtensorMap &tm_k, const CUtensorMap &tm_v,
                                    const uint32_t *mask, void *out, int32_t *coverage,
                                    int64_t batch, int64_t tokens, int hq, int hkv, float scale_log2,
                                    cudaStream_t stream, int64_t i_lo = 0, int64_t i_hi = -1,
                                    unsigned long long *empty_rows = nullptr);

cudaError_t launch_flop_count(const uint32_t *mask, int64_t batch, int64_t hq, int64_t tokens,
                              int64_t *counts, cudaStream_t stream);

} // namespace sale_b200
