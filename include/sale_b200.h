/*
 * sale_b200.h — C ABI of the B200-native SALE prefill path (sm_100a).
 *
 * The drop-in boundary for the reference's hot path (the header-only
 * `namespace sale` in /root/reference/proj/include/sale). Every entry point
 * names the reference function it replaces (file:line). Plain pointers and
 * sizes only; no torch / C++ types. All status codes are int:
 *
 *   0  SALE_B200_OK
 *   1  SALE_B200_INVALID_ARGUMENT   (reference throws std::invalid_argument)
 *   2  SALE_B200_DOMAIN_ERROR       (reference throws std::domain_error)
 *   3  SALE_B200_OUT_OF_RANGE       (reference throws std::out_of_range)
 *   4  SALE_B200_CUDA_ERROR
 *   5  SALE_B200_UNSUPPORTED        (valid for the reference, not on this path:
 *                                    see DESIGN.md "Scope")
 *   6  SALE_B200_FORMAT_ERROR       (reference throws sale::TensorFileError; the
 *                                    message carries "(offset N)" like its what())
 *   7  SALE_B200_IO_ERROR           (reference throws std::runtime_error: cannot
 *                                    open / write failed)
 *
 * Device data layout (all device pointers, caller-allocated):
 *   q            bf16 [B][N][Hq][128]      rows padded with zeros past head_dim
 *   k, v         bf16 [B][N][Hkv][128]
 *   q_codes      int8 [B][N][Hq][128]      4-bit codes in [-7, 7]
 *   k_codes      int8 [B][N][Hkv][128]
 *   q_scales     f32  [B][Hq][N]           one per token        (quant.hpp:95-104)
 *   k_scales     f32  [B][Hkv][ceil(N/32)] one per key block    (quant.hpp:107-119)
 *   mask_words   u32  [B][Hq][ceil(N/64)][ceil(ceil(N/32)/32)] packed BlockMask
 *                (bit j%32 of word j/32 of row i == BlockMask::get(i, j))
 *   out          bf16 [B][N][Hq][128]
 * Geometry: block_q 64 and block_k 32 (the reference's defaults,
 * selection.hpp:22-23; other block sizes return SALE_B200_UNSUPPORTED) with any
 * valid sink_tokens, local_tokens_min and segment_size (defaults 32 / 128 / 4);
 * Hq a multiple of Hkv (GQA); head_dim <= 128 (the row pitch is always 128).
 *
 * Streams: every call is stream-ordered and asynchronous unless it says
 * otherwise; `stream` is a cudaStream_t (NULL = legacy default stream).
 * A ctx owns workspace (codes, scales, thresholds, the default mask, taus,
 * work-unit tables) shared by its calls: a call issued on a different stream
 * than the previous workspace user first waits (cudaStreamWaitEvent) for that
 * call's work, so calls on several streams are serialized on the device rather
 * than racing. For concurrency, use one ctx per stream. Every entry point runs
 * on the ctx's device and restores the caller's current device.
 */
#ifndef SALE_B200_H
#define SALE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SALE_B200_OK 0
#define SALE_B200_INVALID_ARGUMENT 1
#define SALE_B200_DOMAIN_ERROR 2
#define SALE_B200_OUT_OF_RANGE 3
#define SALE_B200_CUDA_ERROR 4
#define SALE_B200_UNSUPPORTED 5
#define SALE_B200_FORMAT_ERROR 6
#define SALE_B200_IO_ERROR 7

typedef struct sale_b200_ctx sale_b200_ctx;

/* Mirrors sale::SelectionConfig (selection.hpp:18-38) minus the per-head tau. */
typedef struct {
    int64_t sink_tokens;      /* 32  */
    int64_t local_tokens_min; /* 128 */
    int64_t segment_size;     /* 4   */
    int64_t block_q;          /* 64  */
    int64_t block_k;          /* 32  */
} sale_b200_selection_config;

/* Problem shape shared by the stage entry points. head_dim is the logical d
 * (1..128) used for 1/sqrt(d); storage rows are always 128 wide. */
typedef struct {
    int64_t batch;
    int64_t tokens;
    int64_t q_heads;
    int64_t kv_heads;
    int64_t head_dim;
} sale_b200_shape;

/* Optional parity outputs of the Selection-Pass (any pointer may be NULL).
 * running_max / exp_sum / bound: f64 [B][Hq][N] for query blocks with a
 * non-empty middle region (selection.hpp:246-251), untouched elsewhere.
 * block_max: int32 [B][Hq][N][ceil(N/32)], the per-row integer maximum of every
 * estimated middle block (quant.hpp:170-179), untouched elsewhere. */
typedef struct {
    double *running_max;
    double *exp_sum;
    double *bound;
    int32_t *block_max;
} sale_b200_select_debug;

/* ---- context ------------------------------------------------------------ */
int sale_b200_ctx_create(int device, sale_b200_ctx **out);
void sale_b200_ctx_destroy(sale_b200_ctx *ctx);
/* Message of the last failing call on ctx (or of ctx creation when ctx==NULL). */
const char *sale_b200_last_error(const sale_b200_ctx *ctx);
int sale_b200_version(void);
void sale_b200_default_config(sale_b200_selection_config *cfg);

/* ---- stage 1: quantization ----------------------------------------------
 * Replaces quantize_per_token (quant.hpp:95) when group_rows == 1 and
 * quantize_per_key_block (quant.hpp:107) when group_rows == 32, for every
 * (batch, head) of x [B][N][H][128] in one launch. */
int sale_b200_quantize(sale_b200_ctx *ctx, const void *x, int64_t batch, int64_t tokens,
                       int64_t heads, int64_t group_rows, int8_t *codes, float *scales,
                       void *stream);
/* Fused Q (per token) + K (per key block) quantization in ONE launch. */
int sale_b200_quantize_qk(sale_b200_ctx *ctx, const void *q, const void *k,
                          const sale_b200_shape *shape, int8_t *q_codes, float *q_scales,
                          int8_t *k_codes, float *k_scales, void *stream);

/* ---- stage 2: Selection-Pass --------------------------------------------
 * Replaces selection_pass (selection.hpp:211) for every (batch, q head):
 * sink_local_index_set (:92) + compute_sink_local_stats (:129) +
 * threshold_bound (:168) + approx_weight_block / max_then_dequantize
 * (quant.hpp:136-179) + segment_aggregate (:182). taus: HOST array of q_heads
 * doubles (per-head tau, runner.hpp:59-60). */
int sale_b200_select(sale_b200_ctx *ctx, const void *q, const void *k, const int8_t *q_codes,
                     const float *q_scales, const int8_t *k_codes, const float *k_scales,
                     const sale_b200_shape *shape, const double *taus,
                     const sale_b200_selection_config *cfg, uint32_t *mask_words,
                     const sale_b200_select_debug *dbg, void *stream);

/* ---- stage 3: Computation-Pass ------------------------------------------
 * Replaces block_sparse_attention (sparse_attention.hpp:37); with
 * mask_words == NULL it is the all-true mask, i.e. full_attention
 * (attention.hpp:18). coverage (optional): int32 [B][Hq][N] attended tokens per
 * row (SparseAttentionOutput::coverage).
 * A row that attends no token returns SALE_B200_DOMAIN_ERROR naming the first
 * such row, as the reference throws std::domain_error (sparse_attention.hpp:
 * 88-90): with a caller mask the call therefore waits for the kernel
 * (synchronous, like the reference). mask_words == NULL is asynchronous. The
 * prefill entry points never check: the Selection-Pass always keeps the sink
 * block, which every row attends. */
int sale_b200_sparse_attention(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                               const sale_b200_shape *shape, const uint32_t *mask_words,
                               void *out, int32_t *coverage, void *stream);

/* ---- accounting ----------------------------------------------------------
 * Replaces flop_accounting (sparse_attention.hpp:101): counts (device int64
 * [B][Hq][3]) = computed, skipped, total causal blocks per head. */
int sale_b200_flop_count(sale_b200_ctx *ctx, const uint32_t *mask_words, int64_t batch,
                         int64_t q_heads, int64_t tokens, int64_t *counts, void *stream);

/* ---- whole prefill --------------------------------------------------------
 * The run_pipeline stage composition (runner.hpp:63-80) on device buffers:
 * quantize -> select -> sparse attention, with codes / scales / thresholds /
 * mask in ctx-owned workspace. mask_out (optional, device) receives the mask. */
int sale_b200_prefill(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                      const sale_b200_shape *shape, const double *taus,
                      const sale_b200_selection_config *cfg, void *out, uint32_t *mask_out,
                      void *stream);
/* One query-block range [i_lo, i_hi) of sale_b200_prefill (a GPU's share when
 * a (batch, KV group) unit is split across GPUs, K/V replicated; SURVEY.md
 * §8(e)): writes the mask and output rows of the range only. Boundaries must
 * be 0, nq or odd query blocks. The results of the range equal those of the
 * whole-sequence call. */
int sale_b200_prefill_range(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                            const sale_b200_shape *shape, const double *taus,
                            const sale_b200_selection_config *cfg, int64_t i_lo, int64_t i_hi,
                            void *out, uint32_t *mask_out, void *stream);
/* sale_b200_sparse_attention restricted to query blocks [i_lo, i_hi). */
int sale_b200_sparse_attention_range(sale_b200_ctx *ctx, const void *q, const void *k,
                                     const void *v, const sale_b200_shape *shape,
                                     const uint32_t *mask_words, int64_t i_lo, int64_t i_hi,
                                     void *out, int32_t *coverage, void *stream);
/* Same, end to end from HOST buffers (bf16 bit patterns, uint16): H2D copies,
 * the three stages and the D2H copy of out, synchronous on return. */
int sale_b200_prefill_host(sale_b200_ctx *ctx, const uint16_t *q, const uint16_t *k,
                           const uint16_t *v, const sale_b200_shape *shape, const double *taus,
                           const sale_b200_selection_config *cfg, uint16_t *out);

/* ---- orchestration above the stages (runner.hpp, calibrate.hpp) ---------- */

/* l1_error (calibrate.hpp:20-29) for every (batch, q head): sum over tokens and
 * the first head_dim channels of |ref - approx| in double, divided by the
 * token count. ref / approx: device bf16 [B][N][Hq][128] (e.g. the dense and the
 * sparse output). out: HOST double [B*Hq]. Synchronous. */
int sale_b200_l1_error(sale_b200_ctx *ctx, const void *ref, const void *approx,
                       const sale_b200_shape *shape, double *out);

/* One head of a RunReport (report.hpp:12-23). */
typedef struct {
    int64_t head;             /* b * Hq + h */
    double tau;
    double sparsity;          /* skipped / total causal blocks */
    double err;               /* l1_error(dense, sparse) */
    int64_t computed_blocks, skipped_blocks, total_blocks;
    int64_t coverage_min, coverage_max;
    double coverage_mean;
} sale_b200_head_report;
/* StageTiming (report.hpp:26-38), device-event times of the whole batch. */
typedef struct {
    double quantization_ms, selection_ms, computation_ms, dense_ms;
} sale_b200_stage_timing;

/* run_pipeline (runner.hpp:37-108) for every (batch, q head) at once:
 * quantization, selection (or the all-true mask when dense_mask != 0, i.e.
 * RunOptions::dense_mask), block-sparse computation with coverage, the dense
 * baseline, flop accounting, l1 error and coverage statistics. q/k/v device;
 * taus HOST [Hq]; reports HOST [B*Hq]; timing HOST (may be NULL). Synchronous. */
int sale_b200_run_pipeline(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                           const sale_b200_shape *shape, const double *taus,
                           const sale_b200_selection_config *cfg, int dense_mask,
                           sale_b200_head_report *reports, sale_b200_stage_timing *timing);

/* SweepRow (runner.hpp:110-114). */
typedef struct {
    double tau;
    double sparsity; /* mean over all (batch, q head) */
    double err;      /* max over all (batch, q head) */
} sale_b200_sweep_row;
/* sweep_thresholds (runner.hpp:119-165): quantization and the dense baseline
 * once, then per tau (applied to every head) selection + sparse computation +
 * accounting + l1. taus HOST [n_taus] in (0,1); rows HOST [n_taus]. */
int sale_b200_sweep_thresholds(sale_b200_ctx *ctx, const void *q, const void *k, const void *v,
                               const sale_b200_shape *shape, const double *taus, int64_t n_taus,
                               const sale_b200_selection_config *cfg, sale_b200_sweep_row *rows);

/* CalibrationSettings (calibrate.hpp:56-68) minus the selection geometry. */
typedef struct {
    double theta;         /* 0.4   */
    double tau0;          /* 0.008 */
    int64_t max_halvings; /* 30    */
} sale_b200_calibration_settings;
/* HeadCalibration (calibrate.hpp:38-44); flag 0 converged, 1 floor-reached. */
typedef struct {
    int64_t layer, head;
    double tau;
    int32_t flag;
    int64_t halvings;
} sale_b200_head_calibration;
/* calibrate_model (calibrate.hpp:149-175) with calibrate_head's greedy halving
 * ladder (:121-145) for every q head at once: sample s is the device q/k/v
 * triple q_samples[s], k_samples[s], v_samples[s] (batch must be 1; all samples
 * share the shape). Quantization and the dense baseline are computed once per
 * sample; every rung runs selection + sparse computation + l1 for all heads
 * with per-head taus; a head stops at its first tau whose worst-sample error
 * is <= theta. out HOST [Hq] (head = q head index, layer = 0). Synchronous. */
int sale_b200_calibrate(sale_b200_ctx *ctx, const void *const *q_samples,
                        const void *const *k_samples, const void *const *v_samples,
                        int64_t n_samples, const sale_b200_shape *shape,
                        const sale_b200_calibration_settings *settings,
                        const sale_b200_selection_config *cfg, sale_b200_head_calibration *out);

/* ---- file formats (host; docs/formats.md; errors: sale_b200_last_error(NULL)) */

/* .tns header (tensor_file.hpp:98-125): heads, tokens, dim and dtype tag (1 =
 * float32 as in the reference; 2 = bf16, this path's extension). */
int sale_b200_tensor_file_info(const char *path, uint32_t *heads, uint32_t *tokens,
                               uint32_t *dim, uint32_t *dtype);
/* read_tensor_file (tensor_file.hpp:98-158) into this path's layout: HOST bf16
 * [1][N][heads][128] q, k, v (RNE from float32, rows zero-padded past dim),
 * i.e. an MHA shape (kv_heads = q_heads). Same validation and error offsets as
 * the reference (magic, version, dtype, zero counts, truncation, non-finite
 * values, trailing bytes). */
int sale_b200_tensor_file_read_bf16(const char *path, uint16_t *q, uint16_t *k, uint16_t *v);
/* write_tensor_file (tensor_file.hpp:69-96) from HOST bf16 [1][N][heads][128]:
 * dtype 1 writes the bf16 values as float32 (byte-identical to the reference
 * writer for bf16-valued inputs), dtype 2 writes bf16 payloads. */
int sale_b200_tensor_file_write(const char *path, const uint16_t *q, const uint16_t *k,
                                const uint16_t *v, uint32_t heads, uint32_t tokens, uint32_t dim,
                                uint32_t dtype);
/* write_mask_dump (mask_io.hpp:28-69) from packed HOST mask words
 * [B][Hq][ceil(N/64)][W]: one RLE record per (batch, head), head index
 * b * Hq + h, tau taus[b * Hq + h] (float32). Byte-identical to the reference. */
int sale_b200_mask_dump_write(const char *path, const uint32_t *mask_words, int64_t batch,
                              int64_t heads, int64_t tokens, const float *taus);
/* read_mask_dump (mask_io.hpp:71-125) back into packed HOST words: first call
 * with mask_words == NULL to get the record count and the grid (all records
 * must share nq / nk); heads / taus receive each record's head index and tau. */
int sale_b200_mask_dump_read(const char *path, int64_t *records, int64_t *nq, int64_t *nk,
                             uint32_t *mask_words, uint32_t *heads, float *taus);

/* ---- device memory helpers (so host code needs no CUDA headers) -----------
 * Synchronous allocation / copies on ctx's device. */
int sale_b200_device_alloc(sale_b200_ctx *ctx, uint64_t bytes, void **out);
int sale_b200_device_free(sale_b200_ctx *ctx, void *ptr);
int sale_b200_copy_to_device(sale_b200_ctx *ctx, void *dst, const void *src, uint64_t bytes);
int sale_b200_copy_to_host(sale_b200_ctx *ctx, void *dst, const void *src, uint64_t bytes);
int sale_b200_memset(sale_b200_ctx *ctx, void *dst, int value, uint64_t bytes);
int sale_b200_synchronize(sale_b200_ctx *ctx);

/* ---- instrumentation -----------------------------------------------------
 * With timing enabled, sale_b200_prefill records CUDA events on its stream
 * between kernels; sale_b200_stage_times waits for the last one and returns
 * ms[5] = quantize, base mask, sink-local stats, estimator, attention. */
int sale_b200_set_timing(sale_b200_ctx *ctx, int enable);
/* Estimator wait-time counters (cycles, summed over CTAs): counters[8] =
 * MMA-issuer loop, A wait, K-stage waits, accumulator waits, stages,
 * epilogue loop (warp 4), epilogue accumulator waits, 0; then counters[8..15]
 * = sink-local-stats phase cycles (staging, dots, logit store, block max,
 * running max, exp sums, combine) and the CTA count. Reads and resets;
 * enable != 0 turns collection on for later launches. counters may be NULL
 * (then it must hold 16 entries otherwise). */
int sale_b200_estimator_profile(sale_b200_ctx *ctx, int enable, uint64_t *counters);

/* Diagnostics: cycle counters of the attention kernel (16 entries): softmax
 * loop, S-ready waits, softmax compute, tiles (one softmax warp, summed over
 * CTAs); MMA loop, K / P / V waits, CTAs; [10] epilogue. Reads and resets;
 * enable != 0 turns collection on for later launches. */
int sale_b200_attention_profile(sale_b200_ctx *ctx, int enable, uint64_t *counters);
int sale_b200_stage_times(sale_b200_ctx *ctx, float *ms);

/* ---- synthetic workload (host, not the hot path) --------------------------
 * workloads.hpp:125-159 sink_local_head / :104-112 gaussian_head for one head
 * (kind 0 gaussian, 1 sink_local), fp32 [n][d] each, bit-identical to the
 * reference generator. */
int sale_b200_workload_head_f32(int kind, uint64_t seed, int64_t n, int64_t d, int64_t head,
                                float *q, float *k, float *v);
/* GQA extension written as bf16 [B][N][H][128] host arrays
 * (rows zero-padded past d): KV head g of batch b is the reference head g of
 * seed+b; query head r>0 of the group adds fresh N(0,1) noise to the same
 * planted terms. threads <= 0 means all cores. */
int sale_b200_workload_gqa_bf16(int kind, uint64_t seed, const sale_b200_shape *shape,
                                uint16_t *q, uint16_t *k, uint16_t *v, int threads);
/* Same for the KV heads [kv_begin, kv_begin + shape->kv_heads) of a model with
 * `total_kv_heads` KV heads (and their q heads): one rank's shard. */
int sale_b200_workload_gqa_shard_bf16(int kind, uint64_t seed, const sale_b200_shape *shape,
                                      int64_t kv_begin, uint16_t *q, uint16_t *k, uint16_t *v,
                                      int threads);

#ifdef __cplusplus
}
#endif

#endif /* SALE_B200_H */
