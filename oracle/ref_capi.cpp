// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper over the UNMODIFIED reference headers
// (/root/reference/proj/include/sale/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libsale_ref.so. Nothing here re-implements an algorithm: every
// entry point converts flat buffers into the reference's own types and calls
// the reference function named in its comment. Used to pin oracle/sale_oracle.c
// and as the reference CPU arm of bench.py (--impl reference / cpu_baseline).
#include <sale/attention.hpp>
#include <sale/block_grid.hpp>
#include <sale/calibrate.hpp>
#include <sale/mask_io.hpp>
#include <sale/tensor_file.hpp>
#include <sale/quant.hpp>
#include <sale/runner.hpp>
#include <sale/selection.hpp>
#include <sale/sparse_attention.hpp>
#include <sale/workloads.hpp>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

using namespace sale;

namespace {

DenseMatrix to_matrix(const float *p, int64_t rows, int64_t cols) {
    DenseMatrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
    std::memcpy(m.data().data(), p, sizeof(float) * static_cast<std::size_t>(rows * cols));
    return m;
}

HeadInput to_head(const float *q, const float *k, const float *v, int64_t n, int64_t d) {
    return HeadInput{to_matrix(q, n, d), to_matrix(k, n, d),
                     v ? to_matrix(v, n, d) : DenseMatrix(static_cast<std::size_t>(n),
                                                          static_cast<std::size_t>(d))};
}

SelectionConfig to_config(double tau, int64_t sink, int64_t local, int64_t seg, int64_t bq,
                          int64_t bk) {
    SelectionConfig c;
    c.tau = tau;
    c.sink_tokens = static_cast<std::size_t>(sink);
    c.local_tokens_min = static_cast<std::size_t>(local);
    c.segment_size = static_cast<std::size_t>(seg);
    c.block_q = static_cast<std::size_t>(bq);
    c.block_k = static_cast<std::size_t>(bk);
    return c;
}

template <typename F> int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument &) {
        return 1;
    } catch (const std::domain_error &) {
        return 2;
    } catch (const std::out_of_range &) {
        return 3;
    } catch (...) {
        return 9;
    }
}

void export_quant(const QuantizedMatrix &q, int8_t *codes, float *scales) {
    for (std::size_t r = 0; r < q.rows(); ++r)
        for (std::size_t c = 0; c < q.cols(); ++c) codes[r * q.cols() + c] = q.code(r, c);
    for (std::size_t g = 0; g < q.num_groups(); ++g) scales[g] = q.group_scale(g);
}

QuantizedMatrix import_quant(const int8_t *codes, const float *scales, int64_t rows, int64_t cols,
                             ScaleGrouping grouping, int64_t group_rows) {
    QuantizedMatrix q(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols), grouping,
                      static_cast<std::size_t>(group_rows));
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) q.code(r, c) = codes[r * cols + c];
    for (std::size_t g = 0; g < q.num_groups(); ++g) q.group_scale(g) = scales[g];
    return q;
}

} // namespace

extern "C" {

// quant.hpp:95 quantize_per_token
int ref_quantize_per_token(const float *x, int64_t rows, int64_t cols, int8_t *codes,
                           float *scales) {
    return guarded([&] { export_quant(quantize_per_token(to_matrix(x, rows, cols)), codes, scales); });
}

// quant.hpp:107 quantize_per_key_block
int ref_quantize_per_key_block(const float *x, int64_t rows, int64_t cols, int64_t block_q,
                               int64_t block_k, int8_t *codes, float *scales) {
    return guarded([&] {
        const BlockGrid grid(static_cast<std::size_t>(rows), static_cast<std::size_t>(block_q),
                             static_cast<std::size_t>(block_k));
        export_quant(quantize_per_key_block(to_matrix(x, rows, cols), grid), codes, scales);
    });
}

// selection.hpp:92 sink_local_index_set; returns count or -status
int64_t ref_sink_local_index_set(int64_t i, int64_t tokens, int64_t sink, int64_t local,
                                 int64_t seg, int64_t bq, int64_t bk, int64_t *out) {
    int64_t n = 0;
    const int st = guarded([&] {
        const BlockGrid grid(static_cast<std::size_t>(tokens), static_cast<std::size_t>(bq),
                             static_cast<std::size_t>(bk));
        const auto set = sink_local_index_set(static_cast<std::size_t>(i), grid,
                                              to_config(0.004, sink, local, seg, bq, bk));
        for (std::size_t j : set) out[n++] = static_cast<int64_t>(j);
    });
    return st ? -st : n;
}

// selection.hpp:129 compute_sink_local_stats
int ref_sink_local_stats(const float *q, const float *k, int64_t n, int64_t d, int64_t bq,
                         int64_t bk, int64_t i, const int64_t *blocks, int64_t nblocks,
                         double *m, double *l) {
    return guarded([&] {
        const HeadInput in = to_head(q, k, nullptr, n, d);
        const BlockGrid grid(static_cast<std::size_t>(n), static_cast<std::size_t>(bq),
                             static_cast<std::size_t>(bk));
        std::vector<std::size_t> bl(blocks, blocks + nblocks);
        const SinkLocalStats s = compute_sink_local_stats(in, static_cast<std::size_t>(i), bl, grid);
        for (std::size_t r = 0; r < s.running_max.size(); ++r) {
            m[r] = s.running_max[r];
            l[r] = s.exp_sum[r];
        }
    });
}

// selection.hpp:168 threshold_bound
double ref_threshold_bound(double tau, double m, double l) { return threshold_bound(tau, m, l); }

// selection.hpp:211 selection_pass; mask uint8 [nq][nk]
int ref_selection_pass(const float *q, const float *k, int64_t n, int64_t d, const int8_t *qcodes,
                       const float *qscales, const int8_t *kcodes, const float *kscales,
                       double tau, int64_t sink, int64_t local, int64_t seg, int64_t bq,
                       int64_t bk, uint8_t *mask) {
    return guarded([&] {
        const HeadInput in = to_head(q, k, nullptr, n, d);
        const SelectionConfig cfg = to_config(tau, sink, local, seg, bq, bk);
        const QuantizedMatrix q4 = import_quant(qcodes, qscales, n, d, ScaleGrouping::PerToken, 1);
        const QuantizedMatrix k4 =
            import_quant(kcodes, kscales, n, d, ScaleGrouping::PerKeyBlock, bk);
        const BlockMask m = selection_pass(in, q4, k4, cfg);
        for (std::size_t i = 0; i < m.query_blocks(); ++i)
            for (std::size_t j = 0; j < m.key_blocks(); ++j)
                mask[i * m.key_blocks() + j] = m.get(i, j) ? 1 : 0;
    });
}

// sparse_attention.hpp:37 block_sparse_attention
int ref_block_sparse_attention(const float *q, const float *k, const float *v, int64_t n,
                               int64_t d, const uint8_t *mask, int64_t bq, int64_t bk, float *out,
                               int64_t *coverage) {
    return guarded([&] {
        const HeadInput in = to_head(q, k, v, n, d);
        const BlockGrid grid(static_cast<std::size_t>(n), static_cast<std::size_t>(bq),
                             static_cast<std::size_t>(bk));
        BlockMask m(grid.num_query_blocks(), grid.num_key_blocks());
        for (std::size_t i = 0; i < m.query_blocks(); ++i)
            for (std::size_t j = 0; j < m.key_blocks(); ++j)
                m.set(i, j, mask[i * m.key_blocks() + j] != 0);
        const SparseAttentionOutput o = block_sparse_attention(in, m, grid);
        std::memcpy(out, o.output.data().data(), sizeof(float) * static_cast<std::size_t>(n * d));
        if (coverage)
            for (int64_t r = 0; r < n; ++r) coverage[r] = static_cast<int64_t>(o.coverage[r]);
    });
}

// attention.hpp:18 full_attention
int ref_full_attention(const float *q, const float *k, const float *v, int64_t n, int64_t d,
                       float *out) {
    return guarded([&] {
        const DenseMatrix o = full_attention(to_head(q, k, v, n, d));
        std::memcpy(out, o.data().data(), sizeof(float) * static_cast<std::size_t>(n * d));
    });
}

// sparse_attention.hpp:101 flop_accounting
int ref_flop_accounting(const uint8_t *mask, int64_t n, int64_t bq, int64_t bk, int64_t *counts) {
    return guarded([&] {
        const BlockGrid grid(static_cast<std::size_t>(n), static_cast<std::size_t>(bq),
                             static_cast<std::size_t>(bk));
        BlockMask m(grid.num_query_blocks(), grid.num_key_blocks());
        for (std::size_t i = 0; i < m.query_blocks(); ++i)
            for (std::size_t j = 0; j < m.key_blocks(); ++j)
                m.set(i, j, mask[i * m.key_blocks() + j] != 0);
        const FlopCounts c = flop_accounting(m, grid);
        counts[0] = static_cast<int64_t>(c.computed_blocks);
        counts[1] = static_cast<int64_t>(c.skipped_blocks);
        counts[2] = static_cast<int64_t>(c.total_blocks);
    });
}

// workloads.hpp:125 sink_local_head / :161 needle_head / gaussian_head via the
// public generators. kind: 0 gaussian, 1 sink_local. Writes q,k,v [n][d].
int ref_workload_head(int kind, uint64_t seed, int64_t n, int64_t d, int64_t head, float *q,
                      float *k, float *v) {
    return guarded([&] {
        WorkloadSpec spec;
        spec.seed = seed;
        spec.tokens = static_cast<std::size_t>(n);
        spec.head_dim = static_cast<std::size_t>(d);
        spec.heads = static_cast<std::size_t>(head + 1);
        spec.kind = kind == 0 ? WorkloadKind::Gaussian : WorkloadKind::SinkLocal;
        spec.validate();
        const HeadInput h = kind == 0 ? detail::gaussian_head(spec, static_cast<std::size_t>(head))
                                      : detail::sink_local_head(spec, static_cast<std::size_t>(head));
        const std::size_t bytes = sizeof(float) * static_cast<std::size_t>(n * d);
        std::memcpy(q, h.query.data().data(), bytes);
        std::memcpy(k, h.key.data().data(), bytes);
        std::memcpy(v, h.value.data().data(), bytes);
    });
}

// The GQA extension of sink_local_head / gaussian_head (the
// product's generator is paper_2505_24179_b200/csrc/workload.cpp, pinned to
// this one by tests/test_abi.py) built from the reference's own Rng,
// head_rng, fill_normal, random_unit and generators (workloads.hpp:17-159):
// KV group g = reference head g (its K, V and, for r = 0, its Q); query head
// r > 0 of the group = fresh N(0,1) noise from the reference Rng seeded
// seed + kQStream * r (head_rng of head g) plus the same planted terms. Output
// per Q head h (K / V of its group replicated): [q_heads][n][d] fp32, rounded
// to bf16 (RNE) when round_bf16 — the values the B200 path receives. Batch 0.
// Lets bench.py's reference arm build its inputs without the product library.
int ref_workload_gqa_heads(int kind, uint64_t seed, int64_t n, int64_t d, int64_t q_heads,
                           int64_t kv_heads, int round_bf16, int64_t threads, float *q, float *k,
                           float *v) {
    constexpr std::uint64_t kQStream = 0xD1B54A32D192ED03ULL;
    return guarded([&] {
        if (q_heads % kv_heads) throw std::invalid_argument("q_heads % kv_heads");
        const int64_t G = q_heads / kv_heads;
        const std::size_t nd = static_cast<std::size_t>(n * d);
        auto bf16 = [&](float x) {
            if (!round_bf16) return x;
            std::uint32_t u;
            std::memcpy(&u, &x, 4);
            u += 0x7FFFu + ((u >> 16) & 1u);
            u &= 0xFFFF0000u;
            float y;
            std::memcpy(&y, &u, 4);
            return y;
        };
        parallel_for(static_cast<std::size_t>(q_heads), static_cast<std::size_t>(threads),
                     [&](std::size_t h) {
            const std::size_t g = h / G, r = h % G;
            WorkloadSpec spec;
            spec.seed = seed;
            spec.tokens = static_cast<std::size_t>(n);
            spec.head_dim = static_cast<std::size_t>(d);
            spec.heads = g + 1;
            spec.kind = kind == 0 ? WorkloadKind::Gaussian : WorkloadKind::SinkLocal;
            const HeadInput base = kind == 0 ? detail::gaussian_head(spec, g)
                                             : detail::sink_local_head(spec, g);
            DenseMatrix qr = base.query;
            if (r > 0) {
                WorkloadSpec s2 = spec;
                s2.seed = seed + kQStream * r;
                Rng noise = detail::head_rng(s2, g);
                detail::fill_normal(noise, qr);
                if (kind == 1) { // the planted query terms of head g (workloads.hpp:128-158)
                    Rng rng = detail::head_rng(spec, g);
                    for (std::size_t t = 0; t < 3 * nd; ++t) (void)rng.next_normal();
                    const double sqrt_d = std::sqrt(static_cast<double>(d));
                    const double sink_amp = std::sqrt(std::max(spec.sink_logit, 0.0) * sqrt_d);
                    const double local_amp = std::sqrt(std::max(spec.local_logit, 0.0) * sqrt_d);
                    const double rho = std::exp(-1.0 / spec.local_decay_tokens);
                    const double drift = std::sqrt(1.0 - rho * rho);
                    const std::vector<double> sink_dir = detail::random_unit(rng, d);
                    std::vector<double> local_dir = detail::random_unit(rng, d);
                    for (int64_t i = 0; i < n; ++i) {
                        if (i > 0) {
                            double norm2 = 0.0;
                            for (int64_t c = 0; c < d; ++c) {
                                local_dir[c] = rho * local_dir[c] + drift * rng.next_normal() / sqrt_d;
                                norm2 += local_dir[c] * local_dir[c];
                            }
                            const double inv = 1.0 / std::sqrt(norm2 > 0.0 ? norm2 : 1.0);
                            for (auto &x : local_dir) x *= inv;
                        }
                        for (int64_t c = 0; c < d; ++c)
                            qr(i, c) += static_cast<float>(sink_amp * sink_dir[c] + local_amp * local_dir[c]);
                    }
                }
            }
            for (std::size_t e = 0; e < nd; ++e) {
                q[h * nd + e] = bf16(qr.data()[e]);
                k[h * nd + e] = bf16(base.key.data()[e]);
                v[h * nd + e] = bf16(base.value.data()[e]);
            }
        });
    });
}

// runner.hpp:37 run_pipeline over `heads` heads laid out [h][n][d]; one tau for
// every head. Returns the wall time of the call in ms through *wall_ms and the
// summed stage fields (quant, select, compute, dense) in stage_ms[4];
// sparsity per head in sparsity[h]. dense_mask / skip_dense as in RunOptions.
int ref_run_pipeline(const float *q, const float *k, const float *v, int64_t heads, int64_t n,
                     int64_t d, double tau, int64_t threads, double *wall_ms, double *stage_ms,
                     double *sparsity) {
    return guarded([&] {
        std::vector<HeadInput> hs;
        hs.reserve(static_cast<std::size_t>(heads));
        for (int64_t h = 0; h < heads; ++h)
            hs.push_back(to_head(q + h * n * d, k + h * n * d, v + h * n * d, n, d));
        const std::vector<double> taus(static_cast<std::size_t>(heads), tau);
        SelectionConfig cfg;
        RunOptions opt;
        opt.threads = static_cast<std::size_t>(threads);
        const auto t0 = std::chrono::steady_clock::now();
        const RunReport r = run_pipeline(hs, taus, cfg, opt);
        *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count();
        stage_ms[0] = r.timing.quantization_ms;
        stage_ms[1] = r.timing.selection_ms;
        stage_ms[2] = r.timing.computation_ms;
        stage_ms[3] = r.timing.dense_ms;
        for (int64_t h = 0; h < heads; ++h) sparsity[h] = r.head_reports[h].sparsity;
    });
}

// The reference's own parallel_for (parallel.hpp:15) over the hot-path stages
// WITHOUT the dense baseline: quant -> selection_pass -> block_sparse_attention
// for each head (runner.hpp:63-80), threads workers. Wall ms via *wall_ms.
// stage_ms[3] receives the per-stage thread-time summed over heads (quant,
// selection, computation), like runner.hpp:101-106.
int ref_sale_heads(const float *q, const float *k, const float *v, int64_t heads, int64_t n,
                   int64_t d, double tau, int64_t threads, double *wall_ms, double *stage_ms) {
    return guarded([&] {
        std::vector<HeadInput> hs;
        hs.reserve(static_cast<std::size_t>(heads));
        for (int64_t h = 0; h < heads; ++h)
            hs.push_back(to_head(q + h * n * d, k + h * n * d, v + h * n * d, n, d));
        SelectionConfig cfg;
        cfg.tau = tau;
        std::vector<double> st(static_cast<std::size_t>(3 * heads), 0.0);
        using clk = std::chrono::steady_clock;
        auto ms = [](clk::time_point a) {
            return std::chrono::duration<double, std::milli>(clk::now() - a).count();
        };
        const auto t0 = clk::now();
        parallel_for(hs.size(), static_cast<std::size_t>(threads), [&](std::size_t h) {
            const BlockGrid grid(hs[h].seq_len(), cfg.block_q, cfg.block_k);
            auto t = clk::now();
            const QuantizedMatrix q4 = quantize_per_token(hs[h].query);
            const QuantizedMatrix k4 = quantize_per_key_block(hs[h].key, grid);
            st[3 * h] = ms(t);
            t = clk::now();
            const BlockMask mask = selection_pass(hs[h], q4, k4, cfg);
            st[3 * h + 1] = ms(t);
            t = clk::now();
            (void)block_sparse_attention(hs[h], mask, grid);
            st[3 * h + 2] = ms(t);
        });
        *wall_ms = ms(t0);
        for (int i = 0; i < 3; ++i) {
            stage_ms[i] = 0.0;
            for (int64_t h = 0; h < heads; ++h) stage_ms[i] += st[3 * h + i];
        }
    });
}

// run_pipeline (runner.hpp:37) with per-head taus; every HeadReport field
// (report.hpp:12-23) as doubles: out[h*10 + {0 sparsity, 1 err, 2 computed,
// 3 skipped, 4 total, 5 cov_min, 6 cov_max, 7 cov_mean}].
int ref_run_report(const float *q, const float *k, const float *v, int64_t heads, int64_t n,
                   int64_t d, const double *taus, int dense_mask, int64_t threads, double *out) {
    return guarded([&] {
        std::vector<HeadInput> hs;
        for (int64_t h = 0; h < heads; ++h)
            hs.push_back(to_head(q + h * n * d, k + h * n * d, v + h * n * d, n, d));
        const std::vector<double> tv(taus, taus + heads);
        RunOptions opt;
        opt.threads = static_cast<std::size_t>(threads);
        opt.dense_mask = dense_mask != 0;
        const RunReport r = run_pipeline(hs, tv, SelectionConfig{}, opt);
        for (int64_t h = 0; h < heads; ++h) {
            const HeadReport &x = r.head_reports[h];
            double *o = out + 10 * h;
            o[0] = x.sparsity, o[1] = x.err, o[2] = double(x.computed_blocks),
            o[3] = double(x.skipped_blocks), o[4] = double(x.total_blocks);
            o[5] = double(x.coverage_min), o[6] = double(x.coverage_max), o[7] = x.coverage_mean;
        }
    });
}

// sweep_thresholds (runner.hpp:119): rows[t*3 + {tau, sparsity, err}].
int ref_sweep(const float *q, const float *k, const float *v, int64_t heads, int64_t n, int64_t d,
              const double *taus, int64_t n_taus, int64_t threads, double *rows) {
    return guarded([&] {
        std::vector<HeadInput> hs;
        for (int64_t h = 0; h < heads; ++h)
            hs.push_back(to_head(q + h * n * d, k + h * n * d, v + h * n * d, n, d));
        const std::vector<double> tv(taus, taus + n_taus);
        const auto r = sweep_thresholds(hs, tv, SelectionConfig{}, static_cast<std::size_t>(threads));
        for (int64_t t = 0; t < n_taus; ++t) {
            rows[3 * t] = r[t].tau, rows[3 * t + 1] = r[t].sparsity, rows[3 * t + 2] = r[t].err;
        }
    });
}

// calibrate_head (calibrate.hpp:121) over samples laid out [s][n][d].
int ref_calibrate_head(const float *q, const float *k, const float *v, int64_t samples, int64_t n,
                       int64_t d, double theta, double tau0, int64_t max_halvings, double *tau,
                       int32_t *flag, int64_t *halvings) {
    return guarded([&] {
        std::vector<HeadInput> hs;
        for (int64_t s = 0; s < samples; ++s)
            hs.push_back(to_head(q + s * n * d, k + s * n * d, v + s * n * d, n, d));
        CalibrationSettings st;
        st.theta = theta;
        st.tau0 = tau0;
        st.max_halvings = static_cast<std::size_t>(max_halvings);
        const HeadCalibration c = calibrate_head(hs, st);
        *tau = c.tau;
        *flag = c.flag == CalibrationFlag::Converged ? 0 : 1;
        *halvings = static_cast<int64_t>(c.halvings);
    });
}

// write_tensor_file (tensor_file.hpp:69), heads laid out [h][n][d].
int ref_write_tensor_file(const char *path, const float *q, const float *k, const float *v,
                          int64_t heads, int64_t n, int64_t d) {
    return guarded([&] {
        std::vector<HeadInput> hs;
        for (int64_t h = 0; h < heads; ++h)
            hs.push_back(to_head(q + h * n * d, k + h * n * d, v + h * n * d, n, d));
        write_tensor_file(path, hs);
    });
}

// read_tensor_file (tensor_file.hpp:98): 0 and the values ([h][n][d] q, k, v)
// or 6 with the TensorFileError what() in msg.
int ref_read_tensor_file(const char *path, float *q, float *k, float *v, char *msg, int64_t cap) {
    try {
        const auto hs = read_tensor_file(path);
        const std::size_t nd = hs.front().query.data().size();
        for (std::size_t h = 0; h < hs.size(); ++h) {
            std::memcpy(q + h * nd, hs[h].query.data().data(), 4 * nd);
            std::memcpy(k + h * nd, hs[h].key.data().data(), 4 * nd);
            std::memcpy(v + h * nd, hs[h].value.data().data(), 4 * nd);
        }
        return 0;
    } catch (const TensorFileError &e) {
        std::snprintf(msg, static_cast<std::size_t>(cap), "%s", e.what());
        return 6;
    } catch (const std::exception &e) {
        std::snprintf(msg, static_cast<std::size_t>(cap), "%s", e.what());
        return 7;
    }
}

// write_mask_dump (mask_io.hpp:28) from uint8 cells [r][nq][nk].
int ref_write_mask_dump(const char *path, const uint8_t *cells, const uint32_t *heads,
                        const float *taus, int64_t records, int64_t nq, int64_t nk) {
    return guarded([&] {
        std::vector<MaskRecord> recs(static_cast<std::size_t>(records));
        for (int64_t r = 0; r < records; ++r) {
            recs[r].head = heads[r];
            recs[r].tau = taus[r];
            recs[r].mask = BlockMask(static_cast<std::size_t>(nq), static_cast<std::size_t>(nk));
            for (int64_t i = 0; i < nq; ++i)
                for (int64_t j = 0; j < nk; ++j)
                    if (cells[(r * nq + i) * nk + j]) recs[r].mask.set(i, j, true);
        }
        write_mask_dump(path, recs);
    });
}

} // extern "C"
