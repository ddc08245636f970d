// workload.cpp — host-side synthetic inputs (measurement harness, not the hot
// path). Restates the reference generator (workloads.hpp:17-159): splitmix64 +
// Box-Muller streams, Gaussian base, planted sink direction and AR(1)-drifting
// local direction. Compiled with -ffp-contract=off so every double/float
// operation rounds exactly like the reference build; tests pin the output
// bit-for-bit against the reference compiled in oracle/_ref.
//
// splitmix64's state after n draws is seed + n * gamma, so any position of a
// stream can be reached in O(1): the Gaussian base is generated in parallel
// row chunks, and only the d-wide AR(1) recurrence runs sequentially.
#include "sale_b200.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kQStream = 0xD1B54A32D192ED03ULL; // GQA extension: extra query heads

struct Rng { // workloads.hpp:19-42
    uint64_t state;
    explicit Rng(uint64_t s) : state(s) {}
    void skip_normals(uint64_t n) { state += kGamma * (2 * n); }
    uint64_t next_u64() {
        state += kGamma;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double next_uniform() { return (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53; }
    double next_normal() {
        const double u1 = next_uniform();
        const double u2 = next_uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
    }
};

uint64_t head_seed(uint64_t seed, int64_t head) { // workloads.hpp:85-87
    return seed + kGamma * static_cast<uint64_t>(head + 1);
}

std::vector<double> random_unit(Rng &rng, int64_t d) { // workloads.hpp:95-106
    std::vector<double> v(static_cast<size_t>(d));
    double norm2 = 0.0;
    for (auto &x : v) {
        x = rng.next_normal();
        norm2 += x * x;
    }
    const double inv = 1.0 / std::sqrt(norm2 > 0.0 ? norm2 : 1.0);
    for (auto &x : v) x *= inv;
    return v;
}

// Planted terms of one reference head (workloads.hpp:128-158), as the float
// increments the reference adds: pq[i][c] to the query, pk[i][c] to the key,
// pk0[c] additionally to key 0.
struct Planted {
    std::vector<float> pq, pk, pk0;
};

Planted planted_terms(uint64_t seed, int64_t head, int64_t n, int64_t d) {
    const double sink_logit = 14.0, local_logit = 10.0, decay = 64.0; // workloads.hpp:57-59
    Rng rng(head_seed(seed, head));
    rng.skip_normals(static_cast<uint64_t>(3 * n * d)); // Q, K, V Gaussian base
    const double sqrt_d = std::sqrt(static_cast<double>(d));
    const double sink_amp = std::sqrt(std::max(sink_logit, 0.0) * sqrt_d);
    const double local_amp = std::sqrt(std::max(local_logit, 0.0) * sqrt_d);
    const double rho = std::exp(-1.0 / decay);
    const double drift = std::sqrt(1.0 - rho * rho);
    const std::vector<double> sink_dir = random_unit(rng, d);
    std::vector<double> local_dir = random_unit(rng, d);
    Planted p;
    p.pq.resize(static_cast<size_t>(n * d));
    p.pk.resize(static_cast<size_t>(n * d));
    p.pk0.resize(static_cast<size_t>(d));
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
        for (int64_t c = 0; c < d; ++c) {
            const double planted = sink_amp * sink_dir[c] + local_amp * local_dir[c];
            p.pq[i * d + c] = static_cast<float>(planted);
            p.pk[i * d + c] = static_cast<float>(local_amp * local_dir[c]);
            if (i == 0) p.pk0[c] = static_cast<float>(sink_amp * sink_dir[c]);
        }
    }
    return p;
}

uint16_t f32_to_bf16(float f) { // round to nearest even (finite inputs)
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

enum Which { kQ = 0, kK = 1, kV = 2 };

// rows [r0, r1) of one tensor: Gaussian base from `stream` starting at normal
// `offset`, plus planted terms. Writes either fp32 (dst32, pitch d) or bf16
// (dst16 with row stride `pitch16`, zero-padded to 128).
void fill_rows(uint64_t stream, uint64_t offset, int64_t r0, int64_t r1, int64_t d, Which which,
               const Planted *pl, float *dst32, uint16_t *dst16, int64_t pitch16) {
    Rng rng(stream);
    rng.skip_normals(offset + static_cast<uint64_t>(r0 * d));
    for (int64_t i = r0; i < r1; ++i) {
        for (int64_t c = 0; c < d; ++c) {
            float x = static_cast<float>(rng.next_normal());
            if (pl) {
                if (which == kQ) x += pl->pq[i * d + c];
                if (which == kK) {
                    x += pl->pk[i * d + c];
                    if (i == 0) x += pl->pk0[c];
                }
            }
            if (dst32) dst32[i * d + c] = x;
            if (dst16) dst16[i * pitch16 + c] = f32_to_bf16(x);
        }
        if (dst16)
            for (int64_t c = d; c < 128; ++c) dst16[i * pitch16 + c] = 0;
    }
}

template <typename F> void parallel(int64_t n, int threads, F &&f) {
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    threads = static_cast<int>(std::min<int64_t>(threads, std::max<int64_t>(n, 1)));
    std::vector<std::thread> pool;
    std::atomic_int64_t next{0};
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&] {
            for (int64_t i; (i = next.fetch_add(1)) < n;) f(i);
        });
    for (auto &t : pool) t.join();
}

} // namespace

extern "C" {

int sale_b200_workload_head_f32(int kind, uint64_t seed, int64_t n, int64_t d, int64_t head,
                                float *q, float *k, float *v) {
    if (n < 1 || d < 1 || head < 0 || !q || !k || !v) return SALE_B200_INVALID_ARGUMENT;
    if (kind != 0 && kind != 1) return SALE_B200_INVALID_ARGUMENT;
    Planted pl;
    if (kind == 1) pl = planted_terms(seed, head, n, d);
    const uint64_t s = head_seed(seed, head);
    const uint64_t nd = static_cast<uint64_t>(n * d);
    fill_rows(s, 0, 0, n, d, kQ, kind ? &pl : nullptr, q, nullptr, 0);
    fill_rows(s, nd, 0, n, d, kK, kind ? &pl : nullptr, k, nullptr, 0);
    fill_rows(s, 2 * nd, 0, n, d, kV, nullptr, v, nullptr, 0);
    return SALE_B200_OK;
}

int sale_b200_workload_gqa_bf16(int kind, uint64_t seed, const sale_b200_shape *shape, uint16_t *q,
                                uint16_t *k, uint16_t *v, int threads) {
    return sale_b200_workload_gqa_shard_bf16(kind, seed, shape, 0, q, k, v, threads);
}

int sale_b200_workload_gqa_shard_bf16(int kind, uint64_t seed, const sale_b200_shape *shape,
                                      int64_t kv_begin, uint16_t *q, uint16_t *k, uint16_t *v,
                                      int threads) {
    if (!shape || !q || !k || !v || kv_begin < 0) return SALE_B200_INVALID_ARGUMENT;
    const int64_t B = shape->batch, N = shape->tokens, Hq = shape->q_heads, Hkv = shape->kv_heads,
                  d = shape->head_dim;
    if (B < 1 || N < 1 || Hq < 1 || Hkv < 1 || d < 1 || d > 128 || Hq % Hkv)
        return SALE_B200_INVALID_ARGUMENT;
    if (kind != 0 && kind != 1) return SALE_B200_INVALID_ARGUMENT;
    const int64_t G = Hq / Hkv;
    // phase 1: planted terms per (batch, kv head) — the sequential recurrence
    std::vector<Planted> planted(static_cast<size_t>(B * Hkv));
    if (kind == 1)
        parallel(B * Hkv, threads, [&](int64_t t) {
            planted[t] = planted_terms(seed + static_cast<uint64_t>(t / Hkv), kv_begin + t % Hkv, N, d);
        });
    // phase 2: Gaussian base + planted, in row chunks
    const int64_t chunk = 4096;
    const int64_t nchunks = (N + chunk - 1) / chunk;
    const int64_t tensors = Hq + 2 * Hkv; // per batch
    const uint64_t nd = static_cast<uint64_t>(N * d);
    parallel(B * tensors * nchunks, threads, [&](int64_t t) {
        const int64_t ch = t % nchunks;
        const int64_t x = (t / nchunks) % tensors;
        const int64_t b = t / (nchunks * tensors);
        const int64_t r0 = ch * chunk, r1 = std::min(N, r0 + chunk);
        const uint64_t sb = seed + static_cast<uint64_t>(b);
        if (x < Hq) {
            const int64_t g = x / G, r = x % G;
            const Planted *pl = kind == 1 ? &planted[b * Hkv + g] : nullptr;
            const uint64_t hs = head_seed(sb, kv_begin + g);
            const uint64_t stream = r == 0 ? hs : hs + kQStream * static_cast<uint64_t>(r);
            fill_rows(stream, 0, r0, r1, d, kQ, pl, nullptr, q + ((b * N) * Hq + x) * 128, Hq * 128);
        } else {
            const bool is_k = x < Hq + Hkv;
            const int64_t g = is_k ? x - Hq : x - Hq - Hkv;
            const Planted *pl = kind == 1 && is_k ? &planted[b * Hkv + g] : nullptr;
            uint16_t *dst = (is_k ? k : v) + ((b * N) * Hkv + g) * 128;
            fill_rows(head_seed(sb, kv_begin + g), is_k ? nd : 2 * nd, r0, r1, d, is_k ? kK : kV, pl, nullptr,
                      dst, Hkv * 128);
        }
    });
    return SALE_B200_OK;
}

} // extern "C"
