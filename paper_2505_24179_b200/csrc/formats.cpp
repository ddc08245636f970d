// formats.cpp — the reference's file formats on this path's layouts (host
// side; docs/formats.md): the .tns tensor container (tensor_file.hpp) read into
// / written from bf16 [1][N][H][128] arrays, with a bf16 payload tag as an
// extension of the float32 one, and the RLE mask dump (mask_io.hpp) written
// from / read into packed BlockMask words. Byte layouts, validation order and
// error offsets follow the reference so its files and ours interchange.
#include "sale_b200.h"

#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

namespace sale_b200 {
int set_error(sale_b200_ctx *ctx, int code, const std::string &msg);
}

namespace {

using sale_b200::set_error;

constexpr char kTensorMagic[8] = {'S', 'A', 'L', 'E', 'T', 'N', 'S', 'R'};
constexpr char kMaskMagic[8] = {'S', 'A', 'L', 'E', 'M', 'A', 'S', 'K'};
constexpr uint32_t kDtypeF32 = 1, kDtypeBf16 = 2;
constexpr int64_t kPitch = 128;

// TensorFileError: "<message> (offset N)" (tensor_file.hpp:22-33)
int format_error(const std::string &msg, uint64_t offset) {
    return set_error(nullptr, SALE_B200_FORMAT_ERROR, msg + " (offset " + std::to_string(offset) + ")");
}

void put_u32(std::ostream &out, uint32_t v) {
    const unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                                static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
    out.write(reinterpret_cast<const char *>(b), 4);
}
bool get_u32(std::istream &in, uint32_t &v) {
    unsigned char b[4];
    if (!in.read(reinterpret_cast<char *>(b), 4)) return false;
    v = b[0] | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
    return true;
}
float bf16_to_f32(uint16_t h) {
    const uint32_t bits = uint32_t(h) << 16;
    float f;
    std::memcpy(&f, &bits, 4);
    return f;
}
uint16_t f32_to_bf16(float f) { // round to nearest even
    uint32_t bits;
    std::memcpy(&bits, &f, 4);
    if ((bits & 0x7F800000u) == 0x7F800000u) return static_cast<uint16_t>(bits >> 16); // inf / nan
    bits += 0x7FFFu + ((bits >> 16) & 1u);
    return static_cast<uint16_t>(bits >> 16);
}

struct TnsHeader {
    uint32_t heads = 0, tokens = 0, dim = 0, dtype = 0;
};

// tensor_file.hpp:98-125
int read_header(std::ifstream &in, const char *path, TnsHeader &h) {
    if (!in) return set_error(nullptr, SALE_B200_IO_ERROR, std::string("read_tensor_file: cannot open ") + path);
    char magic[8];
    if (!in.read(magic, 8)) return format_error("truncated magic", 0);
    if (std::memcmp(magic, kTensorMagic, 8) != 0) return format_error("bad magic", 0);
    uint32_t version;
    if (!get_u32(in, version)) return format_error("truncated version", 8);
    if (version != 1) return format_error("unsupported version " + std::to_string(version), 8);
    if (!get_u32(in, h.dtype)) return format_error("truncated dtype", 12);
    if (h.dtype != kDtypeF32 && h.dtype != kDtypeBf16)
        return format_error("unsupported dtype tag " + std::to_string(h.dtype), 12);
    if (!get_u32(in, h.heads)) return format_error("truncated head count", 16);
    if (!get_u32(in, h.tokens)) return format_error("truncated token count", 20);
    if (!get_u32(in, h.dim)) return format_error("truncated head dim", 24);
    if (h.heads == 0) return format_error("head count must be >= 1", 16);
    if (h.tokens == 0) return format_error("token count must be >= 1", 20);
    if (h.dim == 0) return format_error("head dim must be >= 1", 24);
    return SALE_B200_OK;
}

} // namespace

extern "C" {

int sale_b200_tensor_file_info(const char *path, uint32_t *heads, uint32_t *tokens, uint32_t *dim,
                               uint32_t *dtype) {
    if (!path) return set_error(nullptr, SALE_B200_INVALID_ARGUMENT, "path is NULL");
    std::ifstream in(path, std::ios::binary);
    TnsHeader h;
    int st = read_header(in, path, h);
    if (st) return st;
    if (heads) *heads = h.heads;
    if (tokens) *tokens = h.tokens;
    if (dim) *dim = h.dim;
    if (dtype) *dtype = h.dtype;
    return SALE_B200_OK;
}

int sale_b200_tensor_file_read_bf16(const char *path, uint16_t *q, uint16_t *k, uint16_t *v) {
    if (!path || !q || !k || !v) return set_error(nullptr, SALE_B200_INVALID_ARGUMENT, "NULL argument");
    std::ifstream in(path, std::ios::binary);
    TnsHeader h;
    int st = read_header(in, path, h);
    if (st) return st;
    if (h.dim > kPitch)
        return set_error(nullptr, SALE_B200_UNSUPPORTED, "head dim > 128 is not supported on the B200 path");
    const uint64_t values = 3ULL * h.heads * h.tokens * h.dim;
    const uint32_t esz = h.dtype == kDtypeF32 ? 4 : 2;
    uint64_t offset = 28;
    std::vector<unsigned char> row(static_cast<size_t>(h.dim) * esz);
    uint16_t *dst3[3] = {q, k, v};
    for (uint32_t hh = 0; hh < h.heads; ++hh) {
        for (int m = 0; m < 3; ++m) { // query, key, value (tensor_file.hpp:133)
            for (uint32_t n = 0; n < h.tokens; ++n) {
                uint16_t *dst = dst3[m] + (static_cast<int64_t>(n) * h.heads + hh) * kPitch;
                const uint64_t row_off = offset;
                if (!in.read(reinterpret_cast<char *>(row.data()), row.size())) {
                    // name the first missing value like the reference (offset of that value)
                    const uint64_t got = static_cast<uint64_t>(in.gcount()) / esz;
                    return format_error("truncated payload: expected " + std::to_string(values) +
                                            (h.dtype == kDtypeF32 ? " float32 values" : " bf16 values"),
                                        row_off + got * esz);
                }
                for (uint32_t c = 0; c < h.dim; ++c) {
                    float f;
                    if (esz == 4) {
                        const uint32_t bits = row[4 * c] | (uint32_t(row[4 * c + 1]) << 8) |
                                              (uint32_t(row[4 * c + 2]) << 16) | (uint32_t(row[4 * c + 3]) << 24);
                        std::memcpy(&f, &bits, 4);
                    } else {
                        f = bf16_to_f32(static_cast<uint16_t>(row[2 * c] | (row[2 * c + 1] << 8)));
                    }
                    if (!std::isfinite(f)) return format_error("non-finite value", row_off + uint64_t(c) * esz);
                    dst[c] = esz == 4 ? f32_to_bf16(f) : static_cast<uint16_t>(row[2 * c] | (row[2 * c + 1] << 8));
                }
                for (int64_t c = h.dim; c < kPitch; ++c) dst[c] = 0;
                offset += row.size();
            }
        }
    }
    char extra;
    if (in.read(&extra, 1)) return format_error("payload longer than header describes", offset);
    return SALE_B200_OK;
}

int sale_b200_tensor_file_write(const char *path, const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                uint32_t heads, uint32_t tokens, uint32_t dim, uint32_t dtype) {
    if (!path || !q || !k || !v) return set_error(nullptr, SALE_B200_INVALID_ARGUMENT, "NULL argument");
    if (heads == 0) return set_error(nullptr, SALE_B200_INVALID_ARGUMENT, "write_tensor_file: no heads");
    if (tokens == 0 || dim == 0) return set_error(nullptr, SALE_B200_INVALID_ARGUMENT, "HeadInput: empty query");
    if (dim > kPitch) return set_error(nullptr, SALE_B200_UNSUPPORTED, "head dim > 128 is not supported");
    if (dtype != kDtypeF32 && dtype != kDtypeBf16)
        return set_error(nullptr, SALE_B200_INVALID_ARGUMENT, "dtype must be 1 (float32) or 2 (bf16)");
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) return set_error(nullptr, SALE_B200_IO_ERROR, std::string("write_tensor_file: cannot open ") + path);
    out.write(kTensorMagic, 8);
    put_u32(out, 1);
    put_u32(out, dtype);
    put_u32(out, heads);
    put_u32(out, tokens);
    put_u32(out, dim);
    const uint16_t *src3[3] = {q, k, v};
    std::vector<unsigned char> row(static_cast<size_t>(dim) * (dtype == kDtypeF32 ? 4 : 2));
    for (uint32_t hh = 0; hh < heads; ++hh)
        for (int m = 0; m < 3; ++m)
            for (uint32_t n = 0; n < tokens; ++n) {
                const uint16_t *src = src3[m] + (static_cast<int64_t>(n) * heads + hh) * kPitch;
                for (uint32_t c = 0; c < dim; ++c) {
                    if (dtype == kDtypeF32) {
                        const uint32_t bits = uint32_t(src[c]) << 16;
                        for (int b = 0; b < 4; ++b) row[4 * c + b] = static_cast<unsigned char>(bits >> (8 * b));
                    } else {
                        row[2 * c] = static_cast<unsigned char>(src[c]);
                        row[2 * c + 1] = static_cast<unsigned char>(src[c] >> 8);
                    }
                }
                out.write(reinterpret_cast<const char *>(row.data()), row.size());
            }
    if (!out) return set_error(nullptr, SALE_B200_IO_ERROR, std::string("write_tensor_file: write failed for ") + path);
    return SALE_B200_OK;
}

int sale_b200_mask_dump_write(const char *path, const uint32_t *mask_words, int64_t batch, int64_t heads,
                              int64_t tokens, const float *taus) {
    if (!path || !mask_words || !taus) return set_error(nullptr, SALE_B200_INVALID_ARGUMENT, "NULL argument");
    if (batch < 1 || heads < 1 || tokens < 1)
        return set_error(nullptr, SALE_B200_INVALID_ARGUMENT, "mask dump: empty shape");
    const int64_t nq = (tokens + 63) / 64, nk = (tokens + 31) / 32, words = (nk + 31) / 32;
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) return set_error(nullptr, SALE_B200_IO_ERROR, std::string("write_mask_dump: cannot open ") + path);
    out.write(kMaskMagic, 8);
    put_u32(out, 1);
    put_u32(out, static_cast<uint32_t>(batch * heads));
    std::vector<uint32_t> runs;
    for (int64_t r = 0; r < batch * heads; ++r) {
        const uint32_t *m = mask_words + r * nq * words;
        put_u32(out, static_cast<uint32_t>(r));
        put_u32(out, static_cast<uint32_t>(nq));
        put_u32(out, static_cast<uint32_t>(nk));
        uint32_t tb;
        std::memcpy(&tb, &taus[r], 4);
        put_u32(out, tb);
        // row-major run-length encoding of the Nq x Nk grid (mask_io.hpp:41-58)
        runs.clear();
        const bool first = m[0] & 1u;
        bool cur = first;
        uint32_t len = 0;
        for (int64_t i = 0; i < nq; ++i)
            for (int64_t j = 0; j < nk; ++j) {
                const bool bit = (m[i * words + (j >> 5)] >> (j & 31)) & 1u;
                if (bit == cur) {
                    ++len;
                } else {
                    runs.push_back(len);
                    cur = bit;
                    len = 1;
                }
            }
        runs.push_back(len);
        out.put(static_cast<char>(first ? 1 : 0));
        put_u32(out, static_cast<uint32_t>(runs.size()));
        for (uint32_t x : runs) put_u32(out, x);
    }
    if (!out) return set_error(nullptr, SALE_B200_IO_ERROR, std::string("write_mask_dump: write failed for ") + path);
    return SALE_B200_OK;
}

int sale_b200_mask_dump_read(const char *path, int64_t *records, int64_t *nq_out, int64_t *nk_out,
                             uint32_t *mask_words, uint32_t *heads, float *taus) {
    if (!path) return set_error(nullptr, SALE_B200_INVALID_ARGUMENT, "path is NULL");
    std::ifstream in(path, std::ios::binary);
    if (!in) return set_error(nullptr, SALE_B200_IO_ERROR, std::string("read_mask_dump: cannot open ") + path);
    char magic[8];
    if (!in.read(magic, 8) || std::memcmp(magic, kMaskMagic, 8) != 0) return format_error("bad mask dump magic", 0);
    uint32_t version, count;
    if (!get_u32(in, version)) return format_error("truncated version", 8);
    if (version != 1) return format_error("unsupported mask dump version", 8);
    if (!get_u32(in, count)) return format_error("truncated record count", 12);
    if (records) *records = count;
    uint64_t offset = 16;
    int64_t words = 0, nq0 = -1, nk0 = -1;
    for (uint32_t rec = 0; rec < count; ++rec) {
        uint32_t head, nq, nk, tb, rc;
        if (!get_u32(in, head)) return format_error("truncated head index", offset);
        if (!get_u32(in, nq)) return format_error("truncated query blocks", offset + 4);
        if (!get_u32(in, nk)) return format_error("truncated key blocks", offset + 8);
        if (!get_u32(in, tb)) return format_error("truncated tau", offset + 12);
        char first;
        if (!in.get(first)) return format_error("truncated first_value", offset + 16);
        if (!get_u32(in, rc)) return format_error("truncated run count", offset + 17);
        offset += 21;
        if (nq0 < 0) {
            nq0 = nq, nk0 = nk, words = (nk + 31) / 32;
            if (nq_out) *nq_out = nq;
            if (nk_out) *nk_out = nk;
            if (!mask_words) return SALE_B200_OK; // size query
        } else if (nq != nq0 || nk != nk0) {
            return set_error(nullptr, SALE_B200_UNSUPPORTED, "mask dump records of different grids");
        }
        if (heads) heads[rec] = head;
        if (taus) std::memcpy(&taus[rec], &tb, 4);
        uint32_t *m = mask_words + static_cast<int64_t>(rec) * nq * words;
        std::memset(m, 0, sizeof(uint32_t) * nq * words);
        const uint64_t total = static_cast<uint64_t>(nq) * nk;
        uint64_t cell = 0;
        bool value = first != 0;
        for (uint32_t r = 0; r < rc; ++r) {
            uint32_t len;
            if (!get_u32(in, len)) return format_error("truncated run length", offset);
            offset += 4;
            if (len == 0) return format_error("zero-length run", offset - 4);
            if (cell + len > total) return format_error("runs exceed grid size", offset - 4);
            if (value)
                for (uint64_t t = cell; t < cell + len; ++t)
                    m[(t / nk) * words + (t % nk) / 32] |= 1u << ((t % nk) % 32);
            cell += len;
            value = !value;
        }
        if (cell != total)
            return format_error("runs cover " + std::to_string(cell) + " of " + std::to_string(total) + " cells",
                                offset);
    }
    return SALE_B200_OK;
}

} // extern "C"
