// exmy_abi.cu -- C ABI (include/exmy.h): host-side argument validation and
// kernel selection.  The library never allocates, frees or synchronises.
#include <climits>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "exmy_launch.cuh"

namespace exmy {
int g_force_generic = 0;
int g_hist_mode = 4;
int g_hist_blocks = 0;
int g_enc_tma = 0;
int g_rowwise_cluster = 0;   // A/B knob: measured slower than two-pass
}  // namespace exmy

using namespace exmy;

namespace {

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

bool fmt_ok(int x, int y) {
    if (x < 0 || x > 8 || y < 0) return false;
    int k = 1 + x + y;
    return k >= 3 && k <= 9;
}

exmy_status check_layout(int64_t rows, int64_t cols, int axis, int64_t *n) {
    if (rows < 0 || cols < 0) return EXMY_E_SHAPE;
    if (axis != EXMY_AXIS_ROWS && axis != EXMY_AXIS_COLS) return EXMY_E_SHAPE;
    if (axis == EXMY_AXIS_ROWS && rows % 8) return EXMY_E_SHAPE;
    if (axis == EXMY_AXIS_COLS && cols % 8) return EXMY_E_SHAPE;
    if (cols && rows > INT64_MAX / cols) return EXMY_E_SHAPE;
    *n = rows * cols;
    return EXMY_OK;
}

bool block_ok(int64_t rows, int64_t cols, int64_t br, int64_t bc) {
    return br >= 1 && bc >= 1 && rows % br == 0 && cols % bc == 0;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

const char *exmy_version(void) { return "exmy-b200 0.2 (sm_100a)"; }

int exmy_specials_words(void) {
    static_assert(EXMY_SPECIALS_WORDS == 2 + SPECIALS_RANGES, "workspace = count + one word per range + flag");
    return EXMY_SPECIALS_WORDS;
}

const char *exmy_status_string(int s) {
    switch (s) {
        case EXMY_OK: return "ok";
        case EXMY_E_FORMAT: return "invalid format (x in [0,8], k=1+x+y in [3,9])";
        case EXMY_E_META: return "metadata out of range (e_max in [0,254])";
        case EXMY_E_SHAPE: return "invalid shape (ROWS needs rows%8==0, COLS cols%8==0)";
        case EXMY_E_DTYPE: return "invalid dtype";
        case EXMY_E_ALIGN: return "misaligned pointer";
        case EXMY_E_CAPACITY: return "invalid specials capacity";
        case EXMY_E_CUDA: return "CUDA launch error";
        case EXMY_E_ARG: return "invalid argument (NULL pointer)";
        case EXMY_E_IO: return "checkpoint file I/O error";
        case EXMY_E_CONTAINER: return "not a valid EXMY container (magic, version or manifest)";
        case EXMY_E_CHECKSUM: return "checkpoint CRC32 mismatch";
    }
    return "unknown status";
}

int exmy_format_valid(int x, int y) { return fmt_ok(x, y) ? 1 : 0; }

int64_t exmy_packed_bytes(int64_t n, int x, int y) {
    if (!fmt_ok(x, y) || n < 0 || n % 8) return -1;
    return n / 8 * (1 + x + y);
}

int exmy_segments(int k, int64_t n, int *widths, int64_t *offsets) {
    if (k < 1 || k > 15 || n < 0 || n % 8) return -1;
    Plan p = make_plan(k, n);
    for (int s = 0; s < p.nseg; ++s) {
        if (widths) widths[s] = p.w[s];
        if (offsets) offsets[s] = p.so.off[s];
    }
    return p.nseg;
}

exmy_status exmy_bias_from_emax(int x, int e_max, int *bias_out) {
    if (x < 0 || x > 8) return EXMY_E_FORMAT;
    if (e_max < 0 || e_max > 254) return EXMY_E_META;
    if (bias_out) *bias_out = (1 << x) + 126 - e_max;
    return EXMY_OK;
}

exmy_status exmy_emax_from_bias(int x, int bias, int *emax_out) {
    if (x < 0 || x > 8) return EXMY_E_FORMAT;
    int e = (1 << x) + 126 - bias;
    if (e < 0 || e > 254) return EXMY_E_META;
    if (emax_out) *emax_out = e;
    return EXMY_OK;
}

int exmy_emax_from_histogram_host(const uint64_t *h) {
    if (!h) return 0;
    for (int b = 254; b >= 0; --b)
        if (h[b]) return b;
    return 0;
}

exmy_status exmy_choose_x(const uint64_t *h, double budget, int *x_out) {
    if (!h || !x_out) return EXMY_E_ARG;
    int e_max = exmy_emax_from_histogram_host(h);
    uint64_t total = 0;
    for (int b = 1; b <= 254; ++b) total += h[b];
    // cumulative from the top bin downwards
    uint64_t covered = 0;
    int lo = e_max + 1;   // bins [lo, e_max] are covered
    for (int x = 0; x <= 8; ++x) {
        int want_lo = e_max - (1 << x) + 2;
        if (want_lo < 1) want_lo = 1;
        while (lo > want_lo) { --lo; covered += h[lo]; }
        if ((double)covered >= (1.0 - budget) * (double)total) { *x_out = x; return EXMY_OK; }
    }
    *x_out = 8;
    return EXMY_OK;
}

int exmy_debug_force_generic(int on) {
    int prev = g_force_generic;
    if (on >= 0) g_force_generic = on ? 1 : 0;
    return prev;
}

int exmy_debug_hist_mode(int mode) {
    int prev = g_hist_mode;
    if (mode >= 0) g_hist_mode = mode;
    return prev;
}

int exmy_debug_rowwise_cluster(int on) {
    int prev = g_rowwise_cluster;
    if (on >= 0) g_rowwise_cluster = on;
    return prev;
}

int exmy_debug_enc_tma(int on) {
    int prev = g_enc_tma;
    if (on >= 0) g_enc_tma = on;
    return prev;
}

int exmy_debug_hist_blocks(int blocks) {
    int prev = g_hist_blocks;
    if (blocks >= 0) g_hist_blocks = blocks;
    return prev;
}

exmy_status exmy_exponent_histogram(const void *in, int dtype, int64_t n, uint64_t *hist, void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (n < 0) return EXMY_E_SHAPE;
    if (n == 0) return EXMY_OK;
    if (!in || !hist) return EXMY_E_ARG;
    return launch_histogram(static_cast<const uint8_t *>(in), dtype == EXMY_BF16, n,
                            reinterpret_cast<unsigned long long *>(hist), S(stream));
}

exmy_status exmy_max_exponent(const void *in, int dtype, int64_t n, uint8_t *meta, void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (n < 0) return EXMY_E_SHAPE;
    if (!meta) return EXMY_E_ARG;
    if (n == 0) return cudaMemsetAsync(meta, 0, 1, S(stream)) == cudaSuccess ? EXMY_OK : EXMY_E_CUDA;
    if (!in) return EXMY_E_ARG;
    if (!aligned(in, 16)) {   // scalar inputs: the histogram path
        return EXMY_E_ALIGN;
    }
    return launch_max_exponent(static_cast<const uint8_t *>(in), dtype == EXMY_BF16, n, meta, S(stream));
}

exmy_status exmy_emax_from_histogram(const uint64_t *hist, uint8_t *meta, void *stream) {
    if (!hist || !meta) return EXMY_E_ARG;
    return launch_emax(reinterpret_cast<const unsigned long long *>(hist), meta, S(stream));
}

exmy_status exmy_quantize(const void *in, void *out, int dtype, int64_t n, int x, int y, const uint8_t *meta,
                          void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    if (n < 0) return EXMY_E_SHAPE;
    if (n == 0) return EXMY_OK;
    if (!in || !out || !meta) return EXMY_E_ARG;
    return launch_quantize(static_cast<const uint8_t *>(in), static_cast<uint8_t *>(out), dtype == EXMY_BF16, n, x,
                           y, meta, S(stream));
}

exmy_status exmy_encode(const void *in, int dtype, int64_t rows, int64_t cols, int axis, int x, int y,
                        const uint8_t *meta, uint8_t *packed, int64_t *sp_index, uint32_t *sp_bits,
                        uint64_t *sp_count, int64_t sp_capacity, void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    int64_t n = 0;
    exmy_status s = check_layout(rows, cols, axis, &n);
    if (s != EXMY_OK) return s;
    if (sp_capacity < 0) return EXMY_E_CAPACITY;
    if (sp_capacity > 0 && (!sp_index || !sp_bits)) return EXMY_E_ARG;
    cudaStream_t st = S(stream);
    auto *spc = reinterpret_cast<unsigned long long *>(sp_count);
    // with a list to fill the workspace is full-size: zero it all (counts, range counts, fix-up flag)
    const bool full_ws = spc && sp_capacity > 0;
    if (spc && cudaMemsetAsync(spc, 0, sizeof(unsigned long long) * (full_ws ? EXMY_SPECIALS_WORDS : 1), st) !=
                   cudaSuccess)
        return EXMY_E_CUDA;
    if (n == 0) return EXMY_OK;
    if (!in || !packed || !meta) return EXMY_E_ARG;
    // the kernels count the NaN/Inf (ws[0]; tiles holding them go to the fix-up pass, which also counts
    // them per range); the ordered list is written after them
    const SpecialsRanges sr = specials_ranges(rows, cols, full_ws);
    s = launch_encode(static_cast<const uint8_t *>(in), dtype == EXMY_BF16, rows, cols, axis, x, y, meta, packed,
                      nullptr, nullptr, spc, 0, st, sr);
    if (s != EXMY_OK) return s;
    return launch_specials_compact(static_cast<const uint8_t *>(in), dtype == EXMY_BF16, n, 0, sp_index, sp_bits, spc,
                                   sp_capacity, st, sr.len(axis, cols));
}

exmy_status exmy_decode(const uint8_t *packed, int64_t rows, int64_t cols, int axis, int x, int y,
                        const uint8_t *meta, const int64_t *sp_index, const uint32_t *sp_bits,
                        const uint64_t *sp_count, int64_t sp_capacity, void *out, int out_dtype, void *stream) {
    if (out_dtype != EXMY_F32 && out_dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    int64_t n = 0;
    exmy_status s = check_layout(rows, cols, axis, &n);
    if (s != EXMY_OK) return s;
    if (sp_capacity < 0) return EXMY_E_CAPACITY;
    if (n == 0) return EXMY_OK;
    if (!packed || !out || !meta) return EXMY_E_ARG;
    cudaStream_t st = S(stream);
    auto *po = static_cast<uint8_t *>(out);
    const bool obf = out_dtype == EXMY_BF16;
    s = launch_decode(packed, rows, cols, axis, x, y, meta, po, obf, st);
    if (s != EXMY_OK) return s;
    if (sp_count && sp_index && sp_bits && sp_capacity > 0)
        s = launch_specials_scatter(sp_index, sp_bits, reinterpret_cast<const unsigned long long *>(sp_count),
                                    sp_capacity, po, obf, st);
    return s;
}

exmy_status exmy_block_max_exponent(const void *in, int dtype, int64_t rows, int64_t cols, int64_t block_rows,
                                    int64_t block_cols, int y, int scheme, uint8_t *meta, void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (rows < 0 || cols < 0 || !block_ok(rows, cols, block_rows, block_cols)) return EXMY_E_SHAPE;
    if (y < 0 || y > 23 || (scheme != EXMY_SCHEME_MAX_BEFORE && scheme != EXMY_SCHEME_MAX_AFTER)) return EXMY_E_ARG;
    if (rows == 0 || cols == 0) return EXMY_OK;
    if (!in || !meta) return EXMY_E_ARG;
    return launch_block_max(static_cast<const uint8_t *>(in), dtype == EXMY_BF16, rows, cols, block_rows, block_cols,
                            y, scheme, meta, S(stream));
}

exmy_status exmy_quantize_blocked(const void *in, void *out, int dtype, int64_t rows, int64_t cols,
                                  int64_t block_rows, int64_t block_cols, int x, int y, const uint8_t *meta,
                                  void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    if (rows < 0 || cols < 0 || !block_ok(rows, cols, block_rows, block_cols)) return EXMY_E_SHAPE;
    if (rows == 0 || cols == 0) return EXMY_OK;
    if (!in || !out || !meta) return EXMY_E_ARG;
    return launch_quantize_blocked(static_cast<const uint8_t *>(in), static_cast<uint8_t *>(out), dtype == EXMY_BF16,
                                   rows, cols, block_rows, block_cols, x, y, meta, S(stream));
}

exmy_status exmy_encode_blocked(const void *in, int dtype, int64_t rows, int64_t cols, int axis, int64_t block_rows,
                                int64_t block_cols, int x, int y, const uint8_t *meta, uint8_t *packed,
                                int64_t *sp_index, uint32_t *sp_bits, uint64_t *sp_count, int64_t sp_capacity,
                                void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    int64_t n = 0;
    exmy_status s = check_layout(rows, cols, axis, &n);
    if (s != EXMY_OK) return s;
    if (!block_ok(rows, cols, block_rows, block_cols)) return EXMY_E_SHAPE;
    if (sp_capacity < 0) return EXMY_E_CAPACITY;
    if (sp_capacity > 0 && (!sp_index || !sp_bits)) return EXMY_E_ARG;
    cudaStream_t st = S(stream);
    auto *spc = reinterpret_cast<unsigned long long *>(sp_count);
    if (spc && cudaMemsetAsync(spc, 0, sizeof(unsigned long long) * (sp_capacity > 0 ? EXMY_SPECIALS_WORDS : 1), st) !=
                   cudaSuccess)
        return EXMY_E_CUDA;
    if (n == 0) return EXMY_OK;
    if (!in || !packed || !meta) return EXMY_E_ARG;
    s = launch_encode_blocked(static_cast<const uint8_t *>(in), dtype == EXMY_BF16, rows, cols, axis, block_rows,
                              block_cols, x, y, meta, packed, nullptr, nullptr, spc, 0, st);
    if (s != EXMY_OK) return s;
    return launch_specials_compact(static_cast<const uint8_t *>(in), dtype == EXMY_BF16, n, 0, sp_index, sp_bits, spc,
                                   sp_capacity, st);
}

exmy_status exmy_decode_blocked(const uint8_t *packed, int64_t rows, int64_t cols, int axis, int64_t block_rows,
                                int64_t block_cols, int x, int y, const uint8_t *meta, const int64_t *sp_index,
                                const uint32_t *sp_bits, const uint64_t *sp_count, int64_t sp_capacity, void *out,
                                int out_dtype, void *stream) {
    if (out_dtype != EXMY_F32 && out_dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    int64_t n = 0;
    exmy_status s = check_layout(rows, cols, axis, &n);
    if (s != EXMY_OK) return s;
    if (!block_ok(rows, cols, block_rows, block_cols)) return EXMY_E_SHAPE;
    if (sp_capacity < 0) return EXMY_E_CAPACITY;
    if (n == 0) return EXMY_OK;
    if (!packed || !out || !meta) return EXMY_E_ARG;
    cudaStream_t st = S(stream);
    auto *po = static_cast<uint8_t *>(out);
    const bool obf = out_dtype == EXMY_BF16;
    s = launch_decode_blocked(packed, rows, cols, axis, block_rows, block_cols, x, y, meta, po, obf, st);
    if (s != EXMY_OK) return s;
    if (sp_count && sp_index && sp_bits && sp_capacity > 0)
        s = launch_specials_scatter(sp_index, sp_bits, reinterpret_cast<const unsigned long long *>(sp_count),
                                    sp_capacity, po, obf, st);
    return s;
}

exmy_status exmy_encode_rowwise(const void *in, int dtype, int64_t rows, int64_t cols, int axis, int x, int y,
                                int scheme, uint8_t *meta, uint8_t *packed, int64_t *sp_index, uint32_t *sp_bits,
                                uint64_t *sp_count, int64_t sp_capacity, void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    int64_t n = 0;
    exmy_status s = check_layout(rows, cols, axis, &n);
    if (s != EXMY_OK) return s;
    if (scheme != EXMY_SCHEME_MAX_BEFORE && scheme != EXMY_SCHEME_MAX_AFTER) return EXMY_E_ARG;
    if (sp_capacity < 0) return EXMY_E_CAPACITY;
    if (sp_capacity > 0 && (!sp_index || !sp_bits)) return EXMY_E_ARG;
    cudaStream_t st = S(stream);
    auto *spc = reinterpret_cast<unsigned long long *>(sp_count);
    if (spc && cudaMemsetAsync(spc, 0, sizeof(unsigned long long) * (sp_capacity > 0 ? EXMY_SPECIALS_WORDS : 1), st) !=
                   cudaSuccess)
        return EXMY_E_CUDA;
    if (n == 0) return EXMY_OK;
    if (!in || !packed || !meta) return EXMY_E_ARG;
    auto *pin = static_cast<const uint8_t *>(in);
    const bool bf = dtype == EXMY_BF16;
    s = EXMY_E_ALIGN;
    if (axis == EXMY_AXIS_ROWS && !g_force_generic)
        s = launch_encode_rowwise(pin, bf, rows, cols, x, y, scheme, meta, packed, nullptr, nullptr, spc, 0, st);
    if (s == EXMY_E_ALIGN) {   // two launches: row maxima, then the blocked encode
        s = launch_block_max(pin, bf, rows, cols, 1, cols, y, scheme, meta, st);
        if (s != EXMY_OK) return s;
        s = launch_encode_blocked(pin, bf, rows, cols, axis, 1, cols, x, y, meta, packed, nullptr, nullptr, spc, 0, st);
    }
    if (s != EXMY_OK) return s;
    return launch_specials_compact(pin, bf, n, 0, sp_index, sp_bits, spc, sp_capacity, st);
}

exmy_status exmy_decode_rows(const uint8_t *packed, int64_t rows, int64_t cols, int x, int y, const uint8_t *meta,
                             int meta_per_row, const int64_t *row_index, int64_t n_index, void *out, int out_dtype,
                             void *stream) {
    if (out_dtype != EXMY_F32 && out_dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    if (rows < 0 || cols < 0 || cols % 8 || n_index < 0) return EXMY_E_SHAPE;
    if (n_index == 0 || cols == 0) return EXMY_OK;
    if (!packed || !meta || !row_index || !out) return EXMY_E_ARG;
    if (!aligned(out, 16) || !aligned(row_index, 8)) return EXMY_E_ALIGN;
    return launch_decode_rows_gather(packed, rows, cols, x, y, meta, meta_per_row != 0, row_index, n_index,
                                     static_cast<uint8_t *>(out), out_dtype == EXMY_BF16, S(stream));
}

exmy_status exmy_encode_host(const void *host_in, int dtype, int64_t rows, int64_t cols, int axis, int x, int y,
                             void *dev_in, uint64_t *dev_hist, uint8_t *dev_meta, uint8_t *dev_packed,
                             int64_t *sp_index, uint32_t *sp_bits, uint64_t *sp_count, int64_t sp_capacity,
                             uint8_t *host_packed, uint8_t *host_meta, void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    int64_t n = 0;
    exmy_status s = check_layout(rows, cols, axis, &n);
    if (s != EXMY_OK) return s;
    if (n == 0) return EXMY_OK;
    if (!host_in || !dev_in || !dev_hist || !dev_meta || !dev_packed || !host_packed) return EXMY_E_ARG;
    cudaStream_t st = S(stream);
    const size_t es = dtype == EXMY_BF16 ? 2 : 4;
    if (cudaMemcpyAsync(dev_in, host_in, (size_t)n * es, cudaMemcpyHostToDevice, st) != cudaSuccess) return EXMY_E_CUDA;
    if (cudaMemsetAsync(dev_hist, 0, 256 * sizeof(uint64_t), st) != cudaSuccess) return EXMY_E_CUDA;
    if ((s = exmy_exponent_histogram(dev_in, dtype, n, dev_hist, stream)) != EXMY_OK) return s;
    if ((s = exmy_emax_from_histogram(dev_hist, dev_meta, stream)) != EXMY_OK) return s;
    if ((s = exmy_encode(dev_in, dtype, rows, cols, axis, x, y, dev_meta, dev_packed, sp_index, sp_bits, sp_count,
                         sp_capacity, stream)) != EXMY_OK)
        return s;
    const size_t nb = (size_t)(n / 8) * (size_t)(1 + x + y);
    if (cudaMemcpyAsync(host_packed, dev_packed, nb, cudaMemcpyDeviceToHost, st) != cudaSuccess) return EXMY_E_CUDA;
    if (host_meta && cudaMemcpyAsync(host_meta, dev_meta, 1, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return EXMY_E_CUDA;
    return EXMY_OK;
}

exmy_status exmy_decode_host(const uint8_t *host_packed, int64_t rows, int64_t cols, int axis, int x, int y,
                             const uint8_t *meta, const int64_t *sp_index, const uint32_t *sp_bits,
                             const uint64_t *sp_count, int64_t sp_capacity, uint8_t *dev_packed, void *dev_out,
                             int out_dtype, void *host_out, void *stream) {
    if (out_dtype != EXMY_F32 && out_dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    int64_t n = 0;
    exmy_status s = check_layout(rows, cols, axis, &n);
    if (s != EXMY_OK) return s;
    if (n == 0) return EXMY_OK;
    if (!host_packed || !dev_packed || !dev_out || !host_out || !meta) return EXMY_E_ARG;
    cudaStream_t st = S(stream);
    const size_t nb = (size_t)(n / 8) * (size_t)(1 + x + y);
    if (cudaMemcpyAsync(dev_packed, host_packed, nb, cudaMemcpyHostToDevice, st) != cudaSuccess) return EXMY_E_CUDA;
    if ((s = exmy_decode(dev_packed, rows, cols, axis, x, y, meta, sp_index, sp_bits, sp_count, sp_capacity, dev_out,
                         out_dtype, stream)) != EXMY_OK)
        return s;
    const size_t es = out_dtype == EXMY_BF16 ? 2 : 4;
    if (cudaMemcpyAsync(host_out, dev_out, (size_t)n * es, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return EXMY_E_CUDA;
    return EXMY_OK;
}

}  // extern "C"
