// exmy_tu_fscale.cu -- float-scaling block scheme (reading D23): ABI entry
// points (include/exmy.h "float scaling") and their launchers.
#include <climits>
#include <cmath>

#include "exmy_fscale.cuh"
#include "exmy_launch.cuh"

using namespace exmy;

namespace {

inline cudaStream_t S_(void *s) { return reinterpret_cast<cudaStream_t>(s); }

bool fmt_ok(int x, int y) {
    if (x < 0 || x > 8 || y < 0) return false;
    const int k = 1 + x + y;
    return k >= 3 && k <= 9;
}

bool block_ok(int64_t rows, int64_t cols, int64_t br, int64_t bc) {
    return rows >= 0 && cols >= 0 && br >= 1 && bc >= 1 && rows % br == 0 && cols % bc == 0;
}

// G = the largest magnitude of (x, y) at e_max 127, and RN64(1/G)
float grid_top(int x, int y) {
    return x >= 1 ? (float)(2.0 - std::ldexp(1.0, -y)) : (float)(std::ldexp((double)((1 << y) - 1), 1 - y));
}

// the float-scale map of a call: rows / blocks with s_hi = amax / G below
// tchk = 2^-99 / g_min (g_min = the smallest non-zero grid value at e_max 127)
// can produce results below 2^-100, which the kernels evaluate exactly
FsMap fs_map(const float *scale, int64_t rows, int64_t cols, int64_t br, int64_t bc, int x, int y) {
    (void)rows;
    const int lg_gmin = x >= 1 ? 2 - (1 << x) - y : 1 - y;
    const double t = std::ldexp(1.0, -99 - lg_gmin);
    return FsMap{scale, br, bc, cols / bc, t > 3.0e38 ? INFINITY : (float)t, x == 8 ? 1 : 0};
}

unsigned grid1(int64_t work, int per_sm) {
    int64_t b = cdiv(work, 256);
    const int64_t m = (int64_t)num_sms() * per_sm;
    if (b > m) b = m;
    return (unsigned)(b < 1 ? 1 : b);
}

template <int K, bool BF16>
exmy_status enc_k(const uint8_t *in, int64_t R, int64_t C, int axis, int x, int y, const FsMap &M, float G,
                  uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb, unsigned long long *spc, int64_t cap,
                  cudaStream_t st) {
    bool fast = axis == EXMY_AXIS_ROWS && x <= 7 && !g_force_generic && M.bc % 4 == 0 && C % 4 == 0 &&
                aligned(in, 4 * Elem<BF16>::ES);
    for (int s = 0; s < p.nseg; ++s) fast = fast && aligned(packed + p.so.off[s], p.w[s] == 8 ? 4 : 4 * p.w[s]);
    if (fast) {
        const int threads = 256;
        const int64_t CV = C / 4, G8 = R / 8;
        const int64_t gx = cdiv(CV, threads);
        int64_t gy = (int64_t)num_sms() * 2 / gx;
        if (gy < 1) gy = 1;
        if (gy > G8) gy = G8;
        if (gy > 65535) gy = 65535;
        if (gx > INT_MAX) return EXMY_E_SHAPE;
        const dim3 grid((unsigned)gx, (unsigned)gy);
        const bool ws = M.bc % 128 == 0 || M.bc == 32 || M.bc == 64;
        const int lpb = M.bc >= 128 ? 32 : (int)(M.bc / 4);   // lanes per block column in a warp
        if (y == 0) {
            if (ws) k_fs_enc_rows<K, BF16, true, true><<<grid, threads, 0, st>>>(in, R, C, x, y, M, G, packed, p.so, spi, spb, spc, cap, lpb);
            else k_fs_enc_rows<K, BF16, true, false><<<grid, threads, 0, st>>>(in, R, C, x, y, M, G, packed, p.so, spi, spb, spc, cap, 32);
        } else {
            if (ws) k_fs_enc_rows<K, BF16, false, true><<<grid, threads, 0, st>>>(in, R, C, x, y, M, G, packed, p.so, spi, spb, spc, cap, lpb);
            else k_fs_enc_rows<K, BF16, false, false><<<grid, threads, 0, st>>>(in, R, C, x, y, M, G, packed, p.so, spi, spb, spc, cap, 32);
        }
        return launch_status();
    }
    const int64_t ncont = R * C / 8;
    k_fs_encode_generic<BF16, K><<<grid1(ncont, 8), 256, 0, st>>>(in, C, ncont, axis, x, y, M, G, packed, p.so, spi, spb,
                                                                  spc, cap);
    return launch_status();
}

template <bool BF16>
exmy_status enc_dispatch(int k, const uint8_t *in, int64_t R, int64_t C, int axis, int x, int y, const FsMap &M,
                         float G, uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb,
                         unsigned long long *spc, int64_t cap, cudaStream_t st) {
    switch (k) {
        case 3: return enc_k<3, BF16>(in, R, C, axis, x, y, M, G, packed, p, spi, spb, spc, cap, st);
        case 4: return enc_k<4, BF16>(in, R, C, axis, x, y, M, G, packed, p, spi, spb, spc, cap, st);
        case 5: return enc_k<5, BF16>(in, R, C, axis, x, y, M, G, packed, p, spi, spb, spc, cap, st);
        case 6: return enc_k<6, BF16>(in, R, C, axis, x, y, M, G, packed, p, spi, spb, spc, cap, st);
        case 7: return enc_k<7, BF16>(in, R, C, axis, x, y, M, G, packed, p, spi, spb, spc, cap, st);
        case 8: return enc_k<8, BF16>(in, R, C, axis, x, y, M, G, packed, p, spi, spb, spc, cap, st);
        case 9: return enc_k<9, BF16>(in, R, C, axis, x, y, M, G, packed, p, spi, spb, spc, cap, st);
    }
    return EXMY_E_FORMAT;
}

template <int K, bool OBF16>
exmy_status dec_k(const uint8_t *packed, int64_t R, int64_t C, int axis, int x, int y, const FsMap &M, float G,
                  const Plan &p, uint8_t *out, cudaStream_t st) {
    bool fast = axis == EXMY_AXIS_ROWS && M.bc % 4 == 0 && C % 4 == 0 && aligned(out, 4 * Elem<OBF16>::ES);
    for (int s = 0; s < p.nseg; ++s) fast = fast && aligned(packed + p.so.off[s], p.w[s] == 8 ? 4 : 4 * p.w[s]);
    if (fast) {
        const int threads = 256;
        const int64_t CV = C / 4, G8 = R / 8;
        const int64_t gx = cdiv(CV, threads);
        int64_t gy = (int64_t)num_sms() * 2 / gx;
        if (gy < 1) gy = 1;
        if (gy > G8) gy = G8;
        if (gy > 65535) gy = 65535;
        if (gx > INT_MAX) return EXMY_E_SHAPE;
        const dim3 grid((unsigned)gx, (unsigned)gy);
        const bool ws = M.bc % 128 == 0 || M.bc == 32 || M.bc == 64;
        const int lpb = M.bc >= 128 ? 32 : (int)(M.bc / 4);
        if (x <= 7 && !g_force_generic) {
            if (ws) k_fs_dec_rows<K, OBF16, true, true><<<grid, threads, 0, st>>>(packed, R, C, x, y, M, G, p.so, out, lpb);
            else k_fs_dec_rows<K, OBF16, true, false><<<grid, threads, 0, st>>>(packed, R, C, x, y, M, G, p.so, out, 32);
        } else {
            if (ws) k_fs_dec_rows<K, OBF16, false, true><<<grid, threads, 0, st>>>(packed, R, C, x, y, M, G, p.so, out, lpb);
            else k_fs_dec_rows<K, OBF16, false, false><<<grid, threads, 0, st>>>(packed, R, C, x, y, M, G, p.so, out, 32);
        }
        // blocks whose results can fall below 2^-100 (and x = 8): the exact evaluation
        const int64_t nb = (R / M.br) * M.nbc;
        k_fs_dec_fixup<OBF16><<<grid1(nb * 32, 8), 256, 0, st>>>(packed, R, C, axis, x, y, M, G, p.so, p.nseg,
                                                                 make_int4(p.w[0], p.w[1], p.w[2], p.w[3]), out);
        return launch_status();
    }
    const int64_t ncont = R * C / 8;
    k_fs_decode_generic<OBF16><<<grid1(ncont, 8), 256, 0, st>>>(packed, C, ncont, axis, x, y, M, G, p.so, p.nseg,
                                                                make_int4(p.w[0], p.w[1], p.w[2], p.w[3]), out);
    return launch_status();
}

template <bool OBF16>
exmy_status dec_dispatch(int k, const uint8_t *packed, int64_t R, int64_t C, int axis, int x, int y, const FsMap &M,
                         float G, const Plan &p, uint8_t *out, cudaStream_t st) {
    switch (k) {
        case 3: return dec_k<3, OBF16>(packed, R, C, axis, x, y, M, G, p, out, st);
        case 4: return dec_k<4, OBF16>(packed, R, C, axis, x, y, M, G, p, out, st);
        case 5: return dec_k<5, OBF16>(packed, R, C, axis, x, y, M, G, p, out, st);
        case 6: return dec_k<6, OBF16>(packed, R, C, axis, x, y, M, G, p, out, st);
        case 7: return dec_k<7, OBF16>(packed, R, C, axis, x, y, M, G, p, out, st);
        case 8: return dec_k<8, OBF16>(packed, R, C, axis, x, y, M, G, p, out, st);
        case 9: return dec_k<9, OBF16>(packed, R, C, axis, x, y, M, G, p, out, st);
    }
    return EXMY_E_FORMAT;
}

}  // namespace

extern "C" {

exmy_status exmy_block_float_scale(const void *in, int dtype, int64_t rows, int64_t cols, int64_t block_rows,
                                   int64_t block_cols, float *scale, void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!block_ok(rows, cols, block_rows, block_cols)) return EXMY_E_SHAPE;
    if (rows == 0 || cols == 0) return EXMY_OK;
    if (!in || !scale) return EXMY_E_ARG;
    const int V = dtype == EXMY_BF16 ? 8 : 4;
    const int64_t gsz = block_cols / V;
    if (block_rows == 1 && block_cols % V == 0 && cols % V == 0 && gsz <= 32 && (gsz & (gsz - 1)) == 0 &&
        aligned(in, 16)) {   // sub-row blocks: segmented warp reduction (exmy_blocked.cuh)
        const int64_t nvec = rows * cols / V;
        const unsigned g = grid1(nvec / 4, 8);
        if (dtype == EXMY_BF16)
            k_block_max_small<true, 2><<<g, 256, 0, S_(stream)>>>(static_cast<const uint8_t *>(in), nvec, (int)gsz, 0,
                                                                 nullptr, scale);
        else
            k_block_max_small<false, 2><<<g, 256, 0, S_(stream)>>>(static_cast<const uint8_t *>(in), nvec, (int)gsz, 0,
                                                                  nullptr, scale);
        return launch_status();
    }
    const int64_t nb = (rows / block_rows) * (cols / block_cols);
    const unsigned grid = grid1(nb * 32, 8);
    if (dtype == EXMY_BF16)
        k_block_amax<true><<<grid, 256, 0, S_(stream)>>>(static_cast<const uint8_t *>(in), rows, cols, block_rows,
                                                         block_cols, scale);
    else
        k_block_amax<false><<<grid, 256, 0, S_(stream)>>>(static_cast<const uint8_t *>(in), rows, cols, block_rows,
                                                          block_cols, scale);
    return launch_status();
}

exmy_status exmy_quantize_fs(const void *in, void *out, int dtype, int64_t rows, int64_t cols, int64_t block_rows,
                             int64_t block_cols, int x, int y, const float *scale, void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    if (!block_ok(rows, cols, block_rows, block_cols)) return EXMY_E_SHAPE;
    if (rows == 0 || cols == 0) return EXMY_OK;
    if (!in || !out || !scale) return EXMY_E_ARG;
    const int V = dtype == EXMY_BF16 ? 8 : 4;
    if (!aligned(in, 16) || !aligned(out, 16) || (rows * cols) % V) return EXMY_E_ALIGN;
    const FsMap M = fs_map(scale, rows, cols, block_rows, block_cols, x, y);
    const float G = grid_top(x, y);
    const int mode = (cols % V == 0 && block_cols % V == 0) ? ((rows % 8 == 0 && block_cols % (32 * V) == 0) ? 2 : 1) : 0;
    const auto *pi = static_cast<const uint8_t *>(in);
    auto *po = static_cast<uint8_t *>(out);
    const bool fast = x <= 7 && !g_force_generic;
    cudaStream_t st = S_(stream);
#define FS_QUANT(M, GRID)                                                                               \
    do {                                                                                                \
        if (dtype == EXMY_BF16) {                                                                       \
            if (fast) k_fs_quant<true, true, M><<<GRID, 256, 0, st>>>(pi, po, rows, cols, x, y, Mp, G);   \
            else k_fs_quant<true, false, M><<<GRID, 256, 0, st>>>(pi, po, rows, cols, x, y, Mp, G);      \
        } else {                                                                                        \
            if (fast) k_fs_quant<false, true, M><<<GRID, 256, 0, st>>>(pi, po, rows, cols, x, y, Mp, G);  \
            else k_fs_quant<false, false, M><<<GRID, 256, 0, st>>>(pi, po, rows, cols, x, y, Mp, G);     \
        }                                                                                               \
    } while (0)
    const FsMap &Mp = M;
    if (mode >= 1) {
        const int64_t CVv = cols / V;
        const int64_t gx = cdiv(CVv, 256);
        const int64_t ny = mode == 2 ? rows / 8 : rows;
        int64_t gy = (int64_t)num_sms() * 4 / gx;
        if (gy < 1) gy = 1;
        if (gy > ny) gy = ny;
        if (gy > 65535) gy = 65535;
        if (gx > INT_MAX) return EXMY_E_SHAPE;
        const dim3 grid((unsigned)gx, (unsigned)gy);
        if (mode == 2) FS_QUANT(2, grid);
        else FS_QUANT(1, grid);
    } else {
        const unsigned grid = grid1(rows * cols / V, 8);
        FS_QUANT(0, grid);
    }
#undef FS_QUANT
    // blocks whose results can fall below 2^-100 (and x = 8): the exact evaluation
    const int64_t nb = (rows / block_rows) * (cols / block_cols);
    if (dtype == EXMY_BF16) k_fs_quant_fixup<true><<<grid1(nb * 32, 8), 256, 0, st>>>(pi, po, rows, cols, x, y, M, G);
    else k_fs_quant_fixup<false><<<grid1(nb * 32, 8), 256, 0, st>>>(pi, po, rows, cols, x, y, M, G);
    return launch_status();
}

exmy_status exmy_encode_fs(const void *in, int dtype, int64_t rows, int64_t cols, int axis, int64_t block_rows,
                           int64_t block_cols, int x, int y, const float *scale, uint8_t *packed, int64_t *sp_index,
                           uint32_t *sp_bits, uint64_t *sp_count, int64_t sp_capacity, void *stream) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    if (axis != EXMY_AXIS_ROWS && axis != EXMY_AXIS_COLS) return EXMY_E_SHAPE;
    if (!block_ok(rows, cols, block_rows, block_cols)) return EXMY_E_SHAPE;
    if ((axis == EXMY_AXIS_ROWS && rows % 8) || (axis == EXMY_AXIS_COLS && cols % 8)) return EXMY_E_SHAPE;
    if (sp_capacity < 0) return EXMY_E_CAPACITY;
    if (sp_capacity > 0 && (!sp_index || !sp_bits)) return EXMY_E_ARG;
    cudaStream_t st = S_(stream);
    auto *spc = reinterpret_cast<unsigned long long *>(sp_count);
    if (spc && cudaMemsetAsync(spc, 0, sizeof(unsigned long long) * (sp_capacity > 0 ? EXMY_SPECIALS_WORDS : 1), st) !=
                   cudaSuccess)
        return EXMY_E_CUDA;
    if (rows == 0 || cols == 0) return EXMY_OK;
    if (!in || !packed || !scale) return EXMY_E_ARG;
    const int k = 1 + x + y;
    const Plan p = make_plan(k, rows * cols);
    const FsMap M = fs_map(scale, rows, cols, block_rows, block_cols, x, y);
    const float G = grid_top(x, y);
    const auto *pi = static_cast<const uint8_t *>(in);
    exmy_status s = dtype == EXMY_BF16
                        ? enc_dispatch<true>(k, pi, rows, cols, axis, x, y, M, G, packed, p, nullptr, nullptr, spc, 0,
                                             st)
                        : enc_dispatch<false>(k, pi, rows, cols, axis, x, y, M, G, packed, p, nullptr, nullptr, spc, 0,
                                              st);
    if (s != EXMY_OK) return s;
    return launch_specials_compact(pi, dtype == EXMY_BF16, rows * cols, 0, sp_index, sp_bits, spc, sp_capacity, st);
}

exmy_status exmy_decode_fs(const uint8_t *packed, int64_t rows, int64_t cols, int axis, int64_t block_rows,
                           int64_t block_cols, int x, int y, const float *scale, const int64_t *sp_index,
                           const uint32_t *sp_bits, const uint64_t *sp_count, int64_t sp_capacity, void *out,
                           int out_dtype, void *stream) {
    if (out_dtype != EXMY_F32 && out_dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    if (axis != EXMY_AXIS_ROWS && axis != EXMY_AXIS_COLS) return EXMY_E_SHAPE;
    if (!block_ok(rows, cols, block_rows, block_cols)) return EXMY_E_SHAPE;
    if ((axis == EXMY_AXIS_ROWS && rows % 8) || (axis == EXMY_AXIS_COLS && cols % 8)) return EXMY_E_SHAPE;
    if (sp_capacity < 0) return EXMY_E_CAPACITY;
    if (rows == 0 || cols == 0) return EXMY_OK;
    if (!packed || !out || !scale) return EXMY_E_ARG;
    const int k = 1 + x + y;
    const Plan p = make_plan(k, rows * cols);
    const FsMap M = fs_map(scale, rows, cols, block_rows, block_cols, x, y);
    const float G = grid_top(x, y);
    cudaStream_t st = S_(stream);
    auto *po = static_cast<uint8_t *>(out);
    const bool obf = out_dtype == EXMY_BF16;
    exmy_status s = obf ? dec_dispatch<true>(k, packed, rows, cols, axis, x, y, M, G, p, po, st)
                        : dec_dispatch<false>(k, packed, rows, cols, axis, x, y, M, G, p, po, st);
    if (s != EXMY_OK) return s;
    if (sp_count && sp_index && sp_bits && sp_capacity > 0)
        s = launch_specials_scatter(sp_index, sp_bits, reinterpret_cast<const unsigned long long *>(sp_count),
                                    sp_capacity, po, obf, st);
    return s;
}

}  // extern "C"
