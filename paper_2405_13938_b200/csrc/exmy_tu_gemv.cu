// exmy_tu_gemv.cu -- decode fused into a matrix-vector product (SURVEY 8(f)
// row 3; exmy_gemv.cuh has the kernel and its reading).
#include <climits>

#include "exmy_gemv.cuh"
#include "exmy_launch.cuh"

using namespace exmy;

namespace {

bool gemv_fmt_ok(int x, int y) { return x >= 0 && x <= 8 && y >= 0 && 1 + x + y >= 3 && 1 + x + y <= 9; }

template <int K, int M>
exmy_status launch_gemv_bulk(const uint8_t *packed, int64_t N, int64_t Kc, const SegOffsets &so, int x, int y,
                             const uint8_t *meta, int per_row, const float *act, int64_t lda, float *out, int64_t ldo,
                             cudaStream_t st) {
    constexpr int smem = gemv_bulk_smem<K>();   // table + alignment slack + the stages
    static unsigned long long configured = 0;
    static int occ = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !(configured & (1ull << dev))) {
        cudaFuncSetAttribute(k_gemv_rows_bulk<K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        occ = occupancy(k_gemv_rows_bulk<K, M>, GEMV_THREADS, smem);
        if (dev >= 0 && dev < 64) configured |= 1ull << dev;
    }
    int64_t blocks = N / 8;
    const int64_t maxb = (int64_t)num_sms() * (occ > 0 ? occ : 1);
    if (blocks > maxb) blocks = maxb;
    if (blocks < 1) blocks = 1;
    k_gemv_rows_bulk<K, M><<<(unsigned)blocks, GEMV_THREADS, smem, st>>>(packed, N, Kc, so, x, y, meta, per_row, act,
                                                                          lda, out, ldo);
    return launch_status();
}

int g_gemv_bulk = 1;   // A/B: 0 = register-pipelined kernel for every shape

template <int K, int M>
exmy_status launch_gemv_km(const uint8_t *packed, int64_t N, int64_t Kc, const SegOffsets &so, int x, int y,
                           const uint8_t *meta, int per_row, const float *act, int64_t lda, float *out, int64_t ldo,
                           cudaStream_t st) {
    if (g_gemv_bulk && Kc % 16 == 0 && aligned(packed, 16))
        return launch_gemv_bulk<K, M>(packed, N, Kc, so, x, y, meta, per_row, act, lda, out, ldo, st);
    constexpr int smem = 2 * (128 << K);   // the table plus its alignment slack
    static unsigned long long configured = 0;
    static int occ = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !(configured & (1ull << dev))) {
        cudaFuncSetAttribute(k_gemv_rows<K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        occ = occupancy(k_gemv_rows<K, M>, GEMV_THREADS, smem);
        if (dev >= 0 && dev < 64) configured |= 1ull << dev;
    }
    int64_t blocks = N / 8;
    const int64_t maxb = (int64_t)num_sms() * (occ > 0 ? occ : 1);
    if (blocks > maxb) blocks = maxb;   // persistent: the table is built once per CTA
    if (blocks < 1) blocks = 1;
    k_gemv_rows<K, M><<<(unsigned)blocks, GEMV_THREADS, smem, st>>>(packed, N, Kc, so, x, y, meta, per_row, act, lda,
                                                                     out, ldo);
    return launch_status();
}

template <int K>
exmy_status launch_gemv_k(const uint8_t *packed, int64_t N, int64_t Kc, const SegOffsets &so, int x, int y,
                          const uint8_t *meta, int per_row, const float *act, int64_t M, float *out, cudaStream_t st) {
    // passes of <= 8 activation rows; each pass reads the packed matrix once
    for (int64_t m0 = 0; m0 < M;) {
        const int64_t left = M - m0;
        const int mm = left >= 8 ? 8 : (left >= 4 ? 4 : (left >= 2 ? 2 : 1));
        const float *a = act + m0 * Kc;
        float *o = out + m0 * N;
        exmy_status s;
        switch (mm) {
            case 8: s = launch_gemv_km<K, 8>(packed, N, Kc, so, x, y, meta, per_row, a, Kc, o, N, st); break;
            case 4: s = launch_gemv_km<K, 4>(packed, N, Kc, so, x, y, meta, per_row, a, Kc, o, N, st); break;
            case 2: s = launch_gemv_km<K, 2>(packed, N, Kc, so, x, y, meta, per_row, a, Kc, o, N, st); break;
            default: s = launch_gemv_km<K, 1>(packed, N, Kc, so, x, y, meta, per_row, a, Kc, o, N, st); break;
        }
        if (s != EXMY_OK) return s;
        m0 += mm;
    }
    return EXMY_OK;
}

}  // namespace

extern "C" int exmy_debug_gemv_bulk(int on) {
    const int prev = g_gemv_bulk;
    if (on >= 0) g_gemv_bulk = on;
    return prev;
}

extern "C" exmy_status exmy_gemv(const uint8_t *packed, int64_t rows, int64_t cols, int x, int y,
                                 const uint8_t *meta, int meta_per_row, const int64_t *sp_index,
                                 const uint32_t *sp_bits, const unsigned long long *sp_count, int64_t sp_capacity,
                                 const float *act, int64_t m, float *out, void *stream) {
    if (!gemv_fmt_ok(x, y)) return EXMY_E_FORMAT;
    const int k = 1 + x + y;
    if (k > 8) return EXMY_E_FORMAT;   // the table holds 2^k codes; k = 9 is not supported here
    if (rows < 0 || cols < 0 || m < 0 || rows % 8 || cols % 4) return EXMY_E_SHAPE;
    if (cols && rows > INT64_MAX / cols) return EXMY_E_SHAPE;
    if (rows == 0 || m == 0) return EXMY_OK;
    if (!packed || !meta || !act || !out) return EXMY_E_ARG;
    if (sp_capacity < 0 || (sp_capacity > 0 && (!sp_index || !sp_bits || !sp_count))) return EXMY_E_ARG;
    if (!aligned(packed, 16) || !aligned(act, 16)) return EXMY_E_ALIGN;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (cols == 0) return cudaMemsetAsync(out, 0, (size_t)(m * rows) * sizeof(float), st) == cudaSuccess
                              ? EXMY_OK : EXMY_E_CUDA;
    const Plan p = make_plan(k, rows * cols);
    for (int s = 0; s < p.nseg; ++s)
        if (!aligned(packed + p.so.off[s], 4)) return EXMY_E_ALIGN;
    exmy_status s = EXMY_E_FORMAT;
    switch (k) {
#define GEMV_K(KK) \
        case KK: s = launch_gemv_k<KK>(packed, rows, cols, p.so, x, y, meta, meta_per_row != 0, act, m, out, st); break;
        GEMV_K(3) GEMV_K(4) GEMV_K(5) GEMV_K(6) GEMV_K(7) GEMV_K(8)
#undef GEMV_K
    }
    if (s != EXMY_OK || sp_capacity == 0) return s;
    const int64_t work = sp_capacity * m;
    int64_t blocks = (work + 255) / 256;
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    k_gemv_specials<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, st>>>(sp_index, sp_bits, sp_count, sp_capacity,
                                                                          cols, act, cols, m, out, rows);
    return launch_status();
}
