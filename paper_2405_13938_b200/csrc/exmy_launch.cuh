// exmy_launch.cuh -- host-side helpers shared by the translation units and
// the internal launcher entry points (one TU per op family).
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "exmy.h"
#include "exmy_blocked.cuh"

namespace exmy {

extern int g_force_generic;   // exmy_debug_force_generic
extern int g_hist_mode;       // exmy_debug_hist_mode
extern int g_hist_blocks;     // exmy_debug_hist_blocks
extern int g_enc_tma;         // exmy_debug_enc_tma: ROWS encode through the TMA-staged kernel
extern int g_rowwise_cluster; // exmy_debug_rowwise_cluster: wide-row fused per-row encode on clusters

inline int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}

template <typename KF>
inline int occupancy(KF kernel, int threads, size_t smem) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess || b < 1) b = 1;
    return b;
}

inline exmy_status launch_status() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? EXMY_OK : EXMY_E_CUDA;
}

inline bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Plan {
    int nseg;
    int w[4];
    SegOffsets so;
};

inline Plan make_plan(int k, int64_t n) {
    Plan p{};
    int64_t off = 0;
    for (int w = 8; w >= 1; w >>= 1) {
        if (k & w) {
            p.w[p.nseg] = w;
            p.so.off[p.nseg] = off;
            off += n * w / 8;
            ++p.nseg;
        }
    }
    return p;
}

// launchers (arguments already validated by the ABI layer)
exmy_status launch_histogram(const uint8_t *in, bool bf16, int64_t n, unsigned long long *hist, cudaStream_t st);
exmy_status launch_max_exponent(const uint8_t *in, bool bf16, int64_t n, uint8_t *meta, cudaStream_t st);
exmy_status launch_emax(const unsigned long long *hist, uint8_t *meta, cudaStream_t st);
exmy_status launch_quantize(const uint8_t *in, uint8_t *out, bool bf16, int64_t n, int x, int y,
                            const uint8_t *meta, cudaStream_t st);
// NaN/Inf range bookkeeping of a per-tensor encode (see k_enc_rows_fixup)
struct SpecialsRanges {
    bool defer = false;   // the workspace is full-size: fast kernels defer NaN/Inf tiles to the fix-up pass
    int lg_rows = 0;      // ROWS: range = row group >> lg_rows
    int lg_cols = 10;     // COLS: range = element >> lg_cols
    int64_t len(int axis, int64_t C) const {
        return axis == EXMY_AXIS_ROWS ? 8 * C * ((int64_t)1 << lg_rows) : ((int64_t)1 << lg_cols);
    }
};
SpecialsRanges specials_ranges(int64_t R, int64_t C, bool defer);
exmy_status launch_encode(const uint8_t *in, bool bf16, int64_t R, int64_t C, int axis, int x, int y,
                          const uint8_t *meta, uint8_t *packed, int64_t *spi, uint32_t *spb,
                          unsigned long long *spc, int64_t cap, cudaStream_t st, const SpecialsRanges &sr);
exmy_status launch_specials_sort(int64_t *spi, uint32_t *spb, const unsigned long long *spc, int64_t cap,
                                 cudaStream_t st);
exmy_status launch_specials_compact(const uint8_t *in, bool bf16, int64_t n, int64_t elem_offset, int64_t *spi,
                                    uint32_t *spb, unsigned long long *ws, int64_t cap, cudaStream_t st,
                                    int64_t L = 0);
exmy_status launch_decode(const uint8_t *packed, int64_t R, int64_t C, int axis, int x, int y,
                          const uint8_t *meta, uint8_t *out, bool obf16, cudaStream_t st);
exmy_status launch_specials_scatter(const int64_t *spi, const uint32_t *spb, const unsigned long long *spc,
                                    int64_t cap, uint8_t *out, bool obf16, cudaStream_t st);

// block metadata
exmy_status launch_block_max(const uint8_t *in, bool bf16, int64_t R, int64_t C, int64_t br, int64_t bc, int y,
                             int scheme, uint8_t *meta, cudaStream_t st);
exmy_status launch_quantize_blocked(const uint8_t *in, uint8_t *out, bool bf16, int64_t R, int64_t C, int64_t br,
                                    int64_t bc, int x, int y, const uint8_t *meta, cudaStream_t st);
exmy_status launch_encode_blocked(const uint8_t *in, bool bf16, int64_t R, int64_t C, int axis, int64_t br,
                                  int64_t bc, int x, int y, const uint8_t *meta, uint8_t *packed, int64_t *spi,
                                  uint32_t *spb, unsigned long long *spc, int64_t cap, cudaStream_t st);
exmy_status launch_decode_blocked(const uint8_t *packed, int64_t R, int64_t C, int axis, int64_t br, int64_t bc,
                                  int x, int y, const uint8_t *meta, uint8_t *out, bool obf16, cudaStream_t st);
exmy_status launch_encode_rowwise(const uint8_t *in, bool bf16, int64_t R, int64_t C, int x, int y, int scheme,
                                  uint8_t *meta, uint8_t *packed, int64_t *spi, uint32_t *spb,
                                  unsigned long long *spc, int64_t cap, cudaStream_t st);
exmy_status launch_decode_rows_gather(const uint8_t *packed, int64_t R, int64_t C, int x, int y, const uint8_t *meta,
                                      bool per_row, const int64_t *idx, int64_t nidx, uint8_t *out, bool obf16,
                                      cudaStream_t st);

}  // namespace exmy
