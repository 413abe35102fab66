// exmy_tu_hist.cu -- K1 exponent histogram + K1b e_max launchers.
#include "exmy_launch.cuh"

namespace exmy {

namespace {
template <bool BF16, int MODE>
exmy_status launch_hist_vec(const uint8_t *in, int64_t n, unsigned long long *hist, cudaStream_t st) {
    // the opt-in shared-memory size is a per-device function attribute
    static unsigned long long configured = 0;
    static int occ = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !(configured & (1ull << dev))) {
        cudaFuncSetAttribute(k_hist<BF16, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, HIST_SMEM);
        occ = occupancy(k_hist<BF16, MODE>, HIST_THREADS, HIST_SMEM);
        if (dev >= 0 && dev < 64) configured |= 1ull << dev;
    }
    const int64_t nvec = n / Elem<BF16>::V;
    int64_t blocks = cdiv(cdiv(nvec, 32 * HIST_U), HIST_WARPS);
    if (blocks < 1) blocks = 1;
    int64_t maxb = (int64_t)num_sms() * occ;
    if (blocks > maxb) blocks = maxb;
    if (g_hist_blocks > 0 && blocks > g_hist_blocks) blocks = g_hist_blocks;   // test knob: long per-lane runs
    k_hist<BF16, MODE><<<(unsigned)blocks, HIST_THREADS, HIST_SMEM, st>>>(in, n, hist);
    return launch_status();
}

#ifndef HIST4_U
#define HIST4_U 4   // 16-byte vectors per lane per iteration (double-buffered)
#endif
// MODE 4: CTA-shared lane-column counters (k_hist_cta); returns
// EXMY_E_SHAPE when a CTA's share could overflow its 32-bit counters
template <bool BF16>
exmy_status launch_hist_cta(const uint8_t *in, int64_t n, unsigned long long *hist, cudaStream_t st) {
    static unsigned long long configured = 0;
    static int occ = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !(configured & (1ull << dev))) {
        cudaFuncSetAttribute(k_hist_cta<BF16, HIST4_U>, cudaFuncAttributeMaxDynamicSharedMemorySize, HIST4_SMEM);
        occ = occupancy(k_hist_cta<BF16, HIST4_U>, HIST4_THREADS, HIST4_SMEM);
        if (dev >= 0 && dev < 64) configured |= 1ull << dev;
    }
    const int64_t nvec = n / Elem<BF16>::V;
    int64_t blocks = cdiv(cdiv(nvec, 32 * HIST4_U), HIST4_THREADS / 32);
    if (blocks < 1) blocks = 1;
    int64_t maxb = (int64_t)num_sms() * occ;
    if (blocks > maxb) blocks = maxb;
    if (g_hist_blocks > 0 && blocks > g_hist_blocks) blocks = g_hist_blocks;
    if (cdiv(n, blocks) + 64 >= (int64_t)UINT32_MAX) return EXMY_E_SHAPE;
    k_hist_cta<BF16, HIST4_U><<<(unsigned)blocks, HIST4_THREADS, HIST4_SMEM, st>>>(in, n, hist);
    return launch_status();
}

}  // namespace

exmy_status launch_histogram(const uint8_t *in, bool bf16, int64_t n, unsigned long long *hist, cudaStream_t st) {
    if (!aligned(in, 16)) {
        int64_t blocks = cdiv(n, 256);
        if (blocks > (int64_t)num_sms() * 4) blocks = (int64_t)num_sms() * 4;
        if (bf16) k_hist_scalar<true><<<(unsigned)blocks, 256, 0, st>>>(in, n, hist);
        else k_hist_scalar<false><<<(unsigned)blocks, 256, 0, st>>>(in, n, hist);
        return launch_status();
    }
    if (g_hist_mode == 4) {
        const exmy_status r = bf16 ? launch_hist_cta<true>(in, n, hist, st) : launch_hist_cta<false>(in, n, hist, st);
        if (r != EXMY_E_SHAPE) return r;   // else: the 16-bit epoch kernel below
    }
    switch (g_hist_mode) {
        case 4:
        case 3: return bf16 ? launch_hist_vec<true, 3>(in, n, hist, st) : launch_hist_vec<false, 3>(in, n, hist, st);
        case 0: return bf16 ? launch_hist_vec<true, 0>(in, n, hist, st) : launch_hist_vec<false, 0>(in, n, hist, st);
        case 2: return bf16 ? launch_hist_vec<true, 2>(in, n, hist, st) : launch_hist_vec<false, 2>(in, n, hist, st);
        default: return bf16 ? launch_hist_vec<true, 1>(in, n, hist, st) : launch_hist_vec<false, 1>(in, n, hist, st);
    }
}

exmy_status launch_max_exponent(const uint8_t *in, bool bf16, int64_t n, uint8_t *meta, cudaStream_t st) {
    if (cudaMemsetAsync(meta, 0, 1, st) != cudaSuccess) return EXMY_E_CUDA;
    const int64_t nvec = n / (bf16 ? 8 : 4);
    int64_t blocks = cdiv(nvec, 1024);   // 16 KB chunks
    if (blocks < 1) blocks = 1;
    static int occ = 0;
    if (!occ) occ = occupancy(k_max_exp<true>, 256, 0);
    if (blocks > (int64_t)num_sms() * occ) blocks = (int64_t)num_sms() * occ;
    if (bf16) k_max_exp<true><<<(unsigned)blocks, 256, 0, st>>>(in, n, meta);
    else k_max_exp<false><<<(unsigned)blocks, 256, 0, st>>>(in, n, meta);
    return launch_status();
}

exmy_status launch_emax(const unsigned long long *hist, uint8_t *meta, cudaStream_t st) {
    k_emax<<<1, 256, 0, st>>>(hist, meta);
    return launch_status();
}

}  // namespace exmy
