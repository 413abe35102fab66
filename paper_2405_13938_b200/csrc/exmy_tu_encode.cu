// exmy_tu_encode.cu -- K3 encode launchers (+ K5 specials list).
#include "exmy_launch.cuh"
#include "exmy_tma.cuh"

namespace exmy {

namespace {
template <int K, bool BF16, int MODE>
exmy_status launch_encode_km(const uint8_t *in, int64_t R, int64_t C, int axis, int x, int y, const uint8_t *meta,
                            uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb,
                            unsigned long long *spc, int64_t cap, cudaStream_t st, const SpecialsRanges &sr) {
    const int64_t n = R * C;
    // a full workspace (sr.defer): NaN/Inf tiles are left to the fix-up pass
    unsigned long long *flag = sr.defer ? spc + FIXUP_FLAG_WORD : nullptr;
    bool vec = aligned(in, 16);
    if (axis == EXMY_AXIS_ROWS) {
        // thread tile = 8 rows x 4 columns: 4-element row chunks, 4*w-byte segment stores
        // (8 rows of one row group must span < 4 GiB: the kernel uses 32-bit row offsets)
        vec = aligned(in, 4 * Elem<BF16>::ES) && (C % 4 == 0) && (8 * C * Elem<BF16>::ES <= (int64_t)UINT32_MAX);
        for (int s = 0; s < p.nseg; ++s) vec = vec && aligned(packed + p.so.off[s], p.w[s] == 8 ? 4 : 4 * p.w[s]);
        if (vec && g_enc_tma && aligned(in, 16) && (C % 8 == 0)) {
            // TMA-staged persistent kernel (exmy_tma.cuh): bulk copies need 16-byte rows / offsets
            constexpr int smem = etma_smem<BF16>();
            static int occ = 0;
            if (!occ) {
                cudaFuncSetAttribute(k_enc_rows_tma<K, BF16, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                occ = occupancy(k_enc_rows_tma<K, BF16, MODE>, ETMA_THREADS, smem);
            }
            const int64_t T = (R / 8) * cdiv(C, ETMA_TC);
            int64_t blocks = (int64_t)num_sms() * (occ > 0 ? occ : 1);
            if (blocks > T) blocks = T;
            if (blocks < 1) blocks = 1;
            k_enc_rows_tma<K, BF16, MODE><<<(unsigned)blocks, ETMA_THREADS, smem, st>>>(
                in, R, C, x, y, meta, packed, p.so, spi, spb, spc, cap, g_force_generic);
            return launch_status();
        }
        if (vec) {
            const int threads = BF16 ? EXMY_ENC_ROWS_THREADS : 256;
            static int occ = 0;
            if (!occ) occ = occupancy(k_enc_rows_fast<K, BF16, MODE>, threads, 0);
            const int64_t CV = C / 4, G = R / 8;
            int64_t gx = cdiv(CV, threads);
#ifdef ENC_OCC_CAP   // A/B experiments: CTAs per SM
            int64_t target = (int64_t)num_sms() * (occ < ENC_OCC_CAP ? occ : ENC_OCC_CAP);
#else
            int64_t target = (int64_t)num_sms() * occ;
#endif
            int64_t gy = target / gx;
            if (gy < 1) gy = 1;
            if (gy > G) gy = G;
            if (gy > 65535) gy = 65535;
            if (gx > INT_MAX) return EXMY_E_SHAPE;
            k_enc_rows_fast<K, BF16, MODE><<<dim3((unsigned)gx, (unsigned)gy), threads, 0, st>>>(
                in, R, C, x, y, meta, packed, p.so, spi, spb, spc, cap, g_force_generic, flag);
            if (flag) {
                const int64_t fx = cdiv(CV, 256);
                int64_t fy = (int64_t)num_sms() * 4 / fx;
                if (fy < 1) fy = 1;
                if (fy > G) fy = G;
                if (fy > 65535) fy = 65535;
                k_enc_rows_fixup<K, BF16, MODE><<<dim3((unsigned)fx, (unsigned)fy), 256, 0, st>>>(
                    in, R, C, x, y, meta, packed, p.so, spc, sr.lg_rows);
            }
            return launch_status();
        }
    } else {
        for (int s = 0; s < p.nseg; ++s) vec = vec && aligned(packed + p.so.off[s], p.w[s]);
        if (vec) {
            const int threads = 256;
            static int occ = 0;
            if (!occ) occ = occupancy(k_enc_cols_fast<K, BF16, MODE>, threads, 0);
            int64_t tiles = cdiv(n / 8, 128);
            int64_t blocks = cdiv(tiles, threads / 32);
            int64_t maxb = (int64_t)num_sms() * occ;
            if (blocks > maxb) blocks = maxb;
            k_enc_cols_fast<K, BF16, MODE><<<(unsigned)blocks, threads, 0, st>>>(in, n, x, y, meta, packed, p.so, spi,
                                                                           spb, spc, cap, g_force_generic, flag);
            if (flag)
                k_enc_cols_fixup<K, BF16, MODE><<<(unsigned)blocks, threads, 0, st>>>(in, n, x, y, meta, packed, p.so,
                                                                                spc, sr.lg_cols);
            return launch_status();
        }
    }
    const int64_t ncont = n / 8;
    int64_t blocks = cdiv(ncont, 256);
    int64_t maxb = (int64_t)num_sms() * 8;
    if (blocks > maxb) blocks = maxb;
    k_encode_generic<BF16><<<(unsigned)blocks, 256, 0, st>>>(in, C, ncont, axis, x, y, meta, packed, p.so, p.nseg,
                                                             make_int4(p.w[0], p.w[1], p.w[2], p.w[3]), spi, spb,
                                                             spc, cap);
    return launch_status();
}

// encode mode from (dtype, y): bf16 SIMD pairs for y <= 6, per-element fp32 otherwise
template <int K, bool BF16>
exmy_status launch_encode_k(const uint8_t *in, int64_t R, int64_t C, int axis, int x, int y, const uint8_t *meta,
                            uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb,
                            unsigned long long *spc, int64_t cap, cudaStream_t st, const SpecialsRanges &sr) {
    if (BF16 && y <= 6) {
        if (y == 0)
            return launch_encode_km<K, BF16, (BF16 ? ENC_SIMD_Y0 : ENC_F32_Y0)>(in, R, C, axis, x, y, meta, packed, p,
                                                                               spi, spb, spc, cap, st, sr);
        return launch_encode_km<K, BF16, (BF16 ? ENC_SIMD : ENC_F32)>(in, R, C, axis, x, y, meta, packed, p, spi, spb,
                                                                     spc, cap, st, sr);
    }
    if (y == 0)
        return launch_encode_km<K, BF16, ENC_F32_Y0>(in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr);
    return launch_encode_km<K, BF16, ENC_F32>(in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr);
}

template <bool BF16>
exmy_status encode_dispatch(int k, const uint8_t *in, int64_t R, int64_t C, int axis, int x, int y,
                            const uint8_t *meta, uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb,
                            unsigned long long *spc, int64_t cap, cudaStream_t st, const SpecialsRanges &sr) {
    switch (k) {
        case 3: return launch_encode_k<3, BF16>(in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr);
        case 4: return launch_encode_k<4, BF16>(in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr);
        case 5: return launch_encode_k<5, BF16>(in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr);
        case 6: return launch_encode_k<6, BF16>(in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr);
        case 7: return launch_encode_k<7, BF16>(in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr);
        case 8: return launch_encode_k<8, BF16>(in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr);
        case 9: return launch_encode_k<9, BF16>(in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr);
    }
    return EXMY_E_FORMAT;
}

}  // namespace

exmy_status launch_encode(const uint8_t *in, bool bf16, int64_t R, int64_t C, int axis, int x, int y,
                          const uint8_t *meta, uint8_t *packed, int64_t *spi, uint32_t *spb,
                          unsigned long long *spc, int64_t cap, cudaStream_t st, const SpecialsRanges &sr) {
    const int k = 1 + x + y;
    Plan p = make_plan(k, R * C);
    return bf16 ? encode_dispatch<true>(k, in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr)
                : encode_dispatch<false>(k, in, R, C, axis, x, y, meta, packed, p, spi, spb, spc, cap, st, sr);
}

SpecialsRanges specials_ranges(int64_t R, int64_t C, bool defer) {
    SpecialsRanges sr;
    sr.defer = defer;
    const int64_t G = R / 8, n = R * C;
    sr.lg_rows = 0;   // ROWS fix-up: ranges of 8 C 2^lg_rows elements (whole row groups)
    while (cdiv(G, (int64_t)1 << sr.lg_rows) > SPECIALS_RANGES) ++sr.lg_rows;
    sr.lg_cols = 10;  // COLS fix-up: ranges of 2^lg_cols >= 1024 elements (whole warp tiles)
    while (cdiv(n, (int64_t)1 << sr.lg_cols) > SPECIALS_RANGES) ++sr.lg_cols;
    return sr;
}

exmy_status launch_specials_sort(int64_t *spi, uint32_t *spb, const unsigned long long *spc, int64_t cap,
                                 cudaStream_t st) {
    k_specials_sort<<<1, 1024, 0, st>>>(spi, spb, spc, cap);
    return launch_status();
}

// the index-ordered specials list of a tensor of n elements (see
// k_specials_count / k_specials_write); ws = the sp_count workspace whose
// word 0 the encode kernel filled with the total count
exmy_status launch_specials_compact(const uint8_t *in, bool bf16, int64_t n, int64_t elem_offset, int64_t *spi,
                                    uint32_t *spb, unsigned long long *ws, int64_t cap, cudaStream_t st,
                                    int64_t L) {
    if (n <= 0 || cap <= 0 || !spi || !spb || !ws) return EXMY_OK;
    int64_t nr;
    if (L <= 0) {   // any range length that is a multiple of 8 works when the ranges are counted here
        nr = cdiv(n, 8192);
        if (nr > SPECIALS_RANGES) nr = SPECIALS_RANGES;
        if (nr < 1) nr = 1;
        L = cdiv(cdiv(n, nr), 8) * 8;
    }
    nr = cdiv(n, L);
    static int occ_b = 0, occ_f = 0;
    if (!occ_b) occ_b = occupancy(k_specials_compact<true>, 256, 0);
    if (!occ_f) occ_f = occupancy(k_specials_compact<false>, 256, 0);
    int64_t grid = (int64_t)num_sms() * (bf16 ? occ_b : occ_f);   // co-resident: the grid barrier needs it
    if (grid > nr) grid = nr;
    if (grid < 1) grid = 1;
    int nri = (int)nr;
    void *args[] = {(void *)&in, (void *)&n, (void *)&L, (void *)&nri, (void *)&elem_offset, (void *)&ws,
                    (void *)&spi, (void *)&spb, (void *)&cap};
    const void *fn = bf16 ? (const void *)k_specials_compact<true> : (const void *)k_specials_compact<false>;
    if (cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(256), args, 0, st) != cudaSuccess)
        return EXMY_E_CUDA;
    return EXMY_OK;
}

}  // namespace exmy
