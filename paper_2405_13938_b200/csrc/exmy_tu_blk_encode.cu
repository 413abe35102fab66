// exmy_tu_blk_encode.cu -- encode with block metadata launchers.
#include "exmy_launch.cuh"
#include "exmy_narrow.cuh"

#ifndef RWS_ENABLE
#define RWS_ENABLE 1   // TMA-staged fused per-row encode for rows <= RWS_MAX_ROW_BYTES
#endif

namespace exmy {

namespace {
template <int K, bool BF16, int MODE>
exmy_status launch_enc_blk_km(const uint8_t *in, int64_t R, int64_t C, int axis, int x, int y, const MetaMap &M,
                              uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb, unsigned long long *spc,
                              int64_t cap, cudaStream_t st) {
    const int64_t n = R * C;
    if (axis == EXMY_AXIS_ROWS) {
        bool vec = aligned(in, 4 * Elem<BF16>::ES) && (C % 4 == 0) && (M.bc % 4 == 0) &&
                   (M.br == 1 || M.br % 8 == 0);
        for (int s = 0; s < p.nseg; ++s) vec = vec && aligned(packed + p.so.off[s], p.w[s] == 8 ? 4 : 4 * p.w[s]);
        if (vec && M.br == 1 && M.nbc == 1 && aligned(M.meta, 8) && 8 * C * Elem<BF16>::ES <= (int64_t)UINT32_MAX) {
            // one byte per row: the rows' constants built once per warp (k_enc_rows_rowmeta)
            const int threads = 256;
            static int occ = 0;
            if (!occ) occ = occupancy(k_enc_rows_rowmeta<K, BF16, MODE>, threads, 0);
            const int64_t CV = C / 4, G = R / 8;
            int64_t gx = cdiv(CV, threads);
            int64_t gy = (int64_t)num_sms() * occ / gx;
            if (gy < 1) gy = 1;
            if (gy > G) gy = G;
            if (gy > 65535) gy = 65535;
            if (gx > INT_MAX) return EXMY_E_SHAPE;
            k_enc_rows_rowmeta<K, BF16, MODE><<<dim3((unsigned)gx, (unsigned)gy), threads, 0, st>>>(
                in, R, C, x, y, M.meta, packed, p.so, spi, spb, spc, cap, g_force_generic, M);
            return launch_status();
        }
        if (vec) {
            const int threads = 256;
            static int occ = 0;
            if (!occ) occ = occupancy(k_enc_rows_blk<K, BF16, MODE>, threads, 0);
            const int64_t CV = C / 4, G = R / 8;
            int64_t gx = cdiv(CV, threads);
            int64_t gy = (int64_t)num_sms() * occ / gx;
            if (gy < 1) gy = 1;
            if (gy > G) gy = G;
            if (gy > 65535) gy = 65535;
            if (gx > INT_MAX) return EXMY_E_SHAPE;
            k_enc_rows_blk<K, BF16, MODE><<<dim3((unsigned)gx, (unsigned)gy), threads, 0, st>>>(
                in, R, C, x, y, M, packed, p.so, spi, spb, spc, cap, g_force_generic);
            return launch_status();
        }
    } else {
        bool vec = aligned(in, 16) && (M.bc % 8 == 0);
        for (int s = 0; s < p.nseg; ++s) vec = vec && aligned(packed + p.so.off[s], p.w[s]);
        // one byte per row of 64 .. 512 columns (embedding tables): the narrow-row kernel
        const int64_t gpr = C / 8;
        const int lg = (gpr >= 8 && gpr <= 64 && (gpr & (gpr - 1)) == 0) ? __builtin_ctzll((unsigned long long)gpr) : -1;
        if (vec && lg >= 0 && M.br == 1 && M.bc == C && aligned(M.meta, (size_t)(128 >> lg))) {
            int64_t blocks = cdiv(cdiv(n / 8, 128), 256 / 32);
            const int64_t maxb = (int64_t)num_sms() * 2;
            if (blocks > maxb) blocks = maxb;
#define EXMY_NARROW_ENC(LG)                                                                                    \
    k_enc_cols_narrow<K, BF16, MODE, LG><<<(unsigned)blocks, 256, 0, st>>>(in, n, x, y, M.meta, packed, p.so, spi, \
                                                                          spb, spc, cap, M, C, g_force_generic)
            switch (lg) {
                case 3: EXMY_NARROW_ENC(3); break;
                case 4: EXMY_NARROW_ENC(4); break;
                case 5: EXMY_NARROW_ENC(5); break;
                default: EXMY_NARROW_ENC(6); break;
            }
#undef EXMY_NARROW_ENC
            return launch_status();
        }
        if (vec) {
            const int threads = 256;
            static int occ = 0;
            if (!occ) occ = occupancy(k_enc_cols_blk<K, BF16, MODE>, threads, 0);
            int64_t blocks = cdiv(cdiv(n / 8, 128), threads / 32);
            int64_t maxb = (int64_t)num_sms() * occ;
            if (blocks > maxb) blocks = maxb;
            k_enc_cols_blk<K, BF16, MODE><<<(unsigned)blocks, threads, 0, st>>>(in, n, C, x, y, M, packed, p.so, spi,
                                                                                spb, spc, cap, g_force_generic);
            return launch_status();
        }
    }
    const int64_t ncont = n / 8;
    int64_t blocks = cdiv(ncont, 256);
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    k_encode_generic_blk<BF16, K><<<(unsigned)blocks, 256, 0, st>>>(in, C, ncont, axis, x, y, M, packed, p.so, spi,
                                                                    spb, spc, cap);
    return launch_status();
}

template <int K, bool BF16>
exmy_status launch_enc_blk_k(const uint8_t *in, int64_t R, int64_t C, int axis, int x, int y, const MetaMap &M,
                             uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb, unsigned long long *spc,
                             int64_t cap, cudaStream_t st) {
    if (BF16 && y <= 6) {
        if (y == 0)
            return launch_enc_blk_km<K, BF16, (BF16 ? ENC_SIMD_Y0 : ENC_F32_Y0)>(in, R, C, axis, x, y, M, packed, p,
                                                                                 spi, spb, spc, cap, st);
        return launch_enc_blk_km<K, BF16, (BF16 ? ENC_SIMD : ENC_F32)>(in, R, C, axis, x, y, M, packed, p, spi, spb,
                                                                       spc, cap, st);
    }
    if (y == 0)
        return launch_enc_blk_km<K, BF16, ENC_F32_Y0>(in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st);
    return launch_enc_blk_km<K, BF16, ENC_F32>(in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st);
}

template <bool BF16>
exmy_status enc_blk_dispatch(int k, const uint8_t *in, int64_t R, int64_t C, int axis, int x, int y,
                             const MetaMap &M, uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb,
                             unsigned long long *spc, int64_t cap, cudaStream_t st) {
    switch (k) {
        case 3: return launch_enc_blk_k<3, BF16>(in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st);
        case 4: return launch_enc_blk_k<4, BF16>(in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st);
        case 5: return launch_enc_blk_k<5, BF16>(in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st);
        case 6: return launch_enc_blk_k<6, BF16>(in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st);
        case 7: return launch_enc_blk_k<7, BF16>(in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st);
        case 8: return launch_enc_blk_k<8, BF16>(in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st);
        case 9: return launch_enc_blk_k<9, BF16>(in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st);
    }
    return EXMY_E_FORMAT;
}
template <int K, bool BF16, int MODE>
exmy_status launch_rowwise_km(const uint8_t *in, int64_t R, int64_t C, int x, int y, int scheme, uint8_t *meta,
                              uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb, unsigned long long *spc,
                              int64_t cap, cudaStream_t st) {
#if RWS_ENABLE
    const int64_t rowb = C * Elem<BF16>::ES;
    // wide rows: a cluster of CL CTAs stages a row group in column slabs (distributed shared memory);
    // two stages per CTA (the next row group's slab in flight) when 2 x 8 slab rows fit in 72 KB
    int cl = 0;
    for (int c : {2, 4, 8})
        if (!cl && rowb > RWS_MAX_ROW_BYTES && rowb % (16 * c) == 0 && rowb / c <= RWS_MAX_ROW_BYTES &&
            C % (4 * c) == 0 && g_rowwise_cluster)
            cl = c;
    if (cl && rowb / 8 <= RWS_MAX_ROW_BYTES / 2 && rowb % (16 * 8) == 0 && C % 32 == 0) cl = 8;   // prefer 2 stages
    if (cl) {
        const int nst = (2 * (rowb / cl) <= RWS_MAX_ROW_BYTES) ? 2 : 1;
        const size_t sm = (size_t)(nst * 8 * (rowb / cl));
        // per (kernel variant, device) configuration: the kernels share one pointer type
        static unsigned long long configured[18] = {0};
        static int occ_cl[18] = {0};
        auto launch = [&](auto kern, int CLv, int slot) -> exmy_status {
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev < 0 || dev >= 64 || !(configured[slot] & (1ull << dev))) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(8 * RWS_MAX_ROW_BYTES));
                occ_cl[slot] = occupancy(kern, RWS_THREADS, 8 * RWS_MAX_ROW_BYTES);
                if (dev >= 0 && dev < 64) configured[slot] |= 1ull << dev;
            }
            const int occ_c = occ_cl[slot];
            int64_t blocks = (int64_t)num_sms() * (occ_c > 0 ? occ_c : 1);
            if (blocks > (R / 8) * CLv) blocks = (R / 8) * CLv;
            blocks = blocks / CLv * CLv;
            if (blocks < CLv) blocks = CLv;
            kern<<<(unsigned)blocks, RWS_THREADS, sm, st>>>(in, R, C, x, y, scheme, meta, packed, p.so, spi, spb, spc,
                                                          cap, g_force_generic);
            return launch_status();
        };
        if (nst == 2) {
            if (cl == 2) return launch(k_enc_rowwise_cluster<K, BF16, MODE, 2, 2>, 2, 0);
            if (cl == 4) return launch(k_enc_rowwise_cluster<K, BF16, MODE, 4, 2>, 4, 1);
            return launch(k_enc_rowwise_cluster<K, BF16, MODE, 8, 2>, 8, 2);
        }
        if (cl == 2) return launch(k_enc_rowwise_cluster<K, BF16, MODE, 2, 1>, 2, 3);
        if (cl == 4) return launch(k_enc_rowwise_cluster<K, BF16, MODE, 4, 1>, 4, 4);
        return launch(k_enc_rowwise_cluster<K, BF16, MODE, 8, 1>, 8, 5);
    }
    if (rowb % 16 == 0 && rowb <= RWS_MAX_ROW_BYTES) {   // TMA-staged: each row group read from HBM once
        const size_t sm = (size_t)(8 * rowb);
        static unsigned long long configured = 0;
        static int occ_s = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !(configured & (1ull << dev))) {
            cudaFuncSetAttribute(k_enc_rowwise_smem<K, BF16, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(8 * RWS_MAX_ROW_BYTES));
            occ_s = occupancy(k_enc_rowwise_smem<K, BF16, MODE>, RWS_THREADS, 8 * RWS_MAX_ROW_BYTES);
            if (dev >= 0 && dev < 64) configured |= 1ull << dev;
        }
        const int occ_now = occupancy(k_enc_rowwise_smem<K, BF16, MODE>, RWS_THREADS, sm);
        int64_t blocks = (int64_t)num_sms() * (occ_now > 0 ? occ_now : (occ_s > 0 ? occ_s : 1));
        if (blocks > R / 8) blocks = R / 8;
        if (blocks < 1) blocks = 1;
        k_enc_rowwise_smem<K, BF16, MODE><<<(unsigned)blocks, RWS_THREADS, sm, st>>>(
            in, R, C, x, y, scheme, meta, packed, p.so, spi, spb, spc, cap, g_force_generic);
        return launch_status();
    }
#endif
    static int occ = 0;
    if (!occ) occ = occupancy(k_enc_rowwise_rows<K, BF16, MODE>, RW_THREADS, 0);
    // the two passes of a row group must meet in L2: bound the CTAs in flight
    // so that their working sets (16*C bytes bf16, 32*C fp32) stay well inside it
    const int64_t ws = 8 * C * Elem<BF16>::ES;
    int64_t maxb = (int64_t)(48ll << 20) / (ws > 0 ? ws : 1);
    const int64_t fill = (int64_t)num_sms() * occ;
    if (maxb > fill) maxb = fill;
    if (maxb < num_sms()) maxb = num_sms();
    int64_t blocks = R / 8;
    if (blocks > maxb) blocks = maxb;
    k_enc_rowwise_rows<K, BF16, MODE><<<(unsigned)blocks, RW_THREADS, 0, st>>>(in, R, C, x, y, scheme, meta, packed,
                                                                               p.so, spi, spb, spc, cap,
                                                                               g_force_generic);
    return launch_status();
}

template <int K, bool BF16>
exmy_status launch_rowwise_k(const uint8_t *in, int64_t R, int64_t C, int x, int y, int scheme, uint8_t *meta,
                             uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb, unsigned long long *spc,
                             int64_t cap, cudaStream_t st) {
    if (BF16 && y <= 6) {
        if (y == 0)
            return launch_rowwise_km<K, BF16, (BF16 ? ENC_SIMD_Y0 : ENC_F32_Y0)>(in, R, C, x, y, scheme, meta, packed,
                                                                                 p, spi, spb, spc, cap, st);
        return launch_rowwise_km<K, BF16, (BF16 ? ENC_SIMD : ENC_F32)>(in, R, C, x, y, scheme, meta, packed, p, spi,
                                                                       spb, spc, cap, st);
    }
    if (y == 0)
        return launch_rowwise_km<K, BF16, ENC_F32_Y0>(in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st);
    return launch_rowwise_km<K, BF16, ENC_F32>(in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st);
}

template <bool BF16>
exmy_status rowwise_dispatch(int k, const uint8_t *in, int64_t R, int64_t C, int x, int y, int scheme, uint8_t *meta,
                             uint8_t *packed, const Plan &p, int64_t *spi, uint32_t *spb, unsigned long long *spc,
                             int64_t cap, cudaStream_t st) {
    switch (k) {
        case 3: return launch_rowwise_k<3, BF16>(in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st);
        case 4: return launch_rowwise_k<4, BF16>(in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st);
        case 5: return launch_rowwise_k<5, BF16>(in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st);
        case 6: return launch_rowwise_k<6, BF16>(in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st);
        case 7: return launch_rowwise_k<7, BF16>(in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st);
        case 8: return launch_rowwise_k<8, BF16>(in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st);
        case 9: return launch_rowwise_k<9, BF16>(in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st);
    }
    return EXMY_E_FORMAT;
}
}  // namespace

// returns EXMY_E_ALIGN when the fused kernel does not apply (caller then
// runs block max + blocked encode)
exmy_status launch_encode_rowwise(const uint8_t *in, bool bf16, int64_t R, int64_t C, int x, int y, int scheme,
                                  uint8_t *meta, uint8_t *packed, int64_t *spi, uint32_t *spb,
                                  unsigned long long *spc, int64_t cap, cudaStream_t st) {
    const int k = 1 + x + y;
    const Plan p = make_plan(k, R * C);
    // measured (config-2 rows x 2048..16384 columns): the fused two-pass kernel
    // beats block max + blocked encode while a row group (8 rows) stays within
    // 128 KB; beyond that its second pass misses L2 and the two launches win
    // rows up to 8 x 9 KB: one HBM read (single CTA or a cluster); longer rows: the two launches
    bool vec = aligned(in, 16) && (C % (bf16 ? 8 : 4) == 0) &&
               (C * (bf16 ? 2 : 4) <= (g_rowwise_cluster ? 8 * RWS_MAX_ROW_BYTES : 16384));
    for (int s = 0; s < p.nseg; ++s) vec = vec && aligned(packed + p.so.off[s], p.w[s] == 8 ? 4 : 4 * p.w[s]);
    if (!vec) return EXMY_E_ALIGN;
    return bf16 ? rowwise_dispatch<true>(k, in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st)
                : rowwise_dispatch<false>(k, in, R, C, x, y, scheme, meta, packed, p, spi, spb, spc, cap, st);
}

exmy_status launch_encode_blocked(const uint8_t *in, bool bf16, int64_t R, int64_t C, int axis, int64_t br,
                                  int64_t bc, int x, int y, const uint8_t *meta, uint8_t *packed, int64_t *spi,
                                  uint32_t *spb, unsigned long long *spc, int64_t cap, cudaStream_t st) {
    const int k = 1 + x + y;
    const Plan p = make_plan(k, R * C);
    const MetaMap M{meta, br, bc, C / bc};
    return bf16 ? enc_blk_dispatch<true>(k, in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st)
                : enc_blk_dispatch<false>(k, in, R, C, axis, x, y, M, packed, p, spi, spb, spc, cap, st);
}

}  // namespace exmy
