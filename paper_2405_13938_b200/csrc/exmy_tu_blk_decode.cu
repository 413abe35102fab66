// exmy_tu_blk_decode.cu -- decode / quantize / block max exponent with block
// metadata launchers.
#include <algorithm>
#include "exmy_launch.cuh"
#include "exmy_narrow.cuh"

namespace exmy {

namespace {
template <int K, bool OBF16>
exmy_status launch_dec_blk_k(const uint8_t *packed, int64_t R, int64_t C, int axis, int x, int y, const MetaMap &M,
                             const Plan &p, uint8_t *out, cudaStream_t st) {
    constexpr int V = Elem<OBF16>::V;
    const int64_t n = R * C;
    const int4 widths = make_int4(p.w[0], p.w[1], p.w[2], p.w[3]);
    const bool fmt_fast = !g_force_generic && x <= 7 && (!OBF16 || y <= 7);
    if (fmt_fast && axis == EXMY_AXIS_ROWS) {
        bool vec = aligned(out, 16) && (C % V == 0) && (M.bc % V == 0) && (M.br == 1 || M.br % 8 == 0);
        for (int s = 0; s < p.nseg; ++s) {
            const size_t a = p.w[s] == 8 ? (size_t)V : (size_t)((V * p.w[s]) < 16 ? V * p.w[s] : 16);
            vec = vec && aligned(packed + p.so.off[s], a);
        }
        if (vec) {
            const int threads = 256;
            static int occ = 0;
            if (!occ) occ = occupancy(k_dec_rows_blk<K, OBF16>, threads, 0);
            const int64_t CV = C / V, G = R / 8;
            int64_t gx = cdiv(CV, threads);
            int64_t gy = (int64_t)num_sms() * occ / gx;
            if (gy < 1) gy = 1;
            if (gy > G) gy = G;
            if (gy > 65535) gy = 65535;
            if (gx > INT_MAX) return EXMY_E_SHAPE;
            k_dec_rows_blk<K, OBF16><<<dim3((unsigned)gx, (unsigned)gy), threads, 0, st>>>(packed, R, C, x, y, M, p.so,
                                                                                          out, p.nseg, widths);
            return launch_status();
        }
    } else if (fmt_fast) {
        bool vec = aligned(out, 16) && (M.bc % 8 == 0);
        for (int s = 0; s < p.nseg; ++s) vec = vec && aligned(packed + p.so.off[s], p.w[s]);
        const int64_t gpr = C / 8;
        const int lg = (gpr >= 8 && gpr <= 64 && (gpr & (gpr - 1)) == 0) ? __builtin_ctzll((unsigned long long)gpr) : -1;
        if (vec && lg >= 0 && M.br == 1 && M.bc == C && aligned(M.meta, (size_t)(128 >> lg))) {
            int64_t blocks = cdiv(cdiv(n / 8, 128), 256 / 32);
            const int64_t maxb = (int64_t)num_sms() * 2;
            if (blocks > maxb) blocks = maxb;
#define EXMY_NARROW_DEC(LG)                                                                                          \
    k_dec_cols_narrow<K, OBF16, LG><<<(unsigned)blocks, 256, 0, st>>>(packed, n, x, y, M.meta, p.so, out, M, C, p.nseg, \
                                                                     widths)
            switch (lg) {
                case 3: EXMY_NARROW_DEC(3); break;
                case 4: EXMY_NARROW_DEC(4); break;
                case 5: EXMY_NARROW_DEC(5); break;
                default: EXMY_NARROW_DEC(6); break;
            }
#undef EXMY_NARROW_DEC
            return launch_status();
        }
        if (vec) {
            const int threads = 256;
            static int occ = 0;
            if (!occ) occ = occupancy(k_dec_cols_blk<K, OBF16>, threads, 0);
            int64_t blocks = cdiv(cdiv(n / 8, 128), threads / 32);
            int64_t maxb = (int64_t)num_sms() * occ;
            if (blocks > maxb) blocks = maxb;
            k_dec_cols_blk<K, OBF16><<<(unsigned)blocks, threads, 0, st>>>(packed, n, C, x, y, M, p.so, out, p.nseg,
                                                                           widths);
            return launch_status();
        }
    }
    const int64_t ncont = n / 8;
    int64_t blocks = cdiv(ncont, 256);
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    k_decode_generic_blk<OBF16><<<(unsigned)blocks, 256, 0, st>>>(packed, C, ncont, axis, x, y, M, p.so, p.nseg,
                                                                  widths, out);
    return launch_status();
}

template <bool OBF16>
exmy_status dec_blk_dispatch(int k, const uint8_t *packed, int64_t R, int64_t C, int axis, int x, int y,
                             const MetaMap &M, const Plan &p, uint8_t *out, cudaStream_t st) {
    switch (k) {
        case 3: return launch_dec_blk_k<3, OBF16>(packed, R, C, axis, x, y, M, p, out, st);
        case 4: return launch_dec_blk_k<4, OBF16>(packed, R, C, axis, x, y, M, p, out, st);
        case 5: return launch_dec_blk_k<5, OBF16>(packed, R, C, axis, x, y, M, p, out, st);
        case 6: return launch_dec_blk_k<6, OBF16>(packed, R, C, axis, x, y, M, p, out, st);
        case 7: return launch_dec_blk_k<7, OBF16>(packed, R, C, axis, x, y, M, p, out, st);
        case 8: return launch_dec_blk_k<8, OBF16>(packed, R, C, axis, x, y, M, p, out, st);
        case 9: return launch_dec_blk_k<9, OBF16>(packed, R, C, axis, x, y, M, p, out, st);
    }
    return EXMY_E_FORMAT;
}
template <int K, bool OBF16>
exmy_status launch_gather_k(const uint8_t *packed, int64_t R, int64_t C, int x, int y, const uint8_t *meta,
                            bool per_row, const int64_t *idx, int64_t nidx, uint8_t *out, cudaStream_t st) {
    const Plan p = make_plan(K, R * C);
    const int fmt_fast = (!g_force_generic && x <= 7 && (!OBF16 || y <= 7)) ? 1 : 0;
    const int threads = 256;
    static int occ = 0;
    if (!occ) occ = occupancy(k_dec_gather<K, OBF16, true>, threads, 0);
    int64_t blocks = cdiv(cdiv(nidx * (C / 8), 128), threads / 32);
    int64_t maxb = (int64_t)num_sms() * occ;
    if (blocks > maxb) blocks = maxb;
    if (blocks < 1) blocks = 1;
    if (per_row)
        k_dec_gather<K, OBF16, true><<<(unsigned)blocks, threads, 0, st>>>(packed, C, x, y, meta, idx, nidx, p.so,
                                                                         out, fmt_fast);
    else
        k_dec_gather<K, OBF16, false><<<(unsigned)blocks, threads, 0, st>>>(packed, C, x, y, meta, idx, nidx, p.so,
                                                                          out, fmt_fast);
    return launch_status();
}

template <bool OBF16>
exmy_status gather_dispatch(int k, const uint8_t *packed, int64_t R, int64_t C, int x, int y, const uint8_t *meta,
                            bool per_row, const int64_t *idx, int64_t nidx, uint8_t *out, cudaStream_t st) {
    switch (k) {
        case 3: return launch_gather_k<3, OBF16>(packed, R, C, x, y, meta, per_row, idx, nidx, out, st);
        case 4: return launch_gather_k<4, OBF16>(packed, R, C, x, y, meta, per_row, idx, nidx, out, st);
        case 5: return launch_gather_k<5, OBF16>(packed, R, C, x, y, meta, per_row, idx, nidx, out, st);
        case 6: return launch_gather_k<6, OBF16>(packed, R, C, x, y, meta, per_row, idx, nidx, out, st);
        case 7: return launch_gather_k<7, OBF16>(packed, R, C, x, y, meta, per_row, idx, nidx, out, st);
        case 8: return launch_gather_k<8, OBF16>(packed, R, C, x, y, meta, per_row, idx, nidx, out, st);
        case 9: return launch_gather_k<9, OBF16>(packed, R, C, x, y, meta, per_row, idx, nidx, out, st);
    }
    return EXMY_E_FORMAT;
}
}  // namespace

exmy_status launch_decode_rows_gather(const uint8_t *packed, int64_t R, int64_t C, int x, int y, const uint8_t *meta,
                                      bool per_row, const int64_t *idx, int64_t nidx, uint8_t *out, bool obf16,
                                      cudaStream_t st) {
    const int k = 1 + x + y;
    return obf16 ? gather_dispatch<true>(k, packed, R, C, x, y, meta, per_row, idx, nidx, out, st)
                 : gather_dispatch<false>(k, packed, R, C, x, y, meta, per_row, idx, nidx, out, st);
}

exmy_status launch_decode_blocked(const uint8_t *packed, int64_t R, int64_t C, int axis, int64_t br, int64_t bc,
                                  int x, int y, const uint8_t *meta, uint8_t *out, bool obf16, cudaStream_t st) {
    const int k = 1 + x + y;
    const Plan p = make_plan(k, R * C);
    const MetaMap M{meta, br, bc, C / bc};
    return obf16 ? dec_blk_dispatch<true>(k, packed, R, C, axis, x, y, M, p, out, st)
                 : dec_blk_dispatch<false>(k, packed, R, C, axis, x, y, M, p, out, st);
}

exmy_status launch_quantize_blocked(const uint8_t *in, uint8_t *out, bool bf16, int64_t R, int64_t C, int64_t br,
                                    int64_t bc, int x, int y, const uint8_t *meta, cudaStream_t st) {
    const MetaMap M{meta, br, bc, C / bc};
    const int V = bf16 ? 8 : 4;
    if (aligned(in, 16) && aligned(out, 16) && C % V == 0 && bc % V == 0) {
        const int threads = 256;
        const int64_t CV = C / V;
        if (CV < threads) {   // narrow rows: flat vector numbering (k_quant_blk_flat)
            int64_t blocks = cdiv(R * CV, (int64_t)threads * 4);
            const int64_t maxb = (int64_t)num_sms() * 8;
            if (blocks > maxb) blocks = maxb;
            if (blocks < 1) blocks = 1;
            if (bf16) k_quant_blk_flat<true><<<(unsigned)blocks, threads, 0, st>>>(in, out, R, C, x, y, M, g_force_generic);
            else k_quant_blk_flat<false><<<(unsigned)blocks, threads, 0, st>>>(in, out, R, C, x, y, M, g_force_generic);
            return launch_status();
        }
        int64_t gx = cdiv(CV, threads);
        int64_t gy = (int64_t)num_sms() * 8 / gx;
        if (gy < 1) gy = 1;
        if (gy > R) gy = R;
        if (gy > 65535) gy = 65535;
        if (gx > INT_MAX) return EXMY_E_SHAPE;
        if (bf16) k_quant_blk<true><<<dim3((unsigned)gx, (unsigned)gy), threads, 0, st>>>(in, out, R, C, x, y, M, g_force_generic);
        else k_quant_blk<false><<<dim3((unsigned)gx, (unsigned)gy), threads, 0, st>>>(in, out, R, C, x, y, M, g_force_generic);
        return launch_status();
    }
    int64_t blocks = cdiv(R * C, 256);
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    if (bf16) k_quant_blk_scalar<true><<<(unsigned)blocks, 256, 0, st>>>(in, out, R, C, x, y, M, g_force_generic);
    else k_quant_blk_scalar<false><<<(unsigned)blocks, 256, 0, st>>>(in, out, R, C, x, y, M, g_force_generic);
    return launch_status();
}

exmy_status launch_block_max(const uint8_t *in, bool bf16, int64_t R, int64_t C, int64_t br, int64_t bc, int y,
                             int scheme, uint8_t *meta, cudaStream_t st) {
    const int V = bf16 ? 8 : 4;
    if (br == 1 && bc % V == 0 && C % V == 0 && bc / V <= 32 && ((bc / V) & (bc / V - 1)) == 0 && aligned(in, 16)) {
        const int64_t nvec = R * C / V;
        int64_t blocks = cdiv(nvec, 256 * 4);
        if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
        if (blocks < 1) blocks = 1;
        const int gsz = (int)(bc / V);
        if (bf16) {
            if (scheme == 0) k_block_max_small<true, 0><<<(unsigned)blocks, 256, 0, st>>>(in, nvec, gsz, y, meta, nullptr);
            else k_block_max_small<true, 1><<<(unsigned)blocks, 256, 0, st>>>(in, nvec, gsz, y, meta, nullptr);
        } else {
            if (scheme == 0) k_block_max_small<false, 0><<<(unsigned)blocks, 256, 0, st>>>(in, nvec, gsz, y, meta, nullptr);
            else k_block_max_small<false, 1><<<(unsigned)blocks, 256, 0, st>>>(in, nvec, gsz, y, meta, nullptr);
        }
        return launch_status();
    }
    const int64_t gsz = bc / V;
    // band kernel when it has >= 4 work items per resident CTA at U >= 2
    // (tall blocks, e.g. 128 x 128, leave too few bands: warp per block below)
    const int64_t resident = (int64_t)num_sms() * 3;   // 256 threads, <= 80 registers at U <= 4
    int u = 8;
    while (u > 1 && (R / br) * cdiv(C / V, (int64_t)256 * u) < 4 * resident) u >>= 1;
    if (br > 1 && bc % V == 0 && gsz <= 16 && (gsz & (gsz - 1)) == 0 && C % (32 * V) == 0 && aligned(in, 16) &&
        (R / br) * cdiv(C / V, (int64_t)256 * u) >= 4 * resident && u >= 2) {
        const int64_t blocks = std::max<int64_t>(1, (R / br) * cdiv(C / V, (int64_t)256 * u));
        if (blocks > INT_MAX) return EXMY_E_SHAPE;
        auto go = [&](auto kern) {
            kern<<<(unsigned)blocks, 256, 0, st>>>(in, R, C, br, (int)gsz, y, scheme, meta);
            return launch_status();
        };
        if (bf16) {
            switch (u) {
                case 8: return go(k_block_max_band<true, 8>);
                case 4: return go(k_block_max_band<true, 4>);
                default: return go(k_block_max_band<true, 2>);
            }
        }
        switch (u) {
            case 8: return go(k_block_max_band<false, 8>);
            case 4: return go(k_block_max_band<false, 4>);
            default: return go(k_block_max_band<false, 2>);
        }
    }
    const int64_t nb = (R / br) * (C / bc);
    int64_t blocks = cdiv(nb, 8);
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    if (blocks < 1) blocks = 1;
    if (bf16) k_block_max<true><<<(unsigned)blocks, 256, 0, st>>>(in, R, C, br, bc, y, scheme, meta);
    else k_block_max<false><<<(unsigned)blocks, 256, 0, st>>>(in, R, C, br, bc, y, scheme, meta);
    return launch_status();
}

}  // namespace exmy
