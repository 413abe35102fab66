// exmy_tu_decode.cu -- K4 decode launchers (+ K5 specials scatter).
#include "exmy_launch.cuh"

namespace exmy {

namespace {
template <int K, bool OBF16, int MODE>
exmy_status launch_decode_km(const uint8_t *packed, int64_t R, int64_t C, int axis, int x, int y,
                            const uint8_t *meta, const Plan &p, uint8_t *out, cudaStream_t st) {
    constexpr int V = Elem<OBF16>::V;
    const int64_t n = R * C;
    bool vec = aligned(out, 16);
    if (axis == EXMY_AXIS_ROWS) {
        vec = vec && (C % V == 0);
        for (int s = 0; s < p.nseg; ++s) {
            size_t a = p.w[s] == 8 ? (size_t)V : (size_t)((V * p.w[s]) < 16 ? V * p.w[s] : 16);
            vec = vec && aligned(packed + p.so.off[s], a);
        }
        if (vec) {
            const int threads = 256;
            static int occ = 0;
            if (!occ) occ = occupancy(k_dec_rows_fast<K, OBF16, MODE>, threads, 0);
            const int64_t CV = C / V, G = R / 8;
            int64_t gx = cdiv(CV, threads);
            // decode is write-bound: 2 CTAs/SM (16 warps) measure ~1.5 % faster than 4
#ifndef DEC_ROWS_OCC
#define DEC_ROWS_OCC 2
#endif
            int64_t target = (int64_t)num_sms() * (occ < DEC_ROWS_OCC ? occ : DEC_ROWS_OCC);
            int64_t gy = target / gx;
            if (gy < 1) gy = 1;
            if (gy > G) gy = G;
            if (gy > 65535) gy = 65535;
            if (gx > INT_MAX) return EXMY_E_SHAPE;
            k_dec_rows_fast<K, OBF16, MODE><<<dim3((unsigned)gx, (unsigned)gy), threads, 0, st>>>(packed, R, C, x, y, meta,
                                                                                               p.so, out);
            return launch_status();
        }
    } else {
        for (int s = 0; s < p.nseg; ++s) vec = vec && aligned(packed + p.so.off[s], p.w[s]);
        if (vec) {
            const int threads = 256;
            static int occ = 0;
            if (!occ) occ = occupancy(k_dec_cols_fast<K, OBF16, MODE>, threads, 0);
            int64_t tiles = cdiv(n / 8, 128);
            int64_t blocks = cdiv(tiles, threads / 32);
            int64_t maxb = (int64_t)num_sms() * occ;
            if (blocks > maxb) blocks = maxb;
            k_dec_cols_fast<K, OBF16, MODE><<<(unsigned)blocks, threads, 0, st>>>(packed, n, x, y, meta, p.so, out);
            return launch_status();
        }
    }
    const int64_t ncont = n / 8;
    int64_t blocks = cdiv(ncont, 256);
    int64_t maxb = (int64_t)num_sms() * 8;
    if (blocks > maxb) blocks = maxb;
    k_decode_generic<OBF16><<<(unsigned)blocks, 256, 0, st>>>(packed, C, ncont, axis, x, y, meta, p.so, p.nseg,
                                                              make_int4(p.w[0], p.w[1], p.w[2], p.w[3]), out,
                                                              g_force_generic);
    return launch_status();
}

// decode mode from the format (no metadata dependence): the multiply path
// needs x <= 7 (and y <= 7 for bf16 output); the debug knob forces generic
template <int K, bool OBF16>
exmy_status launch_decode_k(const uint8_t *packed, int64_t R, int64_t C, int axis, int x, int y,
                            const uint8_t *meta, const Plan &p, uint8_t *out, cudaStream_t st) {
    const bool fast = !g_force_generic && x <= 7 && (!OBF16 || y <= 7);
    return fast ? launch_decode_km<K, OBF16, DEC_FAST>(packed, R, C, axis, x, y, meta, p, out, st)
                : launch_decode_km<K, OBF16, DEC_GENERIC>(packed, R, C, axis, x, y, meta, p, out, st);
}

template <bool OBF16>
exmy_status decode_dispatch(int k, const uint8_t *packed, int64_t R, int64_t C, int axis, int x, int y,
                            const uint8_t *meta, const Plan &p, uint8_t *out, cudaStream_t st) {
    switch (k) {
        case 3: return launch_decode_k<3, OBF16>(packed, R, C, axis, x, y, meta, p, out, st);
        case 4: return launch_decode_k<4, OBF16>(packed, R, C, axis, x, y, meta, p, out, st);
        case 5: return launch_decode_k<5, OBF16>(packed, R, C, axis, x, y, meta, p, out, st);
        case 6: return launch_decode_k<6, OBF16>(packed, R, C, axis, x, y, meta, p, out, st);
        case 7: return launch_decode_k<7, OBF16>(packed, R, C, axis, x, y, meta, p, out, st);
        case 8: return launch_decode_k<8, OBF16>(packed, R, C, axis, x, y, meta, p, out, st);
        case 9: return launch_decode_k<9, OBF16>(packed, R, C, axis, x, y, meta, p, out, st);
    }
    return EXMY_E_FORMAT;
}

}  // namespace

exmy_status launch_decode(const uint8_t *packed, int64_t R, int64_t C, int axis, int x, int y,
                          const uint8_t *meta, uint8_t *out, bool obf16, cudaStream_t st) {
    const int k = 1 + x + y;
    Plan p = make_plan(k, R * C);
    return obf16 ? decode_dispatch<true>(k, packed, R, C, axis, x, y, meta, p, out, st)
                 : decode_dispatch<false>(k, packed, R, C, axis, x, y, meta, p, out, st);
}

exmy_status launch_specials_scatter(const int64_t *spi, const uint32_t *spb, const unsigned long long *spc,
                                    int64_t cap, uint8_t *out, bool obf16, cudaStream_t st) {
    if (obf16) k_specials_scatter<true><<<num_sms(), 256, 0, st>>>(spi, spb, spc, cap, out);
    else k_specials_scatter<false><<<num_sms(), 256, 0, st>>>(spi, spb, spc, cap, out);
    return launch_status();
}

}  // namespace exmy
