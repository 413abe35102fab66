// exmy_narrow.cuh -- COLS packing with one metadata byte per row for NARROW
// rows: embedding tables (config 5: 128 columns; P:622-627's per-row recipe,
// P:481-484 "embedding").  A COLS warp tile is 128 groups of 8 elements; with
// gpr = C / 8 groups per row (a power of two, 8 <= gpr <= 64, i.e. C = 64 ..
// 512) it covers 128 / gpr whole rows whose metadata bytes are contiguous:
// ONE 2..16-byte load per thread serves the tile, and it is software-pipelined
// with the tile's data (the next tile's bytes are in flight while this tile
// is converted).  The general blocked kernels (k_enc_cols_blk /
// k_dec_cols_blk) looked every group's byte up separately, after the data
// had arrived -- a dependent L2 round trip per tile that left config 5's
// recipe at 46 % (encode) / 52 % (decode) of the copy bandwidth.
#pragma once
#include "exmy_blocked.cuh"

namespace exmy {

// the tile's 128 / 2^LG metadata bytes (rows rb0 ...) in up to four words
template <int LG>
__device__ __forceinline__ void load_tile_rowmeta(const uint8_t *meta, int64_t rb0, int64_t nrows, uint32_t (&m)[4]) {
    m[0] = m[1] = m[2] = m[3] = 0;
    constexpr int NB = 128 >> LG;   // 16, 8, 4, 2 bytes
    if (rb0 + NB <= nrows) {
        if constexpr (NB == 16) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(meta + rb0));
            m[0] = v.x; m[1] = v.y; m[2] = v.z; m[3] = v.w;
        } else if constexpr (NB == 8) {
            const uint2 v = __ldg(reinterpret_cast<const uint2 *>(meta + rb0));
            m[0] = v.x; m[1] = v.y;
        } else if constexpr (NB == 4) {
            m[0] = __ldg(reinterpret_cast<const unsigned int *>(meta + rb0));
        } else {
            m[0] = __ldg(reinterpret_cast<const unsigned short *>(meta + rb0));
        }
    } else {   // the ragged last tile
        for (int b = 0; b < NB && rb0 + b < nrows; ++b) m[b >> 2] |= (uint32_t)__ldg(meta + rb0 + b) << (8 * (b & 3));
    }
}

__device__ __forceinline__ int rowmeta_byte(const uint32_t (&m)[4], int b) {
    const int e = (int)((m[b >> 2] >> (8 * (b & 3))) & 0xFFu);
    return e > 254 ? 254 : e;
}

template <int K, bool BF16, int MODE, int LG>
__global__ void __launch_bounds__(256, 2) k_enc_cols_narrow(const uint8_t *__restrict__ in, int64_t n, int x, int y,
                                                            const uint8_t *__restrict__ meta,
                                                            uint8_t *__restrict__ packed, SegOffsets so, int64_t *spi,
                                                            uint32_t *spb, unsigned long long *spc, int64_t cap,
                                                            MetaMap M, int64_t C, int force_generic) {
    using EL = Elem<BF16>;
    constexpr int NV = BF16 ? 1 : 2;
    constexpr int NP = EL::V / 2;
    constexpr bool SIMD = (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0);
    const FastP P = make_fast(fmt_of(x, y, 0), BF16, 1);
    const int64_t NG = n / 8, nrows = NG >> LG;
    const int lane = threadIdx.x & 31;
    const int64_t step = (int64_t)gridDim.x * (blockDim.x >> 5) * 128;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint4 nxt[4][NV];
    uint32_t nm[4];
    {
        const int64_t b0 = gw * 128;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t q = b0 + 32 * u + lane;
#pragma unroll
            for (int t = 0; t < NV; ++t)
                nxt[u][t] = q < NG ? ldg_nc_v4(in + q * 8 * EL::ES + 16 * t) : make_uint4(0, 0, 0, 0);
        }
        if (b0 < NG) load_tile_rowmeta<LG>(meta, b0 >> LG, nrows, nm);
    }
    for (int64_t base = gw * 128; base < NG; base += step) {
        uint4 r[4][NV];
        uint32_t mt[4] = {nm[0], nm[1], nm[2], nm[3]};
        const int64_t bn = base + step;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t qn = bn + 32 * u + lane;
#pragma unroll
            for (int t = 0; t < NV; ++t) {
                r[u][t] = nxt[u][t];
                nxt[u][t] = qn < NG ? ldg_nc_v4(in + qn * 8 * EL::ES + 16 * t) : make_uint4(0, 0, 0, 0);
            }
        }
        if (bn < NG) load_tile_rowmeta<LG>(meta, bn >> LG, nrows, nm);
        uint32_t cp[4][4];
        uint32_t amax = 0;
        bool ok = !force_generic;
        // the tile's <= 16 rows' encode constants: lane l computes row l's, every
        // group takes its row's by shuffles
        const RowP Rl = make_rowp<SIMD>(rowmeta_byte(mt, lane & ((128 >> LG) - 1)), x, y);
        const uint32_t ra = SIMD ? Rl.lo2 : Rl.lo, rb = SIMD ? Rl.k3 : Rl.k3f;
        const int rok = Rl.ok ? 1 : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t q = base + 32 * u + lane;
            const int src = (32 * u + lane) >> LG;
            RowP Rp;
            const uint32_t a_ = __shfl_sync(0xFFFFFFFFu, ra, src), b_ = __shfl_sync(0xFFFFFFFFu, rb, src);
            Rp.ok = __shfl_sync(0xFFFFFFFFu, rok, src) != 0;
            if (SIMD) {
                Rp.lo2 = a_; Rp.k3 = b_; Rp.lo = Rp.k3f = 0;
            } else {
                Rp.lo = a_; Rp.k3f = b_; Rp.lo2 = Rp.k3 = 0;
            }
            ok = ok && (Rp.ok || q >= NG);
#pragma unroll
            for (int t = 0; t < NV; ++t) {
                uint32_t c2[NP];
                const uint32_t ww[4] = {r[u][t].x, r[u][t].y, r[u][t].z, r[u][t].w};
                vec_codes_r<K, BF16, MODE, 4>(ww, c2, P, Rp, amax);
#pragma unroll
                for (int p = 0; p < NP; ++p) cp[u][t * NP + p] = c2[p];
            }
        }
        if (ok && !amax_special<BF16, MODE>(amax, P)) {
            uint32_t RL[8], RH[8];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint32_t y01 = prmt(cp[0][t], cp[1][t], 0x6420), y23 = prmt(cp[2][t], cp[3][t], 0x6420);
                RL[2 * t] = prmt(y01, y23, 0x6420);
                RL[2 * t + 1] = prmt(y01, y23, 0x7531);
                if (K == 9) {
                    const uint32_t h01 = prmt(cp[0][t] >> 1, cp[1][t] >> 1, 0x6420);
                    const uint32_t h23 = prmt(cp[2][t] >> 1, cp[3][t] >> 1, 0x6420);
                    RH[2 * t] = prmt(h01, h23, 0x6420);
                    RH[2 * t + 1] = prmt(h01, h23, 0x7531);
                }
            }
            cols_fast_store<K, 0>(RL, RH, cp, packed, so, base + lane, NG);
        } else {   // NaN/Inf, huge values or metadata outside the fast ranges: the integer path
            for (int u = 0; u < 4; ++u) {
                const int64_t q = base + 32 * u + lane;
                if (q < NG) enc_container_generic_blk<BF16, K>(in, C, q, 1, x, y, M, packed, so, spi, spb, spc, cap);
            }
        }
    }
}

// the raw packed words of a COLS warp tile (lane's groups q0 + 32u): per
// segment, W == 8: 8 words; W < 8: W words -- loaded as cols_fast_load does
template <int K>
__host__ __device__ constexpr int cols_raw_words() {
    int t = 0;
    for (int s = 0; s < seg_count(K); ++s) t += seg_width(K, s) == 8 ? 8 : seg_width(K, s);
    return t;
}

template <int K, int S, int OFF>
__device__ __forceinline__ void cols_load_raw(uint32_t (&raw)[cols_raw_words<K>()], const uint8_t *packed,
                                              const SegOffsets &so, int64_t q0, int64_t NG) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S);
        const uint8_t *seg = packed + so.off[S];
        if constexpr (W == 8) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t q = q0 + 32 * u;
                const uint2 t = q < NG ? __ldg((const uint2 *)(seg + 8 * q)) : make_uint2(0, 0);
                raw[OFF + u] = t.x;
                raw[OFF + 4 + u] = t.y;
            }
        } else {
#pragma unroll
            for (int q = 0; q < W; ++q) raw[OFF + q] = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t q = q0 + 32 * u;
                if (q < NG) {
                    if constexpr (W == 4) raw[OFF + u] = __ldg((const unsigned int *)(seg + 4 * q));
                    else if constexpr (W == 2)
                        raw[OFF + (u >> 1)] |= (uint32_t)__ldg((const unsigned short *)(seg + 2 * q)) << (16 * (u & 1));
                    else raw[OFF + 0] |= (uint32_t)__ldg((const unsigned char *)(seg + q)) << (8 * u);
                }
            }
        }
        cols_load_raw<K, S + 1, OFF + (W == 8 ? 8 : W)>(raw, packed, so, q0, NG);
    }
}

template <int K, int S, int OFF>
__device__ __forceinline__ void cols_unpack_raw(const uint32_t (&raw)[cols_raw_words<K>()], uint32_t (&RL)[8],
                                                uint32_t (&RH)[8]) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S);
        if constexpr (W == 8) {
            uint32_t *dst = (K == 9) ? RH : RL;
            const uint32_t a0 = prmt(raw[OFF], raw[OFF + 1], 0x5140), a1 = prmt(raw[OFF + 2], raw[OFF + 3], 0x5140);
            const uint32_t a2 = prmt(raw[OFF], raw[OFF + 1], 0x7362), a3 = prmt(raw[OFF + 2], raw[OFF + 3], 0x7362);
            dst[0] = prmt(a0, a1, 0x5410); dst[1] = prmt(a0, a1, 0x7632);
            dst[2] = prmt(a2, a3, 0x5410); dst[3] = prmt(a2, a3, 0x7632);
            const uint32_t b0 = prmt(raw[OFF + 4], raw[OFF + 5], 0x5140), b1 = prmt(raw[OFF + 6], raw[OFF + 7], 0x5140);
            const uint32_t b2 = prmt(raw[OFF + 4], raw[OFF + 5], 0x7362), b3 = prmt(raw[OFF + 6], raw[OFF + 7], 0x7362);
            dst[4] = prmt(b0, b1, 0x5410); dst[5] = prmt(b0, b1, 0x7632);
            dst[6] = prmt(b2, b3, 0x5410); dst[7] = prmt(b2, b3, 0x7632);
        } else {
            uint32_t in[W];
#pragma unroll
            for (int q = 0; q < W; ++q) in[q] = raw[OFF + q];
            swar_unpack4<W, LO>(in, RL);
        }
        cols_unpack_raw<K, S + 1, OFF + (W == 8 ? 8 : W)>(raw, RL, RH);
    }
}

template <int K, bool OBF16, int LG>
__global__ void __launch_bounds__(256, 2) k_dec_cols_narrow(const uint8_t *__restrict__ packed, int64_t n, int x,
                                                            int y, const uint8_t *__restrict__ meta, SegOffsets so,
                                                            uint8_t *__restrict__ out, MetaMap M, int64_t C, int nseg,
                                                            int4 widths) {
    constexpr int TW = cols_raw_words<K>();
    const int64_t NG = n / 8, nrows = NG >> LG;
    const int lane = threadIdx.x & 31;
    const int64_t step = (int64_t)gridDim.x * (blockDim.x >> 5) * 128;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint32_t nxt[TW], nm[4];
    if (gw * 128 < NG) {
        cols_load_raw<K, 0, 0>(nxt, packed, so, gw * 128 + lane, NG);
        load_tile_rowmeta<LG>(meta, (gw * 128) >> LG, nrows, nm);
    }
    for (int64_t base = gw * 128; base < NG; base += step) {
        uint32_t raw[TW];
#pragma unroll
        for (int q = 0; q < TW; ++q) raw[q] = nxt[q];
        const uint32_t mt[4] = {nm[0], nm[1], nm[2], nm[3]};
        const int64_t bn = base + step;
        if (bn < NG) {
            cols_load_raw<K, 0, 0>(nxt, packed, so, bn + lane, NG);
            load_tile_rowmeta<LG>(meta, bn >> LG, nrows, nm);
        }
        uint32_t RL[8], RH[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { RL[i] = 0; RH[i] = 0; }
        cols_unpack_raw<K, 0, 0>(raw, RL, RH);
        // the tile's <= 16 rows' decode factors: lane l computes row l's, every
        // group takes its row's by a shuffle (not one factor per group)
        const RowD Dl = make_rowd(rowmeta_byte(mt, lane & ((128 >> LG) - 1)), x);
        const uint32_t dsc = OBF16 ? Dl.s_bf2 : __float_as_uint(Dl.s_f);
        const int dok = Dl.ok ? 1 : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t q = base + 32 * u + lane;
            const int src = (32 * u + lane) >> LG;
            RowD D;
            const uint32_t sc = __shfl_sync(0xFFFFFFFFu, dsc, src);
            D.ok = __shfl_sync(0xFFFFFFFFu, dok, src) != 0;
            D.s_bf2 = sc;
            D.s_f = __uint_as_float(sc);
            if (q >= NG) continue;
            if (!D.ok) {
                dec_container_generic_blk<OBF16>(packed, C, q, 1, x, y, M, so, nseg, widths, out);
                continue;
            }
            if (OBF16) {
                uint32_t o[4];
                const uint32_t sel = (uint32_t)u | ((uint32_t)(4 + u) << 4);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    uint32_t cp = prmt(RL[2 * t], RL[2 * t + 1], sel);
                    cp = (cp & 0xFFu) | ((cp & 0xFF00u) << 8);
                    if (K == 9) {
                        uint32_t ch = prmt(RH[2 * t], RH[2 * t + 1], sel);
                        cp |= ((ch & 0xFFu) | ((ch & 0xFF00u) << 8)) << 1;
                    }
                    o[t] = dec_pair_bf16_r<K>(cp, y, D);
                }
                stg_v4(out + q * 16, make_uint4(o[0], o[1], o[2], o[3]));
            } else {
                uint32_t o[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    uint32_t code = (RL[i] >> (8 * u)) & 0xFFu;
                    if (K == 9) code |= ((RH[i] >> (8 * u)) & 0xFFu) << 1;
                    o[i] = dec_f32_r<K>(code, y, D);
                }
                stg_v4(out + q * 32, make_uint4(o[0], o[1], o[2], o[3]));
                stg_v4(out + q * 32 + 16, make_uint4(o[4], o[5], o[6], o[7]));
            }
        }
    }
}

}  // namespace exmy
