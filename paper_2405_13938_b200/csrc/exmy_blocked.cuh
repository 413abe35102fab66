// exmy_blocked.cuh -- block metadata:
// per-block maximum exponent (before / after rounding) and quantize /
// encode / decode where every (block_rows x block_cols) tile of the tensor
// carries its own metadata byte.  The per-element arithmetic is that of
// exmy_fast.cuh; only the quantities that depend on e_max (the subnormal
// clamp, the exponent offset, the decode scale) become per row / per group.
#pragma once
#include "exmy_fast.cuh"

namespace exmy {

// block (i, j) of a (R, C) tensor tiled by (br x bc) owns meta[i * nbc + j]
struct MetaMap {
    const uint8_t *meta;
    int64_t br, bc, nbc;
};

__device__ __forceinline__ int meta_at(const MetaMap &M, int64_t r, int64_t c) {
    const int e = __ldg(M.meta + (r / M.br) * M.nbc + c / M.bc);
    return e > 254 ? 254 : e;
}

__device__ __forceinline__ Fmt fmt_of(int x, int y, int e) {
    Fmt F;
    F.x = x; F.y = y; F.e_max = e;
    F.top = (1 << x) - 1;
    F.o = e - F.top;
    F.M = (1u << (x + y)) - 1u;
    return F;
}

// ------------------------------------------------------- per-row params
// The e_max-dependent constants of the encode fast paths (see FastP).
struct RowP {
    uint32_t lo2, k3;           // bf16 lanes
    uint32_t lo, k3f;           // fp32
    bool ok;                    // fast preconditions hold for this e_max
};

template <bool SIMD>
__device__ __forceinline__ RowP make_rowp(int e, int x, int y) {
    RowP R;
    const int o1 = e - ((1 << x) - 1) + 1;   // o + 1
    R.ok = (o1 >= 1) && (e <= (SIMD ? 246 : 230) + y);
    const uint32_t u1 = (uint32_t)o1;
    if (SIMD) {
        R.lo2 = u1 * (0x80u * 0x00010001u);
        R.k3 = u1 * ((1u << y) * 0x00010001u);
        R.lo = R.k3f = 0;
    } else {
        R.lo = u1 << 23;
        R.k3f = u1 << y;
        R.lo2 = R.k3 = 0;
    }
    return R;
}

template <int K, bool Y0, bool SIGN = true>
__device__ __forceinline__ uint32_t enc_pair_bf16_r(uint32_t w, const FastP &P, const RowP &R, uint32_t &amax) {
    const uint32_t a2 = w & 0x7FFF7FFFu;
    const uint32_t ev = w & 0x7F807F80u;
    const uint32_t ecl = vmax_u16x2(ev, R.lo2);
    uint32_t c, t;
    if (Y0) {   // D6: y = 0 ties to the even fp32 exponent (see exmy_fast.cuh)
        t = ecl >> 7;
        c = ecl + P.k2 + ((~(t | (ev >> 7))) & 0x00010001u);
    } else {
        t = ecl >> P.sh_b;
        c = ecl + P.k2;
    }
    const uint32_t s = hadd2_bf16(a2, c);
    uint32_t code = s - c + t - R.k3;
    code = vmin_u16x2(code, P.m2);
    if (SIGN) code |= (w >> (16 - K)) & ((1u << (K - 1)) * 0x00010001u);
    amax = vmax_u16x2(amax, a2);
    return code;
}

template <int K, bool Y0, bool SIGN = true>
__device__ __forceinline__ uint32_t enc_f32_fast_r(uint32_t u, const FastP &P, const RowP &R, uint32_t &amax) {
    const uint32_t a = u & 0x7FFFFFFFu;
    const uint32_t ev = u & 0x7F800000u;
    const uint32_t ecl = max(ev, R.lo);
    uint32_t c = ecl + P.k2f;
    if (Y0) c += (~((ecl | ev) >> 23)) & 1u;
    const uint32_t s = __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(c)));
    uint32_t code = s - c + (ecl >> P.sh_f) - R.k3f;
    code = min(code, (1u << (K - 1)) - 1u);
    if (SIGN) code |= (u >> (32 - K)) & (1u << (K - 1));
    amax = max(amax, a);
    return code;
}

template <int K, bool BF16, int MODE, int NW, bool SIGN = true>
__device__ __forceinline__ void vec_codes_r(const uint32_t (&w)[NW], uint32_t (&cp)[BF16 ? NW : NW / 2],
                                            const FastP &P, const RowP &R, uint32_t &amax) {
    constexpr int NP = BF16 ? NW : NW / 2;
    if constexpr (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0) {
#pragma unroll
        for (int t = 0; t < NP; ++t) cp[t] = enc_pair_bf16_r<K, MODE == ENC_SIMD_Y0, SIGN>(w[t], P, R, amax);
    } else {
#pragma unroll
        for (int t = 0; t < NP; ++t) {
            const uint32_t lo = enc_f32_fast_r<K, MODE == ENC_F32_Y0, SIGN>(wordvec_elem<BF16, NW>(w, 2 * t), P, R, amax);
            const uint32_t hi = enc_f32_fast_r<K, MODE == ENC_F32_Y0, SIGN>(wordvec_elem<BF16, NW>(w, 2 * t + 1), P, R, amax);
            cp[t] = lo | (hi << 16);
        }
    }
}

// ---------------------------------------------------- generic containers
// one container on the integer path, metadata looked up per element
template <bool BF16, int K>
__device__ __noinline__ void enc_container_generic_blk(const uint8_t *__restrict__ in, int64_t C, int64_t idx, int axis,
                                                       int x, int y, const MetaMap M, uint8_t *packed,
                                                       const SegOffsets so, int64_t *spi, uint32_t *spb,
                                                       unsigned long long *spc, int64_t cap) {
    uint32_t c[8];
    int64_t e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        e[i] = lane_elem(idx, i, C, axis);
        const Fmt F = fmt_of(x, y, meta_at(M, e[i] / C, e[i] % C));
        c[i] = enc_elem(load_elem_scalar<BF16>(in, e[i]), F, e[i], spi, spb, spc, cap);
    }
    int hi = K;
#pragma unroll
    for (int s = 0; s < seg_count(K); ++s) {
        const int w = seg_width(K, s), lo = hi - w;
        uint8_t *seg = packed + so.off[s];
        if (w == 8) {
            for (int i = 0; i < 8; ++i) seg[e[i]] = (uint8_t)(c[i] >> lo);
        } else {
            uint32_t cont = 0;
            for (int i = 0; i < 8; ++i) cont |= ((c[i] >> lo) & ((1u << w) - 1u)) << (w * i);
            for (int b = 0; b < w; ++b) seg[idx * w + b] = (uint8_t)(cont >> (8 * b));
        }
        hi = lo;
    }
}

template <bool BF16, int K>
__global__ void k_encode_generic_blk(const uint8_t *__restrict__ in, int64_t C, int64_t ncont, int axis, int x, int y,
                                     MetaMap M, uint8_t *__restrict__ packed, SegOffsets so, int64_t *spi,
                                     uint32_t *spb, unsigned long long *spc, int64_t cap) {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < ncont;
         idx += (int64_t)gridDim.x * blockDim.x)
        enc_container_generic_blk<BF16, K>(in, C, idx, axis, x, y, M, packed, so, spi, spb, spc, cap);
}

// ---------------------------------------------------- encode ROWS (blocked)
// Same tiles as k_enc_rows_fast (8 rows x 4 columns).  Host guarantees
// bc % 4 == 0 (the 4 columns share a block column) and br == 1 or br % 8 == 0.
// metadata bytes of the 8 rows of row group g in this thread's block column
// (br == 1: one per row; br % 8 == 0: the same byte for all 8)
__device__ __forceinline__ void load_tile_meta(const uint8_t *mcol, int64_t g, const MetaMap &M, uint32_t (&e)[8]) {
    if (M.br == 1) {
        if (M.nbc == 1 && ((reinterpret_cast<uintptr_t>(mcol) & 7) == 0)) {
            const uint2 v = __ldg(reinterpret_cast<const uint2 *>(mcol + 8 * g));
#pragma unroll
            for (int i = 0; i < 4; ++i) { e[i] = (v.x >> (8 * i)) & 0xFFu; e[4 + i] = (v.y >> (8 * i)) & 0xFFu; }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) e[i] = __ldg(mcol + (8 * g + i) * M.nbc);
        }
    } else {
        const uint32_t v = __ldg(mcol + ((8 * g) / M.br) * M.nbc);
#pragma unroll
        for (int i = 0; i < 8; ++i) e[i] = v;
    }
}

template <int K, bool BF16, int MODE>
// CTAs per SM (measured, config 2 per-row: encode 2 > 3; decode 2: e3m3
// 159 -> 132 us, fp32 out 288 -> 229 us vs unbounded registers)
#ifndef ENC_ROWS_BLK_MINB
#define ENC_ROWS_BLK_MINB 2
#endif
#ifndef DEC_ROWS_BLK_MINB
#define DEC_ROWS_BLK_MINB 2
#endif
__global__ void __launch_bounds__(256, ENC_ROWS_BLK_MINB) k_enc_rows_blk(const uint8_t *__restrict__ in, int64_t R, int64_t C,
                                                                   int x, int y, MetaMap M,
                                                                   uint8_t *__restrict__ packed, SegOffsets so,
                                                                   int64_t *spi, uint32_t *spb,
                                                                   unsigned long long *spc, int64_t cap,
                                                                   int force_generic) {
    using EL = Elem<BF16>;
    constexpr int NW = BF16 ? 2 : 4;
    constexpr bool SIMD = (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0);
    const FastP P = make_fast(fmt_of(x, y, 0), BF16, 1);   // e_max-independent constants only
    const int64_t CV = C / 4, G = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= CV) return;
    const int64_t c0 = j * 4;
    const uint8_t *mcol = M.meta + c0 / M.bc;      // block column of this thread
    const uint8_t *src = in + c0 * EL::ES;
    const int64_t rstride = C * EL::ES;
    // software pipeline: next tile's data and metadata in flight
    uint32_t nw[8][NW], nm[8];
    int64_t g = blockIdx.y;
    if (g < G) {
#pragma unroll
        for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * g + i) * rstride, nw[i]);
        load_tile_meta(mcol, g, M, nm);
    }
    for (; g < G; g += gridDim.y) {
        uint32_t w[8][NW], em[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            em[i] = nm[i];
#pragma unroll
            for (int q = 0; q < NW; ++q) w[i][q] = nw[i][q];
        }
        const int64_t gn = g + gridDim.y;
        if (gn < G) {
#pragma unroll
            for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * gn + i) * rstride, nw[i]);
            load_tile_meta(mcol, gn, M, nm);
        }
        bool ok = !force_generic;
        uint32_t cp[8][2];
        uint32_t amax = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const RowP Rp = make_rowp<SIMD>(em[i] > 254u ? 254 : (int)em[i], x, y);
            ok = ok && Rp.ok;
            vec_codes_r<K, BF16, MODE, NW>(w[i], cp[i], P, Rp, amax);
        }
        if (ok && !amax_special<BF16, MODE>(amax, P)) {
            uint32_t RL[1][8], RH[1][8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                RL[0][i] = prmt(cp[i][0], cp[i][1], 0x6420);
                RH[0][i] = (K == 9) ? prmt(cp[i][0] >> 1, cp[i][1] >> 1, 0x6420) : 0u;
            }
            rows_fast_store<K, 1, 0>(RL, RH, packed, so, g, C, c0);
        } else {
            for (int v = 0; v < 4; ++v)
                enc_container_generic_blk<BF16, K>(in, C, g * C + c0 + v, 0, x, y, M, packed, so, spi, spb, spc, cap);
        }
    }
}

// ROWS encode with ONE METADATA BYTE PER ROW (the paper's recipe):
// a CTA works on one row group at a time, so its 8 metadata bytes are one
// uniform 8-byte load (prefetched with the tile) and each row's constants
// (subnormal clamp, exponent offset) take 4 SIMD ops per 32 elements (PRMT
// the byte into both 16-bit lanes, clamp, two IMADs) instead of make_rowp's
// scalar chain per element vector (k_enc_rows_blk) or 16 shuffles per tile.
template <int K, bool BF16, int MODE>
__global__ void __launch_bounds__(256, (BF16 && K <= 7) ? 3 : 2)
    k_enc_rows_rowmeta(const uint8_t *__restrict__ in, int64_t R, int64_t C, int x, int y,
                       const uint8_t *__restrict__ meta, uint8_t *__restrict__ packed, SegOffsets so, int64_t *spi,
                       uint32_t *spb, unsigned long long *spc, int64_t cap, int force_generic, MetaMap M) {
    using EL = Elem<BF16>;
    constexpr int NW = BF16 ? 2 : 4;
    constexpr bool SIMD = (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0);
    const FastP P = make_fast(fmt_of(x, y, 0), BF16, 1);   // e_max-independent constants only
    const int64_t CV = C / 4, G = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= CV) return;
    const int64_t c0 = j * 4;
    const uint8_t *src = in + c0 * EL::ES;
    const int64_t rstride = C * EL::ES;
    const uint32_t rs32 = (uint32_t)rstride;
    // row constants from the byte e: u = o + 1 = e - (top - 1); SIMD lanes
    // lo2 = u << 7, k3 = u << y; fp32 lo = u << 23, k3f = u << y
    const uint32_t top1 = (uint32_t)((1 << x) - 2) * (SIMD ? 0x00010001u : 1u);
    // fast preconditions on every byte: top <= e <= (SIMD ? 246 : 230) + y
    const uint32_t emin4 = (uint32_t)((1 << x) - 1) * 0x01010101u;
    const int ehi = (SIMD ? 246 : 230) + y;
    const uint32_t emax4 = (uint32_t)(ehi > 255 ? 255 : ehi) * 0x01010101u;
    uint32_t nw[8][NW];
    uint2 nm = make_uint2(0u, 0u);
    int64_t g = blockIdx.y;
    if (g < G) {
#pragma unroll
        for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * g + i) * rstride, nw[i]);
        nm = __ldg(reinterpret_cast<const uint2 *>(meta) + g);
    }
    for (; g < G; g += gridDim.y) {
        uint32_t w[8][NW];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < NW; ++q) w[i][q] = nw[i][q];
        const uint2 em = nm;
        const int64_t gn = g + gridDim.y;
        if (gn < G) {
            const uint8_t *pb = src + 8 * gn * rstride;
#pragma unroll
            for (int i = 0; i < 8; ++i) load4<BF16>(pb + (uint32_t)i * rs32, nw[i]);
            nm = __ldg(reinterpret_cast<const uint2 *>(meta) + gn);
        }
        const uint32_t mn = __vminu4(em.x, em.y), mx = __vmaxu4(em.x, em.y);
        const bool ok = !force_generic && (__vcmpgeu4(mn, emin4) & __vcmpleu4(mx, emax4)) == 0xFFFFFFFFu;
        uint32_t cp[8][2];
        uint32_t amax = 0;
        constexpr bool LATE_SIGN = BF16 ? (SIMD && K <= 8) : K <= 7;   // signs per row, as k_enc_rows_fast
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t word = i < 4 ? em.x : em.y;
            RowP Rp;
            if (SIMD) {   // e in both 16-bit lanes
                const uint32_t u2 = prmt(word, 0u, 0x4040u | (uint32_t)(i & 3) | ((uint32_t)(i & 3) << 8)) - top1;
                Rp.lo2 = u2 << 7;
                Rp.k3 = u2 << y;
                Rp.lo = Rp.k3f = 0;
            } else {
                const uint32_t u = ((word >> (8 * (i & 3))) & 0xFFu) - top1;
                Rp.lo = u << 23;
                Rp.k3f = u << y;
                Rp.lo2 = Rp.k3 = 0;
            }
            Rp.ok = true;
            vec_codes_r<K, BF16, MODE, NW, !LATE_SIGN>(w[i], cp[i], P, Rp, amax);
        }
        if (ok && !amax_special<BF16, MODE>(amax, P)) {
            uint32_t RL[1][8], RH[1][8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                RL[0][i] = prmt(cp[i][0], cp[i][1], 0x6420);
                if constexpr (LATE_SIGN) {
                    uint32_t sb;
                    if constexpr (NW == 2) sb = sign_bytes(w[i][0], w[i][NW - 1]);
                    else sb = sign_bytes_f32(w[i][0], w[i][1 % NW], w[i][2 % NW], w[i][3 % NW]);
                    RL[0][i] |= sb & ((1u << (K - 1)) * 0x01010101u);
                }
                RH[0][i] = (K == 9) ? prmt(cp[i][0] >> 1, cp[i][1] >> 1, 0x6420) : 0u;
            }
            rows_fast_store<K, 1, 0>(RL, RH, packed, so, g, C, c0);
        } else {
            for (int v = 0; v < 4; ++v)
                enc_container_generic_blk<BF16, K>(in, C, g * C + c0 + v, 0, x, y, M, packed, so, spi, spb, spc, cap);
        }
    }
}

// ---------------------------------------------------- encode COLS (blocked)
// groups of 8 consecutive elements of one row; host guarantees bc % 8 == 0.
// Row of group q: q / gpr, computed with an fp64 reciprocal and corrected.
__device__ __forceinline__ int64_t div_rcp(int64_t q, int64_t d, double inv) {
    int64_t r = (int64_t)((double)q * inv);
    if (r * d > q) --r;
    else if ((r + 1) * d <= q) ++r;
    return r;
}

// metadata of COLS group q (8 consecutive elements of one row) without
// 64-bit integer divisions: row, block row and block column via reciprocals
struct GroupMeta {
    int64_t gpr, bc8;
    double inv_gpr, inv_br, inv_bc8;
    int gpr_shift;   // log2(gpr) when gpr is a power of two (e.g. 128-column tables), else -1
    __device__ __forceinline__ GroupMeta(const MetaMap &M, int64_t C) {
        gpr = C / 8;
        bc8 = M.bc / 8;
        gpr_shift = (gpr > 0 && (gpr & (gpr - 1)) == 0) ? __ffsll(gpr) - 1 : -1;
        inv_gpr = 1.0 / (double)gpr;
        inv_br = 1.0 / (double)M.br;
        inv_bc8 = 1.0 / (double)bc8;
    }
    __device__ __forceinline__ int at_row(const MetaMap &M, int64_t row, int64_t gcol) const {
        const int64_t brow = M.br == 1 ? row : div_rcp(row, M.br, inv_br);
        const int64_t bcol = bc8 == gpr ? 0 : div_rcp(gcol, bc8, inv_bc8);
        const int e = __ldg(M.meta + brow * M.nbc + bcol);
        return e > 254 ? 254 : e;
    }
    __device__ __forceinline__ int at(const MetaMap &M, int64_t q) const {
        const int64_t row = gpr_shift >= 0 ? (q >> gpr_shift) : div_rcp(q, gpr, inv_gpr);
        return at_row(M, row, q - row * gpr);
    }
    // blocks spanning whole rows (bc == C) and rows of >= 128 groups: a warp
    // tile covers at most rows rb and rb+1, so two metadata bytes serve it
    __device__ __forceinline__ bool whole_rows() const { return bc8 == gpr && gpr >= 128; }
    __device__ __forceinline__ int row_meta(const MetaMap &M, int64_t row) const {
        const int64_t brow = M.br == 1 ? row : div_rcp(row, M.br, inv_br);
        const int e = __ldg(M.meta + brow * M.nbc);
        return e > 254 ? 254 : e;
    }
    // warp tile of 128 groups starting at `base`: when a row holds >= 128
    // groups the tile spans at most two rows, so one division per tile
    // serves all of its groups
    __device__ __forceinline__ int at_tile(const MetaMap &M, int64_t base, int64_t rb, int64_t qs, int t) const {
        if (gpr < 128) return at(M, base + t);
        const int64_t c = qs + t;
        const bool cross = c >= gpr;
        return at_row(M, rb + (cross ? 1 : 0), cross ? c - gpr : c);
    }
};

template <int K, bool BF16, int MODE>
__global__ void __launch_bounds__(256, 2) k_enc_cols_blk(const uint8_t *__restrict__ in, int64_t n, int64_t C, int x,
                                                      int y, MetaMap M, uint8_t *__restrict__ packed, SegOffsets so,
                                                      int64_t *spi, uint32_t *spb, unsigned long long *spc,
                                                      int64_t cap, int force_generic) {
    using EL = Elem<BF16>;
    constexpr int NV = BF16 ? 1 : 2;
    constexpr int NP = EL::V / 2;
    constexpr bool SIMD = (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0);
    const FastP P = make_fast(fmt_of(x, y, 0), BF16, 1);
    const int64_t NG = n / 8;
    const GroupMeta GM(M, C);
    const int lane = threadIdx.x & 31;
    const int64_t step = (int64_t)gridDim.x * (blockDim.x >> 5) * 128;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    // software pipeline (as k_enc_cols_fast): the next tile's groups are in
    // flight while this tile is converted and packed
    uint4 nxt[4][NV];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t q = gw * 128 + 32 * u + lane;
#pragma unroll
        for (int t = 0; t < NV; ++t)
            nxt[u][t] = q < NG ? ldg_nc_v4(in + q * 8 * EL::ES + 16 * t) : make_uint4(0, 0, 0, 0);
    }
    for (int64_t base = gw * 128; base < NG; base += step) {
        const int64_t rb = div_rcp(base, GM.gpr, GM.inv_gpr), qs = base - rb * GM.gpr;
        uint4 r[4][NV];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t qn = base + step + 32 * u + lane;
#pragma unroll
            for (int t = 0; t < NV; ++t) {
                r[u][t] = nxt[u][t];
                nxt[u][t] = qn < NG ? ldg_nc_v4(in + qn * 8 * EL::ES + 16 * t) : make_uint4(0, 0, 0, 0);
            }
        }
        uint32_t cp[4][4];
        uint32_t amax = 0;
        bool ok = !force_generic;
#pragma unroll
        // whole-row blocks: the tile's two possible rows' parameters, once per tile
        const bool wr = GM.whole_rows();
        const int64_t split = GM.gpr - qs;   // tile groups t < split lie in row rb
        RowP R0, R1;
        if (wr) {
            R0 = make_rowp<SIMD>(GM.row_meta(M, rb), x, y);
            R1 = make_rowp<SIMD>(rb + 1 < NG / GM.gpr ? GM.row_meta(M, rb + 1) : 0, x, y);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t q = base + 32 * u + lane;
            const bool in_range = q < NG;
            RowP Rp;
            if (wr) {
                Rp = (32 * u + lane) < split ? R0 : R1;
            } else {
                Rp = make_rowp<SIMD>(in_range ? GM.at_tile(M, base, rb, qs, 32 * u + lane) : 0, x, y);
            }
            ok = ok && (Rp.ok || !in_range);
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
        } else {
            for (int u = 0; u < 4; ++u) {
                const int64_t q = base + 32 * u + lane;
                if (q < NG) enc_container_generic_blk<BF16, K>(in, C, q, 1, x, y, M, packed, so, spi, spb, spc, cap);
            }
        }
    }
}

// ------------------------------------------------------- decode (blocked)
struct RowD {
    uint32_t s_bf2;   // 2^o as a bf16 pair
    float s_f;        // 2^o as fp32
    bool ok;          // o <= 127 (one multiply)
};

__device__ __forceinline__ RowD make_rowd(int e, int x) {
    RowD D;
    const int o = e - ((1 << x) - 1);
    D.ok = o <= 127;
    const int oc = o > 127 ? 127 : o;
    D.s_bf2 = (oc >= -133 ? bf16_pow2(oc) : 0u) * 0x00010001u;
    D.s_f = pow2f_exact(oc < -149 ? -149 : oc);
    return D;
}

template <int K>
__device__ __forceinline__ uint32_t dec_pair_bf16_r(uint32_t cp, int y, const RowD &D) {
    const uint32_t mag = cp & (((1u << (K - 1)) - 1u) * 0x00010001u);
    const uint32_t v = hmul2_bf16(mag << (7 - y), D.s_bf2);
    return v | ((cp << (16 - K)) & 0x80008000u);
}
template <int K>
__device__ __forceinline__ uint32_t dec_f32_r(uint32_t code, int y, const RowD &D) {
    const uint32_t mag = code & ((1u << (K - 1)) - 1u);
    const float f = __fmul_rn(__uint_as_float(mag << (23 - y)), D.s_f);
    return __float_as_uint(f) | ((code << (32 - K)) & 0x80000000u);
}

template <bool OBF16>
__device__ __noinline__ void dec_container_generic_blk(const uint8_t *__restrict__ packed, int64_t C, int64_t idx,
                                                       int axis, int x, int y, const MetaMap M, const SegOffsets so,
                                                       int nseg, int4 widths, uint8_t *out) {
    const int wd[4] = {widths.x, widths.y, widths.z, widths.w};
    uint32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = lane_elem(idx, i, C, axis);
    int hi = 1 + x + y;
    for (int s = 0; s < nseg; ++s) {
        const int w = wd[s], lo = hi - w;
        const uint8_t *seg = packed + so.off[s];
        if (w == 8) {
            for (int i = 0; i < 8; ++i) c[i] |= (uint32_t)seg[e[i]] << lo;
        } else {
            uint32_t cont = 0;
            for (int b = 0; b < w; ++b) cont |= (uint32_t)seg[idx * w + b] << (8 * b);
            for (int i = 0; i < 8; ++i) c[i] |= ((cont >> (w * i)) & ((1u << w) - 1u)) << lo;
        }
        hi = lo;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const Fmt F = fmt_of(x, y, meta_at(M, e[i] / C, e[i] % C));
        if (OBF16) {
            const uint16_t h = (uint16_t)dec_code_generic<8>(c[i], F);
            memcpy(out + 2 * e[i], &h, 2);
        } else {
            const uint32_t v = dec_code_generic<24>(c[i], F);
            memcpy(out + 4 * e[i], &v, 4);
        }
    }
}

template <bool OBF16>
__global__ void k_decode_generic_blk(const uint8_t *__restrict__ packed, int64_t C, int64_t ncont, int axis, int x,
                                     int y, MetaMap M, SegOffsets so, int nseg, int4 widths,
                                     uint8_t *__restrict__ out) {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < ncont;
         idx += (int64_t)gridDim.x * blockDim.x)
        dec_container_generic_blk<OBF16>(packed, C, idx, axis, x, y, M, so, nseg, widths, out);
}

// ROWS, 8 rows x (4*NH) columns per thread (NH = 2 for bf16 out, 1 fp32);
// host guarantees bc % (4*NH) == 0, br == 1 or br % 8 == 0, x <= 7 (and
// y <= 7 for bf16 out).
template <int K, bool OBF16>
__global__ void __launch_bounds__(256, DEC_ROWS_BLK_MINB) k_dec_rows_blk(const uint8_t *__restrict__ packed, int64_t R, int64_t C, int x,
                                                      int y, MetaMap M, SegOffsets so, uint8_t *__restrict__ out,
                                                      int nseg, int4 widths) {
    using EL = Elem<OBF16>;
    constexpr int V = EL::V, NH = V / 4, TW = tile_words(K, NH);
    const int64_t CV = C / V, G = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= CV) return;
    const int64_t c0 = j * V;
    const uint8_t *mcol = M.meta + c0 / M.bc;
    uint32_t nxt[TW], nm[8];
    int64_t g = blockIdx.y;
    if (g < G) {
        rows_load_raw<K, NH, 0>(nxt, packed, so, g, C, c0);
        load_tile_meta(mcol, g, M, nm);
    }
    for (; g < G; g += gridDim.y) {
        uint32_t raw[TW], em[8];
#pragma unroll
        for (int q = 0; q < TW; ++q) raw[q] = nxt[q];
#pragma unroll
        for (int i = 0; i < 8; ++i) em[i] = nm[i];
        if (g + gridDim.y < G) {
            rows_load_raw<K, NH, 0>(nxt, packed, so, g + gridDim.y, C, c0);
            load_tile_meta(mcol, g + gridDim.y, M, nm);
        }
        RowD D[8];
        bool ok = true;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            D[i] = make_rowd(em[i] > 254u ? 254 : (int)em[i], x);
            ok = ok && D[i].ok;
        }
        if (!ok) {
            for (int v = 0; v < V; ++v)
                dec_container_generic_blk<OBF16>(packed, C, g * C + c0 + v, 0, x, y, M, so, nseg, widths, out);
            continue;
        }
        uint32_t RL[NH][8], RH[NH][8];
#pragma unroll
        for (int h = 0; h < NH; ++h)
#pragma unroll
            for (int i = 0; i < 8; ++i) { RL[h][i] = 0; RH[h][i] = 0; }
        rows_unpack_raw<K, NH, 0>(raw, RL, RH);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t o[4];
            if (OBF16) {
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    o[2 * h] = dec_pair_bf16_r<K>(pair_from_lanes<K>(RL[h][i], RH[h][i], 0x4140), y, D[i]);
                    o[2 * h + 1] = dec_pair_bf16_r<K>(pair_from_lanes<K>(RL[h][i], RH[h][i], 0x4342), y, D[i]);
                }
            } else {
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    uint32_t code = (RL[0][i] >> (8 * v)) & 0xFFu;
                    if (K == 9) code |= ((RH[0][i] >> (8 * v)) & 0xFFu) << 1;
                    o[v] = dec_f32_r<K>(code, y, D[i]);
                }
            }
            stg_v4(out + ((8 * g + i) * C + c0) * EL::ES, make_uint4(o[0], o[1], o[2], o[3]));
        }
    }
}

// COLS: lane handles groups q = base + 32u + lane (one metadata per group);
// host guarantees bc % 8 == 0 and the same format conditions.
template <int K, bool OBF16>
// 3 CTAs / SM (80 registers): per-row COLS decode e3m3 238 -> 187 us
#ifndef DEC_COLS_BLK_MINB
#define DEC_COLS_BLK_MINB 3
#endif
__global__ void __launch_bounds__(256, DEC_COLS_BLK_MINB) k_dec_cols_blk(const uint8_t *__restrict__ packed, int64_t n,
                                                                         int64_t C, int x, int y, MetaMap M,
                                                                         SegOffsets so, uint8_t *__restrict__ out,
                                                                         int nseg, int4 widths) {
    const int64_t NG = n / 8;
    const GroupMeta GM(M, C);
    const int lane = threadIdx.x & 31;
    const int64_t step = (int64_t)gridDim.x * (blockDim.x >> 5) * 128;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int64_t base = gw * 128; base < NG; base += step) {
        const int64_t rb = div_rcp(base, GM.gpr, GM.inv_gpr), qs = base - rb * GM.gpr;
        uint32_t RL[8], RH[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { RL[i] = 0; RH[i] = 0; }
        cols_fast_load<K, 0>(RL, RH, packed, so, base + lane, NG);
        const bool wr = GM.whole_rows();
        const int64_t split = GM.gpr - qs;
        RowD D0, D1;
        if (wr) {
            D0 = make_rowd(GM.row_meta(M, rb), x);
            D1 = make_rowd(rb + 1 < NG / GM.gpr ? GM.row_meta(M, rb + 1) : 0, x);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t q = base + 32 * u + lane;
            if (q >= NG) continue;
            const RowD D = wr ? ((32 * u + lane) < split ? D0 : D1) : make_rowd(GM.at_tile(M, base, rb, qs, 32 * u + lane), x);
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

// ----------------------------------------------------- quantize (blocked)
// 2D: thread = one 16-byte vector of one row (vector-aligned rows, host
// guarantees C % V == 0 and bc % V == 0 so a vector never straddles blocks).
template <bool BF16>
__global__ void __launch_bounds__(256) k_quant_blk(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                   int64_t R, int64_t C, int x, int y, MetaMap M, int force_generic) {
    using EL = Elem<BF16>;
    const int64_t CV = C / EL::V;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= CV) return;
    const int64_t c0 = j * EL::V;
    const uint8_t *mcol = M.meta + c0 / M.bc;   // this thread's block column (one division per thread)
    for (int64_t r = blockIdx.y; r < R; r += gridDim.y) {
        const uint4 v = ldg_nc_v4(in + (r * C + c0) * EL::ES);
        const int64_t rb = M.br == 1 ? r : r / M.br;
        const int em = __ldg(mcol + rb * M.nbc);
        const Fmt F = fmt_of(x, y, em > 254 ? 254 : em);
        const FastP P = make_fast(F, BF16, force_generic);
        const DecPath DP = make_dec_path(F, force_generic);
        uint32_t o[4];
        uint32_t flag = 0;
        const bool fast = BF16 ? P.enc_simd : P.enc_f32;
        if (fast) {
#pragma unroll
            for (int t = 0; t < 4; ++t)
                o[t] = BF16 ? quant_pair_bf16(word_of(v, t), P, flag) : quant_f32_fast(word_of(v, t), P, flag);
            flag &= 0x80008000u;
        }
        if (!fast || flag) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint32_t w = word_of(v, t);
                if (BF16) {
                    const uint32_t lo = quantize_elem<true>(w << 16, F, DP);
                    const uint32_t hi = quantize_elem<true>(w & 0xFFFF0000u, F, DP);
                    o[t] = (lo & 0xFFFFu) | (hi << 16);
                } else {
                    o[t] = quantize_elem<false>(w, F, DP);
                }
            }
        }
        stg_v4(out + (r * C + c0) * EL::ES, make_uint4(o[0], o[1], o[2], o[3]));
    }
}

// Narrow rows (C / V < 256 vectors, e.g. 128-column embedding tables): the
// 2D mapping above would leave most of a CTA's threads without a column.
// Here vectors are numbered over the whole tensor (row-major), a CTA takes
// one contiguous chunk of 4 x 256 vectors per iteration, and each vector
// finds its row by one 32-bit division (64-bit beyond 2^32 vectors).
template <bool BF16>
__global__ void __launch_bounds__(256) k_quant_blk_flat(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                        int64_t R, int64_t C, int x, int y, MetaMap M,
                                                        int force_generic) {
    using EL = Elem<BF16>;
    constexpr int U = 4;
    const int64_t CV = C / EL::V, nvec = R * CV;
    const bool small = nvec < (1ll << 32);
    const int64_t cstep = (int64_t)gridDim.x * blockDim.x * U;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < nvec; base += cstep) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t vi = base + (int64_t)u * blockDim.x;
            v[u] = vi < nvec ? ldg_nc_v4(in + vi * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t vi = base + (int64_t)u * blockDim.x;
            if (vi >= nvec) continue;
            const int64_t r = small ? (int64_t)((uint32_t)vi / (uint32_t)CV) : vi / CV;
            const int64_t c0 = (vi - r * CV) * EL::V;
            const int64_t rb = M.br == 1 ? r : r / M.br;
            const int64_t cb = M.nbc == 1 ? 0 : c0 / M.bc;
            const int em = __ldg(M.meta + rb * M.nbc + cb);
            const Fmt F = fmt_of(x, y, em > 254 ? 254 : em);
            const FastP P = make_fast(F, BF16, force_generic);
            uint32_t o[4];
            uint32_t flag = 0;
            const bool fast = BF16 ? P.enc_simd : P.enc_f32;
            if (fast) {
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    o[t] = BF16 ? quant_pair_bf16(word_of(v[u], t), P, flag) : quant_f32_fast(word_of(v[u], t), P, flag);
                flag &= 0x80008000u;
            }
            if (!fast || flag) {
                const DecPath DP = make_dec_path(F, force_generic);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const uint32_t w = word_of(v[u], t);
                    if (BF16) {
                        const uint32_t lo = quantize_elem<true>(w << 16, F, DP);
                        const uint32_t hi = quantize_elem<true>(w & 0xFFFF0000u, F, DP);
                        o[t] = (lo & 0xFFFFu) | (hi << 16);
                    } else {
                        o[t] = quantize_elem<false>(w, F, DP);
                    }
                }
            }
            stg_v4(out + vi * 16, make_uint4(o[0], o[1], o[2], o[3]));
        }
    }
}

template <bool BF16>
__global__ void k_quant_blk_scalar(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, int64_t R, int64_t C,
                                   int x, int y, MetaMap M, int force_generic) {
    const int64_t n = R * C;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const Fmt F = fmt_of(x, y, meta_at(M, i / C, i % C));
        const DecPath DP = make_dec_path(F, force_generic);
        if (BF16) {
            uint16_t b;
            memcpy(&b, in + 2 * i, 2);
            const uint16_t o = (uint16_t)quantize_elem<true>((uint32_t)b << 16, F, DP);
            memcpy(out + 2 * i, &o, 2);
        } else {
            uint32_t u;
            memcpy(&u, in + 4 * i, 4);
            const uint32_t o = quantize_elem<false>(u, F, DP);
            memcpy(out + 4 * i, &o, 4);
        }
    }
}

// --------------------------------------------------- block max exponent
// biased exponent of |v| (finite, fp32 bits a) rounded RTNE to y mantissa
// bits in its own binade, clamped to [0, 254]
__device__ __forceinline__ int exp_after_rounding(uint32_t a, int y) {
    if (a == 0u) return 0;
    if (a >= 0x00800000u) {   // normal: integer RTNE at bit 23-y, carry lands in the exponent
        if (y >= 23) return (int)(a >> 23);
        const int sh = 23 - y;
        const uint32_t t = a + ((1u << (sh - 1)) - 1u) + ((a >> sh) & 1u);
        const int e = (int)(t >> 23);
        return e > 254 ? 254 : e;
    }
    // fp32 subnormal: own binade is below 2^-126; only a carry to 2^-126 (exp 1) matters
    const int L = 32 - __clz(a);          // significant bits, 1..23
    const int p = L - 1 - y;              // rounding position
    if (p <= 0 || L < 23) return 0;
    const uint32_t t = a + ((1u << (p - 1)) - 1u) + ((a >> p) & 1u);
    return t >= (1u << 23) ? 1 : 0;
}

// Sub-row blocks (1 x bc, bc / V in {1, 2, 4, 8, 16, 32}: "a sub row",
// P:230-241, the small blocks e2m1 / e1m2 want): one thread per
// 16-byte vector, four vectors in flight, and the bc / V lanes holding a
// block combine their maxima with xor-shuffles; the group's first lane
// writes the block's byte (MODE 0 / 1: exponent before / after rounding) or
// its fp32 maximum (MODE 2, float scaling).  A warp-per-block kernel would
// leave most lanes idle for such blocks.
template <bool BF16, int MODE>
__global__ void __launch_bounds__(256) k_block_max_small(const uint8_t *__restrict__ in, int64_t nvec, int gsz,
                                                         int y, uint8_t *__restrict__ meta, float *__restrict__ amax_out) {
    constexpr int U = 4;
    const int lane = threadIdx.x & 31;
    // a CTA reads one contiguous chunk of U x 256 vectors per iteration (as
    // k_quant_fast); a warp's 32 consecutive vectors per u hold whole blocks
    const int64_t stride = blockDim.x;
    const int gshift = __ffs(gsz) - 1;   // gsz is a power of two
    for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x * U + (threadIdx.x - lane); v0 < nvec;
         v0 += (int64_t)gridDim.x * blockDim.x * U) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t vi = v0 + u * stride + lane;
            r[u] = vi < nvec ? ldg_nc_v4(in + vi * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t vb = v0 + u * stride;
            if (vb >= nvec) break;   // warp-uniform
            uint32_t am = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint32_t w = word_of(r[u], t);
                if (BF16) {
                    const uint32_t lo = (w << 16) & 0x7FFF0000u, hi = w & 0x7FFF0000u;
                    if (lo < 0x7F800000u) am = max(am, lo);
                    if (hi < 0x7F800000u) am = max(am, hi);
                } else {
                    const uint32_t a = w & 0x7FFFFFFFu;
                    if (a < 0x7F800000u) am = max(am, a);
                }
            }
            for (int o = 1; o < gsz; o <<= 1) am = max(am, __shfl_xor_sync(0xFFFFFFFFu, am, o));
            const int64_t vi = vb + lane;
            if ((lane & (gsz - 1)) == 0 && vi < nvec) {
                const int64_t b = vi >> gshift;
                if (MODE == 2) {
                    amax_out[b] = __uint_as_float(am);
                } else {
                    const int e = MODE == 0 ? (int)(am >> 23) : exp_after_rounding(am, y);
                    meta[b] = (uint8_t)(e > 254 ? 254 : e);
                }
            }
        }
    }
}

// bf16: 16-bit-lane max of the magnitudes with the NaN/Inf lanes zeroed;
// fp32: max of the finite magnitudes
template <bool BF16>
__device__ __forceinline__ void bmax_acc(uint32_t &am2, const uint4 &q) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const uint32_t w = word_of(q, t);
        if (BF16) {
            const uint32_t a2 = w & 0x7FFF7FFFu;
            const uint32_t sp = (a2 + 0x00800080u) & 0x80008000u;   // bit 15 of special lanes
            am2 = vmax_u16x2(am2, a2 & ~((sp >> 15) * 0xFFFFu));
        } else {
            const uint32_t a = w & 0x7FFFFFFFu;
            am2 = max(am2, a < 0x7F800000u ? a : 0u);
        }
    }
}

// 2-D blocks whose rows are short (br x bc, bc / V = gsz in {1..16}, e.g.
// 32 x 32 tiles): a CTA owns a band of br rows x a chunk of 256*U vectors
// (U = 8: 16384 bf16 columns; the launcher picks the largest U in 8,4,2
// that still gives >= 4 work items per resident CTA, else k_block_max) and
// streams it row by row -- one contiguous
// 256*U*16-byte span of a row per step, the next row's span in flight while
// this one is folded into U per-thread maxima (thread t: vectors t + 256u,
// fixed across the band).  At the band's end the gsz lanes of each block
// combine with xor-shuffles.  (A warp per span of 8 rows x 512 B reached
// 69 % of copy at 32 x 32: short strided bursts.)
template <bool BF16, int U>
__global__ void __launch_bounds__(256) k_block_max_band(const uint8_t *__restrict__ in, int64_t R, int64_t C,
                                                        int64_t br, int gsz, int y, int scheme,
                                                        uint8_t *__restrict__ meta) {
    constexpr int V = Elem<BF16>::V;
    constexpr int64_t ES = Elem<BF16>::ES;
    const int lane = threadIdx.x & 31;
    const int64_t CV = C / V;
    const int64_t nch = (CV + 256 * U - 1) / (256 * U);   // column chunks per band
    const int64_t nbands = R / br, nwork = nbands * nch;
    const int64_t nbc = CV / gsz;                      // blocks per block row
    for (int64_t wk = blockIdx.x; wk < nwork; wk += gridDim.x) {
        const int64_t band = wk / nch, v0 = (wk % nch) * 256 * U + threadIdx.x;
        const uint8_t *base = in + (band * br * C) * ES + v0 * 16;
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ok[u] = v0 + 256 * u < CV;
        uint32_t am[U];
        uint4 nx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            am[u] = 0;
            nx[u] = ok[u] ? ldg_nc_v4(base + 256 * 16 * u) : make_uint4(0, 0, 0, 0);
        }
        for (int64_t i = 0; i < br; ++i) {
            uint4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = nx[u];
            if (i + 1 < br) {
                const uint8_t *nb = base + (i + 1) * C * ES;
#pragma unroll
                for (int u = 0; u < U; ++u) nx[u] = ok[u] ? ldg_nc_v4(nb + 256 * 16 * u) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) bmax_acc<BF16>(am[u], r[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t amax = BF16 ? max(am[u] & 0xFFFFu, am[u] >> 16) << 16 : am[u];
            for (int o = 1; o < gsz; o <<= 1) amax = max(amax, __shfl_xor_sync(0xFFFFFFFFu, amax, o));
            if ((lane & (gsz - 1)) == 0 && ok[u]) {
                const int e = scheme == 0 ? (int)(amax >> 23) : exp_after_rounding(amax, y);
                meta[band * nbc + (v0 + 256 * u) / gsz] = (uint8_t)(e > 254 ? 254 : e);
            }
        }
    }
}

// one warp per block: max |finite| over the block, then the scheme's exponent.
// 16-byte path: U independent loads per lane in flight (one per iteration
// left the SM short of bytes in flight: 94 us for config 2's rows vs the
// histogram's 81 us over the same bytes).  Rows of >= 32 vectors: the warp
// walks each row; shorter block rows (e.g. 128 x 128 tiles, 16 / 32 vectors a row):
// the lanes cover several rows at once over the block's flattened vectors
// (a warp per row left 28 of 32 lanes idle and serialised the rows).
template <bool BF16>
__global__ void __launch_bounds__(256) k_block_max(const uint8_t *__restrict__ in, int64_t R, int64_t C, int64_t br,
                                                   int64_t bc, int y, int scheme, uint8_t *__restrict__ meta) {
    constexpr int U = 8;
    const int lane = threadIdx.x & 31;
    const int64_t nbc = C / bc, nb = (R / br) * nbc;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    constexpr int V = Elem<BF16>::V;
    constexpr int64_t ES = Elem<BF16>::ES;
    const bool vec = (bc % V == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) && (C % V == 0);
    const int64_t nv = bc / V;
    const bool flat = vec && (nv % 32 != 0 || (br > 1 && nv < 32 * U)) && br * nv < (1ll << 31);
    for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += warps) {
        const int64_t r0 = (b / nbc) * br, c0 = (b % nbc) * bc;
        const uint8_t *blk = in + (r0 * C + c0) * ES;
        uint32_t amax = 0;   // max finite magnitude bits (fp32 convention)
        if (flat) {
            const uint32_t tot = (uint32_t)(br * nv), nv32 = (uint32_t)nv;
            uint32_t am2 = 0;
            for (uint32_t f0 = 0; f0 < tot; f0 += 32 * U) {
                uint4 r[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t f = f0 + 32 * u + lane;
                    const uint32_t i = f / nv32;
                    r[u] = f < tot ? ldg_nc_v4(blk + (int64_t)i * C * ES + (int64_t)(f - i * nv32) * 16)
                                   : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) bmax_acc<BF16>(am2, r[u]);
            }
            amax = BF16 ? max(am2 & 0xFFFFu, am2 >> 16) << 16 : am2;
        } else {
            for (int64_t i = 0; i < br; ++i) {
                const uint8_t *row = blk + i * C * ES;
                if (vec) {
                    uint32_t am2 = 0;
                    for (int64_t v0 = 0; v0 < nv; v0 += 32 * U) {
                        uint4 r[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int64_t v = v0 + 32 * u + lane;
                            r[u] = v < nv ? ldg_nc_v4(row + v * 16) : make_uint4(0, 0, 0, 0);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) bmax_acc<BF16>(am2, r[u]);
                    }
                    if (BF16) am2 = max(am2 & 0xFFFFu, am2 >> 16) << 16;
                    amax = max(amax, am2);
                } else {
                    for (int64_t c = lane; c < bc; c += 32) {
                        const uint32_t a = load_elem_scalar<BF16>(row, c) & 0x7FFFFFFFu;
                        if (a < 0x7F800000u) amax = max(amax, a);
                    }
                }
            }
        }
        amax = __reduce_max_sync(0xFFFFFFFFu, amax);
        if (lane == 0) {
            int e = scheme == 0 ? (int)(amax >> 23) : exp_after_rounding(amax, y);
            meta[b] = (uint8_t)(e > 254 ? 254 : e);
        }
    }
}

}  // namespace exmy

namespace exmy {

// ------------------------------------------- row gather-decode (COLS layout)
// decode an arbitrary list of rows (embedding lookup).
// In the COLS layout row r's containers are groups r*gpr .. r*gpr+gpr-1, a
// contiguous byte range per segment, so a looked-up row reads exactly its
// own n*k/8 bytes.  Output row i = decode(source row idx[i]).
template <int K, int S>
__device__ __forceinline__ void cols_gather_load(uint32_t (&RL)[8], uint32_t (&RH)[8], const uint8_t *packed,
                                                 const SegOffsets &so, const int64_t (&src)[4], const bool (&ok)[4]) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S);
        const uint8_t *seg = packed + so.off[S];
        if constexpr (W == 8) {
            uint32_t a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint2 t = ok[u] ? __ldg((const uint2 *)(seg + 8 * src[u])) : make_uint2(0, 0);
                a[u] = t.x;
                b[u] = t.y;
            }
            uint32_t *dst = (K == 9) ? RH : RL;
            const uint32_t a0 = prmt(a[0], a[1], 0x5140), a1 = prmt(a[2], a[3], 0x5140);
            const uint32_t a2 = prmt(a[0], a[1], 0x7362), a3 = prmt(a[2], a[3], 0x7362);
            dst[0] = prmt(a0, a1, 0x5410); dst[1] = prmt(a0, a1, 0x7632);
            dst[2] = prmt(a2, a3, 0x5410); dst[3] = prmt(a2, a3, 0x7632);
            const uint32_t b0 = prmt(b[0], b[1], 0x5140), b1 = prmt(b[2], b[3], 0x5140);
            const uint32_t b2 = prmt(b[0], b[1], 0x7362), b3 = prmt(b[2], b[3], 0x7362);
            dst[4] = prmt(b0, b1, 0x5410); dst[5] = prmt(b0, b1, 0x7632);
            dst[6] = prmt(b2, b3, 0x5410); dst[7] = prmt(b2, b3, 0x7632);
        } else {
            uint32_t in[W];
#pragma unroll
            for (int q = 0; q < W; ++q) in[q] = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (ok[u]) {
                    if constexpr (W == 4) in[u] = __ldg((const unsigned int *)(seg + 4 * src[u]));
                    else if constexpr (W == 2)
                        in[u >> 1] |= (uint32_t)__ldg((const unsigned short *)(seg + 2 * src[u])) << (16 * (u & 1));
                    else in[0] |= (uint32_t)__ldg((const unsigned char *)(seg + src[u])) << (8 * u);
                }
            }
            swar_unpack4<W, LO>(in, RL);
        }
        cols_gather_load<K, S + 1>(RL, RH, packed, so, src, ok);
    }
}

template <int K, bool OBF16, bool PERROW>
__global__ void __launch_bounds__(256) k_dec_gather(const uint8_t *__restrict__ packed, int64_t C, int x, int y,
                                                    const uint8_t *__restrict__ meta, const int64_t *__restrict__ idx,
                                                    int64_t nidx, SegOffsets so, uint8_t *__restrict__ out,
                                                    int fmt_fast) {
    const int64_t gpr = C / 8, NG = nidx * gpr;
    const double inv = 1.0 / (double)gpr;
    const int lane = threadIdx.x & 31;
    const int64_t step = (int64_t)gridDim.x * (blockDim.x >> 5) * 128;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    RowD D0;
    if (!PERROW) D0 = make_rowd(min((int)__ldg(meta), 254), x);
    for (int64_t base = gw * 128; base < NG; base += step) {
        int64_t src[4];
        bool ok[4];
        RowD D[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t q = base + 32 * u + lane;
            ok[u] = q < NG;
            const int64_t i = ok[u] ? div_rcp(q, gpr, inv) : 0;
            const int64_t r = ok[u] ? __ldg(idx + i) : 0;
            src[u] = r * gpr + (q - i * gpr);
            D[u] = PERROW ? make_rowd(ok[u] ? min((int)__ldg(meta + r), 254) : 127, x) : D0;
            D[u].ok = D[u].ok && fmt_fast;
        }
        uint32_t RL[8], RH[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { RL[i] = 0; RH[i] = 0; }
        cols_gather_load<K, 0>(RL, RH, packed, so, src, ok);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t q = base + 32 * u + lane;
            if (!OBF16) {
                uint32_t o[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    uint32_t code = (RL[i] >> (8 * u)) & 0xFFu;
                    if (K == 9) code |= ((RH[i] >> (8 * u)) & 0xFFu) << 1;
                    o[i] = D[u].ok ? dec_f32_r<K>(code, y, D[u])
                                   : dec_code_generic<24>(code, fmt_of(x, y, PERROW ? min((int)__ldg(meta + (src[u] / gpr)), 254) : min((int)__ldg(meta), 254)));
                }
                const int64_t g0 = base + 32 * u;   // 512-byte full-sector stores (see k_dec_cols_fast)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int srcl = 16 * h + (lane >> 1);
                    const bool hi = lane & 1;
                    uint32_t v[4];
#pragma unroll
                    for (int k2 = 0; k2 < 4; ++k2) {
                        const uint32_t a = __shfl_sync(0xFFFFFFFFu, o[k2], srcl);
                        const uint32_t b = __shfl_sync(0xFFFFFFFFu, o[4 + k2], srcl);
                        v[k2] = hi ? b : a;
                    }
                    if (g0 + srcl < NG) stg_v4(out + (g0 * 32) + (32 * h + lane) * 16, make_uint4(v[0], v[1], v[2], v[3]));
                }
                continue;
            }
            if (q >= NG) continue;
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
                if (D[u].ok) {
                    o[t] = dec_pair_bf16_r<K>(cp, y, D[u]);
                } else {
                    const Fmt F = fmt_of(x, y, PERROW ? min((int)__ldg(meta + (src[u] / gpr)), 254) : min((int)__ldg(meta), 254));
                    o[t] = dec_code_generic<8>(cp & 0xFFFFu, F) | (dec_code_generic<8>(cp >> 16, F) << 16);
                }
            }
            stg_v4(out + q * 16, make_uint4(o[0], o[1], o[2], o[3]));
        }
    }
}

}  // namespace exmy

namespace exmy {

// ------------------------------------- fused per-row metadata + encode (ROWS)
// "a CTA owns whole rows, so the block max fuses into one
// encode pass".  One CTA per row group of 8 rows: pass 1 reduces the 8 row
// maxima (16-byte loads), pass 2 re-reads the same rows -- now L2-resident,
// the CTAs' working set is ~16*C bytes each -- and encodes them with the
// per-row constants.  HBM reads the input once.

// ROWS container (g, c) on the integer path with the 8 rows' e_max given
template <bool BF16, int K>
__device__ __noinline__ void enc_container_generic_rows8(const uint8_t *__restrict__ in, int64_t C, int64_t g,
                                                         int64_t c, int x, int y, const int *e8, uint8_t *packed,
                                                         const SegOffsets so, int64_t *spi, uint32_t *spb,
                                                         unsigned long long *spc, int64_t cap) {
    uint32_t cd[8];
    int64_t e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        e[i] = (8 * g + i) * C + c;
        cd[i] = enc_elem(load_elem_scalar<BF16>(in, e[i]), fmt_of(x, y, e8[i]), e[i], spi, spb, spc, cap);
    }
    const int64_t idx = g * C + c;
    int hi = K;
#pragma unroll
    for (int s = 0; s < seg_count(K); ++s) {
        const int w = seg_width(K, s), lo = hi - w;
        uint8_t *seg = packed + so.off[s];
        if (w == 8) {
            for (int i = 0; i < 8; ++i) seg[e[i]] = (uint8_t)(cd[i] >> lo);
        } else {
            uint32_t cont = 0;
            for (int i = 0; i < 8; ++i) cont |= ((cd[i] >> lo) & ((1u << w) - 1u)) << (w * i);
            for (int b = 0; b < w; ++b) seg[idx * w + b] = (uint8_t)(cont >> (8 * b));
        }
        hi = lo;
    }
}

// running max of finite magnitudes (fp32-convention bits) of one 16-byte vector
template <bool BF16>
__device__ __forceinline__ uint32_t vec_max_mag(const uint4 &v, uint32_t m) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (BF16) {
            const uint32_t a2 = w[q] & 0x7FFF7FFFu;
            const uint32_t sp = (a2 + 0x00800080u) & 0x80008000u;
            m = vmax_u16x2(m, a2 & ~((sp >> 15) * 0xFFFFu));
        } else {
            const uint32_t a = w[q] & 0x7FFFFFFFu;
            m = max(m, a < 0x7F800000u ? a : 0u);
        }
    }
    return m;
}

#ifndef RW_THREADS_N
#define RW_THREADS_N 512
#endif
constexpr int RW_THREADS = RW_THREADS_N;
#ifndef RW_HINT
#define RW_HINT 1   // L2 eviction priorities: pass 1 evict_last, pass 2 evict_first
#endif

template <int K, bool BF16, int MODE>
__global__ void __launch_bounds__(RW_THREADS) k_enc_rowwise_rows(const uint8_t *__restrict__ in, int64_t R, int64_t C,
                                                                 int x, int y, int scheme, uint8_t *__restrict__ meta,
                                                                 uint8_t *__restrict__ packed, SegOffsets so,
                                                                 int64_t *spi, uint32_t *spb,
                                                                 unsigned long long *spc, int64_t cap,
                                                                 int force_generic) {
    using EL = Elem<BF16>;
    constexpr int NW = BF16 ? 2 : 4;
    constexpr bool SIMD = (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0);
    __shared__ uint32_t s_m[RW_THREADS / 32][8];
    __shared__ int s_e[8];
    const FastP P = make_fast(fmt_of(x, y, 0), BF16, 1);
    const int64_t G = R / 8, CV16 = C / EL::V, CV4 = C / 4;
    const int64_t rstride = C * EL::ES;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t pol_keep = RW_HINT ? l2_policy_evict_last() : 0, pol_drop = RW_HINT ? l2_policy_evict_first() : 0;
    for (int64_t g = blockIdx.x; g < G; g += gridDim.x) {
        // ---- pass 1: row maxima
        uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const uint8_t *rg = in + 8 * g * rstride;
        for (int64_t j = tid; j < CV16; j += RW_THREADS) {
            uint4 v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                v[i] = RW_HINT ? ldg_nc_v4_pol(rg + i * rstride + j * 16, pol_keep) : ldg_nc_v4(rg + i * rstride + j * 16);
#pragma unroll
            for (int i = 0; i < 8; ++i) m[i] = vec_max_mag<BF16>(v[i], m[i]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t mm = BF16 ? max((m[i] & 0xFFFFu) << 16, m[i] & 0xFFFF0000u) : m[i];
            const uint32_t r = __reduce_max_sync(0xFFFFFFFFu, mm);
            if (lane == 0) s_m[warp][i] = r;
        }
        __syncthreads();
        if (tid < 8) {
            uint32_t r = 0;
#pragma unroll
            for (int w = 0; w < RW_THREADS / 32; ++w) r = max(r, s_m[w][tid]);
            int e = scheme == 0 ? (int)(r >> 23) : exp_after_rounding(r, y);
            e = e > 254 ? 254 : e;
            s_e[tid] = e;
            meta[8 * g + tid] = (uint8_t)e;
        }
        __syncthreads();
        int e8[8];
        RowP Rp[8];
        bool ok = !force_generic;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            e8[i] = s_e[i];
            Rp[i] = make_rowp<SIMD>(e8[i], x, y);
            ok = ok && Rp[i].ok;
        }
        // ---- pass 2: encode the row group (8 x 4 tiles), input now in L2
        for (int64_t jj = tid; jj < CV4; jj += RW_THREADS) {
            const int64_t c0 = jj * 4;
            uint32_t w[8][NW];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if constexpr (RW_HINT) {   // second read of the row group: last use
                    if constexpr (BF16) {
                        const uint2 t = ldg_nc_v2_pol(rg + i * rstride + c0 * EL::ES, pol_drop);
                        w[i][0] = t.x; w[i][1] = t.y;
                    } else {
                        const uint4 t = ldg_nc_v4_pol(rg + i * rstride + c0 * EL::ES, pol_drop);
                        w[i][0] = t.x; w[i][1] = t.y; w[i][2] = t.z; w[i][3] = t.w;
                    }
                } else {
                    load4<BF16>(rg + i * rstride + c0 * EL::ES, w[i]);
                }
            }
            uint32_t cp[8][2];
            uint32_t amax = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) vec_codes_r<K, BF16, MODE, NW>(w[i], cp[i], P, Rp[i], amax);
            if (ok && !amax_special<BF16, MODE>(amax, P)) {
                uint32_t RL[1][8], RH[1][8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    RL[0][i] = prmt(cp[i][0], cp[i][1], 0x6420);
                    RH[0][i] = (K == 9) ? prmt(cp[i][0] >> 1, cp[i][1] >> 1, 0x6420) : 0u;
                }
                rows_fast_store<K, 1, 0>(RL, RH, packed, so, g, C, c0);
            } else {
                for (int v = 0; v < 4; ++v)
                    enc_container_generic_rows8<BF16, K>(in, C, g, c0 + v, x, y, e8, packed, so, spi, spb, spc, cap);
            }
        }
        __syncthreads();   // s_e / s_m reused by the next row group
    }
}

// ------------------- fused per-row metadata + encode, TMA-staged (ROWS)
// Rows up to RWS_MAX_ROW_BYTES: the CTA's row group (8 rows) is copied into
// shared memory by bulk asynchronous copies (cp.async.bulk, one per row,
// completion counted on an mbarrier), so pass 1 (the 8 row maxima) and pass 2
// (the encode) both read shared memory: HBM is read exactly once and no L2
// residency is assumed.  Several CTAs per SM overlap one CTA's copy with
// another's passes.
constexpr int RWS_THREADS = 256;
constexpr int64_t RWS_MAX_ROW_BYTES = 9216;   // 8 rows <= 72 KB of shared memory: 3 CTAs per SM

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "RWS_WAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra RWS_WAIT%=;\n\t}" ::"r"(bar), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// one row group (8 rows starting at row 8g of a C-column tensor `in`):
// stage, row maxima -> meta[8g..8g+7], encode.  Called by every thread of the
// CTA with the same arguments; `phase` is the mbarrier parity of this use.
template <int K, bool BF16, int MODE>
__device__ __forceinline__ void rws_row_group(const uint8_t *__restrict__ in, int64_t C, int64_t g, int x, int y,
                                              int scheme, uint8_t *__restrict__ meta, uint8_t *__restrict__ packed,
                                              const SegOffsets &so, int64_t *spi, uint32_t *spb,
                                              unsigned long long *spc, int64_t cap, int force_generic,
                                              const FastP &P, uint8_t *rws_sm, uint32_t sbase, uint32_t bar,
                                              uint32_t phase, uint32_t (*s_m)[8], int *s_e) {
    using EL = Elem<BF16>;
    constexpr int NW = BF16 ? 2 : 4;
    constexpr bool SIMD = (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0);
    const uint32_t rowb = (uint32_t)(C * EL::ES);
    const int CV16 = (int)(rowb / 16), CV4 = (int)(C / 4);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {   // the row group's 8 rows -> shared memory (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of the buffer
        mbar_expect_tx(bar, 8u * rowb);
#pragma unroll
        for (int i = 0; i < 8; ++i) bulk_g2s(sbase + i * rowb, in + (8 * g + i) * (int64_t)rowb, rowb, bar);
    }
    mbar_wait(bar, phase);
    // ---- pass 1: row maxima from shared memory
    uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = tid; j < CV16; j += RWS_THREADS) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint4 v = *reinterpret_cast<const uint4 *>(rws_sm + i * rowb + j * 16);
            m[i] = vec_max_mag<BF16>(v, m[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t mm = BF16 ? max((m[i] & 0xFFFFu) << 16, m[i] & 0xFFFF0000u) : m[i];
        const uint32_t r = __reduce_max_sync(0xFFFFFFFFu, mm);
        if (lane == 0) s_m[warp][i] = r;
    }
    __syncthreads();
    if (tid < 8) {
        uint32_t r = 0;
#pragma unroll
        for (int w = 0; w < RWS_THREADS / 32; ++w) r = max(r, s_m[w][tid]);
        int e = scheme == 0 ? (int)(r >> 23) : exp_after_rounding(r, y);
        e = e > 254 ? 254 : e;
        s_e[tid] = e;
        meta[8 * g + tid] = (uint8_t)e;
    }
    __syncthreads();
    int e8[8];
    bool ok = !force_generic;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        e8[i] = s_e[i];
        ok = ok && make_rowp<SIMD>(e8[i], x, y).ok;
    }
    // ---- pass 2: encode the row group (8 x 4 tiles) from shared memory
    for (int jj = tid; jj < CV4; jj += RWS_THREADS) {
        const int c0 = jj * 4;
        uint32_t w[8][NW];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint8_t *sp = rws_sm + i * rowb + c0 * EL::ES;
            if constexpr (BF16) {
                const uint2 t = *reinterpret_cast<const uint2 *>(sp);
                w[i][0] = t.x; w[i][1] = t.y;
            } else {
                const uint4 t = *reinterpret_cast<const uint4 *>(sp);
                w[i][0] = t.x; w[i][1] = t.y; w[i][2] = t.z; w[i][3] = t.w;
            }
        }
        uint32_t cp[8][2];
        uint32_t amax = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) vec_codes_r<K, BF16, MODE, NW>(w[i], cp[i], P, make_rowp<SIMD>(e8[i], x, y), amax);
        if (ok && !amax_special<BF16, MODE>(amax, P)) {
            uint32_t RL[1][8], RH[1][8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                RL[0][i] = prmt(cp[i][0], cp[i][1], 0x6420);
                RH[0][i] = (K == 9) ? prmt(cp[i][0] >> 1, cp[i][1] >> 1, 0x6420) : 0u;
            }
            rows_fast_store<K, 1, 0>(RL, RH, packed, so, g, C, c0);
        } else {
            for (int v = 0; v < 4; ++v)
                enc_container_generic_rows8<BF16, K>(in, C, g, c0 + v, x, y, e8, packed, so, spi, spb, spc, cap);
        }
    }
    __syncthreads();   // buffer, s_e and s_m are reused by the next row group
}

template <int K, bool BF16, int MODE>
__global__ void __launch_bounds__(RWS_THREADS) k_enc_rowwise_smem(const uint8_t *__restrict__ in, int64_t R, int64_t C,
                                                                 int x, int y, int scheme, uint8_t *__restrict__ meta,
                                                                 uint8_t *__restrict__ packed, SegOffsets so,
                                                                 int64_t *spi, uint32_t *spb,
                                                                 unsigned long long *spc, int64_t cap,
                                                                 int force_generic) {
    extern __shared__ __align__(16) uint8_t rws_sm[];   // 8 rows of C elements
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ uint32_t s_m[RWS_THREADS / 32][8];
    __shared__ int s_e[8];
    const FastP P = make_fast(fmt_of(x, y, 0), BF16, 1);
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(rws_sm);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    for (int64_t g = blockIdx.x; g < R / 8; g += gridDim.x, phase ^= 1u)
        rws_row_group<K, BF16, MODE>(in, C, g, x, y, scheme, meta, packed, so, spi, spb, spc, cap, force_generic, P,
                                     rws_sm, sbase, bar, phase, s_m, s_e);
}

// ------------ fused per-row metadata + encode for WIDE rows (thread-block
// cluster, distributed shared memory).  A cluster of CL CTAs owns one row
// group (8 rows) at a time; CTA rank r stages the column slab
// [r C / CL, (r + 1) C / CL) of the 8 rows in its shared memory with 8 bulk
// asynchronous copies (cp.async.bulk on an mbarrier), reduces the slab's 8
// row maxima, and the CTAs exchange those partial maxima through distributed
// shared memory (a cluster barrier, then loads from the peers' shared memory
// via map_shared_rank) -- so every CTA knows the row group's 8 metadata bytes
// and encodes its slab from its own shared memory.  HBM is read exactly once
// for rows up to CL x 9 KB (config 2's 32 KB rows: CL = 4), where the
// single-CTA staged kernel stops at 9 KB and the two-pass kernel re-reads
// the rows from L2.  The partial maxima are double-buffered by row-group
// parity: one cluster barrier per row group keeps a peer's slot stable
// until every CTA has read it.
template <int K, bool BF16, int MODE, int CL, int NST>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(RWS_THREADS)
    k_enc_rowwise_cluster(const uint8_t *__restrict__ in, int64_t R, int64_t C, int x, int y, int scheme,
                          uint8_t *__restrict__ meta, uint8_t *__restrict__ packed, SegOffsets so, int64_t *spi,
                          uint32_t *spb, unsigned long long *spc, int64_t cap, int force_generic) {
    using EL = Elem<BF16>;
    constexpr int NW = BF16 ? 2 : 4;
    constexpr bool SIMD = (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0);
    extern __shared__ __align__(16) uint8_t rws_sm[];   // NST stages of 8 rows x C / CL elements
    __shared__ __align__(8) unsigned long long s_bar[NST];
    __shared__ uint32_t s_m[RWS_THREADS / 32][8];
    __shared__ uint32_t s_part[2][8];   // this slab's 8 row maxima (fp32 magnitude bits), by row-group parity
    __shared__ int s_e[8];
    cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
    const int rank = (int)cluster.block_rank();
    const FastP P = make_fast(fmt_of(x, y, 0), BF16, 1);
    const int64_t Cs = C / CL;                              // slab columns
    const uint32_t rowb = (uint32_t)(Cs * EL::ES);          // slab row bytes (staged)
    const uint32_t stb = 8u * rowb;                         // stage bytes
    const int64_t growb = C * EL::ES;                       // tensor row bytes
    const int CV16 = (int)(rowb / 16), CV4 = (int)(Cs / 4);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(rws_sm);
    if (tid == 0) {
        for (int st = 0; st < NST; ++st) mbar_init((uint32_t)__cvta_generic_to_shared(&s_bar[st]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t ncl = gridDim.x / CL, cid = blockIdx.x / CL, G = R / 8;
    // this CTA's slab of row group g -> stage st (async proxy; one thread)
    auto issue = [&](int64_t g, int st) {
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar[st]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, stb);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            bulk_g2s(sbase + st * stb + i * rowb, in + (8 * g + i) * growb + (int64_t)rank * rowb, rowb, bar);
    };
    if (tid == 0 && cid < G) issue(cid, 0);
    uint32_t phase[NST];
#pragma unroll
    for (int st = 0; st < NST; ++st) phase[st] = 0;
    int it = 0;
    for (int64_t g = cid; g < G; g += ncl, ++it) {
        const int st = NST == 2 ? (it & 1) : 0, par = it & 1;
        // double-buffered: the next row group's slab is in flight during this one
        if (NST == 2 && tid == 0 && g + ncl < G) issue(g + ncl, st ^ 1);
        mbar_wait((uint32_t)__cvta_generic_to_shared(&s_bar[st]), phase[st]);
        phase[st] ^= 1u;
        const uint8_t *buf = rws_sm + st * stb;
        // ---- pass 1: the slab's row maxima
        uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int j = tid; j < CV16; j += RWS_THREADS) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint4 v = *reinterpret_cast<const uint4 *>(buf + i * rowb + j * 16);
                m[i] = vec_max_mag<BF16>(v, m[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t mm = BF16 ? max((m[i] & 0xFFFFu) << 16, m[i] & 0xFFFF0000u) : m[i];
            const uint32_t r = __reduce_max_sync(0xFFFFFFFFu, mm);
            if (lane == 0) s_m[warp][i] = r;
        }
        __syncthreads();
        if (tid < 8) {
            uint32_t r = 0;
#pragma unroll
            for (int w = 0; w < RWS_THREADS / 32; ++w) r = max(r, s_m[w][tid]);
            s_part[par][tid] = r;
        }
        cluster.sync();   // every slab's partial maxima are written
        if (tid < 8) {    // the row's maximum over the cluster's slabs (distributed shared memory)
            uint32_t r = 0;
#pragma unroll
            for (int q = 0; q < CL; ++q) r = max(r, *cluster.map_shared_rank(&s_part[par][tid], q));
            int e = scheme == 0 ? (int)(r >> 23) : exp_after_rounding(r, y);
            e = e > 254 ? 254 : e;
            s_e[tid] = e;
            if (rank == 0) meta[8 * g + tid] = (uint8_t)e;
        }
        __syncthreads();
        int e8[8];
        bool ok = !force_generic;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            e8[i] = s_e[i];
            ok = ok && make_rowp<SIMD>(e8[i], x, y).ok;
        }
        // ---- pass 2: encode the slab (8 x 4 tiles) from shared memory
        for (int jj = tid; jj < CV4; jj += RWS_THREADS) {
            const int64_t c0 = (int64_t)rank * Cs + jj * 4;   // tensor column
            uint32_t w[8][NW];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint8_t *sp = buf + i * rowb + jj * 4 * EL::ES;
                if constexpr (BF16) {
                    const uint2 t = *reinterpret_cast<const uint2 *>(sp);
                    w[i][0] = t.x; w[i][1] = t.y;
                } else {
                    const uint4 t = *reinterpret_cast<const uint4 *>(sp);
                    w[i][0] = t.x; w[i][1] = t.y; w[i][2] = t.z; w[i][3] = t.w;
                }
            }
            uint32_t cp[8][2];
            uint32_t amax = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                vec_codes_r<K, BF16, MODE, NW>(w[i], cp[i], P, make_rowp<SIMD>(e8[i], x, y), amax);
            if (ok && !amax_special<BF16, MODE>(amax, P)) {
                uint32_t RL[1][8], RH[1][8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    RL[0][i] = prmt(cp[i][0], cp[i][1], 0x6420);
                    RH[0][i] = (K == 9) ? prmt(cp[i][0] >> 1, cp[i][1] >> 1, 0x6420) : 0u;
                }
                rows_fast_store<K, 1, 0>(RL, RH, packed, so, g, C, c0);
            } else {
                for (int v = 0; v < 4; ++v)
                    enc_container_generic_rows8<BF16, K>(in, C, g, c0 + v, x, y, e8, packed, so, spi, spb, spc, cap);
            }
        }
        __syncthreads();   // this stage and s_e are reused two (one) row groups on
        if (NST == 1 && tid == 0 && g + ncl < G) issue(g + ncl, 0);
    }
    cluster.sync();   // no CTA leaves while a peer may still read its partial maxima
}

}  // namespace exmy
