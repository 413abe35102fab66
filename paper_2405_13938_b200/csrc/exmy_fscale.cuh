// exmy_fscale.cuh -- the float-scaling block scheme (Fig. 2's third scheme,
// "float scaling with maximum exponent of 127"; reading D23 in
// DESIGN.md).  Each block carries one fp32 metadata value, its largest finite
// magnitude amax = A1 * 2^p (A1 in [1,2)); codes live on the e_max = 127 grid
// whose top is G.
//   encode: u = RN32(v * RN32(G / A1) * 2^-p)         (FMUL when the factor is
//           a normal fp32, else one fp64 product), code = e_max-127 code of u
//   decode: out = RN32(g amax / G), g the code's exact value at e_max 127.
//           Computed as RN32(g s_hi + RN32(g s_lo)) with s_hi = RN32(amax/G),
//           s_lo = RN32((amax - s_hi G) / G) (one FMUL + one FFMA per
//           element): its relative error <= 2^-47 cannot move a result
//           >= 2^-100 across a rounding boundary, because g amax / G is either
//           an fp32 value (an exact binary fraction has the integer
//           significand M_g M_a / M_G < 2^24) or >= 2^-34 (relative) away
//           from every fp32 midpoint.  Smaller results (fp32 subnormals, tiny
//           maxima) and x = 8 codes below the fp32 range take fs_out_exact,
//           the integer evaluation of the definition.
// so the block maximum decodes to exactly amax.
#pragma once
#include "exmy_blocked.cuh"

namespace exmy {

// block (i, j) of a (R, C) tensor tiled by (br x bc) owns amax[i * nbc + j]
struct FsMap {
    const float *amax;
    int64_t br, bc, nbc;
    float tchk;   // rows / blocks with s_hi < tchk may produce results < 2^-100: per-element check
    int x8;       // x = 8: codes below the fp32 range, every element takes fs_out_exact
};

// RN32(g * amax / G) evaluated with integers (reading D23's definition), for
// the results the FMUL + FFMA decode cannot guarantee.  mag = the code's
// magnitude bits, amax = the block's fp32 maximum (bits, positive).  Returns
// the result's magnitude bits; the caller attaches the code's sign.
//   g = M_g 2^eg, amax = M_a 2^ea, G = M_G 2^eG  ->  (M_g M_a / M_G) 2^(eg+ea-eG),
// the quotient taken to >= 54 bits plus a sticky remainder, then rounded once
// at the fp32 quantum (2^-149 in the subnormal range), ties to even.
__device__ __noinline__ uint32_t fs_out_exact(uint32_t mag, uint32_t amax, int x, int y) {
    if (mag == 0u || amax == 0u) return 0u;
    const int bias = (1 << x) - 1;                               // e_max 127 (D1)
    const uint32_t e = x == 0 ? 0u : (mag >> y), m = mag & ((1u << y) - 1u);
    const uint32_t Mg = e ? ((1u << y) | m) : m;
    const int eg = e ? (int)e - bias - y : 1 - bias - y;
    const uint32_t MG = x >= 1 ? (2u << y) - 1u : (1u << y) - 1u;   // G's integer significand
    const int eG = x >= 1 ? -y : 1 - y;
    const uint32_t Ea = amax >> 23, fa = amax & 0x7FFFFFu;
    const uint32_t Ma = Ea ? (fa | 0x800000u) : fa;
    const int ea = Ea ? (int)Ea - 150 : -149;
    const unsigned long long N = (unsigned long long)Mg * Ma;    // < 2^33, > 0
    const int L = __clzll((long long)N) - 1;                     // N << L in [2^62, 2^63)
    const unsigned long long num = N << L;
    const unsigned long long q = num / MG, rem = num - q * MG;   // q >= 2^53
    const int E0 = eg + ea - eG - L;                             // value = (q + rem / MG) 2^E0
    const int b = 64 - __clzll((long long)q);
    int qe = E0 + b - 24;                                        // quantum of a 24-bit significand
    if (qe < -149) qe = -149;
    const int sh = qe - E0;                                      // >= b - 24
    if (sh > b) return 0u;                                       // below half the quantum
    unsigned long long kept, r;
    if (sh >= 64) {
        kept = 0ull;
        r = q;
    } else {
        kept = q >> sh;
        r = q & ((1ull << sh) - 1ull);
    }
    const unsigned long long half = 1ull << (sh - 1);
    if (r > half || (r == half && (rem != 0ull || (kept & 1ull)))) ++kept;
    if (kept >= (1ull << 24)) {                                  // carry into the next binade
        kept >>= 1;
        ++qe;
    }
    if (kept >= (1ull << 23)) return ((uint32_t)(qe + 150) << 23) | ((uint32_t)kept - 0x800000u);
    return (uint32_t)kept;                                       // fp32 subnormal (qe = -149)
}

__device__ __forceinline__ uint32_t fs_amax_at(const FsMap &S, int64_t r, int64_t c) {
    return __float_as_uint(__ldg(S.amax + (r / S.br) * S.nbc + c / S.bc)) & 0x7FFFFFFFu;
}

// block row of tensor row r without a 64-bit division in the common cases
// (per-row blocks, block rows a multiple of the 8-row tile)
__device__ __forceinline__ int64_t fs_rb(const FsMap &S, int64_t r) {
    if (S.br == 1) return r;
    if ((r >> 31) == 0 && (S.br >> 31) == 0) return (int64_t)((uint32_t)r / (uint32_t)S.br);
    return r / S.br;
}

// amax = A1 * 2^p, A1 in [1, 2) (a subnormal amax is normalised); amax != 0
__device__ __forceinline__ void fs_split(uint32_t a, float &A1, int &p) {
    const int E = (int)(a >> 23);
    if (E == 0) {
        const int hb = 31 - __clz(a);   // highest set bit, < 23
        const int s = 23 - hb;
        A1 = __uint_as_float(0x3F800000u | ((a << s) & 0x7FFFFFu));
        p = -126 - s;
    } else {
        A1 = __uint_as_float(0x3F800000u | (a & 0x7FFFFFu));
        p = E - 127;
    }
}

__device__ __forceinline__ double fs_pow2d(int e) {   // e in [-1022, 1023]
    return __longlong_as_double((long long)(e + 1023) << 52);
}

// encode factor of one block
struct FsE {
    float rr;     // RN32(G/A1) * 2^-p when that is a normal fp32 (mode 1)
    float r1;     // RN32(G/A1)
    int p;
    int mode;     // 0: amax = 0 (u = v * 0), 1: fp32 multiply, 2: fp64 product
};

__device__ __forceinline__ FsE fs_enc(uint32_t amax, float G) {
    FsE q;
    if (amax == 0u) {
        q.mode = 0; q.rr = q.r1 = 0.f; q.p = 0;
        return q;
    }
    float A1;
    fs_split(amax, A1, q.p);
    q.r1 = __fdiv_rn(G, A1);   // in (G/2, G] with G in [1, 2): exponent -1 or 0 (x = 0, y = 1: G = 1)
    // r1 * 2^-p is a normal fp32 for -126 <= e(r1) - p <= 127
    q.mode = (q.p >= -126 && q.p <= 125) ? 1 : 2;
    q.rr = q.mode == 1 ? __fmul_rn(q.r1, __uint_as_float((uint32_t)(127 - q.p) << 23)) : 0.f;   // exact
    return q;
}

// scaled fp32 pattern of a finite input pattern v
__device__ __forceinline__ uint32_t fs_in(uint32_t v, const FsE &q) {
    if (q.mode == 1) return __float_as_uint(__fmul_rn(__uint_as_float(v), q.rr));
    if (q.mode == 0) return v & 0x80000000u;
    const double prod = (double)__uint_as_float(v) * (double)q.r1;   // exact (24 x 24 bits)
    return __float_as_uint(__double2float_rn(prod * fs_pow2d(-q.p)));  // exact scaling, one rounding
}

// decode factors of one block: s_hi + s_lo ~ amax / G (reading D23)
struct FsD {
    float hi, lo;
};

__device__ __forceinline__ FsD fs_dec(uint32_t amax, float G) {
    FsD d;
    const float a = __uint_as_float(amax);
    d.hi = __fdiv_rn(a, G);
    if (amax >= 0x0D800000u) {   // amax >= 2^-100: the residual a - hi G is an fp32 (exact FMA)
        d.lo = __fdiv_rn(__fmaf_rn(-d.hi, G, a), G);
    } else {                     // tiny amax: exact residual in fp64, quotient rounded once
        const double r = fma(-(double)d.hi, (double)G, (double)a);
        d.lo = __double2float_rn(__ddiv_rn(r, (double)G));
    }
    return d;
}

// RN32(g s_hi + RN32(g s_lo)) computed on |g| (hi + lo >= 0: the result is
// >= 0) with g's sign attached, so a zero result keeps the code's sign
__device__ __forceinline__ uint32_t fs_out(uint32_t gbits, const FsD &d) {
    const float g = __uint_as_float(gbits & 0x7FFFFFFFu);
    return __float_as_uint(__fmaf_rn(g, d.hi, __fmul_rn(g, d.lo))) | (gbits & 0x80000000u);
}

__device__ __forceinline__ uint32_t f32_to_bf16_bits(uint32_t f) {   // RTNE, finite input (no carry past Inf:
    return (f + 0x7FFFu + ((f >> 16) & 1u)) >> 16;                     // |f| <= amax < 2^128 rounds to <= max)
}

// ------------------------------------------------------------ block max
// one warp per block: the largest finite magnitude (fp32 bits) -> amax[b]
template <bool BF16>
__global__ void __launch_bounds__(256) k_block_amax(const uint8_t *__restrict__ in, int64_t R, int64_t C, int64_t br,
                                                    int64_t bc, float *__restrict__ amax_out) {
    const int lane = threadIdx.x & 31;
    const int64_t nbc = C / bc, nb = (R / br) * nbc;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    constexpr int V = Elem<BF16>::V;
    const bool vec = (bc % V == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) && (C % V == 0);
    for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += warps) {
        const int64_t r0 = (b / nbc) * br, c0 = (b % nbc) * bc;
        uint32_t am = 0;
        for (int64_t i = 0; i < br; ++i) {
            const uint8_t *row = in + ((r0 + i) * C + c0) * Elem<BF16>::ES;
            if (vec) {
                for (int64_t v = lane; v < bc / V; v += 32) {
                    const uint4 q = ldg_nc_v4(row + v * 16);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const uint32_t w = word_of(q, t);
                        if (BF16) {
                            const uint32_t lo = (w << 16) & 0x7FFF0000u, hi = w & 0x7FFF0000u;
                            if (lo < 0x7F800000u) am = max(am, lo);
                            if (hi < 0x7F800000u) am = max(am, hi);
                        } else {
                            const uint32_t a = w & 0x7FFFFFFFu;
                            if (a < 0x7F800000u) am = max(am, a);
                        }
                    }
                }
            } else {
                for (int64_t c = lane; c < bc; c += 32) {
                    const uint32_t a = load_elem_scalar<BF16>(row, c) & 0x7FFFFFFFu;
                    if (a < 0x7F800000u) am = max(am, a);
                }
            }
        }
        am = __reduce_max_sync(0xFFFFFFFFu, am);
        if (lane == 0) amax_out[b] = __uint_as_float(am);
    }
}

// ------------------------------------------------------ generic containers
template <bool BF16, int K>
__device__ __noinline__ void fs_enc_container(const uint8_t *__restrict__ in, int64_t C, int64_t idx, int axis, int x,
                                              int y, const FsMap S, float G, uint8_t *packed, const SegOffsets so,
                                              int64_t *spi, uint32_t *spb, unsigned long long *spc, int64_t cap) {
    const Fmt F = fmt_of(x, y, 127);
    uint32_t c[8];
    int64_t e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        e[i] = lane_elem(idx, i, C, axis);
        const uint32_t v = load_elem_scalar<BF16>(in, e[i]);
        if (is_special_f32(v)) {
            push_special(e[i], v, spi, spb, spc, cap);
            c[i] = 0u;
        } else {
            c[i] = enc_code_generic(fs_in(v, fs_enc(fs_amax_at(S, e[i] / C, e[i] % C), G)), F);
        }
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
__global__ void k_fs_encode_generic(const uint8_t *__restrict__ in, int64_t C, int64_t ncont, int axis, int x, int y,
                                    FsMap S, float G, uint8_t *__restrict__ packed, SegOffsets so, int64_t *spi,
                                    uint32_t *spb, unsigned long long *spc, int64_t cap) {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < ncont;
         idx += (int64_t)gridDim.x * blockDim.x)
        fs_enc_container<BF16, K>(in, C, idx, axis, x, y, S, G, packed, so, spi, spb, spc, cap);
}

template <bool OBF16>
__device__ __noinline__ void fs_dec_container(const uint8_t *__restrict__ packed, int64_t C, int64_t idx, int axis,
                                              int x, int y, const FsMap S, float G, const SegOffsets so, int nseg,
                                              int4 widths, uint8_t *out) {
    const int wd[4] = {widths.x, widths.y, widths.z, widths.w};
    const Fmt F = fmt_of(x, y, 127);
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
        const uint32_t am = fs_amax_at(S, e[i] / C, e[i] % C);
        uint32_t o = fs_out(dec_code_generic<24>(c[i], F), fs_dec(am, G));
        const uint32_t mag = c[i] & F.M;
        if (mag != 0u && (S.x8 || (o & 0x7FFFFFFFu) < 0x0D800000u))   // results < 2^-100: the definition itself
            o = fs_out_exact(mag, am, x, y) | (o & 0x80000000u);
        if (OBF16) {
            const uint16_t h = (uint16_t)f32_to_bf16_bits(o);
            memcpy(out + 2 * e[i], &h, 2);
        } else {
            memcpy(out + 4 * e[i], &o, 4);
        }
    }
}

template <bool OBF16>
__global__ void k_fs_decode_generic(const uint8_t *__restrict__ packed, int64_t C, int64_t ncont, int axis, int x, int y,
                                    FsMap S, float G, SegOffsets so, int nseg, int4 widths,
                                    uint8_t *__restrict__ out) {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < ncont;
         idx += (int64_t)gridDim.x * blockDim.x)
        fs_dec_container<OBF16>(packed, C, idx, axis, x, y, S, G, so, nseg, widths, out);
}

// ------------------------------------------------------------ emulation
// out = decode(encode(v)) in v's dtype; one 16-byte vector per thread, whose
// elements share one block when bc % V == 0 (else per element).  FAST: the
// e_max-127 grid rounding by the one-addition fp32 trick (x <= 7), else the
// integer code path.
template <bool BF16, bool FAST>
__device__ __forceinline__ uint32_t fs_quant_elem(uint32_t u, const FsE &fe, const FsD &fd, const Fmt &F,
                                                  const FastP &P, const FsMap &S, uint32_t am) {
    (void)S;
    (void)am;   // results below 2^-100 are redone exactly by k_fs_quant_fixup
    if (is_special_f32(u)) return u;
    const uint32_t us = fs_in(u, fe);
    uint32_t g;
    if (FAST) {
        uint32_t flag = 0;
        g = quant_f32_fast(us, P, flag);
    } else {
        g = dec_code_generic<24>(enc_code_generic(us, F), F);
    }
    const uint32_t o = fs_out(g, fd);
    return BF16 ? (f32_to_bf16_bits(o) << 16) : o;
}

// the exact float-scaled emulation of one finite input pattern: the
// e_max-127 code of the scaled value, then RN32(g amax / G) by integers
__device__ __noinline__ uint32_t fs_quant_exact(uint32_t u, uint32_t am, float G, int x, int y) {
    const Fmt F = fmt_of(x, y, 127);
    const uint32_t code = enc_code_generic(fs_in(u, fs_enc(am, G)), F);
    return fs_out_exact(code & F.M, am, x, y) | ((code >> (x + y)) << 31);
}

template <bool BF16>
__device__ __forceinline__ void fs_put(uint32_t (&w)[4], int v, uint32_t o) {
    if (BF16) {
        const uint32_t h = o >> 16;
        w[v >> 1] = (v & 1) ? ((w[v >> 1] & 0xFFFFu) | (h << 16)) : ((w[v >> 1] & 0xFFFF0000u) | h);
    } else {
        w[v] = o;
    }
}

// MODE 2 (host: C % V == 0, R % 8 == 0, bc % (32 V) == 0): 2-D grid, a
// thread takes one 16-byte column vector of 8 consecutive rows; a warp's 32
// vectors share a block column, so lanes 0..7 compute the 8 rows' factors
// and broadcast them.  MODE 1 (C % V == 0, bc % V == 0): the same grid one
// row at a time, factors per thread.  MODE 0: one vector per thread, the
// block looked up per element.
template <bool BF16, bool FAST, int MODE>
__global__ void __launch_bounds__(256) k_fs_quant(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, int64_t R,
                                                  int64_t C, int x, int y, FsMap S, float G) {
    using EL = Elem<BF16>;
    constexpr int V = EL::V;
    const Fmt F = fmt_of(x, y, 127);
    const FastP P = make_fast(F, false, 0);
    if (MODE == 2) {
        const int64_t CVv = C / V;
        const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const bool act = j < CVv;
        const int lane = threadIdx.x & 31;
        const float *scol = S.amax + ((act ? j : 0) * V) / S.bc;
        for (int64_t g = blockIdx.y; g < R / 8; g += gridDim.y) {
            const uint32_t am0 = __float_as_uint(__ldg(scol + fs_rb(S, 8 * g + (lane & 7)) * S.nbc)) & 0x7FFFFFFFu;
            const FsE fe0 = fs_enc(am0, G);
            const FsD fd0 = fs_dec(am0, G);
            uint4 q[8];
            if (act) {
#pragma unroll
                for (int i = 0; i < 8; ++i) q[i] = ldg_nc_v4(in + ((8 * g + i) * C + j * V) * EL::ES);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                FsE fe;
                fe.rr = __shfl_sync(0xFFFFFFFFu, fe0.rr, i);
                fe.r1 = __shfl_sync(0xFFFFFFFFu, fe0.r1, i);
                fe.p = __shfl_sync(0xFFFFFFFFu, fe0.p, i);
                fe.mode = __shfl_sync(0xFFFFFFFFu, fe0.mode, i);
                FsD fd;
                fd.hi = __shfl_sync(0xFFFFFFFFu, fd0.hi, i);
                fd.lo = __shfl_sync(0xFFFFFFFFu, fd0.lo, i);
                const uint32_t am = __shfl_sync(0xFFFFFFFFu, am0, i);
                if (!act) continue;
                uint32_t w[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
#pragma unroll
                for (int v = 0; v < V; ++v)
                    fs_put<BF16>(w, v, fs_quant_elem<BF16, FAST>(vec_elem<BF16>(q[i], v), fe, fd, F, P, S, am));
                stg_v4(out + ((8 * g + i) * C + j * V) * EL::ES, make_uint4(w[0], w[1], w[2], w[3]));
            }
        }
    } else if (MODE == 1) {
        const int64_t CVv = C / V;
        const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (j >= CVv) return;
        const float *scol = S.amax + (j * V) / S.bc;
        for (int64_t r = blockIdx.y; r < R; r += gridDim.y) {
            const int64_t off = (r * C + j * V) * EL::ES;
            const uint4 q = ldg_nc_v4(in + off);
            const uint32_t am = __float_as_uint(__ldg(scol + fs_rb(S, r) * S.nbc)) & 0x7FFFFFFFu;
            const FsE fe = fs_enc(am, G);
            const FsD fd = fs_dec(am, G);
            uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int v = 0; v < V; ++v)
                fs_put<BF16>(w, v, fs_quant_elem<BF16, FAST>(vec_elem<BF16>(q, v), fe, fd, F, P, S, am));
            stg_v4(out + off, make_uint4(w[0], w[1], w[2], w[3]));
        }
    } else {
        const int64_t nvec = R * C / V;
        for (int64_t vi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; vi < nvec;
             vi += (int64_t)gridDim.x * blockDim.x) {
            const uint4 q = ldg_nc_v4(in + vi * 16);
            uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int64_t e = vi * V + v;
                const uint32_t am = fs_amax_at(S, e / C, e % C);
                fs_put<BF16>(w, v, fs_quant_elem<BF16, FAST>(vec_elem<BF16>(q, v), fs_enc(am, G), fs_dec(am, G), F, P, S, am));
            }
            stg_v4(out + vi * 16, make_uint4(w[0], w[1], w[2], w[3]));
        }
    }
}

// ------------------------------------------------------- encode ROWS fast
// 8-row x 4-column tiles as k_enc_rows_fast (host: bc % 4 == 0, so the 4
// columns of a row share a block).  WSHARE (host: bc % 128 == 0, or bc = 32 /
// 64): a warp's 128 columns span 1, 2 or 4 block columns, so 8 x that many
// lanes compute the 8 rows' factors once and broadcast them (one division per
// lane instead of eight);
// otherwise each thread computes its 8.  The scaled patterns go through the
// fp32 one-addition code path at e_max 127.  Tiles with NaN/Inf, amax = 0 or
// an extreme amax take the integer path.
template <int K, bool BF16, bool Y0, bool WSHARE>
__global__ void __launch_bounds__(256, 2) k_fs_enc_rows(const uint8_t *__restrict__ in, int64_t R, int64_t C, int x,
                                                        int y, FsMap S, float G, uint8_t *__restrict__ packed,
                                                        SegOffsets so, int64_t *spi, uint32_t *spb,
                                                        unsigned long long *spc, int64_t cap, int lpb) {
    using EL = Elem<BF16>;
    constexpr int NW = BF16 ? 2 : 4;
    const Fmt F = fmt_of(x, y, 127);
    const FastP P = make_fast(F, false, 0);
    const int64_t CV = C / 4, G8 = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (!WSHARE && j >= CV) return;
    const bool act = j < CV;               // WSHARE: whole warps stay for the shuffles
    const int lane = threadIdx.x & 31;
    const int64_t c0 = (act ? j : 0) * 4;
    const uint8_t *src = in + c0 * EL::ES;
    const int64_t rstride = C * EL::ES;
    const float *scol = S.amax + c0 / S.bc;   // this thread's block column
    // WSHARE: lanes (8q .. 8q+7) compute the 8 rows' factors of the warp's
    // q-th block column (lpb lanes per block column); lane t reads row i from
    // lane i + 8 (t / lpb)
    const int nbw = 32 / lpb, qb = (lane >> 3) < nbw ? (lane >> 3) : 0, src8 = 8 * (lane / lpb);
    int64_t pcol = ((j - lane) * 4 + (int64_t)qb * lpb * 4) / S.bc;
    if (pcol >= S.nbc) pcol = S.nbc - 1;   // lanes past the right edge of a partial warp
    const float *scol_w = S.amax + pcol;
    uint32_t nxt[8][NW];
    int64_t g = blockIdx.y;
    if (g < G8 && act) {
#pragma unroll
        for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * g + i) * rstride, nxt[i]);
    }
    for (; g < G8; g += gridDim.y) {
        uint32_t w[8][NW];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < NW; ++q) w[i][q] = nxt[i][q];
        const int64_t gn = g + gridDim.y;
        if (gn < G8 && act) {
#pragma unroll
            for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * gn + i) * rstride, nxt[i]);
        }
        float rr[8];
        bool ok = true;
        if (WSHARE) {
            const FsE fe = fs_enc(__float_as_uint(__ldg(scol_w + fs_rb(S, 8 * g + (lane & 7)) * S.nbc)) & 0x7FFFFFFFu, G);
            ok = __all_sync(0xFFFFFFFFu, fe.mode == 1);
#pragma unroll
            for (int i = 0; i < 8; ++i) rr[i] = __shfl_sync(0xFFFFFFFFu, fe.rr, i + src8);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const FsE fe = fs_enc(__float_as_uint(__ldg(scol + fs_rb(S, 8 * g + i) * S.nbc)) & 0x7FFFFFFFu, G);
                ok = ok && fe.mode == 1;
                rr[i] = fe.rr;
            }
        }
        if (!act) continue;
        uint32_t vmax = 0, amax = 0;
        uint32_t cp[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t cd[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint32_t u = wordvec_elem<BF16, NW>(w[i], v);
                vmax = max(vmax, u & 0x7FFFFFFFu);
                cd[v] = enc_f32_fast<K, Y0>(__float_as_uint(__fmul_rn(__uint_as_float(u), rr[i])), P, amax);
            }
            cp[i][0] = cd[0] | (cd[1] << 16);
            cp[i][1] = cd[2] | (cd[3] << 16);
        }
        if (ok && vmax < 0x7F800000u) {
            uint32_t RL[1][8], RH[1][8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                RL[0][i] = prmt(cp[i][0], cp[i][1], 0x6420);
                RH[0][i] = (K == 9) ? prmt(cp[i][0] >> 1, cp[i][1] >> 1, 0x6420) : 0u;
            }
            rows_fast_store<K, 1, 0>(RL, RH, packed, so, g, C, c0);
        } else {
            for (int v = 0; v < 4; ++v)
                fs_enc_container<BF16, K>(in, C, g * C + c0 + v, 0, x, y, S, G, packed, so, spi, spb, spc, cap);
        }
    }
}

// ------------------------------------------------------- decode ROWS fast
// 8-row x 4-column tiles; codes -> e_max-127 fp32 values (one multiply for
// x <= 7) -> g s_hi + RN32(g s_lo) (FMUL + FFMA) -> RN16 for bf16 output.
// Row factors shared across the warp as in k_fs_enc_rows; a CTA barrier per
// row group, as k_dec_rows_fast.
template <int K, bool OBF16, bool FAST, bool WSHARE>
__global__ void __launch_bounds__(256) k_fs_dec_rows(const uint8_t *__restrict__ packed, int64_t R, int64_t C, int x,
                                                     int y, FsMap S, float G, SegOffsets so,
                                                     uint8_t *__restrict__ out, int lpb) {
    using EL = Elem<OBF16>;
    constexpr int TW = tile_words(K, 1);
    const Fmt F = fmt_of(x, y, 127);
    const FastP P = make_fast(F, false, 0);
    const int64_t CV = C / 4, G8 = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = j < CV;
    const int lane = threadIdx.x & 31;
    const int64_t c0 = (act ? j : 0) * 4;
    const float *scol = S.amax + c0 / S.bc;
    const int nbw = 32 / lpb, qb = (lane >> 3) < nbw ? (lane >> 3) : 0, src8 = 8 * (lane / lpb);
    int64_t pcol = ((j - lane) * 4 + (int64_t)qb * lpb * 4) / S.bc;
    if (pcol >= S.nbc) pcol = S.nbc - 1;   // lanes past the right edge of a partial warp
    const float *scol_w = S.amax + pcol;
    uint32_t nxt[TW];
    int64_t g = blockIdx.y;
    if (g < G8 && act) rows_load_raw<K, 1, 0>(nxt, packed, so, g, C, c0);
    for (; g < G8; g += gridDim.y) {
        uint32_t raw[TW];
#pragma unroll
        for (int q = 0; q < TW; ++q) raw[q] = nxt[q];
        __syncthreads();
        if (g + gridDim.y < G8 && act) rows_load_raw<K, 1, 0>(nxt, packed, so, g + gridDim.y, C, c0);
        float hi[8], lo[8];
        if (WSHARE) {
            const FsD fd = fs_dec(__float_as_uint(__ldg(scol_w + fs_rb(S, 8 * g + (lane & 7)) * S.nbc)) & 0x7FFFFFFFu, G);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                hi[i] = __shfl_sync(0xFFFFFFFFu, fd.hi, i + src8);
                lo[i] = __shfl_sync(0xFFFFFFFFu, fd.lo, i + src8);
            }
        } else if (act) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const FsD fd = fs_dec(__float_as_uint(__ldg(scol + fs_rb(S, 8 * g + i) * S.nbc)) & 0x7FFFFFFFu, G);
                hi[i] = fd.hi;
                lo[i] = fd.lo;
            }
        }
        if (!act) continue;
        uint32_t RL[1][8], RH[1][8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { RL[0][i] = 0; RH[0][i] = 0; }
        rows_unpack_raw<K, 1, 0>(raw, RL, RH);
        // (blocks whose results can fall below 2^-100, and x = 8, are redone
        // exactly afterwards by k_fs_dec_fixup)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t o[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                uint32_t code = (RL[0][i] >> (8 * v)) & 0xFFu;
                if (K == 9) code |= ((RH[0][i] >> (8 * v)) & 0xFFu) << 1;
                const uint32_t gb = FAST ? dec_f32_fast<K, false>(code, P, y) : dec_code_generic<24>(code, F);
                const float gf = __uint_as_float(gb & 0x7FFFFFFFu);
                const uint32_t r = __float_as_uint(__fmaf_rn(gf, hi[i], __fmul_rn(gf, lo[i])));
                o[v] = r | ((code << (32 - K)) & 0x80000000u);
            }
            uint8_t *dst = out + ((8 * g + i) * C + c0) * EL::ES;
            if (OBF16)
                stg_v2(dst, f32_to_bf16_bits(o[0]) | (f32_to_bf16_bits(o[1]) << 16),
                       f32_to_bf16_bits(o[2]) | (f32_to_bf16_bits(o[3]) << 16));
            else
                stg_v4(dst, make_uint4(o[0], o[1], o[2], o[3]));
        }
    }
}

// ------------------------------------------------ exact small results
// The fast float-scale kernels decode with FMUL + FFMA, exact for results
// >= 2^-100 (reading D23).  A block can produce smaller ones only when
// amax * g_min / G < 2^-99 (g_min = the smallest non-zero grid value), i.e.
// amax < tchk * G, and x = 8 codes lie below the fp32 range: those blocks are
// redone here with the integer evaluation of the definition.  One warp per
// block; a block that needs nothing costs one metadata load, so the pass is
// a few microseconds on ordinary tensors (and the fast kernels keep their
// round-1 register budgets).
__device__ __forceinline__ bool fs_block_needs_exact(const FsMap &S, float G, int64_t b) {
    if (S.x8) return true;
    const float a = __uint_as_float(__float_as_uint(__ldg(S.amax + b)) & 0x7FFFFFFFu);
    return a > 0.f && a < S.tchk * G * 1.0625f;   // conservative
}

template <bool BF16>
__global__ void __launch_bounds__(256) k_fs_quant_fixup(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                        int64_t R, int64_t C, int x, int y, FsMap S, float G) {
    const int lane = threadIdx.x & 31;
    const int64_t nb = (R / S.br) * S.nbc, warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += warps) {
        if (!fs_block_needs_exact(S, G, b)) continue;
        const uint32_t am = __float_as_uint(__ldg(S.amax + b)) & 0x7FFFFFFFu;
        const int64_t r0 = (b / S.nbc) * S.br, c0 = (b % S.nbc) * S.bc;
        for (int64_t k = lane; k < S.br * S.bc; k += 32) {
            const int64_t e = (r0 + k / S.bc) * C + c0 + k % S.bc;
            const uint32_t u = load_elem_scalar<BF16>(in, e);
            if (is_special_f32(u)) continue;   // passed through by the main kernel
            const uint32_t o = fs_quant_exact(u, am, G, x, y);
            if (BF16) {
                const uint16_t h = (uint16_t)f32_to_bf16_bits(o);
                memcpy(out + 2 * e, &h, 2);
            } else {
                memcpy(out + 4 * e, &o, 4);
            }
        }
    }
}

// decode: every container (8 codes) touching a block that needs the exact
// evaluation is decoded again by fs_dec_container (whose per-element check
// covers all of its blocks); a container shared by two such blocks is
// written twice with the same bytes
template <bool OBF16>
__global__ void __launch_bounds__(256) k_fs_dec_fixup(const uint8_t *__restrict__ packed, int64_t R, int64_t C,
                                                      int axis, int x, int y, FsMap S, float G, SegOffsets so,
                                                      int nseg, int4 widths, uint8_t *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nb = (R / S.br) * S.nbc, warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += warps) {
        if (!fs_block_needs_exact(S, G, b)) continue;
        const int64_t r0 = (b / S.nbc) * S.br, c0 = (b % S.nbc) * S.bc;
        if (axis == 0) {   // ROWS: container (g, c) holds rows 8g..8g+7 of column c
            const int64_t g0 = r0 / 8, g1 = (r0 + S.br + 7) / 8, nc = g1 - g0;
            for (int64_t k = lane; k < nc * S.bc; k += 32)
                fs_dec_container<OBF16>(packed, C, (g0 + k / S.bc) * C + c0 + k % S.bc, 0, x, y, S, G, so, nseg,
                                        widths, out);
        } else {           // COLS: container q holds elements 8q .. 8q+7 of one row
            const int64_t per_row = (c0 % 8 + S.bc + 7) / 8;
            for (int64_t k = lane; k < S.br * per_row; k += 32) {
                const int64_t r = r0 + k / per_row;
                fs_dec_container<OBF16>(packed, C, (r * C + c0) / 8 + k % per_row, 1, x, y, S, G, so, nseg, widths,
                                        out);
            }
        }
    }
}

}  // namespace exmy
