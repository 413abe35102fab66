// exmy_fast.cuh -- the fast (vectorised, SWAR) encode / decode / quantize
// kernels.  Same results as the integer generic path (exmy_device.cuh) bit
// for bit; every kernel checks the fast-path preconditions on the device
// (warp-uniform, from the metadata byte) and falls back per tile.
//
// Encode: one addition does the rounding.  For |v| in binade Ecl (clamped
// to [o+1, e_max+1]) the grid quantum is q = 2^(Ecl-127-y) (subnormal
// region: Ecl = o+1).  With C = 2^7 q as a bf16 (or 2^23 q as an fp32),
// ulp(C) = q and |v| < 2^(y+1) q <= C, so RN(|v| + C) = C + RTNE_q(|v|)
// exactly (ties to an even significand = even code, y >= 1), and the
// count of quanta is bits(RN(|v|+C)) - bits(C).  The code is that count
// plus (Ecl-o-1) << y (the implicit bit is in the count).  A carry out of
// the binade lands on the next exponent code; saturation is one min.
// For y = 0 (reading D6) a tie goes to the even fp32 exponent (the paper's
// Eigen RTNE extended to zero mantissa bits): without help the addition
// sends every y = 0 tie up (count 2 is the even significand), so C is moved
// by one quantum where the binade's exponent is even; taking that parity
// from (clamped | unclamped) exponent keeps the flush tie (half the smallest
// non-zero value, one binade below the clamp) at zero (D8).  bf16 inputs run
// two elements per 32-bit register (16-bit SIMD lanes, HADD2.BF16) for
// y <= 6.
//
// Decode: the magnitude code shifted into a bf16/fp32 bit pattern is the
// value scaled by 2^-o (code exponent 0 lands on subnormals); one
// multiply by 2^o (RN, subnormals kept) gives RTNE(exact value) (D21).
//
// Packing: codes are moved into byte-lane registers (4 containers x one
// element each) and the power-of-2 segments are built with shift/LOP3
// masks and PRMT byte transposes (SWAR) -- about 2 ops per element for
// k = 7 instead of 3 ops per element per segment.
#pragma once
#include "exmy_kernels.cuh"

namespace exmy {

// ---------------------------------------------------------- SIMD helpers
__device__ __forceinline__ uint32_t vmax_u16x2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t vmin_u16x2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t hadd2_bf16(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t hsub2_bf16(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t hmul2_bf16(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) { return __byte_perm(a, b, s); }

template <int S>
__device__ __forceinline__ uint32_t shl_s(uint32_t v) {   // shift left by S (right if S < 0)
    if constexpr (S >= 0) return v << S;
    else return v >> (-S);
}

// ------------------------------------------------------- fast parameters
struct FastP {
    // encode / quantize
    bool enc_simd;      // bf16 16-bit-lane path usable (bf16 input, y <= 6)
    bool enc_f32;       // per-element fp32 path usable
    bool y0;            // parity fix needed
    uint32_t lo2, hi2;  // clamp bounds on the exponent field (bf16 lanes)
    uint32_t k2, k3;    // (7-y)<<7, (o+1)<<y per lane (bf16 lanes)
    uint32_t m2;        // M per lane
    uint32_t lo, hi, k2f, k3f;   // fp32 variants
    int sh_b, sh_f;     // 7-y, 23-y
    // decode
    bool dec_fast;      // fp32 out: x <= 7
    bool dec_fast_bf;   // bf16 out: x <= 7, y <= 7
    bool two_mul;       // o > 127
    uint32_t s1_bf2, s2_bf2;   // 2^min(o,127), 2^(o-127) as bf16 pairs
    float s1_f, s2_f;
    uint32_t big2;      // bf16 lanes: 0x8000 - (248+y)<<7, tile fallback threshold bias
    uint32_t bigf;      // fp32: (232+y)<<23
    uint32_t maxv2;     // largest grid magnitude as bf16 lanes (quantize)
    uint32_t maxvf;     // ... as fp32 bits
};

__device__ __forceinline__ uint32_t bf16_pow2(int e) {   // e in [-133, 127]
    return e >= -126 ? (uint32_t)(e + 127) << 7 : (1u << (e + 133));
}

__device__ __forceinline__ FastP make_fast(const Fmt &F, bool bf16_in, int force_generic) {
    FastP P;
    const int x = F.x, y = F.y, o = F.o, e = F.e_max;
    const bool base = !force_generic && o >= 0;
    P.enc_simd = base && bf16_in && y <= 6 && e <= 246 + y;
    P.enc_f32 = base && y <= 22 && e <= 230 + y;
    P.y0 = (y == 0);
    P.lo2 = ((uint32_t)(o + 1) << 7) * 0x00010001u;
    P.hi2 = ((uint32_t)(e + 1) << 7) * 0x00010001u;
    P.k2 = ((uint32_t)(7 - (y > 7 ? 7 : y)) << 7) * 0x00010001u;
    P.k3 = ((uint32_t)(o + 1) << y) * 0x00010001u;
    P.m2 = F.M * 0x00010001u;
    P.lo = (uint32_t)(o + 1) << 23;
    P.hi = (uint32_t)(e + 1) << 23;
    P.k2f = (uint32_t)(23 - y) << 23;
    P.k3f = (uint32_t)(o + 1) << y;
    P.sh_b = 7 - (y > 7 ? 7 : y);
    // Without an upper clamp on the exponent, C = 2^(E-127+7-y) overflows only
    // for E > 247+y (bf16) / 231+y (fp32); tiles holding such magnitudes (or
    // NaN/Inf) take the generic path.  Below that, magnitudes above the grid
    // saturate through min(code, M).
    P.big2 = (0x8000u - ((uint32_t)(248 + (y > 7 ? 7 : y)) << 7)) * 0x00010001u;
    P.bigf = (uint32_t)(232 + y) << 23;
    P.sh_f = 23 - y;
    P.dec_fast = !force_generic && x <= 7;
    P.dec_fast_bf = P.dec_fast && y <= 7;
    P.two_mul = o > 127;
    const int e1 = o > 127 ? 127 : o, e2 = o > 127 ? o - 127 : 0;
    P.s1_bf2 = (e1 >= -133 ? bf16_pow2(e1) : 0u) * 0x00010001u;
    P.s2_bf2 = bf16_pow2(e2) * 0x00010001u;
    P.s1_f = pow2f_exact(e1 < -149 ? -149 : e1);
    P.s2_f = pow2f_exact(e2);
    // largest grid magnitude as bf16 / fp32 bits (quantize saturation); only
    // used when the fast encode preconditions hold (o >= 0, y <= 22)
    uint32_t mv, mvf;
    const uint32_t yb = (uint32_t)(y > 7 ? 7 : y);
    if (x == 0) {   // (2^y - 1) 2^(e_max-126-y) = (2 - 2^(1-y)) 2^(e_max-128) ... normalised below
        if (e >= 1) {
            mv = ((uint32_t)e << 7) | ((((1u << yb) - 1u) << (8 - yb)) & 0x7Fu);
            mvf = ((uint32_t)e << 23) | ((((1u << y) - 1u) << (24 - y)) & 0x7FFFFFu);
        } else {    // e_max = 0: a subnormal in both containers
            mv = (1u << 7) - (1u << (7 - yb));
            mvf = (1u << 23) - (1u << (23 - y));
        }
    } else {
        mv = ((uint32_t)e << 7) | ((((1u << yb) - 1u) << (7 - yb)) & 0x7Fu);
        mvf = ((uint32_t)e << 23) | ((((1u << y) - 1u) << (23 - y)) & 0x7FFFFFu);
    }
    P.maxvf = mvf;
    P.maxv2 = mv * 0x00010001u;
    return P;
}

// ------------------------------------------------------- code computation
// Encode modes (chosen on the host from (dtype, y); e_max is checked on the
// device): bf16 SIMD pairs for y in 1..6 / y = 0, per-element fp32 FADD for
// fp32 inputs and bf16 with y >= 7.
enum EncMode { ENC_SIMD = 0, ENC_SIMD_Y0 = 1, ENC_F32 = 2, ENC_F32_Y0 = 3 };

// two bf16 elements (one 32-bit word) -> two k-bit codes in 16-bit lanes;
// amax accumulates the largest magnitude seen (NaN/Inf test at the end)
template <int K, bool Y0, bool SIGN = true>
__device__ __forceinline__ uint32_t enc_pair_bf16(uint32_t w, const FastP &P, uint32_t &amax) {
    const uint32_t a2 = w & 0x7FFF7FFFu;
    const uint32_t ev = w & 0x7F807F80u;
    uint32_t ecl = vmax_u16x2(ev, P.lo2);   // subnormal region -> binade o+1
    uint32_t c, t;
    if (Y0) {   // y = 0: shift is 7; move C by one quantum where the binade's exponent is even (D6)
        t = ecl >> 7;
        c = ecl + P.k2 + ((~(t | (ev >> 7))) & 0x00010001u);
    } else {
        t = ecl >> P.sh_b;
        c = ecl + P.k2;
    }
    const uint32_t s = hadd2_bf16(a2, c);
    uint32_t code = s - c + t - P.k3;
    code = vmin_u16x2(code, P.m2);
    if (SIGN) code |= (w >> (16 - K)) & ((1u << (K - 1)) * 0x00010001u);
    amax = vmax_u16x2(amax, a2);
    return code;
}
// The signs of the 4 bf16 elements in words w0, w1 as bytes 0x00 / 0xFF
// (prmt's sign-replicating selectors 8 + b on the high bytes 1, 3, 5, 7), in
// the byte order of prmt(cp0, cp1, 0x6420): the codes of a row's 4 elements
// get their sign bits with ONE LOP3 per row instead of a shift and a LOP3
// per pair -- the ROWS encode is bound by the ALU pipe.
__device__ __forceinline__ uint32_t sign_bytes(uint32_t w0, uint32_t w1) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, 0xFDB9;" : "=r"(d) : "r"(w0), "r"(w1));
    return d;
}
// the same for 4 fp32 elements (sign in byte 3 of each word): 3 PRMTs
__device__ __forceinline__ uint32_t sign_bytes_f32(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
    uint32_t a, b;
    asm("prmt.b32 %0, %1, %2, 0x00FB;" : "=r"(a) : "r"(w0), "r"(w1));
    asm("prmt.b32 %0, %1, %2, 0x00FB;" : "=r"(b) : "r"(w2), "r"(w3));
    return prmt(a, b, 0x5410);
}
// any lane at or above the fallback threshold (NaN/Inf, or huge values)
__device__ __forceinline__ bool amax_special_bf16(uint32_t amax, const FastP &P) {
    return ((amax + P.big2) & 0x80008000u) != 0u;
}

// one fp32 pattern -> k-bit code
template <int K, bool Y0, bool SIGN = true>
__device__ __forceinline__ uint32_t enc_f32_fast(uint32_t u, const FastP &P, uint32_t &amax) {
    const uint32_t a = u & 0x7FFFFFFFu;
    const uint32_t ev = u & 0x7F800000u;
    const uint32_t ecl = max(ev, P.lo);
    uint32_t c = ecl + P.k2f;
    if (Y0) c += (~((ecl | ev) >> 23)) & 1u;   // D6: y = 0 ties to the even fp32 exponent
    const uint32_t s = __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(c)));
    uint32_t code = s - c + (ecl >> P.sh_f) - P.k3f;
    code = min(code, (1u << (K - 1)) - 1u);
    if (SIGN) code |= (u >> (32 - K)) & (1u << (K - 1));
    amax = max(amax, a);
    return code;
}

// quantize two bf16 elements directly in bf16 arithmetic (value, not code)
__device__ __forceinline__ uint32_t quant_pair_bf16(uint32_t w, const FastP &P, uint32_t &flag) {
    const uint32_t a2 = w & 0x7FFF7FFFu;
    const uint32_t ev = w & 0x7F807F80u;
    const uint32_t ecl = vmax_u16x2(ev, P.lo2);
    uint32_t c = ecl + P.k2;
    if (P.y0) c += (~((ecl | ev) >> 7)) & 0x00010001u;
    const uint32_t s = hadd2_bf16(a2, c);
    uint32_t q = hsub2_bf16(s, c);            // exact (Sterbenz): RTNE_q(|v|)
    q = vmin_u16x2(q, P.maxv2);
    flag |= a2 + P.big2;                      // NaN/Inf or C-overflow range -> generic
    return q | (w & 0x80008000u);
}

// ------------------------------------------------------ decode helpers
// code pair (16-bit lanes) -> bf16 pair
// TWO: o > 127, the scale 2^o is applied as an exact 2^127 then 2^(o-127)
template <int K, bool TWO = false>
__device__ __forceinline__ uint32_t dec_pair_bf16(uint32_t cp, const FastP &P, int y) {
    uint32_t mag = cp & (((1u << (K - 1)) - 1u) * 0x00010001u);
    uint32_t b = mag << (7 - y);
    uint32_t v = hmul2_bf16(b, P.s1_bf2);
    if (TWO) v = hmul2_bf16(v, P.s2_bf2);
    return v | ((cp << (16 - K)) & 0x80008000u);
}

template <int K, bool TWO = false>
__device__ __forceinline__ uint32_t dec_f32_fast(uint32_t code, const FastP &P, int y) {
    uint32_t mag = code & ((1u << (K - 1)) - 1u);
    float f = __uint_as_float(mag << (23 - y));
    f = __fmul_rn(f, P.s1_f);
    if (TWO) f = __fmul_rn(f, P.s2_f);
    return __float_as_uint(f) | ((code << (32 - K)) & 0x80000000u);
}

// ------------------------------------------------------------ SWAR pack
// R[8]: byte-lane registers; byte l of R[i] = bits of element i of container
// l (4 containers).  Produces the 4 containers of segment (W, LO) as W words.
template <int W, int LO>
__device__ __forceinline__ void swar_pack4(const uint32_t (&R)[8], uint32_t (&out)[W]) {
    if constexpr (W == 1) {
        uint32_t b = 0;
        b |= shl_s<0 - LO>(R[0]) & (0x01010101u << 0);
        b |= shl_s<1 - LO>(R[1]) & (0x01010101u << 1);
        b |= shl_s<2 - LO>(R[2]) & (0x01010101u << 2);
        b |= shl_s<3 - LO>(R[3]) & (0x01010101u << 3);
        b |= shl_s<4 - LO>(R[4]) & (0x01010101u << 4);
        b |= shl_s<5 - LO>(R[5]) & (0x01010101u << 5);
        b |= shl_s<6 - LO>(R[6]) & (0x01010101u << 6);
        b |= shl_s<7 - LO>(R[7]) & (0x01010101u << 7);
        out[0] = b;
    } else if constexpr (W == 2) {
        uint32_t lo = 0, hi = 0;
        lo |= shl_s<0 - LO>(R[0]) & (0x03030303u << 0);
        lo |= shl_s<2 - LO>(R[1]) & (0x03030303u << 2);
        lo |= shl_s<4 - LO>(R[2]) & (0x03030303u << 4);
        lo |= shl_s<6 - LO>(R[3]) & (0x03030303u << 6);
        hi |= shl_s<0 - LO>(R[4]) & (0x03030303u << 0);
        hi |= shl_s<2 - LO>(R[5]) & (0x03030303u << 2);
        hi |= shl_s<4 - LO>(R[6]) & (0x03030303u << 4);
        hi |= shl_s<6 - LO>(R[7]) & (0x03030303u << 6);
        out[0] = prmt(lo, hi, 0x5140);
        out[1] = prmt(lo, hi, 0x7362);
    } else {
        static_assert(W == 4, "");
        uint32_t N[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            N[j] = (shl_s<-LO>(R[2 * j]) & 0x0F0F0F0Fu) | (shl_s<4 - LO>(R[2 * j + 1]) & 0xF0F0F0F0u);
        const uint32_t t0 = prmt(N[0], N[1], 0x5140), t1 = prmt(N[2], N[3], 0x5140);
        const uint32_t t2 = prmt(N[0], N[1], 0x7362), t3 = prmt(N[2], N[3], 0x7362);
        out[0] = prmt(t0, t1, 0x5410);
        out[1] = prmt(t0, t1, 0x7632);
        out[2] = prmt(t2, t3, 0x5410);
        out[3] = prmt(t2, t3, 0x7632);
    }
}

// inverse: OR the segment's bits back into byte-lane registers R[8]
template <int W, int LO>
__device__ __forceinline__ void swar_unpack4(const uint32_t (&in)[W], uint32_t (&R)[8]) {
    if constexpr (W == 1) {
        const uint32_t b = in[0];
        R[0] |= shl_s<LO - 0>(b & (0x01010101u << 0));
        R[1] |= shl_s<LO - 1>(b & (0x01010101u << 1));
        R[2] |= shl_s<LO - 2>(b & (0x01010101u << 2));
        R[3] |= shl_s<LO - 3>(b & (0x01010101u << 3));
        R[4] |= shl_s<LO - 4>(b & (0x01010101u << 4));
        R[5] |= shl_s<LO - 5>(b & (0x01010101u << 5));
        R[6] |= shl_s<LO - 6>(b & (0x01010101u << 6));
        R[7] |= shl_s<LO - 7>(b & (0x01010101u << 7));
    } else if constexpr (W == 2) {
        const uint32_t lo = prmt(in[0], in[1], 0x6420), hi = prmt(in[0], in[1], 0x7531);
        R[0] |= shl_s<LO - 0>(lo & (0x03030303u << 0));
        R[1] |= shl_s<LO - 2>(lo & (0x03030303u << 2));
        R[2] |= shl_s<LO - 4>(lo & (0x03030303u << 4));
        R[3] |= shl_s<LO - 6>(lo & (0x03030303u << 6));
        R[4] |= shl_s<LO - 0>(hi & (0x03030303u << 0));
        R[5] |= shl_s<LO - 2>(hi & (0x03030303u << 2));
        R[6] |= shl_s<LO - 4>(hi & (0x03030303u << 4));
        R[7] |= shl_s<LO - 6>(hi & (0x03030303u << 6));
    } else {
        static_assert(W == 4, "");
        const uint32_t t0 = prmt(in[0], in[1], 0x5140), t1 = prmt(in[2], in[3], 0x5140);
        const uint32_t t2 = prmt(in[0], in[1], 0x7362), t3 = prmt(in[2], in[3], 0x7362);
        const uint32_t N[4] = {prmt(t0, t1, 0x5410), prmt(t0, t1, 0x7632), prmt(t2, t3, 0x5410),
                               prmt(t2, t3, 0x7632)};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            R[2 * j] |= shl_s<LO>(N[j] & 0x0F0F0F0Fu);
            R[2 * j + 1] |= shl_s<LO - 4>(N[j] & 0xF0F0F0F0u);
        }
    }
}

}  // namespace exmy

namespace exmy {

__device__ __forceinline__ uint32_t quant_f32_fast(uint32_t u, const FastP &P, uint32_t &flag) {
    const uint32_t a = u & 0x7FFFFFFFu;
    const uint32_t ev = u & 0x7F800000u;
    const uint32_t ecl = max(ev, P.lo);
    uint32_t c = ecl + P.k2f;
    if (P.y0) c += (~((ecl | ev) >> 23)) & 1u;
    const float s = __fadd_rn(__uint_as_float(a), __uint_as_float(c));
    uint32_t q = __float_as_uint(__fsub_rn(s, __uint_as_float(c)));   // exact
    q = min(q, P.maxvf);
    flag |= (a >= P.bigf) ? 0x80000000u : 0u;
    return q | (u & 0x80000000u);
}

__device__ __forceinline__ uint32_t word_of(const uint4 &r, int t) {
    return t == 0 ? r.x : t == 1 ? r.y : t == 2 ? r.z : r.w;
}

// codes of NW input words (bf16: 2 elements per word, fp32: 1) as 16-bit-lane
// pairs cp[t] = codes (2t, 2t+1).  The fast paths accumulate a NaN/Inf flag;
// the generic path records specials itself (idx0 = index of element 0).
template <bool BF16, int NW>
__device__ __forceinline__ uint32_t wordvec_elem(const uint32_t (&w)[NW], int v) {
    if (BF16) return (v & 1) ? (w[v >> 1] & 0xFFFF0000u) : (w[v >> 1] << 16);
    return w[v];
}

template <int K, bool BF16, int MODE, int NW, bool SIGN = true>
__device__ __forceinline__ void vec_codes(const uint32_t (&w)[NW], uint32_t (&cp)[BF16 ? NW : NW / 2],
                                          const FastP &P, uint32_t &amax) {
    constexpr int NP = BF16 ? NW : NW / 2;
    if constexpr (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0) {
        static_assert(BF16, "SIMD encode needs bf16 input");
#pragma unroll
        for (int t = 0; t < NP; ++t) cp[t] = enc_pair_bf16<K, MODE == ENC_SIMD_Y0, SIGN>(w[t], P, amax);
    } else {
#pragma unroll
        for (int t = 0; t < NP; ++t) {
            uint32_t lo = enc_f32_fast<K, MODE == ENC_F32_Y0, SIGN>(wordvec_elem<BF16, NW>(w, 2 * t), P, amax);
            uint32_t hi = enc_f32_fast<K, MODE == ENC_F32_Y0, SIGN>(wordvec_elem<BF16, NW>(w, 2 * t + 1), P, amax);
            cp[t] = lo | (hi << 16);
        }
    }
}

template <bool BF16, int MODE>
__device__ __forceinline__ bool amax_special(uint32_t amax, const FastP &P) {
    if constexpr (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0) return amax_special_bf16(amax, P);
    else return amax >= P.bigf;
}

// A tile whose fast-path flag fired because of NaN/Inf only (no finite
// magnitude in the C-overflow range): its codes are the fast ones with the
// special lanes set to 0 (D9's in-band placeholder), so NaN-heavy tensors
// keep the vector path; returns the number of specials (the ordered list is
// written afterwards by the compaction kernels), or -1 if the tile needs the
// integer path.  cp as from vec_codes (16-bit lanes: codes 2t, 2t+1).
template <int K, bool BF16, int MODE, int NW>
__device__ __forceinline__ int mask_special_codes(const uint32_t (&w)[NW], uint32_t (&cp)[BF16 ? NW : NW / 2],
                                                  const FastP &P) {
    constexpr int NP = BF16 ? NW : NW / 2;
    int n = 0;
    bool bad = false;
#pragma unroll
    for (int t = 0; t < NP; ++t) {
        uint32_t sp;   // bit 15 / 31: element 2t / 2t+1 is NaN/Inf
        if (BF16) {
            const uint32_t a2 = w[t] & 0x7FFF7FFFu;
            sp = (a2 + 0x00800080u) & 0x80008000u;
            if constexpr (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0) {
                bad = bad || (((a2 + P.big2) & 0x80008000u) & ~sp) != 0u;
                // a NaN/Inf lane's arithmetic can borrow across the 16-bit lane
                // boundary: recompute the pair with that lane zeroed
                if (sp) {
                    const uint32_t keep = ~((sp >> 15) * 0xFFFFu);
                    uint32_t am = 0;
                    cp[t] = enc_pair_bf16<K, MODE == ENC_SIMD_Y0>(w[t] & keep, P, am);
                }
            } else   // y >= 7: per-element fp32 path on the widened elements
                bad = bad || (!(sp & 0x8000u) && (a2 << 16) >= P.bigf) ||
                      (!(sp & 0x80000000u) && (a2 & 0xFFFF0000u) >= P.bigf);
        } else {
            const uint32_t a0 = w[2 * t] & 0x7FFFFFFFu, a1 = w[2 * t + 1] & 0x7FFFFFFFu;
            const bool s0 = a0 >= 0x7F800000u, s1 = a1 >= 0x7F800000u;
            sp = (s0 ? 0x8000u : 0u) | (s1 ? 0x80000000u : 0u);
            bad = bad || (!s0 && a0 >= P.bigf) || (!s1 && a1 >= P.bigf);
        }
        cp[t] &= ~((sp >> 15) * 0xFFFFu);
        n += __popc(sp);
    }
    return bad ? -1 : n;
}

// a warp that deferred a tile raises the fix-up flag once (kernel end)
__device__ __forceinline__ void raise_fixup_flag(unsigned long long *flag, bool deferred) {
    const unsigned m = __activemask();
    const unsigned b = __ballot_sync(m, deferred);
    if (b && (threadIdx.x & 31) == __ffs(m) - 1) atomicOr(flag, 1ull);
}

// add a thread's count of specials to *spc once per warp (kernel end)
__device__ __forceinline__ void flush_special_count(unsigned long long *spc, unsigned long long nsp) {
    const unsigned m = __activemask();
    const unsigned long long t = __reduce_add_sync(m, (unsigned)nsp);
    if (spc && t && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(spc, t);
}

template <bool BF16, int MODE>
__device__ __forceinline__ bool enc_fast_ok(const Fmt &F, int force_generic) {
    if (force_generic || F.o < 0) return false;
    return (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0) ? (F.e_max <= 246 + F.y) : (F.e_max <= 230 + F.y);
}

// 4 consecutive elements of a row: bf16 -> 2 words (8 B), fp32 -> 4 words (16 B)
template <bool BF16>
__device__ __forceinline__ void load4(const uint8_t *p, uint32_t (&w)[BF16 ? 2 : 4]) {
    if constexpr (BF16) {
        uint2 t;
#if defined(EXMY_LD_HINT) && EXMY_LD_HINT == 1   // A/B builds only: 256-byte L2 prefetch
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.u32 {%0,%1}, [%2];" : "=r"(t.x), "=r"(t.y) : "l"(p));
#elif defined(EXMY_LD_HINT) && EXMY_LD_HINT == 2   // A/B builds only: L2 evict_first policy
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                     : "=r"(t.x), "=r"(t.y) : "l"(p), "l"(pol));
#else
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(t.x), "=r"(t.y) : "l"(p));
#endif
        w[0] = t.x; w[1] = t.y;
    } else {
        uint4 t = ldg_nc_v4(p);
        w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
    }
}

// One container (8 elements) on the integer generic path, stored with plain
// byte stores; kept out of line so the fast paths' register allocation does
// not pay for it (it runs only for tiles holding NaN/Inf, or for metadata
// outside the fast preconditions).
template <bool BF16, int K>
__device__ __noinline__ void enc_container_generic(const uint8_t *__restrict__ in, int64_t C, int64_t idx, int axis,
                                                   const Fmt F, uint8_t *packed, const SegOffsets so, int64_t *spi,
                                                   uint32_t *spb, unsigned long long *spc, int64_t cap) {
    uint32_t c[8];
    int64_t e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        e[i] = lane_elem(idx, i, C, axis);
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

// ---------------------------------------------------------- encode ROWS
template <int K, int NH, int S>
__device__ __forceinline__ void rows_fast_store(const uint32_t (&RL)[NH][8], const uint32_t (&RH)[NH][8],
                                                uint8_t *packed, const SegOffsets &so, int64_t g, int64_t C,
                                                int64_t c0) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S);
        uint8_t *seg = packed + so.off[S];
        if constexpr (W == 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                uint32_t w[NH];
#pragma unroll
                for (int h = 0; h < NH; ++h) w[h] = (K == 9) ? RH[h][i] : RL[h][i];
                store_words<NH>(seg + (8 * g + i) * C + c0, w);
            }
        } else {
            uint32_t w[NH * W];
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                uint32_t out[W];
                swar_pack4<W, LO>(RL[h], out);
#pragma unroll
                for (int q = 0; q < W; ++q) w[h * W + q] = out[q];
            }
            store_words<NH * W>(seg + (g * C + c0) * W, w);
        }
        rows_fast_store<K, NH, S + 1>(RL, RH, packed, so, g, C, c0);
    }
}

// Thread tile: 8 rows (one row group g) x 4 adjacent columns.  Every store
// of a segment is then one instruction per thread covering whole sectors
// across the warp (4 containers x w bytes: 16/8/4 B); a 32-byte per-thread
// store split in two instructions made L2 write partial sectors back twice.
// A CTA barrier per row group for bf16 input with k >= 8 (its byte-wide
// segment is stored row-major, 4 bytes per thread per row): measured on
// config 2, e4m3 178 -> 145 us, e3m5 196 -> 160 us; for k <= 7 and fp32 input
// the barrier costs 5-10 %, so those run without it.
template <int K, bool BF16>
__host__ __device__ constexpr bool enc_rows_bar() { return BF16 && K >= 8; }

template <int K, bool BF16, int MODE>
#ifndef EXMY_ENC_ROWS_MINB   // A/B builds only: bf16 ROWS encode CTAs per SM, CTA size
#define EXMY_ENC_ROWS_MINB 3
#endif
#ifndef EXMY_ENC_ROWS_THREADS
#define EXMY_ENC_ROWS_THREADS 256
#endif
__global__ void __launch_bounds__(BF16 ? EXMY_ENC_ROWS_THREADS : 256, BF16 ? EXMY_ENC_ROWS_MINB : 2) k_enc_rows_fast(const uint8_t *__restrict__ in, int64_t R, int64_t C, int x,
                                                       int y, const uint8_t *__restrict__ meta,
                                                       uint8_t *__restrict__ packed, SegOffsets so, int64_t *spi,
                                                       uint32_t *spb, unsigned long long *spc, int64_t cap,
                                                       int force_generic, unsigned long long *defer_flag) {
    const bool defer = defer_flag != nullptr;
    using EL = Elem<BF16>;
    constexpr int NW = BF16 ? 2 : 4;   // words per 4 elements
    const Fmt F = load_fmt(x, y, meta);
    const FastP P = make_fast(F, BF16, force_generic);
    const int64_t CV = C / 4, G = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    constexpr bool BAR = enc_rows_bar<K, BF16>();
    if (!BAR && j >= CV) return;
    const bool act = j < CV;   // with barriers, idle threads stay for them
    const int64_t c0 = j * 4;
    const uint8_t *src = in + c0 * EL::ES;
    const int64_t rstride = C * EL::ES;
    const uint32_t rs32 = (uint32_t)rstride;
    if (!enc_fast_ok<BF16, MODE>(F, force_generic)) {   // metadata outside the fast preconditions
        if (!act) return;
        for (int64_t g = blockIdx.y; g < G; g += gridDim.y)
            for (int v = 0; v < 4; ++v)
                enc_container_generic<BF16, K>(in, C, g * C + c0 + v, 0, F, packed, so, spi, spb, spc, cap);
        return;
    }
    // software pipeline: the next tile's 8 row chunks are in flight while
    // this tile is converted and packed
    bool deferred = false;   // a tile with NaN/Inf (or huge values) left to k_enc_rows_fixup
    uint32_t nxt[8][NW];
    int64_t g = blockIdx.y;
    if (g < G && act) {
#pragma unroll
        for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * g + i) * rstride, nxt[i]);
    }
    for (; g < G; g += gridDim.y) {
        uint32_t w[8][NW];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < NW; ++q) w[i][q] = nxt[i][q];
        if constexpr (BAR) __syncthreads();
        const int64_t gn = g + gridDim.y;
        if (gn < G && act) {
            if constexpr (BF16) {
                // one 64-bit base and 32-bit row offsets (the launcher guarantees
                // 8 * rstride < 2^32): no local-memory reloads at the 80-register
                // cap, e3m3 139.0 -> 137.9 us, e6m0 160.7 -> 150.3 us (fp32 input
                // does not spill and measured 1 % slower this way)
                const uint8_t *pb = src + 8 * gn * rstride;
#pragma unroll
                for (int i = 0; i < 8; ++i) load4<BF16>(pb + (uint32_t)i * rs32, nxt[i]);
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * gn + i) * rstride, nxt[i]);
            }
        }
        if (!act) continue;
        uint32_t cp[8][2];
        uint32_t amax = 0;
        // bf16 lanes, k <= 8: codes without sign, the signs added per row below
        // (fp32 input: the same with 3 PRMTs per row for the 4 elements' signs)
        constexpr bool LATE_SIGN = BF16 ? (K <= 8 && (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0)) : K <= 7;
#pragma unroll
        for (int i = 0; i < 8; ++i) vec_codes<K, BF16, MODE, NW, !LATE_SIGN>(w[i], cp[i], P, amax);
        if (!amax_special<BF16, MODE>(amax, P)) {
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
        } else if (defer) {   // NaN/Inf (or huge values): k_enc_rows_fixup encodes this tile
            deferred = true;
        } else {   // no workspace: the integer path here (round-1 behaviour)
            for (int v = 0; v < 4; ++v)
                enc_container_generic<BF16, K>(in, C, g * C + c0 + v, 0, F, packed, so, spi, spb, spc, cap);
        }
    }
    if (defer) raise_fixup_flag(defer_flag, deferred);
}

// ---------------------------------------------------------- encode COLS
template <int K, int S>
__device__ __forceinline__ void cols_fast_store(const uint32_t (&RL)[8], const uint32_t (&RH)[8],
                                                const uint32_t (&cp)[4][4], uint8_t *packed, const SegOffsets &so,
                                                int64_t q0, int64_t NG) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S);
        uint8_t *seg = packed + so.off[S];
        if constexpr (W == 8) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t q = q0 + 32 * u;
                if (q < NG) {
                    constexpr int SH = (K == 9) ? 1 : 0;
                    const uint32_t w0 = prmt(cp[u][0] >> SH, cp[u][1] >> SH, 0x6420);
                    const uint32_t w1 = prmt(cp[u][2] >> SH, cp[u][3] >> SH, 0x6420);
                    stg_v2(seg + 8 * q, w0, w1);
                }
            }
        } else {
            uint32_t out[W];
            swar_pack4<W, LO>(RL, out);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t q = q0 + 32 * u;
                if (q < NG) {
                    if constexpr (W == 4) *(uint32_t *)(seg + 4 * q) = out[u];
                    else if constexpr (W == 2) *(uint16_t *)(seg + 2 * q) = (uint16_t)(out[u >> 1] >> (16 * (u & 1)));
                    else seg[q] = (uint8_t)(out[0] >> (8 * u));
                }
            }
        }
        cols_fast_store<K, S + 1>(RL, RH, cp, packed, so, q0, NG);
    }
}

template <int K, bool BF16, int MODE>
__global__ void __launch_bounds__(256) k_enc_cols_fast(const uint8_t *__restrict__ in, int64_t n, int x, int y,
                                                       const uint8_t *__restrict__ meta, uint8_t *__restrict__ packed,
                                                       SegOffsets so, int64_t *spi, uint32_t *spb,
                                                       unsigned long long *spc, int64_t cap, int force_generic,
                                                       unsigned long long *defer_flag) {
    const bool defer = defer_flag != nullptr;
    using EL = Elem<BF16>;
    constexpr int NV = BF16 ? 1 : 2;   // 16-byte vectors per group of 8
    constexpr int NP = EL::V / 2;      // pairs per vector
    const Fmt F = load_fmt(x, y, meta);
    const FastP P = make_fast(F, BF16, force_generic);
    const int64_t NG = n / 8;
    const int lane = threadIdx.x & 31;
    const int64_t step = (int64_t)gridDim.x * (blockDim.x >> 5) * 128;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (!enc_fast_ok<BF16, MODE>(F, force_generic)) {
        for (int64_t base = gw * 128; base < NG; base += step)
            for (int u = 0; u < 4; ++u) {
                const int64_t q = base + 32 * u + lane;
                if (q < NG) enc_container_generic<BF16, K>(in, 0, q, 1, F, packed, so, spi, spb, spc, cap);
            }
        return;
    }
    bool deferred = false;   // a warp tile with NaN/Inf (or huge values) left to k_enc_cols_fixup
    uint4 nxt[4][NV];
    int64_t base = gw * 128;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t q = base + 32 * u + lane;
#pragma unroll
        for (int t = 0; t < NV; ++t)
            nxt[u][t] = q < NG ? ldg_nc_v4(in + q * 8 * EL::ES + 16 * t) : make_uint4(0, 0, 0, 0);
    }
    for (; base < NG; base += step) {
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
        uint32_t cp[4][4];   // group u, pair t (elements 2t, 2t+1)
        uint32_t amax = 0;
        // bf16 lanes, k <= 8: signs merged per byte-lane word below (as ROWS)
        constexpr bool LATE_SIGN = BF16 && K <= 7 && (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0);   // k = 8: the 8-bit segment stores from cp
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int t = 0; t < NV; ++t) {
                uint32_t c2[NP];
                const uint32_t ww[4] = {r[u][t].x, r[u][t].y, r[u][t].z, r[u][t].w};
                vec_codes<K, BF16, MODE, 4, !LATE_SIGN>(ww, c2, P, amax);
#pragma unroll
                for (int p = 0; p < NP; ++p) cp[u][t * NP + p] = c2[p];
            }
        }
        if (!amax_special<BF16, MODE>(amax, P)) {
            uint32_t RL[8], RH[8];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint32_t y01 = prmt(cp[0][t], cp[1][t], 0x6420), y23 = prmt(cp[2][t], cp[3][t], 0x6420);
                RL[2 * t] = prmt(y01, y23, 0x6420);
                RL[2 * t + 1] = prmt(y01, y23, 0x7531);
                if constexpr (LATE_SIGN) {
                    // sign bytes of elements 2t / 2t+1 of groups 0..3 (word t of each
                    // group: bytes 1 and 3 hold the signs; selectors 8 + b replicate them)
                    uint32_t s01, s23;
                    asm("prmt.b32 %0, %1, %2, 0xFBD9;" : "=r"(s01) : "r"(word_of(r[0][0], t)), "r"(word_of(r[1][0], t)));
                    asm("prmt.b32 %0, %1, %2, 0xFBD9;" : "=r"(s23) : "r"(word_of(r[2][0], t)), "r"(word_of(r[3][0], t)));
                    constexpr uint32_t SM = (1u << (K - 1)) * 0x01010101u;
                    RL[2 * t] |= prmt(s01, s23, 0x5410) & SM;
                    RL[2 * t + 1] |= prmt(s01, s23, 0x7632) & SM;
                }
                if (K == 9) {
                    const uint32_t h01 = prmt(cp[0][t] >> 1, cp[1][t] >> 1, 0x6420);
                    const uint32_t h23 = prmt(cp[2][t] >> 1, cp[3][t] >> 1, 0x6420);
                    RH[2 * t] = prmt(h01, h23, 0x6420);
                    RH[2 * t + 1] = prmt(h01, h23, 0x7531);
                }
            }
            cols_fast_store<K, 0>(RL, RH, cp, packed, so, base + lane, NG);
        } else if (defer) {   // NaN/Inf (or huge values): k_enc_cols_fixup encodes this warp tile
            deferred = true;
        } else {
            for (int u = 0; u < 4; ++u) {
                const int64_t q = base + 32 * u + lane;
                if (q < NG) enc_container_generic<BF16, K>(in, 0, q, 1, F, packed, so, spi, spb, spc, cap);
            }
        }
    }
    if (defer) raise_fixup_flag(defer_flag, deferred);
}

}  // namespace exmy

namespace exmy {

// ---------------------------------------------------------- decode helpers
// pair of codes (16-bit lanes) from byte-lane registers
template <int K>
__device__ __forceinline__ uint32_t pair_from_lanes(uint32_t rl, uint32_t rh, uint32_t sel) {
    uint32_t p = prmt(rl, 0u, sel);
    if (K == 9) p |= prmt(rh, 0u, sel) << 1;
    return p;
}

// pair of codes -> pair of output words (bf16: one word; fp32: two words)
template <int K>
__device__ __forceinline__ uint32_t dec_pair_to_bf16(uint32_t cp, const FastP &P, const Fmt &F) {
    if (P.dec_fast_bf) return P.two_mul ? dec_pair_bf16<K, true>(cp, P, F.y) : dec_pair_bf16<K, false>(cp, P, F.y);
    return dec_code_generic<8>(cp & 0xFFFFu, F) | (dec_code_generic<8>(cp >> 16, F) << 16);
}
template <int K>
__device__ __forceinline__ uint32_t dec_to_f32(uint32_t code, const FastP &P, const Fmt &F) {
    if (P.dec_fast) return dec_f32_fast<K>(code, P, F.y);
    return dec_code_generic<24>(code, F);
}

// ---------------------------------------------------------- decode ROWS
// Raw packed words of one 8-row x (4*NH)-column tile, all segments: loaded
// one tile ahead (software pipeline) and unpacked into byte lanes after.
__host__ __device__ constexpr int seg_words(int k, int s, int nh) {
    return seg_width(k, s) == 8 ? 8 * nh : nh * seg_width(k, s);
}
__host__ __device__ constexpr int seg_word_off(int k, int s, int nh) {
    int o = 0;
    for (int t = 0; t < s; ++t) o += seg_words(k, t, nh);
    return o;
}
__host__ __device__ constexpr int tile_words(int k, int nh) { return seg_word_off(k, seg_count(k), nh); }

template <int K, int NH, int S>
__device__ __forceinline__ void rows_load_raw(uint32_t (&raw)[tile_words(K, NH)], const uint8_t *packed,
                                              const SegOffsets &so, int64_t g, int64_t C, int64_t c0) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S), OFF = seg_word_off(K, S, NH);
        const uint8_t *seg = packed + so.off[S];
        if constexpr (W == 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                uint32_t w[NH];
                load_words<NH>(seg + (8 * g + i) * C + c0, w);
#pragma unroll
                for (int h = 0; h < NH; ++h) raw[OFF + i * NH + h] = w[h];
            }
        } else {
            uint32_t w[NH * W];
            load_words<NH * W>(seg + (g * C + c0) * W, w);
#pragma unroll
            for (int q = 0; q < NH * W; ++q) raw[OFF + q] = w[q];
        }
        rows_load_raw<K, NH, S + 1>(raw, packed, so, g, C, c0);
    }
}

template <int K, int NH, int S>
__device__ __forceinline__ void rows_unpack_raw(const uint32_t (&raw)[tile_words(K, NH)], uint32_t (&RL)[NH][8],
                                                uint32_t (&RH)[NH][8]) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S), OFF = seg_word_off(K, S, NH);
        if constexpr (W == 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    if (K == 9) RH[h][i] = raw[OFF + i * NH + h];
                    else RL[h][i] = raw[OFF + i * NH + h];
                }
        } else {
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                uint32_t in[W];
#pragma unroll
                for (int q = 0; q < W; ++q) in[q] = raw[OFF + h * W + q];
                swar_unpack4<W, LO>(in, RL[h]);
            }
        }
        rows_unpack_raw<K, NH, S + 1>(raw, RL, RH);
    }
}

// DEC_FAST2: the fast path with o > 127 (two multiplies); kernels launched
// as DEC_FAST switch to it on the device (warp-uniform, once per launch)
enum DecMode { DEC_FAST = 0, DEC_GENERIC = 1, DEC_FAST2 = 2 };

template <int K, bool OBF16, int MODE>
__device__ __forceinline__ uint32_t dec_pair_bf16_m(uint32_t cp, const FastP &P, const Fmt &F) {
    if constexpr (MODE == DEC_FAST) return dec_pair_bf16<K, false>(cp, P, F.y);
    else if constexpr (MODE == DEC_FAST2) return dec_pair_bf16<K, true>(cp, P, F.y);
    else return dec_code_generic<8>(cp & 0xFFFFu, F) | (dec_code_generic<8>(cp >> 16, F) << 16);
}
template <int K, int MODE>
__device__ __forceinline__ uint32_t dec_f32_m(uint32_t code, const FastP &P, const Fmt &F) {
    if constexpr (MODE == DEC_FAST) return dec_f32_fast<K, false>(code, P, F.y);
    else if constexpr (MODE == DEC_FAST2) return dec_f32_fast<K, true>(code, P, F.y);
    else return dec_code_generic<24>(code, F);
}

#ifndef DEC_ROWS_BAR
#define DEC_ROWS_BAR 1
#endif
// DEC_ROWS_BAR: a CTA barrier per row group keeps the CTA's warps writing one
// contiguous run together; the write-bound decode gains when the warps of a
// CTA do not drift apart (config 2, e3m3: 139.8 -> 128.1 us, 84 -> 92 % of
// the copy peak; fp32 output 239.6 -> 213.5 us)
template <int K, bool OBF16, int MODE>
__device__ __forceinline__ void dec_rows_body(const uint8_t *__restrict__ packed, int64_t R, int64_t C,
                                              SegOffsets so, uint8_t *__restrict__ out, const Fmt &F,
                                              const FastP &P) {
    using EL = Elem<OBF16>;
    constexpr int V = EL::V, NH = V / 4, TW = tile_words(K, NH);
    const int64_t CV = C / V, G = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
#if DEC_ROWS_BAR
    const bool act = j < CV;
#else
    if (j >= CV) return;
    constexpr bool act = true;
#endif
    const int64_t c0 = j * V;
    uint32_t nxt[TW];
    int64_t g = blockIdx.y;
    if (g < G && act) rows_load_raw<K, NH, 0>(nxt, packed, so, g, C, c0);
    for (; g < G; g += gridDim.y) {
        uint32_t raw[TW];
#pragma unroll
        for (int q = 0; q < TW; ++q) raw[q] = nxt[q];
#if DEC_ROWS_BAR
        __syncthreads();
#endif
        if (g + gridDim.y < G && act) rows_load_raw<K, NH, 0>(nxt, packed, so, g + gridDim.y, C, c0);
        if (!act) continue;
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
                    o[2 * h] = dec_pair_bf16_m<K, OBF16, MODE>(pair_from_lanes<K>(RL[h][i], RH[h][i], 0x4140), P, F);
                    o[2 * h + 1] = dec_pair_bf16_m<K, OBF16, MODE>(pair_from_lanes<K>(RL[h][i], RH[h][i], 0x4342), P, F);
                }
            } else {
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    uint32_t code = (RL[0][i] >> (8 * v)) & 0xFFu;
                    if (K == 9) code |= ((RH[0][i] >> (8 * v)) & 0xFFu) << 1;
                    o[v] = dec_f32_m<K, MODE>(code, P, F);
                }
            }
            stg_v4(out + ((8 * g + i) * C + c0) * EL::ES, make_uint4(o[0], o[1], o[2], o[3]));
        }
    }
}

template <int K, bool OBF16, int MODE>
__global__ void __launch_bounds__(256) k_dec_rows_fast(const uint8_t *__restrict__ packed, int64_t R, int64_t C,
                                                       int x, int y, const uint8_t *__restrict__ meta, SegOffsets so,
                                                       uint8_t *__restrict__ out) {
    const Fmt F = load_fmt(x, y, meta);
    const FastP P = make_fast(F, false, 0);
    if (MODE == DEC_FAST && P.two_mul) dec_rows_body<K, OBF16, DEC_FAST2>(packed, R, C, so, out, F, P);
    else dec_rows_body<K, OBF16, MODE>(packed, R, C, so, out, F, P);
}

// ---------------------------------------------------------- decode COLS
template <int K, int S>
__device__ __forceinline__ void cols_fast_load(uint32_t (&RL)[8], uint32_t (&RH)[8], const uint8_t *packed,
                                               const SegOffsets &so, int64_t q0, int64_t NG) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S);
        const uint8_t *seg = packed + so.off[S];
        if constexpr (W == 8) {
            uint32_t a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t q = q0 + 32 * u;
                uint2 t = q < NG ? __ldg((const uint2 *)(seg + 8 * q)) : make_uint2(0, 0);
                a[u] = t.x;
                b[u] = t.y;
            }
            // 4x4 byte transposes: group-major words -> element-major byte lanes
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
                const int64_t q = q0 + 32 * u;
                if (q < NG) {
                    if constexpr (W == 4) in[u] = __ldg((const unsigned int *)(seg + 4 * q));
                    else if constexpr (W == 2)
                        in[u >> 1] |= (uint32_t)__ldg((const unsigned short *)(seg + 2 * q)) << (16 * (u & 1));
                    else in[0] |= (uint32_t)__ldg((const unsigned char *)(seg + q)) << (8 * u);
                }
            }
            swar_unpack4<W, LO>(in, RL);
        }
        cols_fast_load<K, S + 1>(RL, RH, packed, so, q0, NG);
    }
}

template <int K, bool OBF16, int MODE>
__device__ __forceinline__ void dec_cols_body(const uint8_t *__restrict__ packed, int64_t n, SegOffsets so,
                                              uint8_t *__restrict__ out, const Fmt &F, const FastP &P) {
    const int64_t NG = n / 8;
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int64_t base = gw * 128; base < NG; base += warps_total * 128) {
        uint32_t RL[8], RH[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { RL[i] = 0; RH[i] = 0; }
        cols_fast_load<K, 0>(RL, RH, packed, so, base + lane, NG);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t q = base + 32 * u + lane;
            if (!OBF16) {
                // fp32 out: 32 B per group.  Lanes swap halves through shuffles
                // so each store instruction writes 512 contiguous bytes (whole
                // sectors); a per-lane 32 B store split in two instructions
                // leaves half-written sectors that L2 writes back twice.
                uint32_t o[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    uint32_t code = (RL[i] >> (8 * u)) & 0xFFu;
                    if (K == 9) code |= ((RH[i] >> (8 * u)) & 0xFFu) << 1;
                    o[i] = dec_f32_m<K, MODE>(code, P, F);
                }
                const int64_t g0 = base + 32 * u;            // first group of this warp row
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int src = 16 * h + (lane >> 1);
                    const bool hi = lane & 1;
                    uint32_t v[4];
#pragma unroll
                    for (int k2 = 0; k2 < 4; ++k2) {
                        const uint32_t a = __shfl_sync(0xFFFFFFFFu, o[k2], src);
                        const uint32_t b = __shfl_sync(0xFFFFFFFFu, o[4 + k2], src);
                        v[k2] = hi ? b : a;
                    }
                    if (g0 + src < NG) stg_v4(out + (g0 * 32) + (32 * h + lane) * 16, make_uint4(v[0], v[1], v[2], v[3]));
                }
                continue;
            }
            if (q >= NG) continue;
            {
                uint32_t o[4];
                const uint32_t sel = (uint32_t)u | ((uint32_t)(4 + u) << 4);   // bytes 0, 1 <- lanes, masked
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    uint32_t cp = prmt(RL[2 * t], RL[2 * t + 1], sel);
                    cp = (cp & 0xFFu) | ((cp & 0xFF00u) << 8);
                    if (K == 9) {
                        uint32_t ch = prmt(RH[2 * t], RH[2 * t + 1], sel);
                        cp |= ((ch & 0xFFu) | ((ch & 0xFF00u) << 8)) << 1;
                    }
                    o[t] = dec_pair_bf16_m<K, OBF16, MODE>(cp, P, F);
                }
                stg_v4(out + q * 16, make_uint4(o[0], o[1], o[2], o[3]));
            }
        }
    }
}

template <int K, bool OBF16, int MODE>
__global__ void __launch_bounds__(256) k_dec_cols_fast(const uint8_t *__restrict__ packed, int64_t n, int x, int y,
                                                       const uint8_t *__restrict__ meta, SegOffsets so,
                                                       uint8_t *__restrict__ out) {
    const Fmt F = load_fmt(x, y, meta);
    const FastP P = make_fast(F, false, 0);
    if (MODE == DEC_FAST && P.two_mul) dec_cols_body<K, OBF16, DEC_FAST2>(packed, n, so, out, F, P);
    else dec_cols_body<K, OBF16, MODE>(packed, n, so, out, F, P);
}

// -------------------------------------------------------------- quantize
template <bool BF16>
__global__ void __launch_bounds__(256) k_quant_fast(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                    int64_t n, int x, int y, const uint8_t *__restrict__ meta,
                                                    int force_generic) {
    using EL = Elem<BF16>;
    const Fmt F = load_fmt(x, y, meta);
    const FastP P = make_fast(F, BF16, force_generic);
    const DecPath DP = make_dec_path(F, force_generic);
    const int64_t nvec = n / EL::V;
    constexpr int U = 4;
    const bool fast = BF16 ? P.enc_simd : P.enc_f32;
    // a CTA owns one contiguous chunk of U*256 vectors (16 KB in, 16 KB out)
    // per iteration (vector = chunk*U*256 + u*256 + tid), chunks grid-strided,
    // and a barrier per chunk keeps its warps reading and writing the chunk
    // together (config 2 bf16: 181 -> 170 us, 90 -> 96 % of the copy peak;
    // fp32 383 -> 353 us)
    const int64_t stride = blockDim.x;
    const int64_t cstep = (int64_t)gridDim.x * blockDim.x * U;
    const int64_t base0 = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x;
    // software pipeline: the next U vectors are in flight while these are processed
    uint4 nxt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t vi = base0 + u * stride;
        if (vi < nvec) nxt[u] = ldg_nc_v4(in + vi * 16);
    }
    for (int64_t base = base0; base < nvec + threadIdx.x; base += cstep) {   // CTA-uniform trip count
        __syncthreads();
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            r[u] = nxt[u];
            const int64_t vn = base + cstep + u * stride;
            if (vn < nvec) nxt[u] = ldg_nc_v4(in + vn * 16);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t vi = base + u * stride;
            if (vi >= nvec) continue;
            uint32_t o[4];
            uint32_t flag = 0;
            if (fast) {
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    o[t] = BF16 ? quant_pair_bf16(word_of(r[u], t), P, flag) : quant_f32_fast(word_of(r[u], t), P, flag);
                flag &= 0x80008000u;
            }
            if (!fast || flag) {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const uint32_t w = word_of(r[u], t);
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
    if (blockIdx.x == 0) {
        for (int64_t i = nvec * EL::V + threadIdx.x; i < n; i += blockDim.x) {
            if (BF16) {
                const uint32_t u = (uint32_t)((const uint16_t *)in)[i] << 16;
                ((uint16_t *)out)[i] = (uint16_t)quantize_elem<true>(u, F, DP);
            } else {
                ((uint32_t *)out)[i] = quantize_elem<false>(((const uint32_t *)in)[i], F, DP);
            }
        }
    }
}

// ------------------------------------------------ deferred NaN/Inf tiles
// The fast encode kernels skip every tile holding NaN/Inf (or a magnitude
// outside the fast range) and raise a flag; this pass -- one launch that
// returns at once while the flag is down -- re-reads the tensor, encodes
// exactly those tiles (fast codes with the NaN/Inf lanes set to code 0, D9's
// in-band placeholder, or the integer path for huge values), and counts the
// NaN/Inf per compaction range, so k_specials_compact can skip its counting
// phase.  The main kernels keep no extra registers for the rare case, and a
// NaN-heavy tensor (a diverged gradient) stays on the vector path.
// Workspace (include/exmy.h): ws[0] total, ws[1 + r] range r's count,
// ws[FIXUP_FLAG_WORD] bit 0 = tiles were deferred, bit 1 = ranges counted.
constexpr int FIXUP_FLAG_WORD = 1 + SPECIALS_RANGES;

// add a per-thread count (all lanes of the calling warp in range r) to the
// range's counter, once per warp
__device__ __forceinline__ void fixup_flush(unsigned long long *ws, int64_t r, unsigned c) {
    const unsigned m = __activemask();
    const unsigned t = __reduce_add_sync(m, c);
    if (t && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(ws + 1 + r, (unsigned long long)t);
}

// NaN/Inf count of NW words (bf16: 2 per word, fp32: 1)
template <bool BF16, int NW>
__device__ __forceinline__ int count_specials(const uint32_t (&w)[NW]) {
    int c = 0;
#pragma unroll
    for (int t = 0; t < NW; ++t) {
        if (BF16) c += __popc(((w[t] & 0x7FFF7FFFu) + 0x00800080u) & 0x80008000u);
        else c += (w[t] & 0x7F800000u) == 0x7F800000u;
    }
    return c;
}

// ROWS: the main kernel's tiles; range of row group g = g >> lg_rg
// (ranges of 8 * C * 2^lg_rg elements)
template <int K, bool BF16, int MODE>
__global__ void __launch_bounds__(256, 2) k_enc_rows_fixup(const uint8_t *__restrict__ in, int64_t R, int64_t C, int x,
                                                           int y, const uint8_t *__restrict__ meta,
                                                           uint8_t *__restrict__ packed, SegOffsets so,
                                                           unsigned long long *ws, int lg_rg) {
    if (ws[FIXUP_FLAG_WORD] == 0ull) return;
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicOr(ws + FIXUP_FLAG_WORD, 2ull);
    using EL = Elem<BF16>;
    constexpr int NW = BF16 ? 2 : 4;
    const Fmt F = load_fmt(x, y, meta);
    const FastP P = make_fast(F, BF16, 0);
    const int64_t CV = C / 4, G = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = j < CV;
    const int64_t c0 = (act ? j : 0) * 4;
    const uint8_t *src = in + c0 * EL::ES;
    const int64_t rstride = C * EL::ES;
    int64_t cur = -1;
    unsigned cnt = 0, total = 0;
    uint32_t nxt[8][NW];   // software pipeline: the next tile's rows in flight (a NaN-heavy tensor is all fix-up)
    int64_t g = blockIdx.y;
    if (g < G && act) {
#pragma unroll
        for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * g + i) * rstride, nxt[i]);
    }
    for (; g < G; g += gridDim.y) {
        const int64_t r = g >> lg_rg;   // the same for the whole CTA
        if (r != cur) {
            if (cur >= 0) fixup_flush(ws, cur, cnt);
            cur = r;
            cnt = 0;
        }
        uint32_t w[8][NW];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < NW; ++q) w[i][q] = nxt[i][q];
        const int64_t gn = g + gridDim.y;
        if (gn < G && act) {
#pragma unroll
            for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * gn + i) * rstride, nxt[i]);
        }
        if (!act) continue;
        int ns = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) ns += count_specials<BF16, NW>(w[i]);
        uint32_t cp[8][2];
        bool bad = false;
        if (ns == 32) {   // every element NaN/Inf (a diverged tensor): all codes are the placeholder 0
#pragma unroll
            for (int i = 0; i < 8; ++i) cp[i][0] = cp[i][1] = 0u;
        } else {
            uint32_t amax = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) vec_codes<K, BF16, MODE, NW>(w[i], cp[i], P, amax);
            if (!amax_special<BF16, MODE>(amax, P)) continue;   // the main kernel stored this tile
#pragma unroll
            for (int i = 0; i < 8; ++i) bad = bad || mask_special_codes<K, BF16, MODE, NW>(w[i], cp[i], P) < 0;
        }
        cnt += (unsigned)ns;
        total += (unsigned)ns;
        if (bad) {   // a huge finite magnitude: the integer path (its specials are counted above)
            for (int v = 0; v < 4; ++v)
                enc_container_generic<BF16, K>(in, C, g * C + c0 + v, 0, F, packed, so, nullptr, nullptr, nullptr, 0);
            continue;
        }
        uint32_t RL[1][8], RH[1][8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            RL[0][i] = prmt(cp[i][0], cp[i][1], 0x6420);
            RH[0][i] = (K == 9) ? prmt(cp[i][0] >> 1, cp[i][1] >> 1, 0x6420) : 0u;
        }
        rows_fast_store<K, 1, 0>(RL, RH, packed, so, g, C, c0);
    }
    if (cur >= 0) fixup_flush(ws, cur, cnt);
    flush_special_count(ws, total);   // the total, once per warp
}

// COLS: the main kernel's warp tiles (128 groups = 1024 elements); range of
// warp tile `base` = (8 * base) >> lg_l (ranges of 2^lg_l >= 1024 elements)
template <int K, bool BF16, int MODE>
__global__ void __launch_bounds__(256) k_enc_cols_fixup(const uint8_t *__restrict__ in, int64_t n, int x, int y,
                                                        const uint8_t *__restrict__ meta,
                                                        uint8_t *__restrict__ packed, SegOffsets so,
                                                        unsigned long long *ws, int lg_l) {
    if (ws[FIXUP_FLAG_WORD] == 0ull) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(ws + FIXUP_FLAG_WORD, 2ull);
    using EL = Elem<BF16>;
    constexpr int NV = BF16 ? 1 : 2;
    constexpr int NP = EL::V / 2;
    const Fmt F = load_fmt(x, y, meta);
    const FastP P = make_fast(F, BF16, 0);
    const int64_t NG = n / 8;
    const int lane = threadIdx.x & 31;
    const int64_t step = (int64_t)gridDim.x * (blockDim.x >> 5) * 128;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    unsigned total = 0;
    for (int64_t base = gw * 128; base < NG; base += step) {
        uint4 r[4][NV];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t q = base + 32 * u + lane;
#pragma unroll
            for (int t = 0; t < NV; ++t) r[u][t] = q < NG ? ldg_nc_v4(in + q * 8 * EL::ES + 16 * t) : make_uint4(0, 0, 0, 0);
        }
        uint32_t cp[4][4];
        uint32_t amax = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int t = 0; t < NV; ++t) {
                uint32_t c2[NP];
                const uint32_t ww[4] = {r[u][t].x, r[u][t].y, r[u][t].z, r[u][t].w};
                vec_codes<K, BF16, MODE, 4>(ww, c2, P, amax);
#pragma unroll
                for (int p = 0; p < NP; ++p) cp[u][t * NP + p] = c2[p];
            }
        }
        // the warp tile was deferred iff any lane saw a special / huge value
        if (!__any_sync(0xFFFFFFFFu, amax_special<BF16, MODE>(amax, P))) continue;
        int ns = 0;
        bool bad = false;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int t = 0; t < NV; ++t) {
                const uint32_t ww[4] = {r[u][t].x, r[u][t].y, r[u][t].z, r[u][t].w};
                uint32_t c2[NP];
#pragma unroll
                for (int p = 0; p < NP; ++p) c2[p] = cp[u][t * NP + p];
                ns += count_specials<BF16, 4>(ww);
                bad = bad || mask_special_codes<K, BF16, MODE, 4>(ww, c2, P) < 0;
#pragma unroll
                for (int p = 0; p < NP; ++p) cp[u][t * NP + p] = c2[p];
            }
        }
        fixup_flush(ws, (8 * base) >> lg_l, (unsigned)ns);
        total += (unsigned)ns;
        if (bad) {
            for (int u = 0; u < 4; ++u) {
                const int64_t q = base + 32 * u + lane;
                if (q < NG) enc_container_generic<BF16, K>(in, 0, q, 1, F, packed, so, nullptr, nullptr, nullptr, 0);
            }
            continue;
        }
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
    }
    flush_special_count(ws, total);
}

}  // namespace exmy
