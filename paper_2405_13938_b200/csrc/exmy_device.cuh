// exmy_device.cuh -- per-element eXmY arithmetic and bit-packing helpers for
// the sm_100a kernels.  Product code: shares nothing with oracle/.
//
// Notation follows PAPER.md (P:n) and DESIGN.md readings (Dn):
//   x, y      exponent / mantissa bits, k = 1+x+y
//   e_max     metadata = max biased exponent (fp32 convention)
//   o         = e_max - (2^x - 1): fp32 biased exponent of exponent code 0's
//             successor minus one, i.e. code exponent e maps to fp32
//             biased exponent e + o (bias = 127 - o, D1)
//   M         = 2^(x+y) - 1, the largest magnitude code (saturation, D7)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

namespace exmy {

struct Fmt {
    int x, y;      // format
    int o;         // exponent offset, see header
    int top;       // 2^x - 1, largest exponent code
    uint32_t M;    // largest magnitude code
    int e_max;
};

__device__ __forceinline__ Fmt load_fmt(int x, int y, const uint8_t *meta) {
    Fmt F;
    int e = (int)__ldg(meta);
    e = e > 254 ? 254 : e;   // D4: 255 is not a valid metadata value
    F.x = x; F.y = y; F.e_max = e;
    F.top = (1 << x) - 1;
    F.o = e - F.top;
    F.M = (1u << (x + y)) - 1u;
    return F;
}

// ---------------------------------------------------------------- rounding
// round-to-nearest-even of X / 2^sh, 1 <= sh <= 31
__device__ __forceinline__ uint32_t rtne_shr(uint32_t X, int sh, uint32_t flip = 0u) {
    // ties go up when (q ^ flip) is odd: flip = 0 is ties-to-even on q
    uint32_t q = X >> sh;
    uint32_t r = X & ((1u << sh) - 1u);
    uint32_t h = 1u << (sh - 1);
    return q + (uint32_t)((r > h) | ((r == h) & ((q ^ flip) & 1u)));
}

__device__ __forceinline__ bool is_special_f32(uint32_t u) {
    return (u & 0x7F800000u) == 0x7F800000u;
}

// --------------------------------------------------------------- encode
// Code of a FINITE fp32 pattern u (bf16 inputs are widened exactly, b<<16).
// Integer-only, valid for every (x, y, e_max):  the exact value
// sig * 2^(Ee-150) is rebased onto the code exponent Ep = Ee - o and
// rounded once (RTNE) at the grid quantum; a carry out of the mantissa
// lands naturally in the next exponent code; saturate at M.
__device__ __forceinline__ uint32_t enc_code_generic(uint32_t u, const Fmt &F) {
    uint32_t s = u >> 31;
    uint32_t a = u & 0x7FFFFFFFu;
    int E = (int)(a >> 23);
    uint32_t f = a & 0x7FFFFFu;
    uint32_t sig;
    int Ee;
    if (E == 0) {                       // zero or fp32 subnormal input (D11)
        if (f == 0) return s << (F.x + F.y);
        int t = __clz(f) - 8;           // normalise: 24 - bitlen(f)
        sig = f << t;
        Ee = 1 - t;
    } else {
        sig = f | 0x800000u;
        Ee = E;
    }
    int Ep = Ee - F.o;
    uint32_t mag;
    if (Ep > F.top) {
        mag = F.M;                      // above the top binade: saturate
    } else {
        uint32_t X;
        int sh;
        uint32_t flip = 0u;
        if (F.x > 0 && Ep >= 1) {       // normal target code
            X = ((uint32_t)(Ep - 1) << 23) + sig;
            sh = 23 - F.y;
            // y = 0 (D6): a tie goes to the even fp32 exponent, i.e. up iff
            // Ep + o is odd (q = Ep here); y >= 1: the even code
            if (F.y == 0) flip = (uint32_t)F.o & 1u;
        } else {                        // subnormal target (every code when x=0)
            X = sig;
            sh = 24 - F.y - Ep;
        }
        mag = sh >= 32 ? 0u : rtne_shr(X, sh, flip);
        mag = min(mag, F.M);
    }
    return (s << (F.x + F.y)) | mag;
}

// ---------------------------------------------------------------- decode
// exact value sig * 2^E2 (sig < 2^10) -> IEEE binary with p significand bits
// and 8 exponent bits (fp32: p=24, bf16: p=8), RTNE (D21).  Sign excluded.
template <int P>
__device__ __forceinline__ uint32_t round_exact_to_ieee(uint32_t sig, int E2) {
    if (sig == 0) return 0u;
    int L = 32 - __clz(sig);
    int Eu = E2 + L - 1;                 // unbiased exponent of the value
    if (Eu >= -126) {                    // normal output: L <= 9 <= P bits, exact
        uint32_t ef = (uint32_t)(Eu + 127);
        if (ef >= 255u) return 0xFFu << (P - 1);   // unreachable for k <= 9
        uint32_t mant = (sig << (P - L)) & ((1u << (P - 1)) - 1u);
        return (ef << (P - 1)) | mant;
    }
    int t = E2 + 126 + P - 1;            // value / output quantum = sig * 2^t
    if (t >= 0) return sig << t;
    int sh = -t;
    return sh >= 32 ? 0u : rtne_shr(sig, sh);
}

// generic decode of a k-bit code to fp32 (P=24) or bf16 (P=8) bits
template <int P>
__device__ __forceinline__ uint32_t dec_code_generic(uint32_t code, const Fmt &F) {
    uint32_t s = (code >> (F.x + F.y)) & 1u;
    uint32_t mag = code & F.M;
    uint32_t e = F.x ? (mag >> F.y) : 0u;
    uint32_t m = mag & ((1u << F.y) - 1u);
    uint32_t sig;
    int E2;
    if (e == 0) { sig = m; E2 = F.o - 126 - F.y; }                 // m 2^(1-bias-y)
    else        { sig = (1u << F.y) | m; E2 = (int)e + F.o - 127 - F.y; }
    return (s << (P + 7)) | round_exact_to_ieee<P>(sig, E2);
}

// Fast decode to fp32 (x <= 7): the magnitude code shifted into an fp32
// pattern has exponent field e and mantissa m<<(23-y), i.e. value
// v_e * 2^(127 - ...) with code exponent 0 landing on fp32 subnormals; one
// non-FTZ multiply by 2^o (split 2^127 * 2^(o-127) when o > 127, the first
// factor being exact) gives the RTNE fp32 result of the exact grid value.
struct DecScale { float s1, s2; bool two; };

__device__ __forceinline__ float pow2f_exact(int e) {   // e in [-149, 127]
    return e >= -126 ? __uint_as_float((uint32_t)(e + 127) << 23)
                     : __uint_as_float(1u << (e + 149));
}

__device__ __forceinline__ DecScale make_dec_scale(const Fmt &F) {
    DecScale d;
    d.two = F.o > 127;
    d.s1 = pow2f_exact(d.two ? 127 : F.o);
    d.s2 = pow2f_exact(d.two ? F.o - 127 : 0);
    return d;
}

__device__ __forceinline__ uint32_t dec_mag_fast_f32(uint32_t mag, int y, const DecScale &d) {
    float f = __uint_as_float(mag << (23 - y));
    f = __fmul_rn(f, d.s1);
    if (d.two) f = __fmul_rn(f, d.s2);
    return __float_as_uint(f);
}

// ------------------------------------------------------------ pack plan
__host__ __device__ constexpr int seg_count(int k) {
    return ((k >> 3) & 1) + ((k >> 2) & 1) + ((k >> 1) & 1) + (k & 1);
}
__host__ __device__ constexpr int seg_width(int k, int j) {
    int w = 8;
    for (; w >= 1; w >>= 1) {
        if (k & w) {
            if (j == 0) return w;
            --j;
        }
    }
    return 0;
}
__host__ __device__ constexpr int seg_lo(int k, int j) {
    int hi = k;
    for (int t = 0; t <= j; ++t) hi -= seg_width(k, t);
    return hi;
}

// container of 8 lanes: sum_i ((c_i >> lo) & (2^w-1)) << (w*i)   (D13, D14)
template <int W, int LO>
__device__ __forceinline__ uint32_t pack8(const uint32_t (&c)[8]) {
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r |= ((c[i] >> LO) & ((1u << W) - 1u)) << (W * i);
    return r;
}

template <int W, int LO>
__device__ __forceinline__ void unpack8(uint32_t cont, uint32_t (&c)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] |= ((cont >> (W * i)) & ((1u << W) - 1u)) << LO;
}

// -------------------------------------------------------- memory helpers
__device__ __forceinline__ uint4 ldg_nc_v4(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
// L2 eviction-priority policies (createpolicy) and loads that carry them:
// a kernel that reads data twice (fused per-row max + encode) marks the first
// read evict_last so the second, evict_first, finds it in L2
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint4 ldg_nc_v4_pol(const void *p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint2 ldg_nc_v2_pol(const void *p, uint64_t pol) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
    return r;
}
// EXMY_ST_HINT (A/B builds only, default 0): 1 = st.global.cs (evict-first
// streaming stores), 2 = st.global.L1::no_allocate
#ifndef EXMY_ST_HINT
#define EXMY_ST_HINT 0
#endif
#if EXMY_ST_HINT == 1
#define EXMY_ST_OP "st.global.cs"
#elif EXMY_ST_HINT == 2
#define EXMY_ST_OP "st.global.L1::no_allocate"
#else
#define EXMY_ST_OP "st.global"
#endif
__device__ __forceinline__ void stg_v4(void *p, uint4 v) {
    asm volatile(EXMY_ST_OP ".v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void stg_v2(void *p, uint32_t a, uint32_t b) {
    asm volatile(EXMY_ST_OP ".v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}

}  // namespace exmy
