// exmy_gemv.cuh -- decode fused into a matrix-vector product (SURVEY 8(f)
// row 3, "decode fused into the consumer"; serving decode is "performance
// critical").  out[m, n] = sum_k act[m, k] * W[n, k] for the
// eXmY-packed weight matrix W (N x K, ROWS layout, per-tensor or per-row
// metadata) and a few fp32 activation rows (M <= 8 per pass): the HBM read is
// the packed bytes (k/8 per weight) instead of a decoded bf16 copy.
//
// Decode by table: a CTA holds the 2^k decoded values (exact, the integer
// decode of every code incl. its sign) 32 times in shared memory, copy l in
// bank l, so lane l's lookup of any code is conflict-free and an element
// costs one byte extract + LOP3 (address), one LDS, then M FFMAs.  Per-row
// metadata: the table is built for e_max = 125 (o = 125 - top: every grid
// value of every format is a normal-or-subnormal fp32 number, none
// overflows) and each row's sum is scaled by the exact 2^(e_n - 125) at the
// end -- equal to the dot product of the decoded row unless a partial sum
// over- or underflows in one of the two (reading D26).
//
// Order of the fp32 sums: per thread over its column tiles in order, then a
// xor-butterfly over the warp, then over the 8 warps in order -- deterministic.
// NaN/Inf weights (out of band, D9) are added afterwards by k_gemv_specials.
#pragma once
#include "exmy_blocked.cuh"

namespace exmy {

constexpr int GEMV_THREADS = 256;

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// U column tiles (8 rows x 4 columns each) per thread and iteration, loads
// issued together: the packed bytes in flight per SM must cover HBM latency
template <int K, int M>
__host__ __device__ constexpr int gemv_u() { return M <= 2 ? 4 : (M <= 4 ? 2 : 1); }

template <int K, int M>
__global__ void __launch_bounds__(GEMV_THREADS, M >= 8 ? 1 : 2)
    k_gemv_rows(const uint8_t *__restrict__ packed, int64_t N, int64_t Kc, SegOffsets so, int x, int y,
                const uint8_t *__restrict__ meta, int per_row, const float *__restrict__ act, int64_t lda,
                float *__restrict__ out, int64_t ldo) {
    extern __shared__ __align__(16) uint32_t gsm[];
    constexpr int TW = tile_words(K, 1);
    constexpr int U = gemv_u<K, M>();
    constexpr uint32_t TB = 128u << K;   // table bytes: 2^K codes x 32 lanes x 4 B
    __shared__ float red[GEMV_THREADS / 32][8 * M];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tab = ((uint32_t)__cvta_generic_to_shared(gsm) + TB - 1u) & ~(TB - 1u);
    // per-tensor: the table IS the decode; per-row: decode at e_max = 125, rows rescaled
    const Fmt F = fmt_of(x, y, per_row ? 125 : min((int)meta[0], 254));
    for (int i = threadIdx.x; i < (32 << K); i += GEMV_THREADS)
        sts_u32(tab + 4u * (uint32_t)i, dec_code_generic<24>((uint32_t)(i >> 5), F));
    __syncthreads();
    const uint32_t lsa = tab + 4u * (uint32_t)lane;
    const int64_t CV = Kc / 4, G = N / 8;
    for (int64_t g = blockIdx.x; g < G; g += gridDim.x) {
        float acc[8][M];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int m = 0; m < M; ++m) acc[i][m] = 0.f;
        for (int64_t j0 = threadIdx.x; j0 < CV; j0 += (int64_t)GEMV_THREADS * U) {
            uint32_t raw[U][TW];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t j = j0 + (int64_t)GEMV_THREADS * u;
                if (j < CV) rows_load_raw<K, 1, 0>(raw[u], packed, so, g, Kc, 4 * j);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t j = j0 + (int64_t)GEMV_THREADS * u;
                if (j >= CV) break;
                uint32_t RL[1][8], RH[1][8];
#pragma unroll
                for (int i = 0; i < 8; ++i) { RL[0][i] = 0; RH[0][i] = 0; }
                rows_unpack_raw<K, 1, 0>(raw[u], RL, RH);
                // column by column: 8 weights (one per row) and M activations live,
                // not 32 weights or M float4s (M = 8 spilled)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    float wv[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint32_t r = RL[0][i];
                        const uint32_t off = v == 0 ? (r << 7) : (r >> (8 * v - 7));
                        wv[i] = lds_f32((off & (TB - 128u)) | lsa);
                    }
#pragma unroll
                    for (int m = 0; m < M; ++m) {
                        const float xs = __ldg(act + m * lda + 4 * j + v);
#pragma unroll
                        for (int i = 0; i < 8; ++i) acc[i][m] = fmaf(xs, wv[i], acc[i][m]);
                    }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int m = 0; m < M; ++m) {
                float a = acc[i][m];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
                if (lane == 0) red[warp][i * M + m] = a;
            }
        __syncthreads();
        if (threadIdx.x < 8 * M) {
            const int i = threadIdx.x / M, m = threadIdx.x % M;
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < GEMV_THREADS / 32; ++w) s += red[w][threadIdx.x];
            if (per_row) {   // exact 2^(e_n - 125), e_n in [0, 254]: two factors in [-126, 127]
                const int d = min((int)meta[8 * g + i], 254) - 125;
                const int d1 = d > 127 ? 127 : d;
                s = __fmul_rn(__fmul_rn(s, pow2f_exact(d1)), pow2f_exact(d - d1));
            }
            out[m * ldo + 8 * g + i] = s;
        }
        __syncthreads();
    }
}

// The same product with the packed bytes staged in shared memory by bulk
// asynchronous copies (cp.async.bulk on an mbarrier, issued by one thread,
// two stages of GEMV_CH columns of a row group: k * GEMV_CH bytes each), so
// the bytes in flight per SM no longer depend on registers -- the register
// path above keeps at most U tiles per thread in flight and ran
// latency-bound (config 2, m = 1: 105 us, 2.2 TB/s of packed bytes).
// Needs cols % 16 == 0 (16-byte aligned segment spans); the last chunk of a
// row may be shorter.  Each thread converts the tiles of the stage (4
// columns x 8 rows) from shared memory exactly as the register path does.
constexpr int GEMV_CH = 2048;   // columns per stage
#ifndef GEMV_NST
#define GEMV_NST 2              // stages in flight (A/B: 2, 3, 4 measured equal: the kernel is issue-bound)
#endif

// one stage (cw columns of a row group, segment spans back to back) folded
// into the thread's 8 x M sums; CW > 0: cw == CW known at compile time
// PA (k <= 7): the table has a 256-byte row per code (lane l at word l) on a
// 64 KB-aligned shared address, so a lookup address is ONE prmt -- the code
// byte dropped into byte 1 of the lane's address -- instead of a shift + LOP3
template <int K, int M, int CW, int NT, bool PA = false>
__device__ __forceinline__ void gemv_tiles(uint32_t dst, uint32_t cw, const uint32_t (&jt)[NT], int64_t c0,
                                           uint32_t lsa, const float *__restrict__ act, int64_t lda,
                                           float (&acc)[8][M]) {
    constexpr int TW = tile_words(K, 1);
    constexpr uint32_t TB = 128u << K;
    uint32_t RL[NT][8];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        uint32_t raw[TW];
        uint32_t soff = 0;
        int wo = 0;
#pragma unroll
        for (int sgi = 0; sgi < seg_count(K); ++sgi) {
            const int W = seg_width(K, sgi);
            if (W == 8) {
#pragma unroll
                for (int i = 0; i < 8; ++i) raw[wo + i] = ld_shared_u32(dst + 4u * jt[t] + (soff + (uint32_t)i * cw));
                wo += 8;
            } else {
                const uint32_t pa = dst + 4u * jt[t] * (uint32_t)W;
#pragma unroll
                for (int w = 0; w < W; ++w) raw[wo + w] = ld_shared_u32(pa + (soff + 4u * (uint32_t)w));
                wo += W;
            }
            soff += cw * (uint32_t)W;
        }
        uint32_t L[1][8], H[1][8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { L[0][i] = 0; H[0][i] = 0; }
        rows_unpack_raw<K, 1, 0>(raw, L, H);
#pragma unroll
        for (int i = 0; i < 8; ++i) RL[t][i] = L[0][i];
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int64_t j = c0 / 4 + jt[t];
        float4 xv[M];
#pragma unroll
        for (int m = 0; m < M; ++m) xv[m] = __ldg(reinterpret_cast<const float4 *>(act + m * lda + 4 * j));
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            float wv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t r = RL[t][i];
                if constexpr (PA) {
                    wv[i] = lds_f32(prmt(r, lsa, 0x7604u | ((uint32_t)v << 4)));
                } else {
                    const uint32_t off = v == 0 ? (r << 7) : (r >> (8 * v - 7));
                    wv[i] = lds_f32((off & (TB - 128u)) | lsa);
                }
            }
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const float xs = v == 0 ? xv[m].x : (v == 1 ? xv[m].y : (v == 2 ? xv[m].z : xv[m].w));
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i][m] = fmaf(xs, wv[i], acc[i][m]);
            }
        }
    }
}

// one stage (cw columns of a row group, segment spans back to back) folded
// into the thread's 8 x M sums; CW > 0: cw == CW known at compile time, and
// the thread's CW / 1024 tiles are converted together (independent chains
// of shared-memory loads and ALU work to overlap)
template <int K, int M, int CW, bool PA>
__device__ __forceinline__ void gemv_stage(uint32_t dst, uint32_t cw_rt, int64_t c0, uint32_t lsa,
                                           const float *__restrict__ act, int64_t lda, float (&acc)[8][M]) {
    if constexpr (CW > 0) {
        static_assert(CW % (4 * GEMV_THREADS) == 0, "full stages: whole tiles per thread");
        constexpr int NT = CW / (4 * GEMV_THREADS);
        uint32_t jt[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) jt[t] = threadIdx.x + (uint32_t)(t * GEMV_THREADS);
        gemv_tiles<K, M, CW, NT, PA>(dst, (uint32_t)CW, jt, c0, lsa, act, lda, acc);
    } else {
        for (uint32_t j1 = threadIdx.x; j1 < cw_rt / 4; j1 += GEMV_THREADS) {
            const uint32_t jt[1] = {j1};
            gemv_tiles<K, M, 0, 1, PA>(dst, cw_rt, jt, c0, lsa, act, lda, acc);
        }
    }
}

#ifndef GEMV_PA
#define GEMV_PA 1   // A/B builds: 0 = shift + LOP3 table addresses
#endif
template <int K>
__host__ __device__ constexpr bool gemv_pa() { return GEMV_PA && K <= 7; }
// dynamic shared memory of the bulk kernel: PA needs a 64 KB-aligned table
// (256 B per code) -- 96 KB always holds table + stages whatever the
// window offset of the dynamic block (< 2 KB: reserved + static)
template <int K>
__host__ __device__ constexpr int gemv_bulk_smem() {
    return gemv_pa<K>() ? 98304 : 2 * (128 << K) + GEMV_NST * K * GEMV_CH;
}

#ifndef GEMV_MINB
#define GEMV_MINB 2   // CTAs per SM for m <= 4 (A/B builds)
#endif
template <int K, int M>
__global__ void __launch_bounds__(GEMV_THREADS, M >= 8 ? 1 : (M <= 2 ? GEMV_MINB : 2))
    k_gemv_rows_bulk(const uint8_t *__restrict__ packed, int64_t N, int64_t Kc, SegOffsets so, int x, int y,
                     const uint8_t *__restrict__ meta, int per_row, const float *__restrict__ act, int64_t lda,
                     float *__restrict__ out, int64_t ldo) {
    extern __shared__ __align__(16) uint32_t gsm[];
    constexpr int TW = tile_words(K, 1);
    constexpr uint32_t TB = 128u << K;
    constexpr uint32_t STB = (uint32_t)K * GEMV_CH;   // bytes of one stage: k bytes per column (8 rows)
    __shared__ float red[GEMV_THREADS / 32][8 * M];
    __shared__ __align__(8) unsigned long long bars[GEMV_NST];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr bool PA = gemv_pa<K>();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(gsm);
    uint32_t tab, stg0;
    if constexpr (PA) {   // table on the next 64 KB boundary, stages below it if they fit
        tab = (base + 65535u) & ~65535u;
        stg0 = (tab - base >= (uint32_t)GEMV_NST * STB) ? base : tab + (256u << K);
    } else {
        tab = (base + TB - 1u) & ~(TB - 1u);
        stg0 = tab + TB;                               // the stages after the table
    }
    const Fmt F = fmt_of(x, y, per_row ? 125 : min((int)meta[0], 254));
    for (int i = threadIdx.x; i < (32 << K); i += GEMV_THREADS)
        sts_u32(tab + (PA ? 256u * (uint32_t)(i >> 5) + 4u * (uint32_t)(i & 31) : 4u * (uint32_t)i),
                dec_code_generic<24>((uint32_t)(i >> 5), F));
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[0]);
    if (threadIdx.x == 0) {
        for (int b = 0; b < GEMV_NST; ++b) mbar_init(bar0 + 8u * b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t lsa = tab + 4u * (uint32_t)lane;
    const int64_t G = N / 8, nch = (Kc + GEMV_CH - 1) / GEMV_CH;
    const int64_t ng = G > blockIdx.x ? (G - 1 - blockIdx.x) / gridDim.x + 1 : 0;   // row groups of this CTA
    const int64_t nq = ng * nch;                                                       // chunks of this CTA
    // chunk q: row group g = blockIdx.x + (q / nch) * gridDim.x, columns [c0, c0 + cw)
    auto issue = [&](int64_t q) {
        const int64_t g = blockIdx.x + (q / nch) * gridDim.x, c0 = (q % nch) * GEMV_CH;
        const uint32_t cw = (uint32_t)min((int64_t)GEMV_CH, Kc - c0);
        const uint32_t st = (uint32_t)(q % GEMV_NST), bar = bar0 + 8u * st, dst = stg0 + st * STB;
        mbar_expect_tx(bar, (uint32_t)K * cw);
        uint32_t soff = 0;   // segment s's span inside the stage: width W bytes per column
#pragma unroll
        for (int sgi = 0; sgi < seg_count(K); ++sgi) {
            const int W = seg_width(K, sgi);
            const uint8_t *seg = packed + so.off[sgi];
            if (W == 8) {   // row-major bytes: one span per row
                for (int i = 0; i < 8; ++i)
                    bulk_g2s(dst + soff + (uint32_t)i * cw, seg + (8 * g + i) * Kc + c0, cw, bar);
            } else {
                bulk_g2s(dst + soff, seg + (g * Kc + c0) * W, cw * (uint32_t)W, bar);
            }
            soff += cw * (uint32_t)W;
        }
    };
    if (threadIdx.x == 0)
        for (int64_t q = 0; q < GEMV_NST && q < nq; ++q) issue(q);
    float acc[8][M];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int m = 0; m < M; ++m) acc[i][m] = 0.f;
    for (int64_t q = 0; q < nq; ++q) {
        const int64_t g = blockIdx.x + (q / nch) * gridDim.x, ch = q % nch, c0 = ch * GEMV_CH;
        const uint32_t cw = (uint32_t)min((int64_t)GEMV_CH, Kc - c0);
        const uint32_t st = (uint32_t)(q % GEMV_NST), dst = stg0 + st * STB;
        mbar_wait(bar0 + 8u * st, (uint32_t)((q / GEMV_NST) & 1));
        // full stages: the column count is the constant GEMV_CH, so every
        // segment offset in the stage is an immediate of the LDS
        if (cw == GEMV_CH) gemv_stage<K, M, GEMV_CH, PA>(dst, GEMV_CH, c0, lsa, act, lda, acc);
        else gemv_stage<K, M, 0, PA>(dst, cw, c0, lsa, act, lda, acc);
        __syncthreads();   // every thread is done with this stage
        if (threadIdx.x == 0 && q + GEMV_NST < nq) issue(q + GEMV_NST);
        if (ch == nch - 1) {   // row group done: reduce over the CTA, store, restart the sums
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    float a = acc[i][m];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
                    if (lane == 0) red[warp][i * M + m] = a;
                    acc[i][m] = 0.f;
                }
            __syncthreads();
            if (threadIdx.x < 8 * M) {
                const int i = threadIdx.x / M, m = threadIdx.x % M;
                float sum = 0.f;
#pragma unroll
                for (int w = 0; w < GEMV_THREADS / 32; ++w) sum += red[w][threadIdx.x];
                if (per_row) {
                    const int d = min((int)meta[8 * g + i], 254) - 125;
                    const int d1 = d > 127 ? 127 : d;
                    sum = __fmul_rn(__fmul_rn(sum, pow2f_exact(d1)), pow2f_exact(d - d1));
                }
                out[m * ldo + 8 * g + i] = sum;
            }
            __syncthreads();
        }
    }
}

// NaN/Inf weights (the encode's ordered out-of-band list, D9): out[m, n] +=
// act[m, k] * v for each listed (n, k).  Any NaN/Inf term decides the sum
// (x * Inf, Inf + finite, Inf - Inf = NaN), so the order of these additions
// does not matter.
static __global__ void k_gemv_specials(const int64_t *__restrict__ idx, const uint32_t *__restrict__ bits,
                                const unsigned long long *__restrict__ count, int64_t cap, int64_t Kc,
                                const float *__restrict__ act, int64_t lda, int64_t M, float *out, int64_t ldo) {
    const long long cnt = (long long)min((unsigned long long)cap, *count);
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < cnt * M;
         t += (long long)gridDim.x * blockDim.x) {
        const long long s = t / M, m = t % M;
        const int64_t e = idx[s], n = e / Kc, k = e % Kc;
        atomicAdd(out + m * ldo + n, act[m * lda + k] * __uint_as_float(bits[s]));
    }
}

}  // namespace exmy
