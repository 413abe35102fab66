// exmy_tma.cuh -- ROWS encode with the input staged by the Tensor Memory
// Accelerator's bulk copies (cp.async.bulk + mbarrier), persistent CTAs.
//
// k_enc_rows_fast keeps one 8-row tile per thread in flight in registers;
// at the 80-register cap that is ~48 KB of loads in flight per SM, about
// the bandwidth-latency product of one SM's share of HBM, and the loads
// themselves are 8 LSU instructions per tile.  Here one elected thread per
// CTA streams 8 rows x TC columns tiles (16 KB bf16) into an S-deep ring of
// shared-memory stages with 8 bulk copies per tile (completion counted on
// the stage's mbarrier); the 256 threads convert a tile from shared memory
// (one 8-byte LDS per row, conflict-free) while the next S-1 tiles are in
// flight -- S x 16 KB per CTA, with no registers held for them -- then pack
// and store exactly as k_enc_rows_fast (same codes, same bytes).  One CTA
// barrier per tile releases its stage to the producer.
#pragma once
#include "exmy_blocked.cuh"

namespace exmy {

constexpr int ETMA_THREADS = 256;
constexpr int ETMA_TC = 4 * ETMA_THREADS;   // tile columns: 4 per thread

template <bool BF16>
__host__ __device__ constexpr int etma_stages() { return BF16 ? 4 : 3; }
template <bool BF16>
__host__ __device__ constexpr int etma_stage_bytes() { return 8 * ETMA_TC * (BF16 ? 2 : 4); }
template <bool BF16>
__host__ __device__ constexpr int etma_smem() { return etma_stages<BF16>() * etma_stage_bytes<BF16>() + 64; }

template <int K, bool BF16, int MODE>
__global__ void __launch_bounds__(ETMA_THREADS, BF16 ? 3 : 2) k_enc_rows_tma(const uint8_t *__restrict__ in, int64_t R, int64_t C,
                                                               int x, int y, const uint8_t *__restrict__ meta,
                                                               uint8_t *__restrict__ packed, SegOffsets so,
                                                               int64_t *spi, uint32_t *spb, unsigned long long *spc,
                                                               int64_t cap, int force_generic) {
    using EL = Elem<BF16>;
    constexpr int NW = BF16 ? 2 : 4;              // words per 4 elements
    constexpr int S = etma_stages<BF16>();
    constexpr int SB = etma_stage_bytes<BF16>();
    extern __shared__ __align__(128) uint8_t etma_sm[];
    const Fmt F = load_fmt(x, y, meta);
    const FastP P = make_fast(F, BF16, force_generic);
    const int tid = threadIdx.x;
    const int64_t nct = (C + ETMA_TC - 1) / ETMA_TC, T = (R / 8) * nct;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(etma_sm);
    const uint32_t bar0 = sbase + S * SB;          // S mbarriers of 8 bytes after the stages
    const int64_t rowb = C * EL::ES;
    const bool fast = enc_fast_ok<BF16, MODE>(F, force_generic);
    unsigned nsp = 0;

    // tile t -> rows 8g..8g+7, columns [c0, c0 + w) with w = min(TC, C - c0)
    auto issue = [&](int64_t t, int s) {
        const int64_t g = t / nct, c0 = (t - g * nct) * ETMA_TC;
        const int64_t w = min((int64_t)ETMA_TC, C - c0);
        const uint32_t bytes = (uint32_t)(w * EL::ES);
        const uint32_t bar = bar0 + 8 * s;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of the stage
        mbar_expect_tx(bar, 8u * bytes);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            bulk_g2s(sbase + s * SB + i * ETMA_TC * EL::ES, in + (8 * g + i) * rowb + c0 * EL::ES, bytes, bar);
    };

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (fast && tid == 0)
        for (int s = 0; s < S; ++s) {
            const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
            if (t < T) issue(t, s);
        }
    int64_t i = 0;
    for (int64_t t = blockIdx.x; t < T; t += gridDim.x, ++i) {
        const int64_t g = t / nct, c0 = (t - g * nct) * ETMA_TC + 4 * tid;
        const bool act = c0 < C;
        if (!fast) {   // metadata outside the fast preconditions: integer path from global memory
            if (act)
                for (int v = 0; v < 4; ++v)
                    enc_container_generic<BF16, K>(in, C, g * C + c0 + v, 0, F, packed, so, spi, spb, spc, cap);
            continue;
        }
        const int s = (int)(i % S);
        mbar_wait(bar0 + 8 * s, (uint32_t)((i / S) & 1));
        uint32_t w[8][NW];
        if (act) {
            const uint8_t *src = etma_sm + s * SB + 4 * tid * EL::ES;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if constexpr (BF16) {
                    const uint2 v = *reinterpret_cast<const uint2 *>(src + r * ETMA_TC * 2);
                    w[r][0] = v.x;
                    w[r][1] = v.y;
                } else {
                    const uint4 v = *reinterpret_cast<const uint4 *>(src + r * ETMA_TC * 4);
                    w[r][0] = v.x;
                    w[r][1] = v.y;
                    w[r][2] = v.z;
                    w[r][3] = v.w;
                }
            }
        }
        __syncthreads();   // every thread holds its words: the stage goes back to the producer
        if (tid == 0) {
            const int64_t tn = t + (int64_t)S * gridDim.x;
            if (tn < T) issue(tn, s);
        }
        if (!act) continue;
        uint32_t cp[8][2];
        uint32_t amax = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) vec_codes<K, BF16, MODE, NW>(w[r], cp[r], P, amax);
        bool store_fast = !amax_special<BF16, MODE>(amax, P);
        if (!store_fast) {   // NaN/Inf: masked fast codes unless huge finite values need the integer path
            int ns = 0;
#pragma unroll
            for (int r = 0; r < 8 && ns >= 0; ++r) {
                const int m = mask_special_codes<K, BF16, MODE, NW>(w[r], cp[r], P);
                ns = m < 0 ? -1 : ns + m;
            }
            if (ns >= 0) {
                nsp += (unsigned)ns;
                store_fast = true;
            }
        }
        if (store_fast) {
            uint32_t RL[1][8], RH[1][8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                RL[0][r] = prmt(cp[r][0], cp[r][1], 0x6420);
                RH[0][r] = (K == 9) ? prmt(cp[r][0] >> 1, cp[r][1] >> 1, 0x6420) : 0u;
            }
            rows_fast_store<K, 1, 0>(RL, RH, packed, so, g, C, c0);
        } else {
            for (int v = 0; v < 4; ++v)
                enc_container_generic<BF16, K>(in, C, g * C + c0 + v, 0, F, packed, so, spi, spb, spc, cap);
        }
    }
    flush_special_count(spc, nsp);
}

}  // namespace exmy
