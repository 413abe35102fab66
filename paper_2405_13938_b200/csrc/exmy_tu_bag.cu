// exmy_tu_bag.cu -- embedding bag over a COLS-packed table (SURVEY 8(f) row 3:
// "decode fused into a GEMM / embedding-bag prologue"; config 5's consumer;
// reading D25).  Each thread owns one 8-column container of one bag's output
// and walks the bag's indices in order: the container of that row is
// gathered from every segment, decoded in registers and accumulated in fp32,
// so decoded rows never reach HBM -- only the pooled (nbags, cols) result.
#include <climits>

#include "exmy_launch.cuh"

using namespace exmy;

namespace {

constexpr int BAG_UNROLL = 4;   // rows gathered ahead of the in-order accumulation

// the 8 codes of container g (row r, container j) from every segment
template <int K>
__device__ __forceinline__ void bag_codes(const uint8_t *__restrict__ packed, const SegOffsets &so, int64_t C,
                                          int64_t r, int64_t j, uint32_t (&code)[8]) {
    const int64_t g = r * (C / 8) + j;
#pragma unroll
    for (int l = 0; l < 8; ++l) code[l] = 0;
    int hi = K;
#pragma unroll
    for (int s = 0; s < seg_count(K); ++s) {
        const int w = seg_width(K, s), lo = hi - w;
        const uint8_t *seg = packed + so.off[s];
        if (w == 8) {
            const uint2 t = __ldg(reinterpret_cast<const uint2 *>(seg + r * C + j * 8));
#pragma unroll
            for (int l = 0; l < 8; ++l) code[l] |= (((l < 4 ? t.x : t.y) >> (8 * (l & 3))) & 0xFFu) << lo;
        } else {
            uint32_t cont;
            if (w == 4) cont = __ldg(reinterpret_cast<const unsigned int *>(seg + g * 4));
            else if (w == 2) cont = __ldg(reinterpret_cast<const unsigned short *>(seg + g * 2));
            else cont = __ldg(seg + g);
#pragma unroll
            for (int l = 0; l < 8; ++l) code[l] |= ((cont >> (w * l)) & ((1u << w) - 1u)) << lo;
        }
        hi = lo;
    }
}

template <int K, bool PERROW, bool WEIGHTED>
__global__ void __launch_bounds__(256) k_embedding_bag(const uint8_t *__restrict__ packed, int64_t C, int x, int y,
                                                       const uint8_t *__restrict__ meta,
                                                       const int64_t *__restrict__ idx,
                                                       const int64_t *__restrict__ offsets, int64_t nbags,
                                                       const float *__restrict__ weights, int mean, SegOffsets so,
                                                       float *__restrict__ out, int fmt_fast) {
    const int64_t gpr = C / 8, total = nbags * gpr;
    RowD D0;
    int e0 = 0;
    if (!PERROW) {
        e0 = min((int)__ldg(meta), 254);
        D0 = make_rowd(e0, x);
        D0.ok = D0.ok && fmt_fast;
    }
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < total; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = p / gpr, j = p - b * gpr;
        const int64_t i0 = __ldg(offsets + b), i1 = __ldg(offsets + b + 1);
        float acc[8];
#pragma unroll
        for (int l = 0; l < 8; ++l) acc[l] = 0.0f;
        for (int64_t i = i0; i < i1; i += BAG_UNROLL) {
            uint32_t code[BAG_UNROLL][8];
            int64_t rr[BAG_UNROLL];
#pragma unroll
            for (int u = 0; u < BAG_UNROLL; ++u) {   // gathers of the next rows in flight together
                rr[u] = i + u < i1 ? __ldg(idx + i + u) : -1;
                if (rr[u] >= 0) bag_codes<K>(packed, so, C, rr[u], j, code[u]);
            }
#pragma unroll
            for (int u = 0; u < BAG_UNROLL; ++u) {   // accumulation strictly in index order (D25)
                if (rr[u] < 0) break;
                RowD D = D0;
                int e = e0;
                if (PERROW) {
                    e = min((int)__ldg(meta + rr[u]), 254);
                    D = make_rowd(e, x);
                    D.ok = D.ok && fmt_fast;
                }
                const float wgt = WEIGHTED ? __ldg(weights + i + u) : 1.0f;
#pragma unroll
                for (int l = 0; l < 8; ++l) {
                    const uint32_t vb = D.ok ? dec_f32_r<K>(code[u][l], y, D) : dec_code_generic<24>(code[u][l], fmt_of(x, y, e));
                    const float v = __uint_as_float(vb);
                    acc[l] = WEIGHTED ? __fmaf_rn(wgt, v, acc[l]) : __fadd_rn(acc[l], v);
                }
            }
        }
        if (mean && i1 > i0) {
            const float cnt = (float)(i1 - i0);
#pragma unroll
            for (int l = 0; l < 8; ++l) acc[l] = __fdiv_rn(acc[l], cnt);
        }
        float *dst = out + b * C + j * 8;
        stg_v4(dst, make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[1]), __float_as_uint(acc[2]),
                               __float_as_uint(acc[3])));
        stg_v4(dst + 4, make_uint4(__float_as_uint(acc[4]), __float_as_uint(acc[5]), __float_as_uint(acc[6]),
                                   __float_as_uint(acc[7])));
    }
}

template <int K>
exmy_status launch_bag_k(const uint8_t *packed, int64_t C, int x, int y, const uint8_t *meta, bool per_row,
                         const int64_t *idx, const int64_t *offsets, int64_t nbags, const float *weights, int mean,
                         const SegOffsets &so, float *out, cudaStream_t st) {
    const int64_t total = nbags * (C / 8);
    int64_t blocks = cdiv(total, 256);
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    if (blocks < 1) blocks = 1;
    const int fast = (!g_force_generic && x <= 7) ? 1 : 0;
#define BAG_LAUNCH(PR, WT)                                                                                        \
    k_embedding_bag<K, PR, WT><<<(unsigned)blocks, 256, 0, st>>>(packed, C, x, y, meta, idx, offsets, nbags, weights, \
                                                                 mean, so, out, fast)
    if (per_row) {
        if (weights) BAG_LAUNCH(true, true);
        else BAG_LAUNCH(true, false);
    } else {
        if (weights) BAG_LAUNCH(false, true);
        else BAG_LAUNCH(false, false);
    }
#undef BAG_LAUNCH
    return launch_status();
}

bool fmt_ok(int x, int y) {
    if (x < 0 || x > 8 || y < 0) return false;
    const int k = 1 + x + y;
    return k >= 3 && k <= 9;
}

}  // namespace

extern "C" exmy_status exmy_embedding_bag(const uint8_t *packed, int64_t rows, int64_t cols, int x, int y,
                                          const uint8_t *meta, int meta_per_row, const int64_t *indices,
                                          const int64_t *offsets, int64_t nbags, const float *weights, int mode,
                                          float *out, void *stream) {
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    if (rows < 0 || cols < 0 || cols % 8 || nbags < 0) return EXMY_E_SHAPE;
    if (cols && rows > INT64_MAX / cols) return EXMY_E_SHAPE;
    if (mode != 0 && mode != 1) return EXMY_E_ARG;
    if (nbags == 0 || cols == 0) return EXMY_OK;
    if (!packed || !meta || !offsets || !out || (!indices && rows)) return EXMY_E_ARG;
    if (!aligned(packed, 8) || !aligned(out, 16)) return EXMY_E_ALIGN;
    const int k = 1 + x + y;
    const Plan p = make_plan(k, rows * cols);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (k) {
#define BAG_K(KK) \
        case KK: return launch_bag_k<KK>(packed, cols, x, y, meta, meta_per_row != 0, indices, offsets, nbags, weights, mode, p.so, out, st);
        BAG_K(3) BAG_K(4) BAG_K(5) BAG_K(6) BAG_K(7) BAG_K(8) BAG_K(9)
#undef BAG_K
    }
    return EXMY_E_FORMAT;
}
