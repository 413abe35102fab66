// exmy_tu_push.cu -- fused encode + all-gather by remote stores (SURVEY 8(f)
// row 2; "encode before ... network communication"
// "each shard can be independently reconstructed").  A rank encodes its row
// shard and its stores go straight to every destination buffer -- on a
// multi-GPU node the peers' packed buffers mapped over NVLink (CUDA IPC /
// symmetric memory), so the all-gather is the encode's own store stream and
// overlaps the conversion tile by tile; no NCCL call, no staging buffer.
#include <climits>

#include "exmy_launch.cuh"

using namespace exmy;

namespace {

constexpr int PUSH_MAX = 8;
struct PushDst {
    uint8_t *p[PUSH_MAX];
    int n;
};

// one container on the integer path: codes of the shard's elements, stored
// at the container's GLOBAL index in every destination; specials recorded
// once with global element indices
template <bool BF16, int K>
__device__ __noinline__ void push_container_generic(const uint8_t *__restrict__ in, int64_t C, int64_t lidx, int64_t g0,
                                                    const Fmt F, const PushDst D, const SegOffsets so, int64_t *spi,
                                                    uint32_t *spb, unsigned long long *spc, int64_t cap) {
    uint32_t c[8];
    int64_t e[8];
    const int64_t eoff = g0 * 8 * C;   // first element of the shard
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        e[i] = lane_elem(lidx, i, C, EXMY_AXIS_ROWS);
        c[i] = enc_elem(load_elem_scalar<BF16>(in, e[i]), F, eoff + e[i], spi, spb, spc, cap);
    }
    const int64_t gidx = lidx + g0 * C;
    for (int d = 0; d < D.n; ++d) {
        int hi = K;
#pragma unroll
        for (int s = 0; s < seg_count(K); ++s) {
            const int w = seg_width(K, s), lo = hi - w;
            uint8_t *seg = D.p[d] + so.off[s];
            if (w == 8) {
                for (int i = 0; i < 8; ++i) seg[eoff + e[i]] = (uint8_t)(c[i] >> lo);
            } else {
                uint32_t cont = 0;
                for (int i = 0; i < 8; ++i) cont |= ((c[i] >> lo) & ((1u << w) - 1u)) << (w * i);
                for (int b = 0; b < w; ++b) seg[gidx * w + b] = (uint8_t)(cont >> (8 * b));
            }
            hi = lo;
        }
    }
}

// ---- NVLS multicast stores: `mc` is a multicast
// address of the symmetric packed buffer (torch symmetric memory's
// multicast_ptr); one multimem.st reaches every GPU bound to the multicast
// object, the NVSwitch replicating it -- instead of one store per peer.
// multimem.st has no byte or half-word form, so every store here is 4, 8 or
// 16 bytes: a tile's 4 containers of a segment (4w bytes) or a w8 row chunk.
__device__ __forceinline__ void mc_st(uint8_t *p, uint32_t a) {
    asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" ::"l"(p), "r"(a) : "memory");
}
__device__ __forceinline__ void mc_st(uint8_t *p, uint32_t a, uint32_t b) {
    asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void mc_st(uint8_t *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
}

template <int W>
__device__ __forceinline__ void mc_store_words(uint8_t *p, const uint32_t (&w)[W]) {
    if constexpr (W == 1) mc_st(p, w[0]);
    else if constexpr (W == 2) mc_st(p, w[0], w[1]);
    else mc_st(p, w[0], w[1], w[2], w[3]);
}

// rows_fast_store (exmy_fast.cuh) with multicast stores: one tile (8 rows x
// 4 columns) of byte-lane codes RL (low 8 code bits) / RH (bits 8..1, k = 9)
template <int K, int S>
__device__ __forceinline__ void rows_mc_store(const uint32_t (&RL)[1][8], const uint32_t (&RH)[1][8], uint8_t *mc,
                                              const SegOffsets &so, int64_t g, int64_t C, int64_t c0) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S);
        uint8_t *seg = mc + so.off[S];
        if constexpr (W == 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i) mc_st(seg + (8 * g + i) * C + c0, (K == 9) ? RH[0][i] : RL[0][i]);
        } else {
            uint32_t out[W];
            swar_pack4<W, LO>(RL[0], out);
            mc_store_words<W>(seg + (g * C + c0) * W, out);
        }
        rows_mc_store<K, S + 1>(RL, RH, mc, so, g, C, c0);
    }
}

// the integer path of one tile for multicast destinations: codes element by
// element (specials recorded with global indices), then the same SWAR packing
// and 4w-byte multicast stores
template <bool BF16, int K>
__device__ __noinline__ void push_tile_generic_mc(const uint8_t *__restrict__ in, int64_t C, int64_t g, int64_t c0,
                                                  int64_t g0, const Fmt F, uint8_t *mc, const SegOffsets so,
                                                  int64_t *spi, uint32_t *spb, unsigned long long *spc, int64_t cap) {
    const int64_t eoff = g0 * 8 * C;
    uint32_t RL[1][8], RH[1][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint32_t cd[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t e = (8 * g + i) * C + c0 + v;
            cd[v] = enc_elem(load_elem_scalar<BF16>(in, e), F, eoff + e, spi, spb, spc, cap);
        }
        const uint32_t p0 = cd[0] | (cd[1] << 16), p1 = cd[2] | (cd[3] << 16);
        RL[0][i] = prmt(p0, p1, 0x6420);
        RH[0][i] = (K == 9) ? prmt(p0 >> 1, p1 >> 1, 0x6420) : 0u;
    }
    rows_mc_store<K, 0>(RL, RH, mc, so, g + g0, C, c0);
}

// k_enc_rows_fast's tiles (8 rows x 4 columns, one tile ahead in flight);
// every segment store is issued once per destination
template <int K, bool BF16, int MODE, bool MC>
__global__ void __launch_bounds__(256, 2) k_enc_push(const uint8_t *__restrict__ in, int64_t R, int64_t C, int64_t g0,
                                                     int x, int y, const uint8_t *__restrict__ meta, PushDst D,
                                                     SegOffsets so, int64_t *spi, uint32_t *spb,
                                                     unsigned long long *spc, int64_t cap, int force_generic) {
    using EL = Elem<BF16>;
    constexpr int NW = BF16 ? 2 : 4;
    const Fmt F = load_fmt(x, y, meta);
    const FastP P = make_fast(F, BF16, force_generic);
    const int64_t CV = C / 4, G = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= CV) return;
    const int64_t c0 = j * 4;
    const uint8_t *src = in + c0 * EL::ES;
    const int64_t rstride = C * EL::ES;
    if (!enc_fast_ok<BF16, MODE>(F, force_generic)) {
        for (int64_t g = blockIdx.y; g < G; g += gridDim.y) {
            if (MC) {
                push_tile_generic_mc<BF16, K>(in, C, g, c0, g0, F, D.p[0], so, spi, spb, spc, cap);
            } else {
                for (int v = 0; v < 4; ++v)
                    push_container_generic<BF16, K>(in, C, g * C + c0 + v, g0, F, D, so, spi, spb, spc, cap);
            }
        }
        return;
    }
    uint32_t nxt[8][NW];
    int64_t g = blockIdx.y;
    if (g < G) {
#pragma unroll
        for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * g + i) * rstride, nxt[i]);
    }
    for (; g < G; g += gridDim.y) {
        uint32_t w[8][NW];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < NW; ++q) w[i][q] = nxt[i][q];
        const int64_t gn = g + gridDim.y;
        if (gn < G) {
#pragma unroll
            for (int i = 0; i < 8; ++i) load4<BF16>(src + (8 * gn + i) * rstride, nxt[i]);
        }
        uint32_t cp[8][2];
        uint32_t amax = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) vec_codes<K, BF16, MODE, NW>(w[i], cp[i], P, amax);
        if (!amax_special<BF16, MODE>(amax, P)) {
            uint32_t RL[1][8], RH[1][8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                RL[0][i] = prmt(cp[i][0], cp[i][1], 0x6420);
                RH[0][i] = (K == 9) ? prmt(cp[i][0] >> 1, cp[i][1] >> 1, 0x6420) : 0u;
            }
            if (MC) {
                rows_mc_store<K, 0>(RL, RH, D.p[0], so, g + g0, C, c0);   // one store reaches every GPU
            } else {
                for (int d = 0; d < D.n; ++d) rows_fast_store<K, 1, 0>(RL, RH, D.p[d], so, g + g0, C, c0);
            }
        } else if (MC) {
            push_tile_generic_mc<BF16, K>(in, C, g, c0, g0, F, D.p[0], so, spi, spb, spc, cap);
        } else {
            for (int v = 0; v < 4; ++v)
                push_container_generic<BF16, K>(in, C, g * C + c0 + v, g0, F, D, so, spi, spb, spc, cap);
        }
    }
}

template <int K, bool BF16, int MODE>
exmy_status launch_push_km(const uint8_t *in, int64_t R, int64_t C, int64_t g0, int x, int y, const uint8_t *meta,
                           const PushDst &D, const SegOffsets &so, int64_t *spi, uint32_t *spb,
                           unsigned long long *spc, int64_t cap, cudaStream_t st, bool mc) {
    const int threads = 256;
    static int occ = 0;
    if (!occ) occ = occupancy(k_enc_push<K, BF16, MODE, false>, threads, 0);
    const int64_t CV = C / 4, G = R / 8;
    const int64_t gx = cdiv(CV, threads);
    int64_t gy = (int64_t)num_sms() * occ / gx;
    if (gy < 1) gy = 1;
    if (gy > G) gy = G;
    if (gy > 65535) gy = 65535;
    if (gx > INT_MAX) return EXMY_E_SHAPE;
    const dim3 grid((unsigned)gx, (unsigned)gy);
    if (mc)
        k_enc_push<K, BF16, MODE, true><<<grid, threads, 0, st>>>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap,
                                                                  g_force_generic);
    else
        k_enc_push<K, BF16, MODE, false><<<grid, threads, 0, st>>>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap,
                                                                   g_force_generic);
    return launch_status();
}

template <int K, bool BF16>
exmy_status launch_push_k(const uint8_t *in, int64_t R, int64_t C, int64_t g0, int x, int y, const uint8_t *meta,
                          const PushDst &D, const SegOffsets &so, int64_t *spi, uint32_t *spb,
                          unsigned long long *spc, int64_t cap, cudaStream_t st, bool mc) {
    if (BF16 && y <= 6)   // mode choice as exmy_encode
        return y == 0 ? launch_push_km<K, BF16, (BF16 ? ENC_SIMD_Y0 : ENC_F32_Y0)>(in, R, C, g0, x, y, meta, D, so, spi,
                                                                                   spb, spc, cap, st, mc)
                      : launch_push_km<K, BF16, (BF16 ? ENC_SIMD : ENC_F32)>(in, R, C, g0, x, y, meta, D, so, spi, spb,
                                                                             spc, cap, st, mc);
    return y == 0 ? launch_push_km<K, BF16, ENC_F32_Y0>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap, st, mc)
                  : launch_push_km<K, BF16, ENC_F32>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap, st, mc);
}

template <bool BF16>
exmy_status push_dispatch(int k, const uint8_t *in, int64_t R, int64_t C, int64_t g0, int x, int y,
                          const uint8_t *meta, const PushDst &D, const SegOffsets &so, int64_t *spi, uint32_t *spb,
                          unsigned long long *spc, int64_t cap, cudaStream_t st, bool mc) {
    switch (k) {
        case 3: return launch_push_k<3, BF16>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap, st, mc);
        case 4: return launch_push_k<4, BF16>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap, st, mc);
        case 5: return launch_push_k<5, BF16>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap, st, mc);
        case 6: return launch_push_k<6, BF16>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap, st, mc);
        case 7: return launch_push_k<7, BF16>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap, st, mc);
        case 8: return launch_push_k<8, BF16>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap, st, mc);
        case 9: return launch_push_k<9, BF16>(in, R, C, g0, x, y, meta, D, so, spi, spb, spc, cap, st, mc);
    }
    return EXMY_E_FORMAT;
}

bool fmt_ok(int x, int y) {
    if (x < 0 || x > 8 || y < 0) return false;
    const int k = 1 + x + y;
    return k >= 3 && k <= 9;
}

}  // namespace

static exmy_status encode_push_impl(const void *in, int dtype, int64_t rows, int64_t cols, int64_t row0,
                                    int64_t total_rows, int x, int y, const uint8_t *meta, uint8_t *const *dst,
                                    int ndst, int64_t *sp_index, uint32_t *sp_bits, uint64_t *sp_count,
                                    int64_t sp_capacity, void *stream, bool mc) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    if (rows < 0 || cols < 0 || row0 < 0 || total_rows < 0 || row0 + rows > total_rows) return EXMY_E_SHAPE;
    if (rows % 8 || row0 % 8 || total_rows % 8) return EXMY_E_SHAPE;
    if (cols && total_rows > INT64_MAX / cols) return EXMY_E_SHAPE;
    if (ndst < 1 || ndst > PUSH_MAX || !dst) return EXMY_E_ARG;
    if (sp_capacity < 0) return EXMY_E_CAPACITY;
    if (sp_capacity > 0 && (!sp_index || !sp_bits)) return EXMY_E_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    auto *spc = reinterpret_cast<unsigned long long *>(sp_count);
    if (spc && cudaMemsetAsync(spc, 0, sizeof(unsigned long long) * (sp_capacity > 0 ? EXMY_SPECIALS_WORDS : 1), st) !=
                   cudaSuccess)
        return EXMY_E_CUDA;
    if (rows == 0 || cols == 0) return EXMY_OK;
    if (!in || !meta) return EXMY_E_ARG;
    const int k = 1 + x + y;
    const Plan p = make_plan(k, total_rows * cols);   // the WHOLE tensor's segment offsets
    PushDst D{};
    D.n = ndst;
    for (int d = 0; d < ndst; ++d) {
        if (!dst[d]) return EXMY_E_ARG;
        D.p[d] = dst[d];
        for (int s = 0; s < p.nseg; ++s)
            if (!aligned(dst[d] + p.so.off[s], p.w[s] == 8 ? 4 : 4 * p.w[s])) return EXMY_E_ALIGN;
    }
    const auto *pi = static_cast<const uint8_t *>(in);
    if (!aligned(pi, 4 * (dtype == EXMY_BF16 ? 2 : 4)) || cols % 4) return EXMY_E_ALIGN;
    exmy_status s = dtype == EXMY_BF16
                        ? push_dispatch<true>(k, pi, rows, cols, row0 / 8, x, y, meta, D, p.so, nullptr, nullptr, spc,
                                              0, st, mc)
                        : push_dispatch<false>(k, pi, rows, cols, row0 / 8, x, y, meta, D, p.so, nullptr, nullptr, spc,
                                               0, st, mc);
    if (s != EXMY_OK) return s;
    // the shard's list, with global element indices (row0 * cols offset)
    return launch_specials_compact(pi, dtype == EXMY_BF16, rows * cols, row0 * cols, sp_index, sp_bits, spc,
                                   sp_capacity, st);
}

extern "C" exmy_status exmy_encode_push(const void *in, int dtype, int64_t rows, int64_t cols, int64_t row0,
                                        int64_t total_rows, int x, int y, const uint8_t *meta, uint8_t *const *dst,
                                        int ndst, int64_t *sp_index, uint32_t *sp_bits, uint64_t *sp_count,
                                        int64_t sp_capacity, void *stream) {
    return encode_push_impl(in, dtype, rows, cols, row0, total_rows, x, y, meta, dst, ndst, sp_index, sp_bits,
                            sp_count, sp_capacity, stream, false);
}

extern "C" exmy_status exmy_encode_push_multicast(const void *in, int dtype, int64_t rows, int64_t cols,
                                                  int64_t row0, int64_t total_rows, int x, int y, const uint8_t *meta,
                                                  uint8_t *mc_dst, int64_t *sp_index, uint32_t *sp_bits,
                                                  uint64_t *sp_count, int64_t sp_capacity, void *stream) {
    uint8_t *const d[1] = {mc_dst};
    return encode_push_impl(in, dtype, rows, cols, row0, total_rows, x, y, meta, d, 1, sp_index, sp_bits, sp_count,
                            sp_capacity, stream, true);
}

// ------------------------------------------------- pull decode (gather on read)
// The mirror of exmy_encode_push ("decode reads peers'
// packed shards over NVLink"): the whole (nsrc * shard_rows, cols) tensor is
// decoded by one kernel whose tiles read row shard s straight from srcs[s]
// -- on a node, every rank's packed shard mapped into this process -- so the
// all-gather of packed bytes happens in the decode's loads and only the
// decoded output is written locally.  k_dec_rows_fast's tiles (8 rows x
// 4*NH columns, next tile in flight, CTA barrier per row group).
namespace {

struct PullSrc {
    const uint8_t *p[PUSH_MAX];
    int n;
};

template <int K, bool OBF16, int MODE>
__device__ __forceinline__ void pull_body(const PullSrc &S, int64_t shard_rows, int64_t C, const SegOffsets &so,
                                          uint8_t *__restrict__ out, const Fmt &F, const FastP &P) {
    using EL = Elem<OBF16>;
    constexpr int V = EL::V, NH = V / 4, TW = tile_words(K, NH);
    const int64_t CV = C / V, gps = shard_rows / 8, G = gps * S.n;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = j < CV;
    const int64_t c0 = j * V;
    uint32_t nxt[TW];
    int64_t g = blockIdx.y;
    if (g < G && act) {
        const int s = (int)(g / gps);
        rows_load_raw<K, NH, 0>(nxt, S.p[s], so, g - s * gps, C, c0);
    }
    for (; g < G; g += gridDim.y) {
        uint32_t raw[TW];
#pragma unroll
        for (int q = 0; q < TW; ++q) raw[q] = nxt[q];
        __syncthreads();
        const int64_t gn = g + gridDim.y;
        if (gn < G && act) {
            const int s = (int)(gn / gps);
            rows_load_raw<K, NH, 0>(nxt, S.p[s], so, gn - s * gps, C, c0);
        }
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
__global__ void __launch_bounds__(256) k_dec_pull(PullSrc S, int64_t shard_rows, int64_t C, int x, int y,
                                                  const uint8_t *__restrict__ meta, SegOffsets so,
                                                  uint8_t *__restrict__ out) {
    const Fmt F = load_fmt(x, y, meta);
    const FastP P = make_fast(F, false, 0);
    if (MODE == DEC_FAST && P.two_mul) pull_body<K, OBF16, DEC_FAST2>(S, shard_rows, C, so, out, F, P);
    else pull_body<K, OBF16, MODE>(S, shard_rows, C, so, out, F, P);
}

template <int K, bool OBF16>
exmy_status launch_pull_k(const PullSrc &S, int64_t shard_rows, int64_t C, int x, int y, const uint8_t *meta,
                          const SegOffsets &so, uint8_t *out, cudaStream_t st) {
    constexpr int V = Elem<OBF16>::V;
    const int threads = 256;
    const int64_t CV = C / V, G = shard_rows / 8 * S.n;
    const int64_t gx = cdiv(CV, threads);
    int64_t gy = (int64_t)num_sms() * 2 / gx;
    if (gy < 1) gy = 1;
    if (gy > G) gy = G;
    if (gy > 65535) gy = 65535;
    if (gx > INT_MAX) return EXMY_E_SHAPE;
    const dim3 grid((unsigned)gx, (unsigned)gy);
    // the multiply path needs x <= 7 (and y <= 7 for bf16 output), as exmy_decode
    if (!g_force_generic && x <= 7 && (!OBF16 || y <= 7)) {
        k_dec_pull<K, OBF16, DEC_FAST><<<grid, threads, 0, st>>>(S, shard_rows, C, x, y, meta, so, out);
    } else {
        k_dec_pull<K, OBF16, DEC_GENERIC><<<grid, threads, 0, st>>>(S, shard_rows, C, x, y, meta, so, out);
    }
    return launch_status();
}

}  // namespace

extern "C" exmy_status exmy_decode_pull(const uint8_t *const *srcs, int nsrc, int64_t shard_rows, int64_t cols, int x,
                                        int y, const uint8_t *meta, void *out, int out_dtype, void *stream) {
    if (out_dtype != EXMY_F32 && out_dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    if (nsrc < 1 || nsrc > PUSH_MAX || !srcs) return EXMY_E_ARG;
    if (shard_rows < 0 || cols < 0 || shard_rows % 8) return EXMY_E_SHAPE;
    if (cols && shard_rows > INT64_MAX / cols / nsrc) return EXMY_E_SHAPE;
    if (shard_rows == 0 || cols == 0) return EXMY_OK;
    if (!meta || !out) return EXMY_E_ARG;
    const bool obf = out_dtype == EXMY_BF16;
    const int V = obf ? 8 : 4;
    const int k = 1 + x + y;
    const Plan p = make_plan(k, shard_rows * cols);   // every shard is an independent packed tensor
    PullSrc S{};
    S.n = nsrc;
    for (int s = 0; s < nsrc; ++s) {
        if (!srcs[s]) return EXMY_E_ARG;
        S.p[s] = srcs[s];
        for (int q = 0; q < p.nseg; ++q) {
            const size_t a = p.w[q] == 8 ? (size_t)V : (size_t)((V * p.w[q]) < 16 ? V * p.w[q] : 16);
            if (!aligned(srcs[s] + p.so.off[q], a)) return EXMY_E_ALIGN;
        }
    }
    if (!aligned(out, 16) || cols % V) return EXMY_E_ALIGN;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    auto *po = static_cast<uint8_t *>(out);
    switch (k) {
#define PULL_K(KK)                                                                                             \
        case KK: return obf ? launch_pull_k<KK, true>(S, shard_rows, cols, x, y, meta, p.so, po, st)          \
                            : launch_pull_k<KK, false>(S, shard_rows, cols, x, y, meta, p.so, po, st);
        PULL_K(3) PULL_K(4) PULL_K(5) PULL_K(6) PULL_K(7) PULL_K(8) PULL_K(9)
#undef PULL_K
    }
    return EXMY_E_FORMAT;
}
