// exmy_grouped.cuh -- one launch over a table of tensors.
// A model is hundreds of tensors, each under its own metadata byte
// (P:222-226); per-tensor calls cost 2-3 launches and a grid tail each, which
// dominates for the small ones (norms, k/v projections).  Here a whole table
// is reduced, encoded or decoded by grid-stride CTAs over "chunks": work
// units that never straddle tensors (each tensor's count is rounded up to
// whole chunks by the host plan), so a CTA locates its tensor once per chunk
// (binary search over the table by one thread, shared with the CTA).
//
// Per element the arithmetic is exactly the per-tensor kernels' (ROWS
// layout, 8-row x 4-column thread tiles, same fast/generic split), so the
// bytes are bit-identical to exmy_encode / exmy_decode per entry.
#pragma once
#include "exmy_blocked.cuh"

namespace exmy {

constexpr uint32_t GROUP_MAGIC = 0x47594D45u;   // "EMYG"

struct GroupHeader {   // first 64 bytes of a plan (host and device copies identical)
    uint32_t magic;
    int32_t n, dtype, x, y, out_dtype;
    int64_t vec_chunks;    // max pass: chunks of GRP_VEC_CHUNK 16-byte vectors
    int64_t tile_chunks;   // encode: CTA chunks of GRP_TILE_CHUNK 8x4 tiles
    int64_t dtile_chunks;  // decode: CTA chunks of GRP_DTILE_CHUNK 8x(4*dec_nh) tiles
    int32_t dec_nh;        // decode tile width / 4: 2 for bf16 output when every cols % 8 == 0, else 1
    int16_t specials;      // 1 if any entry has a specials counter
    int16_t per_row;       // 1: one metadata byte per row (exmy_group_plan_rows), else one per tensor
    int64_t row_total;     // per-row plans: rows over all non-empty entries (the row max pass's work)
};
static_assert(sizeof(GroupHeader) == 64, "plan header is 64 bytes");

struct GroupEntry {   // one tensor (128 bytes)
    const uint8_t *in;
    uint8_t *out;
    uint8_t *packed;
    uint8_t *meta;
    int64_t *spi;
    uint32_t *spb;
    unsigned long long *spc;
    int64_t cap;
    int64_t rows, cols;
    int64_t vec_begin, tile_begin, dtile_begin;   // first chunk of this tensor in each pass
    int64_t row_begin;                            // per-row plans: first global row of this tensor
    int64_t frg_begin;                            // per-row plans: first staged row group (fused entries)
    int64_t fused;                                // per-row plans: rows fit the TMA-staged fused encode
};
static_assert(sizeof(GroupEntry) == 128, "plan entry is 128 bytes");

// segment byte offsets of an n-element tensor (exmy_segments): widths of k's
// set bits, widest first, each segment n*w/8 bytes
template <int K>
__device__ __forceinline__ SegOffsets grp_so(int64_t n) {
    SegOffsets so;
    const int64_t n8 = n >> 3;
    int acc = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        so.off[s] = (long long)acc * n8;
        if (s < seg_count(K)) acc += seg_width(K, s);
    }
    return so;
}

#ifndef GRP_ENC_MINB
#define GRP_ENC_MINB 2   // encode CTAs per SM (launch bounds)
#endif
#ifndef GRP_DEC_BAR
#define GRP_DEC_BAR 1    // decode: CTA barrier per chunk (config 3: 4.15 -> 3.80 ms)
#endif
#ifndef GRP_ENC_BAR
#define GRP_ENC_BAR 0    // encode: CTA barrier per chunk
#endif
#ifndef GRP_DEC_OCC
#define GRP_DEC_OCC 3    // decode CTAs per SM (measured: 2 -> 4.52 ms, 3 -> 3.85, 4 -> 3.98 on config 3)
#endif

constexpr int GRP_THREADS = 256;
constexpr int GRP_VEC_CHUNK = GRP_THREADS * 4;   // 16 KB of input per max chunk
#ifndef GRP_TPC
#define GRP_TPC 8        // encode: tiles per thread per chunk
#endif
#ifndef GRP_DTPC
#define GRP_DTPC 1       // decode: tiles per thread per chunk
#endif
constexpr int GRP_TILE_CHUNK = GRP_THREADS * GRP_TPC;     // encode: tiles per CTA chunk
constexpr int GRP_DTILE_CHUNK = GRP_THREADS * GRP_DTPC;   // decode: tiles per CTA chunk

// last entry whose first chunk is <= ch (entries without work share their
// successor's begin and are never returned for a valid chunk)
// Chunk -> tensor lookup: binary search for the last entry whose first chunk
// is <= ch (entries without work share their successor's begin and are never
// returned for a valid chunk).  The begin column of the table is staged in
// shared memory at kernel start (8 bytes per entry, up to GRP_SMEM_TAB
// entries) so the search costs shared-memory latency, not a chain of
// dependent global loads in front of every chunk's loads.
constexpr int GRP_SMEM_TAB = 4096;
enum GrpKind { GRP_VEC = 0, GRP_TILE = 1, GRP_DTILE = 2, GRP_ROW = 3, GRP_FRG = 4 };

template <int KIND>
__device__ __forceinline__ int64_t grp_begin(const GroupEntry &e) {
    return KIND == GRP_VEC     ? e.vec_begin
           : KIND == GRP_TILE  ? e.tile_begin
           : KIND == GRP_DTILE ? e.dtile_begin
           : KIND == GRP_ROW   ? e.row_begin
                               : e.frg_begin;
}

__host__ __device__ inline size_t grp_smem_bytes(int n) { return n <= GRP_SMEM_TAB ? (size_t)n * 8 : 0; }

template <int KIND>
__device__ __forceinline__ const int64_t *grp_stage(const GroupEntry *tab, int n, int64_t *sm) {
    if (n > GRP_SMEM_TAB) return nullptr;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = grp_begin<KIND>(tab[i]);
    __syncthreads();
    return sm;
}

template <int KIND>
__device__ __forceinline__ int grp_find(const GroupEntry *tab, const int64_t *sb, int n, int64_t ch) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        const int64_t b = sb ? sb[mid] : grp_begin<KIND>(tab[mid]);
        if (b <= ch) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

template <int WHAT>   // 0: meta bytes, 1: specials counts
__global__ void k_grouped_clear(const GroupEntry *__restrict__ tab, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (WHAT == 0) {
            if (tab[i].meta) *tab[i].meta = 0;
        }
        else if (tab[i].spc) *tab[i].spc = 0ull;
    }
}

// ------------------------------------------------ per-tensor max exponent
// Each thread keeps the running maximum magnitude of the tensor it is on
// (bf16: two 16-bit lanes, NaN/Inf lanes zeroed); the CTA reduces and raises
// the tensor's byte (byte_atomic_max) only when its chunks move to another
// tensor, so a large tensor costs one atomic per CTA, not per chunk.
template <bool BF16>
__device__ __forceinline__ void grp_flush_max(uint8_t *meta, uint32_t amax, uint32_t *wm) {
    uint32_t e = BF16 ? max((amax & 0xFFFFu) >> 7, amax >> 23) : (amax >> 23);
    e = __reduce_max_sync(0xFFFFFFFFu, e);
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t m = 0;
#pragma unroll
        for (int i = 0; i < GRP_THREADS / 32; ++i) m = max(m, wm[i]);
        byte_atomic_max(meta, m > 254u ? 254u : m);
    }
    __syncthreads();
}

template <bool BF16>
__global__ void __launch_bounds__(GRP_THREADS) k_grouped_max(const GroupEntry *__restrict__ tab, int n,
                                                             int64_t nchunks) {
    extern __shared__ int64_t grp_sm[];
    __shared__ int s_e[2];
    __shared__ uint32_t wm[GRP_THREADS / 32];
    const int64_t *sb = grp_stage<GRP_VEC>(tab, n, grp_sm);
    uint32_t amax = 0;
    int cur = -1, it = 0;
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x, it ^= 1) {
        if (threadIdx.x == 0) s_e[it] = grp_find<GRP_VEC>(tab, sb, n, ch);
        __syncthreads();
        const int e = s_e[it];
        if (e != cur) {   // block-uniform
            if (cur >= 0) grp_flush_max<BF16>(tab[cur].meta, amax, wm);
            amax = 0;
            cur = e;
        }
        const uint8_t *in = tab[e].in;
        const int64_t nvec = tab[e].rows * tab[e].cols / Elem<BF16>::V;
        const int64_t v0 = (ch - tab[e].vec_begin) * GRP_VEC_CHUNK + threadIdx.x;
        uint4 r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t vi = v0 + u * GRP_THREADS;
            r[u] = vi < nvec ? ldg_nc_v4(in + vi * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t w = word_of(r[u], q);
                if (BF16) {
                    const uint32_t a2 = w & 0x7FFF7FFFu;
                    const uint32_t sp = (a2 + 0x00800080u) & 0x80008000u;   // lanes with exponent 255
                    amax = vmax_u16x2(amax, a2 & ~((sp >> 15) * 0xFFFFu));
                } else {
                    const uint32_t a = w & 0x7FFFFFFFu;
                    amax = max(amax, a < 0x7F800000u ? a : 0u);
                }
            }
        }
    }
    if (cur >= 0) grp_flush_max<BF16>(tab[cur].meta, amax, wm);
}

// ------------------------------------------------ chunk -> thread tiles
// Encode and decode hand out work per CTA chunk of GRP_TPC (decode:
// GRP_DTPC) steps x 256 tiles: at step s, warp w covers tiles s*256 + 32w .. +31 (one per lane), so
// the CTA's warps sweep one contiguous 256-tile run per step (whole DRAM
// pages read / written together) without any barrier: each warp resolves
// its chunk's tensor itself, galloping forward from the current one (all
// lanes search the same shared-memory words: broadcast reads, no
// divergence), and issues its next tile's loads as soon as its own data has
// arrived.  Inside a chunk the next tile is one add and one compare away.
template <int KIND>
__device__ __forceinline__ int64_t grp_b(const GroupEntry *tab, const int64_t *sb, int i) {
    return sb ? sb[i] : grp_begin<KIND>(tab[i]);
}

template <int KIND>
__device__ __forceinline__ int grp_advance(const GroupEntry *tab, const int64_t *sb, int n, int e, int64_t ch) {
    if (e + 1 >= n || grp_b<KIND>(tab, sb, e + 1) > ch) return e;
    int lo = e + 1, step = 1;   // begin(lo) <= ch
    while (lo + step < n && grp_b<KIND>(tab, sb, lo + step) <= ch) {
        lo += step;
        step <<= 1;
    }
    int hi = min(lo + step, n) - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (grp_b<KIND>(tab, sb, mid) <= ch) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// per-lane cursor over 8 x 4*NH tiles (32-bit tile coordinates: the plan
// bounds rows/8 and cols)
struct GrpCur {
    int64_t ch;    // warp chunk
    int e;         // its tensor
    int sub;       // step of this thread within the chunk (0..GRP_TPC-1)
    int g, c;      // row group, first column of the tile
    int G, C;      // tensor row groups, columns
    int dq, dc;    // step to the thread's next tile of the chunk (+256 tiles): +dq row groups, +dc columns
};

template <int NH, int KIND, bool SKIPF = false>   // SKIPF: fused entries' chunks do no work
__device__ __forceinline__ void grp_chunk(GrpCur &u, const GroupEntry *tab, const int64_t *sb) {
    const int C = (int)tab[u.e].cols;
    const uint32_t CV = (uint32_t)C / (4 * NH);
    const int64_t j = (u.ch - grp_b<KIND>(tab, sb, u.e)) * (KIND == GRP_DTILE ? GRP_DTILE_CHUNK : GRP_TILE_CHUNK) +
                      threadIdx.x;
    const int64_t q = ((j >> 32) == 0) ? (int64_t)((uint32_t)j / CV) : j / CV;   // 32-bit division when it fits
    u.C = C;
    u.G = (SKIPF && tab[u.e].fused) ? 0 : (int)(tab[u.e].rows >> 3);
    u.g = (int)q;
    u.c = (int)(j - q * CV) * (4 * NH);
    u.dq = (int)((uint32_t)GRP_THREADS / CV);
    u.dc = (int)((uint32_t)GRP_THREADS % CV) * (4 * NH);
    u.sub = 0;
}

// next tile of this thread; false when the CTA has no more chunks.  BAR: a
// CTA barrier at each chunk boundary (uniform: every warp takes GRP_TPC
// steps per chunk), which keeps the CTA's warps on the same chunk
template <int NH, int KIND, bool BAR = false, bool SKIPF = false>
__device__ __forceinline__ bool grp_next(GrpCur &u, const GroupEntry *tab, const int64_t *sb, int n,
                                         int64_t nchunks, int64_t wstride) {
    if (++u.sub < (KIND == GRP_DTILE ? GRP_DTPC : GRP_TPC)) {
        u.g += u.dq;
        u.c += u.dc;
        if (u.c >= u.C) {
            u.c -= u.C;
            ++u.g;
        }
        return true;
    }
    u.ch += wstride;
    if (u.ch >= nchunks) return false;
    if (BAR) __syncthreads();
    u.e = grp_advance<KIND>(tab, sb, n, u.e, u.ch);
    grp_chunk<NH, KIND, SKIPF>(u, tab, sb);
    return true;
}

// ------------------------------------------------ per-row max exponent
// Per-row plans ("the maximum exponent of each row"): one warp per row,
// rows numbered across the whole table; consecutive warps of a CTA take
// consecutive rows, so a CTA streams one contiguous run of the table.  Each
// row's byte is written by its warp alone (no clear, no atomics).  Host
// guarantees cols % 8 == 0 (whole 16-byte vectors per row).
constexpr int GRP_ROW_UNROLL = 4;

template <bool BF16, bool SKIPF = false>   // SKIPF: leave the fused entries' rows to k_grouped_rowwise_smem
__global__ void __launch_bounds__(GRP_THREADS) k_grouped_rowmax(const GroupEntry *__restrict__ tab, int n,
                                                                int64_t nrows) {
    extern __shared__ int64_t grp_sm[];
    const int64_t *sb = grp_stage<GRP_ROW>(tab, n, grp_sm);
    const int lane = threadIdx.x & 31;
    const int64_t wstride = (int64_t)gridDim.x * (GRP_THREADS / 32);
    int64_t r = (int64_t)blockIdx.x * (GRP_THREADS / 32) + (threadIdx.x >> 5);
    if (r >= nrows) return;
    int e = grp_find<GRP_ROW>(tab, sb, n, r);
    for (; r < nrows; r += wstride) {
        e = grp_advance<GRP_ROW>(tab, sb, n, e, r);
        if (SKIPF && tab[e].fused) continue;
        const int64_t lr = r - grp_b<GRP_ROW>(tab, sb, e);
        const int64_t C = tab[e].cols;
        const int64_t nv = C * Elem<BF16>::ES / 16;
        const uint8_t *src = tab[e].in + lr * C * Elem<BF16>::ES;
        uint32_t amax = 0;
        for (int64_t v = lane; v < nv; v += 32 * GRP_ROW_UNROLL) {
            uint4 q[GRP_ROW_UNROLL];
#pragma unroll
            for (int u = 0; u < GRP_ROW_UNROLL; ++u) {
                const int64_t vi = v + 32 * u;
                q[u] = vi < nv ? ldg_nc_v4(src + vi * 16) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < GRP_ROW_UNROLL; ++u) {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const uint32_t w = word_of(q[u], t);
                    if (BF16) {
                        const uint32_t a2 = w & 0x7FFF7FFFu;
                        const uint32_t sp = (a2 + 0x00800080u) & 0x80008000u;   // lanes with exponent 255
                        amax = vmax_u16x2(amax, a2 & ~((sp >> 15) * 0xFFFFu));
                    } else {
                        const uint32_t a = w & 0x7FFFFFFFu;
                        amax = max(amax, a < 0x7F800000u ? a : 0u);
                    }
                }
            }
        }
        uint32_t m = BF16 ? max((amax & 0xFFFFu) >> 7, amax >> 23) : (amax >> 23);
        m = __reduce_max_sync(0xFFFFFFFFu, m);
        if (lane == 0) tab[e].meta[lr] = (uint8_t)(m > 254u ? 254u : m);
    }
}

// ------------------------------------------------ encode (ROWS)
// The lane's next tile is loaded while the current one is converted and
// packed (software pipeline, as k_enc_rows_fast).
template <bool BF16, int NW, bool PR>
__device__ __forceinline__ void grp_enc_load(const GroupEntry *tab, const GrpCur &u, uint32_t (&nxt)[8][NW],
                                             uint2 &nm) {
    using EL = Elem<BF16>;
    const uint8_t *src = tab[u.e].in + ((int64_t)8 * u.g * u.C + u.c) * EL::ES;
    const int64_t rs = (int64_t)u.C * EL::ES;
#pragma unroll
    for (int i = 0; i < 8; ++i) load4<BF16>(src + i * rs, nxt[i]);
    if (PR) nm = __ldg(reinterpret_cast<const uint2 *>(tab[u.e].meta) + u.g);   // the tile's 8 row bytes
}

// byte i of a tile's 8 per-row metadata bytes, clamped to 254 (D2)
__device__ __forceinline__ int tile_row_meta(const uint2 &m, int i) {
    const uint32_t b = ((i < 4 ? m.x : m.y) >> (8 * (i & 3))) & 0xFFu;
    return b > 254u ? 254 : (int)b;
}

// PR: per-row metadata (exmy_group_plan_rows): the tile's 8 rows each under
// their own byte, arithmetic as k_enc_rows_blk (exmy_blocked.cuh)
template <int K, bool BF16, int MODE, bool PR, bool SKIPF = false>
__global__ void __launch_bounds__(GRP_THREADS, GRP_ENC_MINB) k_grouped_encode(const GroupEntry *__restrict__ tab,
                                                                              int n, int64_t nchunks, int x, int y,
                                                                              int force_generic) {
    constexpr int NW = BF16 ? 2 : 4;
    constexpr bool SIMD = (MODE == ENC_SIMD || MODE == ENC_SIMD_Y0);
    extern __shared__ int64_t grp_sm[];
    const int64_t *sb = grp_stage<GRP_TILE>(tab, n, grp_sm);
    const int64_t wstride = gridDim.x;
    GrpCur u;
    u.ch = blockIdx.x;
    if (u.ch >= nchunks) return;
    u.e = grp_find<GRP_TILE>(tab, sb, n, u.ch);
    grp_chunk<1, GRP_TILE, SKIPF>(u, tab, sb);
    uint32_t nxt[8][NW];
    uint2 nm = make_uint2(0, 0);
    if (u.g < u.G) grp_enc_load<BF16, NW, PR>(tab, u, nxt, nm);
    int cur = -1;
    FastP P;            // only the fast path's constants stay live; the integer
    bool fast = false;  // path rebuilds its Fmt from the metadata byte
    if (PR) {           // e_max-independent constants only (per-row: RowP per tile row)
        P = make_fast(fmt_of(x, y, 0), BF16, 1);
        fast = !force_generic;
    }
    for (bool more = true; more;) {
        const int te = u.e, tg = u.g, tc = u.c;
        const bool ok = u.g < u.G;
        uint32_t w[8][NW];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < NW; ++q) w[i][q] = nxt[i][q];
        const uint2 em = nm;
        more = grp_next<1, GRP_TILE, GRP_ENC_BAR != 0, SKIPF>(u, tab, sb, n, nchunks, wstride);   // warp-uniform
        if (more && u.g < u.G) grp_enc_load<BF16, NW, PR>(tab, u, nxt, nm);
        if (!PR && te != cur) {   // new tensor: its format constants
            cur = te;
            const Fmt F = load_fmt(x, y, tab[cur].meta);
            P = make_fast(F, BF16, force_generic);
            fast = enc_fast_ok<BF16, MODE>(F, force_generic);
        }
        if (!ok) continue;
        const GroupEntry &E = tab[te];
        const int64_t C = E.cols;
        const SegOffsets so = grp_so<K>(E.rows * C);
        uint32_t amax = 0;
        uint32_t cp[8][2];
        bool tfast = fast;
        if (fast) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (PR) {
                    const RowP Rp = make_rowp<SIMD>(tile_row_meta(em, i), x, y);
                    tfast = tfast && Rp.ok;
                    vec_codes_r<K, BF16, MODE, NW>(w[i], cp[i], P, Rp, amax);
                } else {
                    vec_codes<K, BF16, MODE, NW>(w[i], cp[i], P, amax);
                }
            }
        }
        if (tfast && !amax_special<BF16, MODE>(amax, P)) {
            uint32_t RL[1][8], RH[1][8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                RL[0][i] = prmt(cp[i][0], cp[i][1], 0x6420);
                RH[0][i] = (K == 9) ? prmt(cp[i][0] >> 1, cp[i][1] >> 1, 0x6420) : 0u;
            }
            rows_fast_store<K, 1, 0>(RL, RH, E.packed, so, tg, C, tc);
        } else if (PR) {   // NaN/Inf in the tile or a row's metadata outside the fast range
            const MetaMap M{E.meta, 1, C, 1};
            for (int v = 0; v < 4; ++v)
                enc_container_generic_blk<BF16, K>(E.in, C, (int64_t)tg * C + tc + v, 0, x, y, M, E.packed, so,
                                                   E.spi, E.spb, E.spc, E.cap);
        } else {   // NaN/Inf in the tile or metadata outside the fast range
            const Fmt F = load_fmt(x, y, E.meta);
            for (int v = 0; v < 4; ++v)
                enc_container_generic<BF16, K>(E.in, C, (int64_t)tg * C + tc + v, 0, F, E.packed, so, E.spi, E.spb,
                                               E.spc, E.cap);
        }
    }
}

// ------------------------------------------------ decode (ROWS)
// Tiles of 8 rows x 4*NH columns (NH = 2 for bf16 output: 16-byte stores,
// as k_dec_rows_fast); the lane's next packed words are in flight while the
// current tile is unpacked and converted.
template <int K, bool OBF16, int MODE, int NH>
__device__ __forceinline__ void grp_dec_tile(const uint32_t (&raw)[tile_words(K, NH)], uint8_t *out, int64_t C,
                                             int64_t g, int64_t c0, const Fmt &F, const FastP &P) {
    using EL = Elem<OBF16>;
    uint32_t RL[NH][8], RH[NH][8];
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
        for (int i = 0; i < 8; ++i) { RL[h][i] = 0; RH[h][i] = 0; }
    rows_unpack_raw<K, NH, 0>(raw, RL, RH);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint8_t *dst = out + ((8 * g + i) * C + c0) * EL::ES;
        if (OBF16) {
            uint32_t o[2 * NH];
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                o[2 * h] = dec_pair_bf16_m<K, OBF16, MODE>(pair_from_lanes<K>(RL[h][i], RH[h][i], 0x4140), P, F);
                o[2 * h + 1] = dec_pair_bf16_m<K, OBF16, MODE>(pair_from_lanes<K>(RL[h][i], RH[h][i], 0x4342), P, F);
            }
            if constexpr (NH == 2) stg_v4(dst, make_uint4(o[0], o[1], o[2], o[3]));
            else stg_v2(dst, o[0], o[1]);
        } else {
            uint32_t o[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                uint32_t code = (RL[0][i] >> (8 * v)) & 0xFFu;
                if (K == 9) code |= ((RH[0][i] >> (8 * v)) & 0xFFu) << 1;
                o[v] = dec_f32_m<K, MODE>(code, P, F);
            }
            stg_v4(dst, make_uint4(o[0], o[1], o[2], o[3]));
        }
    }
}

// per-row metadata: row i of the tile scaled by 2^o_i (one multiply, o_i <=
// 127 checked by the caller), arithmetic as k_dec_rows_blk; GEN: the integer
// path (dec_code_generic) under each row's own format, inline (a call to the
// per-container fallback would keep the pipeline registers live across it)
template <int K, bool OBF16, int NH, bool GEN>
__device__ __forceinline__ void grp_dec_tile_r(const uint32_t (&raw)[tile_words(K, NH)], uint8_t *out, int64_t C,
                                               int64_t g, int64_t c0, int x, int y, const uint2 &em) {
    using EL = Elem<OBF16>;
    uint32_t RL[NH][8], RH[NH][8];
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
        for (int i = 0; i < 8; ++i) { RL[h][i] = 0; RH[h][i] = 0; }
    rows_unpack_raw<K, NH, 0>(raw, RL, RH);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const RowD D = make_rowd(tile_row_meta(em, i), x);
        const Fmt F = fmt_of(x, y, tile_row_meta(em, i));
        uint8_t *dst = out + ((8 * g + i) * C + c0) * EL::ES;
        if (OBF16) {
            uint32_t o[2 * NH];
#pragma unroll
            for (int h = 0; h < NH; ++h) {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint32_t cp = pair_from_lanes<K>(RL[h][i], RH[h][i], j ? 0x4342 : 0x4140);
                    o[2 * h + j] = GEN ? dec_code_generic<8>(cp & 0xFFFFu, F) | (dec_code_generic<8>(cp >> 16, F) << 16)
                                       : dec_pair_bf16_r<K>(cp, y, D);
                }
            }
            if constexpr (NH == 2) stg_v4(dst, make_uint4(o[0], o[1], o[2], o[3]));
            else stg_v2(dst, o[0], o[1]);
        } else {
            uint32_t o[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                uint32_t code = (RL[0][i] >> (8 * v)) & 0xFFu;
                if (K == 9) code |= ((RH[0][i] >> (8 * v)) & 0xFFu) << 1;
                o[v] = GEN ? dec_code_generic<24>(code, F) : dec_f32_r<K>(code, y, D);
            }
            stg_v4(dst, make_uint4(o[0], o[1], o[2], o[3]));
        }
    }
}

template <int K, int NH, bool PR>
__device__ __forceinline__ void grp_dec_load(const GroupEntry *tab, const GrpCur &u,
                                             uint32_t (&nxt)[tile_words(K, NH)], uint2 &nm) {
    rows_load_raw<K, NH, 0>(nxt, tab[u.e].packed, grp_so<K>(tab[u.e].rows * tab[u.e].cols), u.g, u.C, u.c);
    if (PR) nm = __ldg(reinterpret_cast<const uint2 *>(tab[u.e].meta) + u.g);
}

template <int K, bool OBF16, int MODE, int NH, bool PR>
__global__ void __launch_bounds__(GRP_THREADS, K < 9 ? GRP_DEC_OCC : 2) k_grouped_decode(const GroupEntry *__restrict__ tab, int n,
                                                                int64_t nchunks, int x, int y) {
    constexpr int TW = tile_words(K, NH);
    static_assert(NH == 1 || OBF16, "fp32 output uses 8x4 tiles");
    extern __shared__ int64_t grp_sm[];
    const int64_t *sb = grp_stage<GRP_DTILE>(tab, n, grp_sm);
    const int64_t wstride = gridDim.x;
    GrpCur u;
    u.ch = blockIdx.x;
    if (u.ch >= nchunks) return;
    u.e = grp_find<GRP_DTILE>(tab, sb, n, u.ch);
    grp_chunk<NH, GRP_DTILE>(u, tab, sb);
    uint32_t nxt[TW];
    uint2 nm = make_uint2(0, 0);
    if (u.g < u.G) grp_dec_load<K, NH, PR>(tab, u, nxt, nm);
    int cur = -1;
    Fmt F;
    FastP P;
    const int omax = 127 + (1 << x) - 1;   // per-row fast path: o = e_max - (2^x - 1) <= 127
    for (bool more = true; more;) {
        const int te = u.e, tg = u.g, tc = u.c;
        const bool ok = u.g < u.G;
        uint32_t raw[TW];
#pragma unroll
        for (int q = 0; q < TW; ++q) raw[q] = nxt[q];
        const uint2 em = nm;
        more = grp_next<NH, GRP_DTILE, GRP_DEC_BAR != 0>(u, tab, sb, n, nchunks, wstride);
        if (more && u.g < u.G) grp_dec_load<K, NH, PR>(tab, u, nxt, nm);
        if (!PR && te != cur) {
            cur = te;
            F = load_fmt(x, y, tab[cur].meta);
            P = make_fast(F, false, 0);
        }
        if (!ok) continue;
        uint8_t *out = tab[te].out;
        const int64_t C = tab[te].cols;
        if (PR) {
            bool tfast = MODE == DEC_FAST;
#pragma unroll
            for (int i = 0; i < 8; ++i) tfast = tfast && tile_row_meta(em, i) <= omax;
            if (tfast) grp_dec_tile_r<K, OBF16, NH, false>(raw, out, C, tg, tc, x, y, em);
            else grp_dec_tile_r<K, OBF16, NH, true>(raw, out, C, tg, tc, x, y, em);
        } else if (MODE == DEC_FAST && P.two_mul) {
            grp_dec_tile<K, OBF16, DEC_FAST2, NH>(raw, out, C, tg, tc, F, P);
        } else {
            grp_dec_tile<K, OBF16, MODE, NH>(raw, out, C, tg, tc, F, P);
        }
    }
}

// ------------------------------------------------ fused per-row max + encode
// Per-row plans, entries whose rows fit the staging limit (`fused`): one CTA
// per row group at a time, the rows staged in shared memory by bulk async
// copies, row maxima and encode from shared memory (rws_row_group,
// exmy_blocked.cuh): each such tensor is read from HBM once.  Units are row
// groups numbered across the fused entries (frg_begin).
__host__ __device__ inline size_t grws_tab_bytes(int n) { return (grp_smem_bytes(n) + 15) & ~(size_t)15; }

template <int K, bool BF16, int MODE>
__global__ void __launch_bounds__(RWS_THREADS) k_grouped_rowwise_smem(const GroupEntry *__restrict__ tab, int n,
                                                                     int64_t nunits, int x, int y,
                                                                     int force_generic) {
    extern __shared__ __align__(16) uint8_t grws_sm[];   // [table begins][8 staged rows]
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ uint32_t s_m[RWS_THREADS / 32][8];
    __shared__ int s_e[8];
    const int64_t *sb = grp_stage<GRP_FRG>(tab, n, reinterpret_cast<int64_t *>(grws_sm));
    uint8_t *buf = grws_sm + grws_tab_bytes(n);
    const FastP P = make_fast(fmt_of(x, y, 0), BF16, 1);
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(buf);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    int e = -1;
    for (int64_t unit = blockIdx.x; unit < nunits; unit += gridDim.x, phase ^= 1u) {
        e = e < 0 ? grp_find<GRP_FRG>(tab, sb, n, unit) : grp_advance<GRP_FRG>(tab, sb, n, e, unit);
        const GroupEntry &E = tab[e];
        rws_row_group<K, BF16, MODE>(E.in, E.cols, unit - grp_b<GRP_FRG>(tab, sb, e), x, y, 0, E.meta, E.packed,
                                     grp_so<K>(E.rows * E.cols), E.spi, E.spb, E.spc, E.cap, force_generic, P, buf,
                                     sbase, bar, phase, s_m, s_e);
    }
}

// ------------------------------------------------ specials (D9) per entry
__global__ void __launch_bounds__(1024) k_grouped_sort(const GroupEntry *__restrict__ tab, int n) {
    __shared__ long long sk[SORT_SMEM];
    __shared__ uint32_t sv[SORT_SMEM];
    for (int e = blockIdx.x; e < n; e += gridDim.x) {
        const GroupEntry &E = tab[e];
        if (!E.spc || E.cap <= 1) continue;
        const long long cnt = (long long)min((unsigned long long)E.cap, *E.spc);
        if (cnt <= 1) continue;
        if (cnt <= SORT_SMEM) {
            for (long long i = threadIdx.x; i < cnt; i += blockDim.x) { sk[i] = E.spi[i]; sv[i] = E.spb[i]; }
            __syncthreads();
            flip_bitonic(sk, sv, cnt);
            for (long long i = threadIdx.x; i < cnt; i += blockDim.x) { E.spi[i] = sk[i]; E.spb[i] = sv[i]; }
            __syncthreads();
        } else {
            flip_bitonic((volatile long long *)E.spi, (volatile uint32_t *)E.spb, cnt);
        }
    }
}

template <bool OBF16>
__global__ void k_grouped_scatter(const GroupEntry *__restrict__ tab, int n) {
    for (int e = blockIdx.x; e < n; e += gridDim.x) {
        const GroupEntry &E = tab[e];
        if (!E.spc || !E.spi || !E.spb || E.cap <= 0) continue;
        const long long cnt = (long long)min((unsigned long long)E.cap, *E.spc);
        for (long long i = threadIdx.x; i < cnt; i += blockDim.x) {
            const uint32_t u = E.spb[i];
            if (OBF16) {
                uint16_t b = (uint16_t)(u >> 16);
                if ((u & 0x7FFFFFu) != 0u && (b & 0x7Fu) == 0u) b |= 0x40u;   // keep NaN a NaN (D9)
                ((uint16_t *)E.out)[E.spi[i]] = b;
            } else {
                ((uint32_t *)E.out)[E.spi[i]] = u;
            }
        }
    }
}

}  // namespace exmy
