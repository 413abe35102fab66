// exmy_kernels.cuh -- sm_100a kernels of the eXmY codec (HBM-bound, no
// tensor cores: the path is elementwise bit manipulation).
//
//   K1  k_hist_*          exponent histogram
//   K1b k_emax            e_max = top populated bin
//   K2  k_quantize        fp -> grid -> fp emulation
//   K3  k_encode_rows / k_encode_cols / k_encode_generic
//                         type conversion + power-of-2 packing
//   K4  k_decode_rows / k_decode_cols / k_decode_generic
//   K5  k_specials_sort / k_specials_scatter   out-of-band NaN/Inf (D9)
#pragma once
#include <cooperative_groups.h>

#include "exmy_device.cuh"

namespace exmy {

struct SegOffsets { long long off[4]; };

template <bool BF16>
struct Elem {
    static constexpr int ES = BF16 ? 2 : 4;   // bytes per element
    static constexpr int V = 16 / ES;         // elements per 16-byte vector
};

// element v of a 16-byte vector as an fp32 bit pattern (bf16 widened exactly)
template <bool BF16>
__device__ __forceinline__ uint32_t vec_elem(const uint4 &r, int v) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    if (BF16) return (v & 1) ? (w[v >> 1] & 0xFFFF0000u) : (w[v >> 1] << 16);
    return w[v];
}

// Out-of-band NaN/Inf (D9).  The per-tensor encode kernels only COUNT them
// here (sp_index == NULL: one warp-aggregated atomic per call site and warp,
// not one per element) and the index-ordered list is written afterwards by
// k_specials_count + k_specials_write (deterministic stream compaction, no
// sort).  The grouped kernels pass their per-entry lists and append directly
// (then k_grouped_sort orders them).
__device__ __forceinline__ void push_special(int64_t idx, uint32_t bits, int64_t *sp_index,
                                             uint32_t *sp_bits, unsigned long long *sp_count,
                                             int64_t cap) {
    if (!sp_count) return;
    if (!sp_index) {
        const unsigned m = __activemask();
        const int lane = threadIdx.x & 31;
        if (lane == __ffs(m) - 1) atomicAdd(sp_count, (unsigned long long)__popc(m));
        return;
    }
    unsigned long long slot = atomicAdd(sp_count, 1ull);
    if ((long long)slot < cap) {
        sp_index[slot] = idx;
        sp_bits[slot] = bits;
    }
}

// code of one element, recording a special if needed
__device__ __forceinline__ uint32_t enc_elem(uint32_t u, const Fmt &F, int64_t idx, int64_t *sp_index,
                                             uint32_t *sp_bits, unsigned long long *sp_count, int64_t cap) {
    if (is_special_f32(u)) {
        push_special(idx, u, sp_index, sp_bits, sp_count, cap);
        return 0u;
    }
    return enc_code_generic(u, F);
}

// ------------------------------------------------------------- K1 hist
// Modes 0-3 (A/B; the default is MODE 4, k_hist_cta below): lane-private
// counters -- warp w, lane l owns 16-bit counters for bins (2*word,
// 2*word+1) in shared word [w][word][l] (bank = lane, no conflicts, no
// atomics).  Counters are flushed before they can overflow.
constexpr int HIST_THREADS = 128;
constexpr int HIST_WARPS = HIST_THREADS / 32;
constexpr int HIST_WORDS_PER_WARP = 128 * 32;                 // 128 words x 32 lanes
constexpr int HIST_SMEM = HIST_WARPS * HIST_WORDS_PER_WARP * 4;  // 64 KB

__device__ __forceinline__ void hist_bump(uint32_t *lanebase, uint32_t b, int mode) {
    // lanebase = &sh[warp][0][lane]; word stride 32 words = 128 bytes
    uint32_t *p = lanebase + ((b >> 1) << 5);
    uint32_t inc = 1u << ((b & 1u) << 4);
    if (mode == 0) {
        *p += inc;
    } else {
        atomicAdd(p, inc);
    }
}

// flush this warp's counters into global hist and zero them
__device__ __forceinline__ void hist_flush_warp(uint32_t *warpbase, int lane, unsigned long long *hist) {
    __syncwarp();
#pragma unroll 1
    for (int wd = lane; wd < 128; wd += 32) {
        uint32_t lo = 0, hi = 0;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) {
            uint32_t v = warpbase[wd * 32 + l];
            lo += v & 0xFFFFu;
            hi += v >> 16;
        }
        if (lo) atomicAdd(hist + 2 * wd, (unsigned long long)lo);
        if (hi) atomicAdd(hist + 2 * wd + 1, (unsigned long long)hi);
    }
    __syncwarp();
    for (int i = lane; i < HIST_WORDS_PER_WARP; i += 32) warpbase[i] = 0;
    __syncwarp();
}

// MODE 2: both counter-word offsets of a bf16 pair from one shift + mask
// (16-bit lanes: ((w >> 1) & 0x3F803F80) = (bin >> 1) * 128 bytes for both
// elements), the increments from the exponent LSBs by select, and
// red.shared on 32-bit shared addresses: 5.5 instead of 7 ops / element.
__device__ __forceinline__ void red_shared_add(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

#ifndef HIST_U
#define HIST_U 12   // 16-byte vectors per lane per iteration, double-buffered: 12 warps/SM (64 KB of
                    // counters per 4 warps) need ~2x12 vectors in flight per lane to cover HBM latency
                    // (config 2 bf16: U=4 114.0 us, 8 105.2, 12 103.1; fp32 200.9 -> 156.6 us)
#endif
// MODE 3 (default until MODE 4, k_hist_cta, below): LANE-PAIR counters.  Lanes 2j and 2j+1 share the 32-bit
// word [bin][j] of their warp's 16 KB (256 bins x 16 words), lane 2j counting
// in the low half and 2j+1 in the high half, so each lane's increment is a
// constant (1 or 0x10000) and an element costs only the bin's byte offset
// (bin * 64: one shift + mask, both bf16 elements of a word at once) and
// its reduction -- MODE 2 spent two more ALU ops per element choosing the
// half by the exponent's LSB and was ALU-bound (ncu: ALU pipe 78 %, issue
// 65 %).  The price: the two lanes of a pair hit the same bank when their
// bins have equal parity (at most 2-way).  Counters stay lane-private, so
// the 16-bit epochs and flushes are MODE 2's.
__device__ __forceinline__ void hist3_flush_warp(uint32_t *warpbase, int lane, unsigned long long *hist) {
    __syncwarp();
#pragma unroll 1
    for (int b = lane; b < 256; b += 32) {
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t v = warpbase[b * 16 + j];
            c += (v & 0xFFFFu) + (v >> 16);
        }
        if (c) atomicAdd(hist + b, (unsigned long long)c);
    }
    __syncwarp();
    for (int i = lane; i < HIST_WORDS_PER_WARP; i += 32) warpbase[i] = 0;
    __syncwarp();
}

template <bool BF16, int MODE>
__global__ void __launch_bounds__(HIST_THREADS) k_hist(const uint8_t *__restrict__ in, int64_t n,
                                                       unsigned long long *__restrict__ hist) {
    extern __shared__ uint32_t hsm[];
    using EL = Elem<BF16>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *warpbase = hsm + warp * HIST_WORDS_PER_WARP;
    uint32_t *lanebase = warpbase + lane;
    // MODE 3: this lane's word of each bin row and its constant half increment
    const uint32_t lane_sa = MODE == 3 ? (uint32_t)__cvta_generic_to_shared(warpbase + (lane >> 1))
                                       : (uint32_t)__cvta_generic_to_shared(lanebase);   // shared-window byte address
    const uint32_t inc3 = (lane & 1) ? 0x10000u : 1u;
    for (int i = threadIdx.x; i < HIST_WARPS * HIST_WORDS_PER_WARP; i += HIST_THREADS) hsm[i] = 0;
    __syncthreads();

    const int64_t nvec = n / EL::V;
    const int64_t warps_total = (int64_t)gridDim.x * HIST_WARPS;
    const int64_t gw = (int64_t)blockIdx.x * HIST_WARPS + warp;
    // each lane may count at most 65535 elements between flushes
    constexpr int64_t EPOCH_VECS = (BF16 ? 8000 : 16000) / HIST_U;   // per lane, in units of HIST_U vectors
    int64_t epoch = 0;
    // warp-uniform loop: iteration t covers vectors (gw + t*warps_total)*32U + 32*u + lane.
    // Loads are double-buffered: the next iteration's U vectors are in flight
    // while this iteration's 8U (bf16) elements update the counters.
    constexpr int U = HIST_U;
    const int64_t step = warps_total * 32 * U;
    uint4 nxt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t vi = gw * 32 * U + 32 * u + lane;
        nxt[u] = vi < nvec ? ldg_nc_v4(in + vi * 16) : make_uint4(0, 0, 0, 0);
    }
    for (int64_t base = gw * 32 * U; base < nvec; base += step) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            r[u] = nxt[u];
            const int64_t vi = base + step + 32 * u + lane;
            nxt[u] = vi < nvec ? ldg_nc_v4(in + vi * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + 32 * u + lane < nvec) {
                const uint32_t w[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (MODE == 3) {
                        if (BF16) {   // both elements' bin * 64 from one shift + mask
                            const uint32_t off = (w[q] >> 1) & 0x3FC03FC0u;
                            red_shared_add(lane_sa + (off & 0xFFFFu), inc3);
                            red_shared_add(lane_sa + (off >> 16), inc3);
                        } else {
                            red_shared_add(lane_sa + ((w[q] >> 17) & 0x3FC0u), inc3);
                        }
                    } else if (BF16 && MODE == 2) {
                        const uint32_t off = (w[q] >> 1) & 0x3F803F80u;   // both elements' word offsets (bytes)
                        const uint32_t inc_lo = (w[q] & 0x80u) ? 0x10000u : 1u;
                        const uint32_t inc_hi = (w[q] & 0x800000u) ? 0x10000u : 1u;
                        red_shared_add(lane_sa + (off & 0xFFFFu), inc_lo);
                        red_shared_add(lane_sa + (off >> 16), inc_hi);
                    } else if (BF16) {
                        hist_bump(lanebase, (w[q] >> 7) & 0xFFu, MODE);
                        hist_bump(lanebase, (w[q] >> 23) & 0xFFu, MODE);
                    } else if (MODE == 2) {
                        const uint32_t wq = w[q];
                        red_shared_add(lane_sa + ((wq >> 17) & 0x3F80u), (wq & 0x800000u) ? 0x10000u : 1u);
                    } else {
                        hist_bump(lanebase, (w[q] >> 23) & 0xFFu, MODE);
                    }
                }
            }
        }
        if (++epoch == EPOCH_VECS) {
            if (MODE == 3) hist3_flush_warp(warpbase, lane, hist);
            else hist_flush_warp(warpbase, lane, hist);
            epoch = 0;
        }
    }
    // scalar tail (n % V elements), block 0 warp 0
    if (blockIdx.x == 0 && warp == 0) {
        int64_t t0 = nvec * EL::V;
        for (int64_t i = t0 + lane; i < n; i += 32) {
            uint32_t u = BF16 ? ((uint32_t)((const uint16_t *)in)[i] << 16) : ((const uint32_t *)in)[i];
            if (MODE == 3) atomicAdd(warpbase + ((u >> 23) & 0xFFu) * 16 + (lane >> 1), inc3);
            else hist_bump(lanebase, (u >> 23) & 0xFFu, 1);
        }
    }
    __syncthreads();
    // block-level reduction: thread t owns bins t and t+128
    for (int b = threadIdx.x; b < 256; b += HIST_THREADS) {
        unsigned long long s = 0;
        if (MODE == 3) {
            for (int w = 0; w < HIST_WARPS; ++w)
                for (int j = 0; j < 16; ++j) {
                    const uint32_t v = hsm[w * HIST_WORDS_PER_WARP + b * 16 + j];
                    s += (v & 0xFFFFu) + (v >> 16);
                }
        } else {
            const uint32_t wd = b >> 1, sh = (b & 1) << 4;
            for (int w = 0; w < HIST_WARPS; ++w)
                for (int l = 0; l < 32; ++l) s += (hsm[w * HIST_WORDS_PER_WARP + wd * 32 + l] >> sh) & 0xFFFFu;
        }
        if (s) atomicAdd(hist + b, s);
    }
}

// MODE 4: ONE counter table per CTA, a column per lane.  Bank conflicts
// only arise between the lanes of one instruction, so every warp of the CTA
// can share one 256-bin x 32-lane table of 32-bit counters: lane l always
// hits bank l (conflict-free, one wavefront per reduction; MODE 3's lane
// pairs cost 2.3 wavefronts each and saturated the shared-memory pipe), the
// increment is the constant 1, and a CTA's table is 32 KB however many
// warps it runs.  The table sits on a 32 KB-aligned shared address, so an
// element's counter address is one LOP3, (bits & 0x7F80) | lane_address,
// for the low bf16 element (two ops for the high one / fp32).  32-bit
// counters: the launcher keeps a CTA's share under 2^32 elements.
constexpr int HIST4_THREADS = 256;
constexpr int HIST4_SMEM = 64 * 1024;   // 32 KB table + its alignment slack

__device__ __forceinline__ void st_shared_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

template <bool BF16, int U>
__global__ void __launch_bounds__(HIST4_THREADS, 3) k_hist_cta(const uint8_t *__restrict__ in, int64_t n,
                                                               unsigned long long *__restrict__ hist) {
    extern __shared__ uint32_t hsm[];
    using EL = Elem<BF16>;
    constexpr int NWARP = HIST4_THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tab = ((uint32_t)__cvta_generic_to_shared(hsm) + 32767u) & ~32767u;
    const uint32_t lsa = tab + 4u * (uint32_t)lane;
    const int64_t nvec = n / EL::V;
    const int64_t warps_total = (int64_t)gridDim.x * NWARP;
    const int64_t gw = (int64_t)blockIdx.x * NWARP + warp;
    const int64_t step = warps_total * 32 * U;
    uint4 nxt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t vi = gw * 32 * U + 32 * u + lane;
        nxt[u] = vi < nvec ? ldg_nc_v4(in + vi * 16) : make_uint4(0, 0, 0, 0);
    }
    // zero the table while the first loads are in flight
    for (int i = threadIdx.x; i < 256 * 32; i += HIST4_THREADS) st_shared_u32(tab + 4u * (uint32_t)i, 0u);
    __syncthreads();
    for (int64_t base = gw * 32 * U; base < nvec; base += step) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            r[u] = nxt[u];
            const int64_t vi = base + step + 32 * u + lane;
            nxt[u] = vi < nvec ? ldg_nc_v4(in + vi * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + 32 * u + lane < nvec) {
                const uint32_t w[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (BF16) red_shared_add((w[q] & 0x7F80u) | lsa, 1u);
                    red_shared_add(((w[q] >> 16) & 0x7F80u) | lsa, 1u);
                }
            }
        }
    }
    // scalar tail (n % V elements), block 0 warp 0
    if (blockIdx.x == 0 && warp == 0) {
        for (int64_t i = nvec * EL::V + lane; i < n; i += 32) {
            const uint32_t u = BF16 ? ((uint32_t)((const uint16_t *)in)[i] << 16) : ((const uint32_t *)in)[i];
            red_shared_add(((u >> 16) & 0x7F80u) | lsa, 1u);
        }
    }
    __syncthreads();
    // bin b = row b: 32 consecutive words, one warp-wide add
    for (int b = warp; b < 256; b += NWARP) {
        const uint32_t c = __reduce_add_sync(0xFFFFFFFFu, ld_shared_u32(tab + 128u * (uint32_t)b + 4u * (uint32_t)lane));
        if (lane == 0 && c) atomicAdd(hist + b, (unsigned long long)c);
    }
}

// misaligned input: plain grid-stride loop with global atomics per warp bin
template <bool BF16>
__global__ void k_hist_scalar(const uint8_t *__restrict__ in, int64_t n, unsigned long long *__restrict__ hist) {
    __shared__ unsigned int sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t u;
        if (BF16) {
            uint16_t b;
            memcpy(&b, in + 2 * i, 2);
            u = (uint32_t)b << 16;
        } else {
            memcpy(&u, in + 4 * i, 4);
        }
        atomicAdd(&sh[(u >> 23) & 0xFFu], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, (unsigned long long)sh[i]);
}

// ------------------------------------------------------------- K1b emax
static __global__ void k_emax(const unsigned long long *__restrict__ hist, uint8_t *__restrict__ meta) {
    __shared__ int wmax[8];
    int t = threadIdx.x;   // 256 threads
    int cand = (t < 255 && hist[t] != 0ull) ? t : 0;
    cand = __reduce_max_sync(0xFFFFFFFFu, (unsigned)cand);
    if ((t & 31) == 0) wmax[t >> 5] = cand;
    __syncthreads();
    if (t == 0) {
        int m = 0;
        for (int i = 0; i < 8; ++i) m = max(m, wmax[i]);
        *meta = (uint8_t)m;
    }
}

// ------------------------------------------------------- value helpers
struct DecPath {
    bool fast_f32;    // x <= 7
    bool fast_bf16;   // x <= 7 and the grid is fp32-exact
    DecScale ds;
};

__device__ __forceinline__ DecPath make_dec_path(const Fmt &F, int force_generic) {
    DecPath p;
    p.fast_f32 = !force_generic && F.x <= 7;
    p.fast_bf16 = p.fast_f32 && (F.e_max + 24 >= (1 << F.x) + F.y);
    p.ds = make_dec_scale(F);
    return p;
}

// code -> fp32 bits
__device__ __forceinline__ uint32_t code_to_f32(uint32_t code, const Fmt &F, const DecPath &P) {
    if (P.fast_f32) {
        uint32_t s = (code >> (F.x + F.y)) & 1u;
        return dec_mag_fast_f32(code & F.M, F.y, P.ds) | (s << 31);
    }
    return dec_code_generic<24>(code, F);
}
// code -> bf16 bits (low 16)
__device__ __forceinline__ uint32_t code_to_bf16(uint32_t code, const Fmt &F, const DecPath &P) {
    if (P.fast_bf16) {
        uint32_t s = (code >> (F.x + F.y)) & 1u;
        float f = __uint_as_float(dec_mag_fast_f32(code & F.M, F.y, P.ds));
        uint16_t h;
        asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(f));
        return (uint32_t)h | (s << 15);
    }
    return dec_code_generic<8>(code, F);
}

// ------------------------------------------------------------ K2 quantize
template <bool BF16>
__device__ __forceinline__ uint32_t quantize_elem(uint32_t u, const Fmt &F, const DecPath &P) {
    // u: fp32 pattern (bf16 widened); returns fp32 bits or bf16 bits
    if (is_special_f32(u)) return BF16 ? (u >> 16) : u;
    uint32_t code = enc_code_generic(u, F);
    return BF16 ? code_to_bf16(code, F, P) : code_to_f32(code, F, P);
}

template <bool BF16>
__global__ void __launch_bounds__(256) k_quantize(const uint8_t *__restrict__ in, uint8_t *__restrict__ out,
                                                  int64_t n, int x, int y, const uint8_t *__restrict__ meta,
                                                  int force_generic) {
    using EL = Elem<BF16>;
    const Fmt F = load_fmt(x, y, meta);
    const DecPath P = make_dec_path(F, force_generic);
    const int64_t nvec = n / EL::V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    constexpr int U = 4;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < nvec; base += stride * U) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int64_t vi = base + u * stride;
            if (vi < nvec) r[u] = ldg_nc_v4(in + vi * 16);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int64_t vi = base + u * stride;
            if (vi < nvec) {
                uint32_t o[4];
                if (BF16) {
                    const uint32_t w[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t lo = quantize_elem<true>(w[q] << 16, F, P);
                        uint32_t hi = quantize_elem<true>(w[q] & 0xFFFF0000u, F, P);
                        o[q] = (lo & 0xFFFFu) | (hi << 16);
                    }
                } else {
                    o[0] = quantize_elem<false>(r[u].x, F, P);
                    o[1] = quantize_elem<false>(r[u].y, F, P);
                    o[2] = quantize_elem<false>(r[u].z, F, P);
                    o[3] = quantize_elem<false>(r[u].w, F, P);
                }
                stg_v4(out + vi * 16, make_uint4(o[0], o[1], o[2], o[3]));
            }
        }
    }
    if (blockIdx.x == 0) {
        for (int64_t i = nvec * EL::V + threadIdx.x; i < n; i += blockDim.x) {
            if (BF16) {
                uint32_t u = (uint32_t)((const uint16_t *)in)[i] << 16;
                ((uint16_t *)out)[i] = (uint16_t)quantize_elem<true>(u, F, P);
            } else {
                ((uint32_t *)out)[i] = quantize_elem<false>(((const uint32_t *)in)[i], F, P);
            }
        }
    }
}

// unaligned quantize: scalar
template <bool BF16>
__global__ void k_quantize_scalar(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, int64_t n, int x,
                                  int y, const uint8_t *__restrict__ meta, int force_generic) {
    const Fmt F = load_fmt(x, y, meta);
    const DecPath P = make_dec_path(F, force_generic);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (BF16) {
            uint16_t b;
            memcpy(&b, in + 2 * i, 2);
            uint16_t o = (uint16_t)quantize_elem<true>((uint32_t)b << 16, F, P);
            memcpy(out + 2 * i, &o, 2);
        } else {
            uint32_t u;
            memcpy(&u, in + 4 * i, 4);
            uint32_t o = quantize_elem<false>(u, F, P);
            memcpy(out + 4 * i, &o, 4);
        }
    }
}

// ---------------------------------------------------------- store helpers
template <int NW>
__device__ __forceinline__ void store_words(uint8_t *p, const uint32_t (&w)[NW]) {
    if constexpr (NW == 1) {
        *(uint32_t *)p = w[0];
    } else if constexpr (NW == 2) {
        stg_v2(p, w[0], w[1]);
    } else if constexpr (NW == 4) {
        stg_v4(p, make_uint4(w[0], w[1], w[2], w[3]));
    } else {
        static_assert(NW == 8, "");
        stg_v4(p, make_uint4(w[0], w[1], w[2], w[3]));
        stg_v4(p + 16, make_uint4(w[4], w[5], w[6], w[7]));
    }
}

template <int NW>
__device__ __forceinline__ void load_words(const uint8_t *p, uint32_t (&w)[NW]) {
    if constexpr (NW == 1) {
        w[0] = __ldg((const unsigned int *)p);
    } else if constexpr (NW == 2) {
        uint2 t = __ldg((const uint2 *)p);
        w[0] = t.x; w[1] = t.y;
    } else if constexpr (NW == 4) {
        uint4 t = ldg_nc_v4(p);
        w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
    } else {
        static_assert(NW == 8, "");
        uint4 t = ldg_nc_v4(p), s = ldg_nc_v4(p + 16);
        w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
        w[4] = s.x; w[5] = s.y; w[6] = s.z; w[7] = s.w;
    }
}

// V containers of width W (bytes) -> words; V*W bytes total
template <int W, int V>
__device__ __forceinline__ void containers_to_words(const uint32_t (&cont)[V], uint32_t (&w)[(V * W) / 4]) {
    if constexpr (W == 4) {
#pragma unroll
        for (int v = 0; v < V; ++v) w[v] = cont[v];
    } else if constexpr (W == 2) {
#pragma unroll
        for (int t = 0; t < V / 2; ++t) w[t] = cont[2 * t] | (cont[2 * t + 1] << 16);
    } else {
#pragma unroll
        for (int t = 0; t < V / 4; ++t)
            w[t] = cont[4 * t] | (cont[4 * t + 1] << 8) | (cont[4 * t + 2] << 16) | (cont[4 * t + 3] << 24);
    }
}

template <int W, int V>
__device__ __forceinline__ void words_to_containers(const uint32_t (&w)[(V * W) / 4], uint32_t (&cont)[V]) {
    if constexpr (W == 4) {
#pragma unroll
        for (int v = 0; v < V; ++v) cont[v] = w[v];
    } else if constexpr (W == 2) {
#pragma unroll
        for (int t = 0; t < V / 2; ++t) { cont[2 * t] = w[t] & 0xFFFFu; cont[2 * t + 1] = w[t] >> 16; }
    } else {
#pragma unroll
        for (int t = 0; t < V / 4; ++t) {
            cont[4 * t] = w[t] & 0xFFu; cont[4 * t + 1] = (w[t] >> 8) & 0xFFu;
            cont[4 * t + 2] = (w[t] >> 16) & 0xFFu; cont[4 * t + 3] = w[t] >> 24;
        }
    }
}

// ------------------------------------------------------- K3 encode ROWS
// Thread tile: 8 rows (one row group g) x V adjacent columns; one 16-byte
// load per row; per segment V containers = V*w contiguous bytes (Fig. 3:
// (8R, C) -> (R, C) per segment).
template <int K, bool BF16, int S>
__device__ __forceinline__ void rows_store_segments(const uint32_t (&c)[8][Elem<BF16>::V], uint8_t *packed,
                                                    const SegOffsets &so, int64_t g, int64_t C, int64_t c0) {
    if constexpr (S < seg_count(K)) {
        constexpr int V = Elem<BF16>::V;
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S);
        uint8_t *seg = packed + so.off[S];
        if constexpr (W == 8) {          // D15 passthrough: row-major bytes
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                uint32_t w[V / 4];
#pragma unroll
                for (int t = 0; t < V / 4; ++t)
                    w[t] = ((c[i][4 * t] >> LO) & 0xFFu) | (((c[i][4 * t + 1] >> LO) & 0xFFu) << 8) |
                           (((c[i][4 * t + 2] >> LO) & 0xFFu) << 16) | (((c[i][4 * t + 3] >> LO) & 0xFFu) << 24);
                store_words<V / 4>(seg + (8 * g + i) * C + c0, w);
            }
        } else {
            uint32_t cont[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                uint32_t col[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) col[i] = c[i][v];
                cont[v] = pack8<W, LO>(col);
            }
            uint32_t w[(V * W) / 4];
            containers_to_words<W, V>(cont, w);
            store_words<(V * W) / 4>(seg + (g * C + c0) * W, w);
        }
        rows_store_segments<K, BF16, S + 1>(c, packed, so, g, C, c0);
    }
}

template <int K, bool BF16>
__global__ void __launch_bounds__(256) k_encode_rows(const uint8_t *__restrict__ in, int64_t R, int64_t C, int x,
                                                     int y, const uint8_t *__restrict__ meta,
                                                     uint8_t *__restrict__ packed, SegOffsets so,
                                                     int64_t *sp_index, uint32_t *sp_bits,
                                                     unsigned long long *sp_count, int64_t cap) {
    using EL = Elem<BF16>;
    constexpr int V = EL::V;
    const Fmt F = load_fmt(x, y, meta);
    const int64_t CV = C / V, G = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= CV) return;
    const int64_t c0 = j * V;
    for (int64_t g = blockIdx.y; g < G; g += gridDim.y) {
        uint4 r[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = ldg_nc_v4(in + ((8 * g + i) * C + c0) * EL::ES);
        uint32_t c[8][V];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int v = 0; v < V; ++v)
                c[i][v] = enc_elem(vec_elem<BF16>(r[i], v), F, (8 * g + i) * C + c0 + v, sp_index, sp_bits,
                                   sp_count, cap);
        rows_store_segments<K, BF16, 0>(c, packed, so, g, C, c0);
    }
}

// ------------------------------------------------------- K3 encode COLS
// COLS == flat groups of 8 consecutive row-major elements, container q.
// A warp tile is 128 groups; lane l handles groups l, l+32, l+64, l+96 so
// every load instruction is a contiguous 512 B (bf16) run and every
// container store a contiguous 32*w B run.
template <int K, bool BF16, int S>
__device__ __forceinline__ void cols_store_segment(const uint32_t (&c)[8], uint8_t *packed, const SegOffsets &so,
                                                   int64_t q) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S);
        uint8_t *seg = packed + so.off[S];
        if constexpr (W == 8) {
            uint32_t a = 0, b = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                a |= ((c[i] >> LO) & 0xFFu) << (8 * i);
                b |= ((c[i + 4] >> LO) & 0xFFu) << (8 * i);
            }
            stg_v2(seg + 8 * q, a, b);
        } else {
            uint32_t cont = pack8<W, LO>(c);
            if constexpr (W == 4) *(uint32_t *)(seg + 4 * q) = cont;
            else if constexpr (W == 2) *(uint16_t *)(seg + 2 * q) = (uint16_t)cont;
            else seg[q] = (uint8_t)cont;
        }
        cols_store_segment<K, BF16, S + 1>(c, packed, so, q);
    }
}

template <int K, bool BF16>
__global__ void __launch_bounds__(256) k_encode_cols(const uint8_t *__restrict__ in, int64_t n, int x, int y,
                                                     const uint8_t *__restrict__ meta, uint8_t *__restrict__ packed,
                                                     SegOffsets so, int64_t *sp_index, uint32_t *sp_bits,
                                                     unsigned long long *sp_count, int64_t cap) {
    using EL = Elem<BF16>;
    constexpr int NV = BF16 ? 1 : 2;   // 16-byte vectors per group
    const Fmt F = load_fmt(x, y, meta);
    const int64_t NG = n / 8;
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int64_t base = gw * 128; base < NG; base += warps_total * 128) {
        uint4 r[4][NV];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int64_t q = base + 32 * u + lane;
            if (q < NG) {
#pragma unroll
                for (int t = 0; t < NV; ++t) r[u][t] = ldg_nc_v4(in + q * 8 * EL::ES + 16 * t);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int64_t q = base + 32 * u + lane;
            if (q < NG) {
                uint32_t c[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    c[i] = enc_elem(vec_elem<BF16>(r[u][i / EL::V], i % EL::V), F, 8 * q + i, sp_index, sp_bits,
                                    sp_count, cap);
                cols_store_segment<K, BF16, 0>(c, packed, so, q);
            }
        }
    }
}

// ---------------------------------------------------- K3 encode generic
// Any alignment, any C (ROWS) -- one thread per container, scalar bytes.
__device__ __forceinline__ int64_t lane_elem(int64_t idx, int i, int64_t C, int axis) {
    if (axis == 0) {
        int64_t g = idx / C, c = idx - g * C;
        return (8 * g + i) * C + c;
    }
    return idx * 8 + i;   // COLS: groups of 8 consecutive row-major elements
}

template <bool BF16>
__device__ __forceinline__ uint32_t load_elem_scalar(const uint8_t *in, int64_t e) {
    if (BF16) {
        uint16_t b;
        memcpy(&b, in + 2 * e, 2);
        return (uint32_t)b << 16;
    }
    uint32_t u;
    memcpy(&u, in + 4 * e, 4);
    return u;
}

template <bool BF16>
__global__ void k_encode_generic(const uint8_t *__restrict__ in, int64_t C, int64_t ncont, int axis, int x, int y,
                                 const uint8_t *__restrict__ meta, uint8_t *__restrict__ packed, SegOffsets so,
                                 int nseg, int4 widths, int64_t *sp_index, uint32_t *sp_bits,
                                 unsigned long long *sp_count, int64_t cap) {
    const Fmt F = load_fmt(x, y, meta);
    const int wd[4] = {widths.x, widths.y, widths.z, widths.w};
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < ncont;
         idx += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c[8];
        int64_t e[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            e[i] = lane_elem(idx, i, C, axis);
            c[i] = enc_elem(load_elem_scalar<BF16>(in, e[i]), F, e[i], sp_index, sp_bits, sp_count, cap);
        }
        int hi = 1 + x + y;
        for (int s = 0; s < nseg; ++s) {
            int w = wd[s], lo = hi - w;
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
}

// ------------------------------------------------------- K4 decode ROWS
template <int K, bool BF16, int S>
__device__ __forceinline__ void rows_load_segments(uint32_t (&c)[8][Elem<BF16>::V], const uint8_t *packed,
                                                   const SegOffsets &so, int64_t g, int64_t C, int64_t c0) {
    if constexpr (S < seg_count(K)) {
        constexpr int V = Elem<BF16>::V;
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S);
        const uint8_t *seg = packed + so.off[S];
        if constexpr (W == 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                uint32_t w[V / 4];
                load_words<V / 4>(seg + (8 * g + i) * C + c0, w);
#pragma unroll
                for (int v = 0; v < V; ++v) c[i][v] |= ((w[v >> 2] >> (8 * (v & 3))) & 0xFFu) << LO;
            }
        } else {
            uint32_t w[(V * W) / 4];
            load_words<(V * W) / 4>(seg + (g * C + c0) * W, w);
            uint32_t cont[V];
            words_to_containers<W, V>(w, cont);
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
                for (int i = 0; i < 8; ++i) c[i][v] |= ((cont[v] >> (W * i)) & ((1u << W) - 1u)) << LO;
        }
        rows_load_segments<K, BF16, S + 1>(c, packed, so, g, C, c0);
    }
}

// V codes -> one 16-byte output vector of out dtype (V = 16/ES of OUT dtype)
template <bool OBF16, int V>
__device__ __forceinline__ uint4 codes_to_vec(const uint32_t (&c)[V], const Fmt &F, const DecPath &P) {
    uint32_t o[4];
    if (OBF16) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            o[q] = code_to_bf16(c[2 * q], F, P) | (code_to_bf16(c[2 * q + 1], F, P) << 16);
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = code_to_f32(c[q], F, P);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

template <int K, bool OBF16>
__global__ void __launch_bounds__(256) k_decode_rows(const uint8_t *__restrict__ packed, int64_t R, int64_t C,
                                                     int x, int y, const uint8_t *__restrict__ meta,
                                                     SegOffsets so, uint8_t *__restrict__ out, int force_generic) {
    using EL = Elem<OBF16>;
    constexpr int V = EL::V;
    const Fmt F = load_fmt(x, y, meta);
    const DecPath P = make_dec_path(F, force_generic);
    const int64_t CV = C / V, G = R / 8;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= CV) return;
    const int64_t c0 = j * V;
    for (int64_t g = blockIdx.y; g < G; g += gridDim.y) {
        uint32_t c[8][V];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int v = 0; v < V; ++v) c[i][v] = 0;
        rows_load_segments<K, OBF16, 0>(c, packed, so, g, C, c0);
#pragma unroll
        for (int i = 0; i < 8; ++i) stg_v4(out + ((8 * g + i) * C + c0) * EL::ES, codes_to_vec<OBF16, V>(c[i], F, P));
    }
}

// ------------------------------------------------------- K4 decode COLS
template <int K, int S>
__device__ __forceinline__ void cols_load_segment(uint32_t (&c)[8], const uint8_t *packed, const SegOffsets &so,
                                                  int64_t q) {
    if constexpr (S < seg_count(K)) {
        constexpr int W = seg_width(K, S), LO = seg_lo(K, S);
        const uint8_t *seg = packed + so.off[S];
        if constexpr (W == 8) {
            uint2 t = __ldg((const uint2 *)(seg + 8 * q));
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                c[i] |= ((t.x >> (8 * i)) & 0xFFu) << LO;
                c[i + 4] |= ((t.y >> (8 * i)) & 0xFFu) << LO;
            }
        } else {
            uint32_t cont;
            if constexpr (W == 4) cont = __ldg((const unsigned int *)(seg + 4 * q));
            else if constexpr (W == 2) cont = __ldg((const unsigned short *)(seg + 2 * q));
            else cont = __ldg((const unsigned char *)(seg + q));
            unpack8<W, LO>(cont, c);
        }
        cols_load_segment<K, S + 1>(c, packed, so, q);
    }
}

template <int K, bool OBF16>
__global__ void __launch_bounds__(256) k_decode_cols(const uint8_t *__restrict__ packed, int64_t n, int x, int y,
                                                     const uint8_t *__restrict__ meta, SegOffsets so,
                                                     uint8_t *__restrict__ out, int force_generic) {
    const Fmt F = load_fmt(x, y, meta);
    const DecPath P = make_dec_path(F, force_generic);
    const int64_t NG = n / 8;
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int64_t base = gw * 128; base < NG; base += warps_total * 128) {
        uint32_t c[4][8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) c[u][i] = 0;
            int64_t q = base + 32 * u + lane;
            if (q < NG) cols_load_segment<K, 0>(c[u], packed, so, q);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int64_t q = base + 32 * u + lane;
            if (q < NG) {
                if (OBF16) {
                    stg_v4(out + q * 16, codes_to_vec<true, 8>(c[u], F, P));
                } else {
                    const uint32_t lo[4] = {c[u][0], c[u][1], c[u][2], c[u][3]};
                    const uint32_t hi[4] = {c[u][4], c[u][5], c[u][6], c[u][7]};
                    stg_v4(out + q * 32, codes_to_vec<false, 4>(lo, F, P));
                    stg_v4(out + q * 32 + 16, codes_to_vec<false, 4>(hi, F, P));
                }
            }
        }
    }
}

// ---------------------------------------------------- K4 decode generic
template <bool OBF16>
__global__ void k_decode_generic(const uint8_t *__restrict__ packed, int64_t C, int64_t ncont, int axis, int x,
                                 int y, const uint8_t *__restrict__ meta, SegOffsets so, int nseg, int4 widths,
                                 uint8_t *__restrict__ out, int force_generic) {
    const Fmt F = load_fmt(x, y, meta);
    const DecPath P = make_dec_path(F, force_generic);
    const int wd[4] = {widths.x, widths.y, widths.z, widths.w};
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < ncont;
         idx += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int64_t e[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) e[i] = lane_elem(idx, i, C, axis);
        int hi = 1 + x + y;
        for (int s = 0; s < nseg; ++s) {
            int w = wd[s], lo = hi - w;
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
            if (OBF16) {
                uint16_t h = (uint16_t)code_to_bf16(c[i], F, P);
                memcpy(out + 2 * e[i], &h, 2);
            } else {
                uint32_t v = code_to_f32(c[i], F, P);
                memcpy(out + 4 * e[i], &v, 4);
            }
        }
    }
}

// ----------------------------------------------------------- K5 specials
// Sort the (index, bits) pairs by index in place, one CTA.  "Flip" bitonic
// network: every compare-exchange is ascending, so the virtual +inf padding
// up to the next power of two never needs storage (pairs whose partner lies
// beyond cnt are skipped).  Shared memory for cnt <= SORT_SMEM, global
// memory otherwise (only pathological NaN/Inf-heavy tensors get there).
constexpr int SORT_SMEM = 4096;

template <typename KeyPtr, typename ValPtr>
__device__ __forceinline__ void flip_bitonic(KeyPtr key, ValPtr val, long long cnt) {
    long long np2 = 1;
    while (np2 < cnt) np2 <<= 1;
    for (long long kk = 2; kk <= np2; kk <<= 1) {
        for (long long jj = kk >> 1; jj > 0; jj >>= 1) {
            for (long long i = threadIdx.x; i < np2; i += blockDim.x) {
                long long l = (jj == (kk >> 1)) ? (i ^ (kk - 1)) : (i ^ jj);
                if (l > i && l < cnt) {
                    if (key[i] > key[l]) {
                        long long tk = key[i]; key[i] = key[l]; key[l] = tk;
                        uint32_t tv = val[i]; val[i] = val[l]; val[l] = tv;
                    }
                }
            }
            __syncthreads();
        }
    }
}

static __global__ void __launch_bounds__(1024) k_specials_sort(int64_t *idx, uint32_t *bits,
                                                        const unsigned long long *count, int64_t cap) {
    __shared__ long long sk[SORT_SMEM];
    __shared__ uint32_t sv[SORT_SMEM];
    const long long cnt = (long long)min((unsigned long long)cap, *count);
    if (cnt <= 1) return;
    if (cnt <= SORT_SMEM) {
        for (long long i = threadIdx.x; i < cnt; i += blockDim.x) { sk[i] = idx[i]; sv[i] = bits[i]; }
        __syncthreads();
        flip_bitonic(sk, sv, cnt);
        for (long long i = threadIdx.x; i < cnt; i += blockDim.x) { idx[i] = sk[i]; bits[i] = sv[i]; }
        return;
    }
    flip_bitonic((volatile long long *)idx, (volatile uint32_t *)bits, cnt);
}

// ------------------------------------------- K5 ordered specials list
// Deterministic stream compaction of the NaN/Inf elements into (index,
// fp32 bits) in ascending index order, after an encode counted them in
// ws[0] (include/exmy.h: sp_count is a workspace of EXMY_SPECIALS_WORDS
// words).  The tensor is cut into nr <= SPECIALS_RANGES contiguous ranges of
// L elements (L % 8 == 0), one CTA each:
//   k_specials_count  ws[1 + b] := number of specials in range b
//   k_specials_write  CTA b writes its specials at positions
//                     sum_{j<b} ws[1+j] + (rank inside the range), the rank
//                     from a CTA-wide exclusive scan, only those < capacity.
// Both phases run in one cooperative launch (k_specials_compact) that returns
// at once when ws[0] == 0 (the usual case: no re-read), and a range whose
// first position is past the capacity is never re-read.
constexpr int SPECIALS_RANGES = 1024;

template <bool BF16>
__device__ __forceinline__ uint32_t elem_bits(const uint8_t *in, int64_t e) {
    return BF16 ? ((uint32_t)((const uint16_t *)in)[e] << 16) : ((const uint32_t *)in)[e];
}

// 8-bit mask of the specials among elements e .. e + 7 (all < n)
template <bool BF16>
__device__ __forceinline__ uint32_t special_mask8(const uint8_t *in, int64_t e, bool vec) {
    uint32_t m = 0;
    if (vec) {
        if (BF16) {
            const uint4 q = ldg_nc_v4(in + e * 2);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint32_t h = ((w[t] & 0x7F807F80u) + 0x00800080u) & 0x80008000u;   // bit 15 / 31: exponent 255
                m |= ((h >> 15) & 1u) << (2 * t) | ((h >> 31) & 1u) << (2 * t + 1);
            }
        } else {
            const uint4 a = ldg_nc_v4(in + e * 4), b = ldg_nc_v4(in + e * 4 + 16);
            const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int t = 0; t < 8; ++t) m |= (uint32_t)((w[t] & 0x7F800000u) == 0x7F800000u) << t;
        }
    } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) m |= (uint32_t)is_special_f32(elem_bits<BF16>(in, e + t)) << t;
    }
    return m;
}

// one cooperative launch of <= nr CTAs (grid-stride over the ranges):
// phase 1 counts every range, a grid-wide barrier, phase 2 writes.  With no
// NaN/Inf (ws[0] == 0) every CTA returns at once: a single short launch.
template <bool BF16>
__global__ void __launch_bounds__(256) k_specials_compact(const uint8_t *__restrict__ in, int64_t n, int64_t L,
                                                          int nr, int64_t elem_offset,
                                                          unsigned long long *__restrict__ ws,
                                                          int64_t *__restrict__ spi, uint32_t *__restrict__ spb,
                                                          int64_t cap) {
    if (ws[0] == 0ull) return;                       // uniform over the grid
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
    const bool vec = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    __shared__ uint32_t wsum[8];
    __shared__ unsigned long long s_prefix;
    // ---- phase 1: ws[1 + b] := specials in range b (already done by an encode fix-up pass: flag bit 1)
    const bool counted = (ws[1 + SPECIALS_RANGES] & 2ull) != 0ull;
    for (int b = counted ? nr : (int)blockIdx.x; b < nr; b += gridDim.x) {
        const int64_t e0 = (int64_t)b * L, e1 = min(n, e0 + L);
        uint32_t c = 0;
        const int64_t full = e0 + ((e1 - e0) / 8) * 8;
        for (int64_t e = e0 + 8 * (int64_t)threadIdx.x; e < full; e += 8 * (int64_t)blockDim.x)
            c += __popc(special_mask8<BF16>(in, e, vec));
        for (int64_t e = full + threadIdx.x; e < e1; e += blockDim.x) c += is_special_f32(elem_bits<BF16>(in, e));
        c = __reduce_add_sync(0xFFFFFFFFu, c);
        if (lane == 0) wsum[warp] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < nw; ++w) t += wsum[w];
            ws[1 + b] = t;
        }
        __syncthreads();
    }
    cooperative_groups::this_grid().sync();
    // ---- phase 2: each range's specials at sum_{j<b} ws[1+j] + rank, up to the capacity
    for (int b = blockIdx.x; b < nr; b += gridDim.x) {
        if (warp == 0) {
            unsigned long long p = 0;
            for (int j = lane; j < b; j += 32) p += ws[1 + j];
#pragma unroll
            for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(0xFFFFFFFFu, p, o);
            if (lane == 0) s_prefix = p;
        }
        __syncthreads();
        const unsigned long long prefix = s_prefix;
        __syncthreads();
        if ((long long)prefix >= cap) break;          // later ranges start even further on
        if (ws[1 + b] == 0ull) continue;
        const int64_t e0 = (int64_t)b * L, e1 = min(n, e0 + L);
        unsigned long long run = prefix;   // position of the chunk's first special
        for (int64_t c0 = e0; c0 < e1; c0 += 8 * (int64_t)blockDim.x) {
            const int64_t e = c0 + 8 * (int64_t)threadIdx.x;
            uint32_t m = 0;
            if (e + 8 <= e1) {
                m = special_mask8<BF16>(in, e, vec);
            } else {
                for (int t = 0; t < 8 && e + t < e1; ++t) m |= (uint32_t)is_special_f32(elem_bits<BF16>(in, e + t)) << t;
            }
            const uint32_t cnt = __popc(m);
            // CTA-wide exclusive scan of cnt (thread order = element order)
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += v;
            }
            if (lane == 31) wsum[warp] = incl;
            __syncthreads();
            uint32_t before = 0, total = 0;
            for (int w = 0; w < nw; ++w) {
                before += (w < warp) ? wsum[w] : 0u;
                total += wsum[w];
            }
            unsigned long long pos = run + before + (incl - cnt);
            while (m) {
                const int t = __ffs(m) - 1;
                m &= m - 1;
                if ((long long)pos < cap) {
                    spi[pos] = elem_offset + e + t;
                    spb[pos] = elem_bits<BF16>(in, e + t);
                }
                ++pos;
            }
            run += total;
            __syncthreads();   // wsum reuse
            if ((long long)run >= cap) break;
        }
    }
}

template <bool OBF16>
__global__ void k_specials_scatter(const int64_t *__restrict__ idx, const uint32_t *__restrict__ bits,
                                   const unsigned long long *__restrict__ count, int64_t cap, uint8_t *out) {
    const long long cnt = (long long)min((unsigned long long)cap, *count);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x) {
        uint32_t u = bits[i];
        if (OBF16) {
            uint16_t b = (uint16_t)(u >> 16);
            if ((u & 0x7FFFFFu) != 0u && (b & 0x7Fu) == 0u) b |= 0x40u;   // keep NaN a NaN (D9)
            ((uint16_t *)out)[idx[i]] = b;
        } else {
            ((uint32_t *)out)[idx[i]] = u;
        }
    }
}

}  // namespace exmy

namespace exmy {

// ------------------------------------------------- K1c tensor max exponent
// meta := max biased exponent field over the finite elements (= the top
// populated histogram bin in [0, 254]) without building the
// histogram: a read-only max reduction.  Grid-wide combination: each CTA
// raises the metadata byte with a compare-and-swap on its enclosing 32-bit
// word (other bytes preserved), skipped when the byte is already >= its max.
__device__ __forceinline__ void byte_atomic_max(uint8_t *p, uint32_t v) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    unsigned int *w = reinterpret_cast<unsigned int *>(a & ~uintptr_t(3));
    const int sh = (int)(a & 3) * 8;
    unsigned int old = *reinterpret_cast<volatile unsigned int *>(w);
    while (((old >> sh) & 0xFFu) < v) {
        const unsigned int nw = (old & ~(0xFFu << sh)) | (v << sh);
        const unsigned int prev = atomicCAS(w, old, nw);
        if (prev == old) break;
        old = prev;
    }
}

template <bool BF16>
__global__ void __launch_bounds__(256) k_max_exp(const uint8_t *__restrict__ in, int64_t n, uint8_t *meta) {
    using EL = Elem<BF16>;
    const int64_t nvec = n / EL::V;
    uint32_t amax = 0;   // bf16: 16-bit lanes of magnitudes; fp32: magnitude bits
    constexpr int U = 4;
    // a CTA reads one contiguous 16 KB chunk per iteration (4 coalesced
    // 16-byte loads per thread), chunks grid-strided: whole DRAM pages per CTA
    const int64_t chunk = (int64_t)blockDim.x * U;
    for (int64_t c0 = (int64_t)blockIdx.x * chunk; c0 < nvec; c0 += (int64_t)gridDim.x * chunk) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t vi = c0 + u * blockDim.x + threadIdx.x;
            r[u] = vi < nvec ? ldg_nc_v4(in + vi * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t w[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (BF16) {
                    // zero the NaN/Inf lanes (exponent 255), then lane-wise max
                    const uint32_t a2 = w[q] & 0x7FFF7FFFu;
                    const uint32_t sp = (a2 + 0x00800080u) & 0x80008000u;   // bit 15 of special lanes
                    const uint32_t keep = ~((sp >> 15) * 0xFFFFu);
                    uint32_t d;
                    asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(amax), "r"(a2 & keep));
                    amax = d;
                } else {
                    const uint32_t a = w[q] & 0x7FFFFFFFu;
                    amax = max(amax, a < 0x7F800000u ? a : 0u);
                }
            }
        }
    }
    if (blockIdx.x == 0) {   // tail elements
        for (int64_t i = nvec * EL::V + threadIdx.x; i < n; i += blockDim.x) {
            const uint32_t u = BF16 ? ((uint32_t)((const uint16_t *)in)[i] << 16) : ((const uint32_t *)in)[i];
            const uint32_t a = u & 0x7FFFFFFFu;
            if (a < 0x7F800000u) {
                if (BF16) {
                    uint32_t d;
                    asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(amax), "r"(a >> 16));
                    amax = d;
                } else {
                    amax = max(amax, a);
                }
            }
        }
    }
    // to an exponent: bf16 lanes -> fp32 convention
    uint32_t e = BF16 ? max((amax & 0xFFFFu) >> 7, amax >> 23) : (amax >> 23);
    e = __reduce_max_sync(0xFFFFFFFFu, e);
    __shared__ uint32_t wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t m = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = max(m, wm[i]);
        if (m > 254u) m = 254u;
        byte_atomic_max(meta, m);
    }
}

}  // namespace exmy
