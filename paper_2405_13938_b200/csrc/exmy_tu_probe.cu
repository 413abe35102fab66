// exmy_tu_probe.cu -- roofline probe ("% of a per-config
// roofline probe: a trivial kernel reading/writing the same bytes per
// element, e.g. read 2 B, write 0.875 B").  Not part of the codec: it
// streams in_bytes of reads and out_bytes of writes with the codec kernels'
// access shape (contiguous 16 KB input chunks per CTA iteration, 16-byte
// vectors, the chunk's share of the output written by the same CTA) and no
// arithmetic beyond an XOR, so its time is the HBM limit for that read:write
// mix on this part.
#include <cstdint>

#include "exmy_launch.cuh"

namespace exmy {
namespace {

constexpr int PROBE_THREADS = 256;
constexpr int PROBE_VECS = 4;                                     // input vectors per thread per chunk
constexpr int64_t PROBE_CHUNK = PROBE_THREADS * PROBE_VECS * 16;  // 16 KB of input per chunk

__global__ void __launch_bounds__(PROBE_THREADS) k_probe(const uint8_t *__restrict__ in, int64_t nchunks,
                                                         uint8_t *__restrict__ out, int64_t out_vecs) {
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        uint4 r[PROBE_VECS];
#pragma unroll
        for (int u = 0; u < PROBE_VECS; ++u)
            r[u] = ldg_nc_v4(in + ch * PROBE_CHUNK + ((int64_t)u * PROBE_THREADS + threadIdx.x) * 16);
        uint4 a = r[0];
#pragma unroll
        for (int u = 1; u < PROBE_VECS; ++u) {
            a.x ^= r[u].x; a.y ^= r[u].y; a.z ^= r[u].z; a.w ^= r[u].w;
        }
        // this chunk's share of the output: vectors [ch*V/N, (ch+1)*V/N)
        const int64_t v0 = ch * out_vecs / nchunks, v1 = (ch + 1) * out_vecs / nchunks;
        for (int64_t v = v0 + threadIdx.x; v < v1; v += PROBE_THREADS)
            stg_v4(out + v * 16, make_uint4(a.x ^ (uint32_t)v, a.y, a.z, a.w));
        __syncthreads();   // the codec kernels' one-contiguous-run-per-step shape
    }
}

}  // namespace
}  // namespace exmy

using namespace exmy;

extern "C" exmy_status exmy_debug_probe(const void *in, int64_t in_bytes, void *out, int64_t out_bytes,
                                        void *stream) {
    if (in_bytes <= 0 || in_bytes % PROBE_CHUNK || out_bytes < 0) return EXMY_E_SHAPE;
    const int64_t nchunks = in_bytes / PROBE_CHUNK;
    if (out_bytes % 16 || out_bytes / 16 > INT64_MAX / nchunks) return EXMY_E_SHAPE;
    if (!in || (out_bytes && !out)) return EXMY_E_ARG;
    if (!aligned(in, 16) || (out && !aligned(out, 16))) return EXMY_E_ALIGN;
    static int occ = 0;
    if (!occ) occ = occupancy(k_probe, PROBE_THREADS, 0);
    int64_t grid = (int64_t)num_sms() * occ;
    if (grid > nchunks) grid = nchunks;
    k_probe<<<(unsigned)grid, PROBE_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t *>(in), nchunks, static_cast<uint8_t *>(out), out_bytes / 16);
    return launch_status();
}
