// exmy_tu_quant.cu -- K2 quantize (emulation) launcher.
#include "exmy_launch.cuh"

namespace exmy {

exmy_status launch_quantize(const uint8_t *in, uint8_t *out, bool bf, int64_t n, int x, int y,
                            const uint8_t *meta, cudaStream_t st) {
    if (aligned(in, 16) && aligned(out, 16)) {
        const int64_t nvec = n / (bf ? 8 : 4);
        int64_t blocks = cdiv(cdiv(nvec, 4), 256);
        if (blocks < 1) blocks = 1;
        static int occ_b = 0, occ_f = 0;
        if (!occ_b) occ_b = occupancy(k_quant_fast<true>, 256, 0);
        if (!occ_f) occ_f = occupancy(k_quant_fast<false>, 256, 0);
        int64_t maxb = (int64_t)num_sms() * (bf ? occ_b : occ_f);
        if (blocks > maxb) blocks = maxb;
        if (bf) k_quant_fast<true><<<(unsigned)blocks, 256, 0, st>>>(in, out, n, x, y, meta, g_force_generic);
        else k_quant_fast<false><<<(unsigned)blocks, 256, 0, st>>>(in, out, n, x, y, meta, g_force_generic);
        return launch_status();
    }
    int64_t blocks = cdiv(n, 256);
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    if (bf) k_quantize_scalar<true><<<(unsigned)blocks, 256, 0, st>>>(in, out, n, x, y, meta, g_force_generic);
    else k_quantize_scalar<false><<<(unsigned)blocks, 256, 0, st>>>(in, out, n, x, y, meta, g_force_generic);
    return launch_status();
}

}  // namespace exmy
