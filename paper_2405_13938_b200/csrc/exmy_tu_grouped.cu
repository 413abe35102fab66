// exmy_tu_grouped.cu -- grouped launch over a tensor table (include/exmy.h,
// "grouped launch"): plan validation and the launchers.
#include <climits>
#include <cstring>

#include "exmy_grouped.cuh"
#include "exmy_launch.cuh"

using namespace exmy;

namespace {

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

bool fmt_ok(int x, int y) {
    if (x < 0 || x > 8 || y < 0) return false;
    const int k = 1 + x + y;
    return k >= 3 && k <= 9;
}

// host copy -> header and entries, checked against the device copy's alignment
exmy_status open_plan(const void *ph, const void *pd, const GroupHeader **h, const GroupEntry **e) {
    if (!ph || !pd) return EXMY_E_ARG;
    if (!aligned(ph, 8) || !aligned(pd, 16)) return EXMY_E_ALIGN;
    const auto *hh = static_cast<const GroupHeader *>(ph);
    if (hh->magic != GROUP_MAGIC || hh->n < 1) return EXMY_E_ARG;
    *h = hh;
    *e = reinterpret_cast<const GroupEntry *>(static_cast<const uint8_t *>(ph) + sizeof(GroupHeader));
    return EXMY_OK;
}

inline const GroupEntry *dev_table(const void *pd) {
    return reinterpret_cast<const GroupEntry *>(static_cast<const uint8_t *>(pd) + sizeof(GroupHeader));
}

template <typename KF>
unsigned grid_for(KF kernel, int threads, int64_t chunks, size_t sm) {
    const int occ = occupancy(kernel, threads, sm);
    int64_t g = (int64_t)num_sms() * occ;
    if (g > chunks) g = chunks;
    return (unsigned)(g < 1 ? 1 : g);
}

template <int K, bool BF16, int MODE, bool PR>
exmy_status launch_genc_kmp(const GroupEntry *tab, const GroupHeader &h, cudaStream_t st) {
    const size_t sm = grp_smem_bytes(h.n);
    const int occ = occupancy(k_grouped_encode<K, BF16, MODE, PR>, GRP_THREADS, sm);
    int64_t g = (int64_t)num_sms() * occ;
    if (g > h.tile_chunks) g = h.tile_chunks;
    k_grouped_encode<K, BF16, MODE, PR><<<(unsigned)g, GRP_THREADS, sm, st>>>(tab, h.n, h.tile_chunks, h.x, h.y,
                                                                               g_force_generic);
    return launch_status();
}

template <int K, bool BF16, int MODE>
exmy_status launch_genc_km(const GroupEntry *tab, const GroupHeader &h, cudaStream_t st) {
    return h.per_row ? launch_genc_kmp<K, BF16, MODE, true>(tab, h, st)
                     : launch_genc_kmp<K, BF16, MODE, false>(tab, h, st);
}

template <int K, bool BF16>
exmy_status launch_genc_k(const GroupEntry *tab, const GroupHeader &h, cudaStream_t st) {
    if (BF16 && h.y <= 6)   // same mode choice as exmy_encode (exmy_tu_encode.cu)
        return h.y == 0 ? launch_genc_km<K, BF16, (BF16 ? ENC_SIMD_Y0 : ENC_F32_Y0)>(tab, h, st)
                        : launch_genc_km<K, BF16, (BF16 ? ENC_SIMD : ENC_F32)>(tab, h, st);
    return h.y == 0 ? launch_genc_km<K, BF16, ENC_F32_Y0>(tab, h, st) : launch_genc_km<K, BF16, ENC_F32>(tab, h, st);
}

template <bool BF16>
exmy_status launch_genc(int k, const GroupEntry *tab, const GroupHeader &h, cudaStream_t st) {
    switch (k) {
        case 3: return launch_genc_k<3, BF16>(tab, h, st);
        case 4: return launch_genc_k<4, BF16>(tab, h, st);
        case 5: return launch_genc_k<5, BF16>(tab, h, st);
        case 6: return launch_genc_k<6, BF16>(tab, h, st);
        case 7: return launch_genc_k<7, BF16>(tab, h, st);
        case 8: return launch_genc_k<8, BF16>(tab, h, st);
        case 9: return launch_genc_k<9, BF16>(tab, h, st);
    }
    return EXMY_E_FORMAT;
}

template <int K, bool OBF16, int MODE, int NH, bool PR>
exmy_status launch_gdec_kmnp(const GroupEntry *tab, const GroupHeader &h, cudaStream_t st) {
    const size_t sm = grp_smem_bytes(h.n);
    const int occ = occupancy(k_grouped_decode<K, OBF16, MODE, NH, PR>, GRP_THREADS, sm);
    // decode is write-bound: GRP_DEC_OCC CTAs/SM (measured on config 3)
    int64_t g = (int64_t)num_sms() * (occ < GRP_DEC_OCC ? occ : GRP_DEC_OCC);
    if (g > h.dtile_chunks) g = h.dtile_chunks;
    k_grouped_decode<K, OBF16, MODE, NH, PR><<<(unsigned)g, GRP_THREADS, sm, st>>>(tab, h.n, h.dtile_chunks, h.x,
                                                                                   h.y);
    return launch_status();
}

template <int K, bool OBF16, int MODE, int NH>
exmy_status launch_gdec_kmn(const GroupEntry *tab, const GroupHeader &h, cudaStream_t st) {
    return h.per_row ? launch_gdec_kmnp<K, OBF16, MODE, NH, true>(tab, h, st)
                     : launch_gdec_kmnp<K, OBF16, MODE, NH, false>(tab, h, st);
}

template <int K, bool OBF16, int MODE>
exmy_status launch_gdec_km(const GroupEntry *tab, const GroupHeader &h, cudaStream_t st) {
    if constexpr (OBF16) {
        if (h.dec_nh == 2) return launch_gdec_kmn<K, OBF16, MODE, 2>(tab, h, st);
    }
    return launch_gdec_kmn<K, OBF16, MODE, 1>(tab, h, st);
}

template <int K, bool OBF16>
exmy_status launch_gdec_k(const GroupEntry *tab, const GroupHeader &h, cudaStream_t st) {
    const bool fast = !g_force_generic && h.x <= 7 && (!OBF16 || h.y <= 7);   // as exmy_decode
    return fast ? launch_gdec_km<K, OBF16, DEC_FAST>(tab, h, st) : launch_gdec_km<K, OBF16, DEC_GENERIC>(tab, h, st);
}

template <bool OBF16>
exmy_status launch_gdec(int k, const GroupEntry *tab, const GroupHeader &h, cudaStream_t st) {
    switch (k) {
        case 3: return launch_gdec_k<3, OBF16>(tab, h, st);
        case 4: return launch_gdec_k<4, OBF16>(tab, h, st);
        case 5: return launch_gdec_k<5, OBF16>(tab, h, st);
        case 6: return launch_gdec_k<6, OBF16>(tab, h, st);
        case 7: return launch_gdec_k<7, OBF16>(tab, h, st);
        case 8: return launch_gdec_k<8, OBF16>(tab, h, st);
        case 9: return launch_gdec_k<9, OBF16>(tab, h, st);
    }
    return EXMY_E_FORMAT;
}

template <int K, bool BF16, int MODE>
exmy_status launch_grws_km(const GroupEntry *tab, const GroupHeader &h, const GroupEntry *host_e, cudaStream_t st) {
    int64_t units = 0, maxrowb = 0, rest = 0;
    for (int i = 0; i < h.n; ++i) {
        const GroupEntry &E = host_e[i];
        if (E.rows * E.cols == 0) continue;
        if (E.fused) {
            units += E.rows / 8;
            maxrowb = E.cols * (BF16 ? 2 : 4) > maxrowb ? E.cols * (BF16 ? 2 : 4) : maxrowb;
        } else {
            rest += E.rows;
        }
    }
    exmy_status s = EXMY_OK;
    if (units) {
        const size_t smax = grws_tab_bytes(GRP_SMEM_TAB) + 8 * (size_t)RWS_MAX_ROW_BYTES;
        static unsigned long long configured = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !(configured & (1ull << dev))) {
            cudaFuncSetAttribute(k_grouped_rowwise_smem<K, BF16, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smax);
            if (dev >= 0 && dev < 64) configured |= 1ull << dev;
        }
        const size_t sm = grws_tab_bytes(h.n) + 8 * (size_t)maxrowb;
        const int occ = occupancy(k_grouped_rowwise_smem<K, BF16, MODE>, RWS_THREADS, sm);
        int64_t g = (int64_t)num_sms() * (occ > 0 ? occ : 1);
        if (g > units) g = units;
        k_grouped_rowwise_smem<K, BF16, MODE><<<(unsigned)g, RWS_THREADS, sm, st>>>(tab, h.n, units, h.x, h.y,
                                                                                      g_force_generic);
        if ((s = launch_status()) != EXMY_OK) return s;
    }
    if (rest) {   // entries with wider rows: row bytes pass + encode, skipping the fused ones
        const size_t sm = grp_smem_bytes(h.n);
        const int64_t cta = cdiv(h.row_total, (int64_t)(GRP_THREADS / 32));
        k_grouped_rowmax<BF16, true><<<grid_for(k_grouped_rowmax<BF16, true>, GRP_THREADS, cta, sm), GRP_THREADS, sm,
                                        st>>>(tab, h.n, h.row_total);
        if ((s = launch_status()) != EXMY_OK) return s;
        const int occ = occupancy(k_grouped_encode<K, BF16, MODE, true, true>, GRP_THREADS, sm);
        int64_t g = (int64_t)num_sms() * occ;
        if (g > h.tile_chunks) g = h.tile_chunks;
        k_grouped_encode<K, BF16, MODE, true, true><<<(unsigned)g, GRP_THREADS, sm, st>>>(tab, h.n, h.tile_chunks,
                                                                                          h.x, h.y, g_force_generic);
        s = launch_status();
    }
    return s;
}

template <int K, bool BF16>
exmy_status launch_grws_k(const GroupEntry *tab, const GroupHeader &h, const GroupEntry *he, cudaStream_t st) {
    if (BF16 && h.y <= 6)   // same mode choice as exmy_encode_rowwise
        return h.y == 0 ? launch_grws_km<K, BF16, (BF16 ? ENC_SIMD_Y0 : ENC_F32_Y0)>(tab, h, he, st)
                        : launch_grws_km<K, BF16, (BF16 ? ENC_SIMD : ENC_F32)>(tab, h, he, st);
    return h.y == 0 ? launch_grws_km<K, BF16, ENC_F32_Y0>(tab, h, he, st) : launch_grws_km<K, BF16, ENC_F32>(tab, h, he, st);
}

template <bool BF16>
exmy_status launch_grws(int k, const GroupEntry *tab, const GroupHeader &h, const GroupEntry *he, cudaStream_t st) {
    switch (k) {
        case 3: return launch_grws_k<3, BF16>(tab, h, he, st);
        case 4: return launch_grws_k<4, BF16>(tab, h, he, st);
        case 5: return launch_grws_k<5, BF16>(tab, h, he, st);
        case 6: return launch_grws_k<6, BF16>(tab, h, he, st);
        case 7: return launch_grws_k<7, BF16>(tab, h, he, st);
        case 8: return launch_grws_k<8, BF16>(tab, h, he, st);
        case 9: return launch_grws_k<9, BF16>(tab, h, he, st);
    }
    return EXMY_E_FORMAT;
}

inline unsigned small_grid(int n, int per) {
    int64_t g = cdiv(n, per);
    return (unsigned)(g < 1 ? 1 : (g > 65535 ? 65535 : g));
}

}  // namespace

extern "C" {

size_t exmy_group_plan_bytes(int n) {
    return n < 1 ? 0 : sizeof(GroupHeader) + (size_t)n * sizeof(GroupEntry);
}

}  // extern "C"

namespace {

exmy_status plan_impl(const exmy_group_entry *entries, int n, int dtype, int x, int y, int out_dtype, int per_row,
                      void *plan, size_t plan_bytes) {
    if (dtype != EXMY_F32 && dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (out_dtype != EXMY_F32 && out_dtype != EXMY_BF16) return EXMY_E_DTYPE;
    if (!fmt_ok(x, y)) return EXMY_E_FORMAT;
    if (n < 1) return EXMY_E_SHAPE;
    if (!entries || !plan || plan_bytes < exmy_group_plan_bytes(n)) return EXMY_E_ARG;
    if (!aligned(plan, 8)) return EXMY_E_ALIGN;
    const int k = 1 + x + y;
    const int V = dtype == EXMY_BF16 ? 8 : 4;
    GroupHeader h{};
    h.magic = GROUP_MAGIC;
    h.n = n;
    h.dtype = dtype;
    h.x = x;
    h.y = y;
    h.out_dtype = out_dtype;
    h.per_row = (int16_t)per_row;
    auto *tab = reinterpret_cast<GroupEntry *>(static_cast<uint8_t *>(plan) + sizeof(GroupHeader));
    // decode tiles 8x8 (16-byte bf16 stores) when every tensor allows them
    h.dec_nh = 1;
    if (out_dtype == EXMY_BF16) {
        h.dec_nh = 2;
        for (int i = 0; i < n; ++i)
            if (entries[i].cols % 8) h.dec_nh = 1;
    }
    int64_t vc = 0, tc = 0, dc = 0, rc = 0, fc = 0;
    const int64_t es = dtype == EXMY_BF16 ? 2 : 4;
    for (int i = 0; i < n; ++i) {
        const exmy_group_entry &a = entries[i];
        if (a.rows < 0 || a.cols < 0 || a.rows % 8 || a.cols % 4) return EXMY_E_SHAPE;
        if (a.cols >= (1 << 30) || a.rows / 8 >= INT_MAX - 64) return EXMY_E_SHAPE;   // 32-bit tile coordinates
        if (a.cols && a.rows > INT64_MAX / 16 / a.cols) return EXMY_E_SHAPE;
        if (a.sp_capacity < 0) return EXMY_E_CAPACITY;
        if (a.sp_capacity > 0 && (!a.sp_index || !a.sp_bits)) return EXMY_E_ARG;
        GroupEntry g{};
        g.in = static_cast<const uint8_t *>(a.in);
        g.out = static_cast<uint8_t *>(a.out);
        g.packed = a.packed;
        g.meta = a.meta;
        g.spi = a.sp_index;
        g.spb = a.sp_bits;
        g.spc = reinterpret_cast<unsigned long long *>(a.sp_count);
        g.cap = a.sp_capacity;
        g.rows = a.rows;
        g.cols = a.cols;
        g.vec_begin = vc;
        g.tile_begin = tc;
        g.dtile_begin = dc;
        g.row_begin = rc;
        g.frg_begin = fc;
        g.fused = 0;
        const int64_t ne = a.rows * a.cols;
        if (ne > 0) {
            if (!a.packed || !a.meta) return EXMY_E_ARG;
            if ((a.in && !aligned(a.in, 16)) || (a.out && !aligned(a.out, 16)) || !aligned(a.packed, 16))
                return EXMY_E_ALIGN;
            if (per_row && (a.cols % 8 || !aligned(a.meta, 8))) return a.cols % 8 ? EXMY_E_SHAPE : EXMY_E_ALIGN;
            rc += a.rows;
            if (per_row && (a.cols * es) % 16 == 0 && a.cols * es <= RWS_MAX_ROW_BYTES) {
                g.fused = 1;
                fc += a.rows / 8;
            }
            vc += cdiv(ne / V, GRP_VEC_CHUNK);
            tc += cdiv((a.rows / 8) * (a.cols / 4), GRP_TILE_CHUNK);
            dc += cdiv((a.rows / 8) * (a.cols / (4 * h.dec_nh)), GRP_DTILE_CHUNK);
        }
        if (g.spc) h.specials = 1;
        std::memcpy(&tab[i], &g, sizeof(g));
    }
    h.vec_chunks = vc;
    h.tile_chunks = tc;
    h.dtile_chunks = dc;
    h.row_total = per_row ? rc : 0;
    std::memcpy(plan, &h, sizeof(h));
    return EXMY_OK;
}

}  // namespace

extern "C" {

exmy_status exmy_group_plan(const exmy_group_entry *entries, int n, int dtype, int x, int y, int out_dtype,
                            void *plan, size_t plan_bytes) {
    return plan_impl(entries, n, dtype, x, y, out_dtype, 0, plan, plan_bytes);
}

exmy_status exmy_group_plan_rows(const exmy_group_entry *entries, int n, int dtype, int x, int y, int out_dtype,
                                 void *plan, size_t plan_bytes) {
    return plan_impl(entries, n, dtype, x, y, out_dtype, 1, plan, plan_bytes);
}

exmy_status exmy_group_max_exponent(const void *plan_host, const void *plan_device, void *stream) {
    const GroupHeader *h;
    const GroupEntry *e;
    exmy_status s = open_plan(plan_host, plan_device, &h, &e);
    if (s != EXMY_OK) return s;
    for (int i = 0; i < h->n; ++i)
        if (e[i].rows * e[i].cols > 0 && !e[i].in) return EXMY_E_ARG;
    cudaStream_t st = S(stream);
    const GroupEntry *tab = dev_table(plan_device);
    if (h->per_row) {   // every row's byte written by its warp: one launch
        if (h->row_total == 0) return EXMY_OK;
        const size_t sm = grp_smem_bytes(h->n);
        const int64_t wpc = GRP_THREADS / 32;
        const int64_t cta = cdiv(h->row_total, wpc);
        if (h->dtype == EXMY_BF16)
            k_grouped_rowmax<true><<<grid_for(k_grouped_rowmax<true>, GRP_THREADS, cta, sm), GRP_THREADS, sm, st>>>(
                tab, h->n, h->row_total);
        else
            k_grouped_rowmax<false><<<grid_for(k_grouped_rowmax<false>, GRP_THREADS, cta, sm), GRP_THREADS, sm,
                                      st>>>(tab, h->n, h->row_total);
        return launch_status();
    }
    k_grouped_clear<0><<<small_grid(h->n, 256), 256, 0, st>>>(tab, h->n);
    if ((s = launch_status()) != EXMY_OK) return s;
    if (h->vec_chunks == 0) return EXMY_OK;
    const size_t sm = grp_smem_bytes(h->n);
    if (h->dtype == EXMY_BF16)
        k_grouped_max<true><<<grid_for(k_grouped_max<true>, GRP_THREADS, h->vec_chunks, sm), GRP_THREADS, sm, st>>>(
            tab, h->n, h->vec_chunks);
    else
        k_grouped_max<false><<<grid_for(k_grouped_max<false>, GRP_THREADS, h->vec_chunks, sm), GRP_THREADS, sm, st>>>(
            tab, h->n, h->vec_chunks);
    return launch_status();
}

exmy_status exmy_group_encode(const void *plan_host, const void *plan_device, void *stream) {
    const GroupHeader *h;
    const GroupEntry *e;
    exmy_status s = open_plan(plan_host, plan_device, &h, &e);
    if (s != EXMY_OK) return s;
    for (int i = 0; i < h->n; ++i)
        if (e[i].rows * e[i].cols > 0 && !e[i].in) return EXMY_E_ARG;
    cudaStream_t st = S(stream);
    const GroupEntry *tab = dev_table(plan_device);
    if (h->specials) {
        k_grouped_clear<1><<<small_grid(h->n, 256), 256, 0, st>>>(tab, h->n);
        if ((s = launch_status()) != EXMY_OK) return s;
    }
    if (h->tile_chunks == 0) return EXMY_OK;
    const int k = 1 + h->x + h->y;
    s = h->dtype == EXMY_BF16 ? launch_genc<true>(k, tab, *h, st) : launch_genc<false>(k, tab, *h, st);
    if (s != EXMY_OK || !h->specials) return s;
    k_grouped_sort<<<small_grid(h->n, 1), 1024, 0, st>>>(tab, h->n);
    return launch_status();
}

exmy_status exmy_group_encode_rowwise(const void *plan_host, const void *plan_device, void *stream) {
    const GroupHeader *h;
    const GroupEntry *e;
    exmy_status s = open_plan(plan_host, plan_device, &h, &e);
    if (s != EXMY_OK) return s;
    if (!h->per_row) return EXMY_E_ARG;
    for (int i = 0; i < h->n; ++i)
        if (e[i].rows * e[i].cols > 0 && !e[i].in) return EXMY_E_ARG;
    cudaStream_t st = S(stream);
    const GroupEntry *tab = dev_table(plan_device);
    if (h->specials) {
        k_grouped_clear<1><<<small_grid(h->n, 256), 256, 0, st>>>(tab, h->n);
        if ((s = launch_status()) != EXMY_OK) return s;
    }
    if (h->row_total == 0) return EXMY_OK;
    const int k = 1 + h->x + h->y;
    s = h->dtype == EXMY_BF16 ? launch_grws<true>(k, tab, *h, e, st) : launch_grws<false>(k, tab, *h, e, st);
    if (s != EXMY_OK || !h->specials) return s;
    k_grouped_sort<<<small_grid(h->n, 1), 1024, 0, st>>>(tab, h->n);
    return launch_status();
}

exmy_status exmy_group_decode(const void *plan_host, const void *plan_device, void *stream) {
    const GroupHeader *h;
    const GroupEntry *e;
    exmy_status s = open_plan(plan_host, plan_device, &h, &e);
    if (s != EXMY_OK) return s;
    for (int i = 0; i < h->n; ++i)
        if (e[i].rows * e[i].cols > 0 && !e[i].out) return EXMY_E_ARG;
    if (h->dtile_chunks == 0) return EXMY_OK;
    cudaStream_t st = S(stream);
    const GroupEntry *tab = dev_table(plan_device);
    const int k = 1 + h->x + h->y;
    const bool obf = h->out_dtype == EXMY_BF16;
    s = obf ? launch_gdec<true>(k, tab, *h, st) : launch_gdec<false>(k, tab, *h, st);
    if (s != EXMY_OK || !h->specials) return s;
    if (obf) k_grouped_scatter<true><<<small_grid(h->n, 1), 256, 0, st>>>(tab, h->n);
    else k_grouped_scatter<false><<<small_grid(h->n, 1), 256, 0, st>>>(tab, h->n);
    return launch_status();
}

}  // extern "C"
