// exmy_ckpt.cpp -- the checkpoint container ("the
// checkpoints half of the paper's library claim": "encoding and
// decoding tensors and checkpoints"; file layout S:369-378).  Host code:
// manifest + per-tensor CRC32 + lazy byte-range reads with pread, so loading
// one tensor touches only its own bytes.
//
//   header   "EXMY" | version u8 = 2 | entry_count u32
//   entry    name_len u16 | name | rank u8 | dims u32 x rank | x u8 | y u8 |
//            scheme u8 | block_kind u8 [+ L u32 | + r u32, c u32] | flags u8 |
//            (offset u64, length u64) for: metadata, each segment (descending
//            width), scale array, specials | crc32 u32
//   payload  sections at their offsets (metadata, segments, scale, specials
//            of one tensor contiguous, in that order)
// flags: bit0 scale present, bit1 specials present, bit2 COLS packing
// (extension: the packing axis), bit3 source dtype bf16 (extension).
// Specials: count x (u64 index, u32 fp32 bits) records, as SPEC's
// "(u64 index, u32 bits) pairs" (version 2; version-1 files, which stored all
// indices then all bits, are still read).  CRC32 (IEEE, reflected
// 0xEDB88320) over the tensor's payload bytes in section order.
//
// The reader trusts nothing in the file: section ranges are checked without
// wrap-around, segment lengths against prod(dims) * w / 8, metadata / scale
// lengths against the block grid, specials indices against the element count;
// allocation failures return E_CONTAINER instead of throwing across the C ABI.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "exmy.h"

namespace {

uint32_t crc_table[256];
bool crc_init_done = false;

void crc_init() {
    if (crc_init_done) return;
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int b = 0; b < 8; ++b) c = (c & 1u) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
        crc_table[i] = c;
    }
    crc_init_done = true;
}

uint32_t crc_update(uint32_t crc, const uint8_t *p, size_t n) {
    crc = ~crc;
    for (size_t i = 0; i < n; ++i) crc = crc_table[(crc ^ p[i]) & 0xFFu] ^ (crc >> 8);
    return ~crc;
}

struct Section {
    uint64_t off = 0, len = 0;
};

struct Entry {
    std::string name;
    int rank = 0;
    uint32_t dims[8] = {0};
    int x = 0, y = 0, scheme = 0, block_kind = 0, axis = 0, bf16 = 0;
    uint32_t bp0 = 0, bp1 = 0;
    int nseg = 0;
    Section meta, seg[4], scale, specials;
    uint32_t crc = 0;
    uint64_t nel = 0;   // prod(dims) (reader)
};

int popcount_k(int k) {
    int n = 0;
    for (int w = 8; w >= 1; w >>= 1) n += (k & w) ? 1 : 0;
    return n;
}

void put(std::vector<uint8_t> &b, const void *p, size_t n) {
    const auto *c = static_cast<const uint8_t *>(p);
    b.insert(b.end(), c, c + n);
}
template <typename T>
void put_le(std::vector<uint8_t> &b, T v) {
    for (size_t i = 0; i < sizeof(T); ++i) b.push_back((uint8_t)((uint64_t)v >> (8 * i)));
}

bool write_all(int fd, const void *p, size_t n, uint64_t off) {
    const auto *c = static_cast<const uint8_t *>(p);
    while (n) {
        const ssize_t w = pwrite(fd, c, n, (off_t)off);
        if (w <= 0) return false;
        c += w;
        off += (uint64_t)w;
        n -= (size_t)w;
    }
    return true;
}

bool read_all(int fd, void *p, size_t n, uint64_t off) {
    auto *c = static_cast<uint8_t *>(p);
    while (n) {
        const ssize_t r = pread(fd, c, n, (off_t)off);
        if (r <= 0) return false;
        c += r;
        off += (uint64_t)r;
        n -= (size_t)r;
    }
    return true;
}

size_t entry_manifest_bytes(const Entry &e) {
    size_t n = 2 + e.name.size() + 1 + 4 * (size_t)e.rank + 4 + (e.block_kind == 3 ? 4 : e.block_kind == 4 ? 8 : 0) + 1;
    n += 16 * (size_t)(1 + e.nseg + 2) + 4;
    return n;
}

void put_entry(std::vector<uint8_t> &b, const Entry &e) {
    put_le<uint16_t>(b, (uint16_t)e.name.size());
    put(b, e.name.data(), e.name.size());
    put_le<uint8_t>(b, (uint8_t)e.rank);
    for (int i = 0; i < e.rank; ++i) put_le<uint32_t>(b, e.dims[i]);
    put_le<uint8_t>(b, (uint8_t)e.x);
    put_le<uint8_t>(b, (uint8_t)e.y);
    put_le<uint8_t>(b, (uint8_t)e.scheme);
    put_le<uint8_t>(b, (uint8_t)e.block_kind);
    if (e.block_kind == 3) put_le<uint32_t>(b, e.bp0);
    if (e.block_kind == 4) {
        put_le<uint32_t>(b, e.bp0);
        put_le<uint32_t>(b, e.bp1);
    }
    const uint8_t flags = (uint8_t)((e.scale.len ? 1 : 0) | (e.specials.len ? 2 : 0) | (e.axis ? 4 : 0) | (e.bf16 ? 8 : 0));
    put_le<uint8_t>(b, flags);
    auto sec = [&](const Section &s) {
        put_le<uint64_t>(b, s.off);
        put_le<uint64_t>(b, s.len);
    };
    sec(e.meta);
    for (int s = 0; s < e.nseg; ++s) sec(e.seg[s]);
    sec(e.scale);
    sec(e.specials);
    put_le<uint32_t>(b, e.crc);
}

constexpr uint8_t kVersion = 2;

// (u64 index, u32 bits) records of a tensor's specials list
std::vector<uint8_t> specials_records(const exmy_ckpt_tensor &a) {
    std::vector<uint8_t> sp;
    sp.reserve((size_t)a.specials_count * 12u);
    for (int64_t j = 0; j < a.specials_count; ++j) {
        put_le<uint64_t>(sp, (uint64_t)a.sp_index[j]);
        put_le<uint32_t>(sp, a.sp_bits[j]);
    }
    return sp;
}

// number of metadata blocks of an entry, or -1 if the block shape does not
// tile the (R, C) view (R = prod(dims[:-1]), C = dims[-1])
int64_t block_count(const Entry &e, uint64_t nel) {
    const uint64_t C = e.rank ? e.dims[e.rank - 1] : 1;
    const uint64_t R = C ? nel / C : 0;
    switch (e.block_kind) {
    case 0: return 1;
    case 1: return (int64_t)R;
    case 2: return (int64_t)C;
    case 3:
        if (e.bp0 == 0 || C % e.bp0) return -1;
        return (int64_t)(R * (C / e.bp0));
    case 4:
        if (e.bp0 == 0 || e.bp1 == 0 || R % e.bp0 || C % e.bp1) return -1;
        return (int64_t)((R / e.bp0) * (C / e.bp1));
    default: return -1;
    }
}

// structural checks of one manifest entry against its own shape
bool entry_consistent(const Entry &e) {
    if (e.x > 8 || 1 + e.x + e.y > 15 || e.scheme > 2 || e.block_kind > 4) return false;
    uint64_t nel = 1;
    for (int d = 0; d < e.rank; ++d)
        if (__builtin_mul_overflow(nel, (uint64_t)e.dims[d], &nel)) return false;
    if (nel % 8) return false;
    const int k = 1 + e.x + e.y;
    int si = 0;
    for (int w = 8; w >= 1; w >>= 1)
        if (k & w) {
            if (e.seg[si].len != nel / 8 * (uint64_t)w) return false;
            ++si;
        }
    const int64_t nb = block_count(e, nel);
    if (nb < 0) return false;
    if (e.scheme == 2) {   // float scaling: one fp32 per block, a fixed metadata byte
        if (e.scale.len != 4u * (uint64_t)nb || e.meta.len > 1) return false;
    } else if (e.meta.len != (uint64_t)nb || e.scale.len != 0) {
        return false;
    }
    if (e.specials.len % 12 || e.specials.len / 12 > nel) return false;
    return true;
}

struct Reader {
    const uint8_t *p, *end;
    bool ok = true;
    template <typename T>
    T get() {
        T v = 0;
        if ((size_t)(end - p) < sizeof(T)) {
            ok = false;
            return v;
        }
        for (size_t i = 0; i < sizeof(T); ++i) v |= (T)((uint64_t)p[i] << (8 * i));
        p += sizeof(T);
        return v;
    }
};

}  // namespace

struct exmy_ckpt {
    int fd = -1;
    int version = 0;
    uint64_t file_size = 0;
    std::vector<Entry> entries;
    uint64_t bytes_read = 0;   // payload bytes read (lazy-read instrumentation)
};

extern "C" {

int64_t exmy_ckpt_write(const char *path, const exmy_ckpt_tensor *t, int n) {
    if (!path || n < 0 || (n > 0 && !t)) return -(int64_t)EXMY_E_ARG;
    crc_init();
    std::vector<Entry> es((size_t)n);
    for (int i = 0; i < n; ++i) {
        const exmy_ckpt_tensor &a = t[i];
        Entry &e = es[(size_t)i];
        if (!a.name || a.rank < 0 || a.rank > 8 || a.x < 0 || a.x > 8 || a.y < 0 || a.scheme < 0 || a.scheme > 2 ||
            a.block_kind < 0 || a.block_kind > 4 || a.meta_bytes < 0 || a.packed_bytes < 0 || a.scale_bytes < 0 ||
            a.specials_count < 0)
            return -(int64_t)EXMY_E_ARG;
        e.name = a.name;
        if (e.name.size() > 65535) return -(int64_t)EXMY_E_ARG;
        for (int j = 0; j < i; ++j)
            if (es[(size_t)j].name == e.name) return -(int64_t)EXMY_E_ARG;   // names unique
        e.rank = a.rank;
        int64_t nel = 1;
        for (int d = 0; d < a.rank; ++d) {
            if (a.dims[d] < 0 || a.dims[d] > 0xFFFFFFFFll) return -(int64_t)EXMY_E_SHAPE;
            e.dims[d] = (uint32_t)a.dims[d];
            nel *= a.dims[d];
        }
        e.x = a.x;
        e.y = a.y;
        e.scheme = a.scheme;
        e.block_kind = a.block_kind;
        e.bp0 = (uint32_t)a.block_p0;
        e.bp1 = (uint32_t)a.block_p1;
        e.axis = a.axis ? 1 : 0;
        e.bf16 = a.src_dtype == EXMY_BF16 ? 1 : 0;
        const int k = 1 + a.x + a.y;
        e.nseg = popcount_k(k);
        if (nel % 8 || a.packed_bytes != nel / 8 * k) return -(int64_t)EXMY_E_SHAPE;
        if ((a.meta_bytes && !a.meta) || (a.packed_bytes && !a.packed) || (a.scale_bytes && !a.scale) ||
            (a.specials_count && (!a.sp_index || !a.sp_bits)))
            return -(int64_t)EXMY_E_ARG;
    }
    // manifest size -> payload offsets
    uint64_t off = 4 + 1 + 4;
    for (auto &e : es) off += entry_manifest_bytes(e);
    for (int i = 0; i < n; ++i) {
        const exmy_ckpt_tensor &a = t[i];
        Entry &e = es[(size_t)i];
        e.meta = {off, (uint64_t)a.meta_bytes};
        off += e.meta.len;
        int64_t nel = 1;
        for (int d = 0; d < a.rank; ++d) nel *= a.dims[d];
        int si = 0;
        for (int w = 8; w >= 1; w >>= 1)
            if ((1 + a.x + a.y) & w) {
                e.seg[si] = {off, (uint64_t)(nel / 8 * w)};
                off += e.seg[si].len;
                ++si;
            }
        e.scale = {off, (uint64_t)a.scale_bytes};
        off += e.scale.len;
        e.specials = {off, (uint64_t)a.specials_count * 12u};
        off += e.specials.len;
        uint32_t c = crc_update(0, static_cast<const uint8_t *>(a.meta), (size_t)a.meta_bytes);
        c = crc_update(c, static_cast<const uint8_t *>(a.packed), (size_t)a.packed_bytes);
        c = crc_update(c, static_cast<const uint8_t *>(a.scale), (size_t)a.scale_bytes);
        const std::vector<uint8_t> sp = specials_records(a);
        e.crc = crc_update(c, sp.data(), sp.size());
    }
    std::vector<uint8_t> head;
    put(head, "EXMY", 4);
    put_le<uint8_t>(head, kVersion);
    put_le<uint32_t>(head, (uint32_t)n);
    for (auto &e : es) put_entry(head, e);
    const int fd = open(path, O_CREAT | O_TRUNC | O_WRONLY, 0644);
    if (fd < 0) return -(int64_t)EXMY_E_IO;
    bool ok = write_all(fd, head.data(), head.size(), 0);
    for (int i = 0; i < n && ok; ++i) {
        const exmy_ckpt_tensor &a = t[i];
        const Entry &e = es[(size_t)i];
        ok = ok && write_all(fd, a.meta, (size_t)e.meta.len, e.meta.off);
        ok = ok && write_all(fd, a.packed, (size_t)a.packed_bytes, e.seg[0].off);
        ok = ok && write_all(fd, a.scale, (size_t)e.scale.len, e.scale.off);
        const std::vector<uint8_t> sp = specials_records(a);
        ok = ok && write_all(fd, sp.data(), sp.size(), e.specials.off);
    }
    if (close(fd) != 0) ok = false;
    return ok ? (int64_t)off : -(int64_t)EXMY_E_IO;
}

static exmy_status ckpt_open_impl(const char *path, exmy_ckpt **out) {
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return EXMY_E_IO;
    struct stat st;
    if (fstat(fd, &st) != 0) {
        close(fd);
        return EXMY_E_IO;
    }
    auto *h = new exmy_ckpt;
    h->fd = fd;
    h->file_size = (uint64_t)st.st_size;
    auto fail = [&](exmy_status s) {
        exmy_ckpt_close(h);
        return s;
    };
    uint8_t hd[9];
    if (!read_all(fd, hd, 9, 0)) return fail(EXMY_E_CONTAINER);
    if (std::memcmp(hd, "EXMY", 4) != 0 || hd[4] < 1 || hd[4] > kVersion) return fail(EXMY_E_CONTAINER);
    h->version = hd[4];
    const uint32_t n = (uint32_t)hd[5] | ((uint32_t)hd[6] << 8) | ((uint32_t)hd[7] << 16) | ((uint32_t)hd[8] << 24);
    // every entry takes at least 2+1+4+1+16*3+4 manifest bytes: a count the
    // file cannot hold is a malformed container, not an allocation to try
    if ((uint64_t)n * 60u > h->file_size) return fail(EXMY_E_CONTAINER);
    // the manifest lies before the first payload byte; read it in growing chunks
    std::vector<uint8_t> man;
    uint64_t want = 4096;
    for (;;) {
        const uint64_t avail = h->file_size > 9 ? h->file_size - 9 : 0;
        const uint64_t len = want < avail ? want : avail;
        man.resize((size_t)len);
        if (len && !read_all(fd, man.data(), (size_t)len, 9)) return fail(EXMY_E_IO);
        Reader r{man.data(), man.data() + man.size()};
        h->entries.clear();
        for (uint32_t i = 0; i < n && r.ok; ++i) {
            Entry e;
            const uint16_t nl = r.get<uint16_t>();
            if ((size_t)(r.end - r.p) < nl) {
                r.ok = false;
                break;
            }
            e.name.assign(reinterpret_cast<const char *>(r.p), nl);
            r.p += nl;
            e.rank = r.get<uint8_t>();
            if (e.rank > 8) return fail(EXMY_E_CONTAINER);
            for (int d = 0; d < e.rank; ++d) e.dims[d] = r.get<uint32_t>();
            e.x = r.get<uint8_t>();
            e.y = r.get<uint8_t>();
            e.scheme = r.get<uint8_t>();
            e.block_kind = r.get<uint8_t>();
            if (e.block_kind == 3) e.bp0 = r.get<uint32_t>();
            if (e.block_kind == 4) {
                e.bp0 = r.get<uint32_t>();
                e.bp1 = r.get<uint32_t>();
            }
            const uint8_t flags = r.get<uint8_t>();
            e.axis = (flags >> 2) & 1;
            e.bf16 = (flags >> 3) & 1;
            if (e.x > 8 || 1 + e.x + e.y > 15) return fail(EXMY_E_CONTAINER);
            e.nseg = popcount_k(1 + e.x + e.y);
            auto sec = [&](Section &s) {
                s.off = r.get<uint64_t>();
                s.len = r.get<uint64_t>();
            };
            sec(e.meta);
            for (int s = 0; s < e.nseg; ++s) sec(e.seg[s]);
            sec(e.scale);
            sec(e.specials);
            e.crc = r.get<uint32_t>();
            h->entries.push_back(e);
        }
        if (r.ok) break;
        if (len == avail) return fail(EXMY_E_CONTAINER);   // truncated manifest
        want *= 4;
    }
    for (auto &e : h->entries) {
        // shape, segment, metadata and specials sizes consistent with the entry
        if (!entry_consistent(e)) return fail(EXMY_E_CONTAINER);
        e.nel = 1;
        for (int d = 0; d < e.rank; ++d) e.nel *= e.dims[d];
        // sections inside the file (no wrap-around), contiguous per tensor
        uint64_t pos = e.meta.off;
        Section *ss[7] = {&e.meta, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        int ns = 1;
        for (int s = 0; s < e.nseg; ++s) ss[ns++] = &e.seg[s];
        ss[ns++] = &e.scale;
        ss[ns++] = &e.specials;
        for (int s = 0; s < ns; ++s) {
            const Section &q = *ss[s];
            if (q.off != pos || q.len > h->file_size || q.off > h->file_size - q.len) return fail(EXMY_E_CONTAINER);
            pos += q.len;
        }
    }
    *out = h;
    return EXMY_OK;
}

exmy_status exmy_ckpt_open(const char *path, exmy_ckpt **out) {
    if (!path || !out) return EXMY_E_ARG;
    *out = nullptr;
    try {
        return ckpt_open_impl(path, out);
    } catch (...) {   // std::bad_alloc and friends never cross the C ABI
        return EXMY_E_CONTAINER;
    }
}

int exmy_ckpt_count(const exmy_ckpt *h) { return h ? (int)h->entries.size() : -1; }

exmy_status exmy_ckpt_info(const exmy_ckpt *h, int i, exmy_ckpt_tensor *info) {
    if (!h || !info || i < 0 || i >= (int)h->entries.size()) return EXMY_E_ARG;
    const Entry &e = h->entries[(size_t)i];
    std::memset(info, 0, sizeof(*info));
    info->name = e.name.c_str();
    info->rank = e.rank;
    for (int d = 0; d < e.rank; ++d) info->dims[d] = e.dims[d];
    info->x = e.x;
    info->y = e.y;
    info->scheme = e.scheme;
    info->block_kind = e.block_kind;
    info->block_p0 = e.bp0;
    info->block_p1 = e.bp1;
    info->axis = e.axis;
    info->src_dtype = e.bf16 ? EXMY_BF16 : EXMY_F32;
    info->meta_bytes = (int64_t)e.meta.len;
    uint64_t pk = 0;
    for (int s = 0; s < e.nseg; ++s) pk += e.seg[s].len;
    info->packed_bytes = (int64_t)pk;
    info->scale_bytes = (int64_t)e.scale.len;
    info->specials_count = (int64_t)(e.specials.len / 12);
    return EXMY_OK;
}

int exmy_ckpt_find(const exmy_ckpt *h, const char *name) {
    if (!h || !name) return -1;
    for (size_t i = 0; i < h->entries.size(); ++i)
        if (h->entries[i].name == name) return (int)i;
    return -1;
}

static exmy_status ckpt_read_impl(exmy_ckpt *h, int i, void *meta, void *packed, void *scale, int64_t *sp_index,
                                  uint32_t *sp_bits) {
    const Entry &e = h->entries[(size_t)i];
    uint64_t pk = 0;
    for (int s = 0; s < e.nseg; ++s) pk += e.seg[s].len;
    if (meta && !read_all(h->fd, meta, (size_t)e.meta.len, e.meta.off)) return EXMY_E_IO;
    if (packed && !read_all(h->fd, packed, (size_t)pk, e.seg[0].off)) return EXMY_E_IO;
    if (scale && !read_all(h->fd, scale, (size_t)e.scale.len, e.scale.off)) return EXMY_E_IO;
    h->bytes_read += (meta ? e.meta.len : 0) + (packed ? pk : 0) + (scale ? e.scale.len : 0);
    const int64_t cnt = (int64_t)(e.specials.len / 12);
    if (cnt && (sp_index || sp_bits)) {
        std::vector<uint8_t> sp((size_t)e.specials.len);
        if (!read_all(h->fd, sp.data(), sp.size(), e.specials.off)) return EXMY_E_IO;
        h->bytes_read += e.specials.len;
        for (int64_t j = 0; j < cnt; ++j) {
            // version 2: (u64, u32) records; version 1: all indices, then all bits
            const size_t io = h->version >= 2 ? (size_t)(12 * j) : (size_t)(8 * j);
            const size_t bo = h->version >= 2 ? (size_t)(12 * j + 8) : (size_t)(8 * cnt + 4 * j);
            uint64_t v = 0;
            for (int b = 0; b < 8; ++b) v |= (uint64_t)sp[io + (size_t)b] << (8 * b);
            uint32_t u = 0;
            for (int b = 0; b < 4; ++b) u |= (uint32_t)sp[bo + (size_t)b] << (8 * b);
            if (v >= e.nel) return EXMY_E_CONTAINER;   // an index outside the tensor
            if (sp_index) sp_index[j] = (int64_t)v;
            if (sp_bits) sp_bits[j] = u;
        }
    }
    return EXMY_OK;
}

exmy_status exmy_ckpt_read(exmy_ckpt *h, int i, void *meta, void *packed, void *scale, int64_t *sp_index,
                           uint32_t *sp_bits) {
    if (!h || i < 0 || i >= (int)h->entries.size()) return EXMY_E_ARG;
    try {
        return ckpt_read_impl(h, i, meta, packed, scale, sp_index, sp_bits);
    } catch (...) {
        return EXMY_E_CONTAINER;
    }
}

exmy_status exmy_ckpt_verify(exmy_ckpt *h, int i) {
    if (!h || i < 0 || i >= (int)h->entries.size()) return EXMY_E_ARG;
    crc_init();
    const Entry &e = h->entries[(size_t)i];
    const uint64_t len = e.specials.off + e.specials.len - e.meta.off;
    std::vector<uint8_t> buf;
    try {
        buf.resize(1u << 20);
    } catch (...) {
        return EXMY_E_CONTAINER;
    }
    uint32_t c = 0;
    for (uint64_t done = 0; done < len;) {
        const size_t n = (size_t)((len - done) < buf.size() ? (len - done) : buf.size());
        if (!read_all(h->fd, buf.data(), n, e.meta.off + done)) return EXMY_E_IO;
        c = crc_update(c, buf.data(), n);
        done += n;
    }
    h->bytes_read += len;
    return c == e.crc ? EXMY_OK : EXMY_E_CHECKSUM;
}

int64_t exmy_ckpt_bytes_read(const exmy_ckpt *h) { return h ? (int64_t)h->bytes_read : -1; }

void exmy_ckpt_close(exmy_ckpt *h) {
    if (!h) return;
    if (h->fd >= 0) close(h->fd);
    delete h;
}

}  // extern "C"
