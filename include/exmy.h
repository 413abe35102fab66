/*
 * exmy.h -- C ABI of the B200 (sm_100a) eXmY tensor codec  (libexmy.so)
 *
 * eXmY (arXiv 2405.13938) is a floating-point format with 1 sign bit, X
 * exponent bits and Y mantissa bits, k = 1+X+Y bits in total, a software
 * defined exponent bias and subnormals (Table 1,
 * P:139-175).  Citations: P:n = PAPER.md line n; Dn = reading n in DESIGN.md.
 *
 * Format descriptor:
 *   x in [0,8], y >= 0, k = 1+x+y in [3,9] on the GPU path (every format of
 *   total width 3..9 bits, 42 formats).
 *   Metadata ("meta") is the per-tensor MAXIMUM BIASED EXPONENT,
 *   one uint8 in DEVICE memory, e_max in [0,254] (D4).  It fixes the bias:
 *   bias = 2^x + 126 - e_max (D1), i.e. the top exponent code 2^x-1 lands on
 *   fp32 biased exponent e_max.  Kernels clamp a device value of 255 to 254.
 *
 * Code layout (D2): [sign(1) | exponent(x) | mantissa(y)], MSB -> LSB.
 *   e >= 1: value = (-1)^s (1 + m/2^y) 2^(e - bias)
 *   e == 0 (and every code when x == 0, D3): value = (-1)^s m 2^(1 - bias - y)
 * Rounding (D5-D8): round to nearest, ties to the code whose LSB
 *   is 0; values beyond the largest magnitude saturate; values
 *   that round to zero keep their sign (D10); fp32 subnormal inputs are exact
 *   (D11).  NaN/Inf are kept out of band (D9).
 *
 * Packed layout (Fig. 3; D12-D16):
 *   a (R,C) row-major tensor with R % 8 == 0 (ROWS) or C % 8 == 0 (COLS) is
 *   split into groups of 8 elements:
 *     ROWS: group (g,c) = elements (8g+i, c), container index g*C + c
 *     COLS: group (r,g) = elements (r, 8g+i), container index r*(C/8) + g
 *   k is decomposed into its set bits, descending (7 = 4+2+1, 9 = 8+1).
 *   Segment j (width w_j) takes code bits [hi_j - w_j, hi_j), hi_0 = k: the
 *   widest segment holds the most significant bits (D13).  For w in {1,2,4}
 *   container = sum_i field_i << (w*i), stored little-endian in w bytes (D14);
 *   for w = 8 the segment is the byte array in row-major element order (D15).
 *   Segments are concatenated in decomposition order; segment j starts at
 *   byte sum_{j'<j} n*w_j'/8; the total is exactly n*k/8 bytes.
 *   A row shard [r0,r1) of segment j is the byte range
 *   off_j + [r0*C*w_j/8, r1*C*w_j/8) (ROWS: r0, r1 multiples of 8) and
 *   decodes on its own.
 *
 * Conventions for every call below:
 *   - Tensor pointers are CUDA DEVICE pointers owned by the caller; the
 *     library never allocates, frees or synchronises.  Every device op is
 *     enqueued on `stream` (a cudaStream_t passed as void*, NULL = legacy
 *     default stream) and returns after the launches.
 *   - Inputs are fp32 (EXMY_F32) or bf16 (EXMY_BF16) bit patterns, row-major
 *     contiguous.  Any alignment is accepted: 16-byte aligned tensors and
 *     segment bases take the vectorised kernels, others a scalar kernel with
 *     identical results.
 *   - n = 0 is a no-op returning EXMY_OK.
 *   - Errors are returned, never aborted on: EXMY_E_FORMAT (x,y out of range,
 *     k not in [3,9]), EXMY_E_SHAPE (ROWS with R%8, COLS with C%8, negative
 *     sizes), EXMY_E_DTYPE, EXMY_E_ARG (NULL pointer where one is required),
 *     EXMY_E_CAPACITY (capacity < 0), EXMY_E_META (host helpers: e_max or
 *     bias out of range), EXMY_E_CUDA (launch error from cudaGetLastError).
 */
#ifndef EXMY_H
#define EXMY_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    EXMY_OK = 0,
    EXMY_E_FORMAT = 1,
    EXMY_E_META = 2,
    EXMY_E_SHAPE = 3,
    EXMY_E_DTYPE = 4,
    EXMY_E_ALIGN = 5,     /* reserved: misaligned tensors take the scalar kernels */
    EXMY_E_CAPACITY = 6,
    EXMY_E_CUDA = 7,
    EXMY_E_ARG = 8,
    EXMY_E_IO = 9,         /* checkpoint file: open / read / write failed */
    EXMY_E_CONTAINER = 10, /* checkpoint file: bad magic, version or manifest */
    EXMY_E_CHECKSUM = 11   /* checkpoint file: CRC32 mismatch */
} exmy_status;

typedef enum { EXMY_F32 = 0, EXMY_BF16 = 1 } exmy_dtype;
typedef enum { EXMY_AXIS_ROWS = 0, EXMY_AXIS_COLS = 1 } exmy_axis;

/* ------------------------------------------------------------ host helpers */

/* Library version string. */
const char *exmy_version(void);

/* Human-readable name of a status code (static storage). */
const char *exmy_status_string(int status);

/* 1 if (x, y) is a GPU-supported format (x in [0,8], k=1+x+y in [3,9]). */
int exmy_format_valid(int x, int y);

/* Packed size in bytes, n*k/8; -1 if the format is invalid or
 * n is negative or not a multiple of 8. */
int64_t exmy_packed_bytes(int64_t n, int x, int y);

/* Segment plan of width k for n elements: writes the widths
 * (descending set bits of k) and byte offsets; returns the segment count,
 * or -1 for k outside [1,15] or bad n.  widths/offsets: host arrays of 4. */
int exmy_segments(int k, int64_t n, int *widths, int64_t *offsets);

/* bias <-> metadata (D1): bias = 2^x + 126 - e_max.  Return EXMY_E_META if
 * the result would leave e_max in [0,254]. */
exmy_status exmy_bias_from_emax(int x, int e_max, int *bias_out);
exmy_status exmy_emax_from_bias(int x, int bias, int *emax_out);

/* e_max of a HOST histogram: the top populated bin in [0,254], 0 if none
 * (max exponent before rounding). */
int exmy_emax_from_histogram_host(const uint64_t *hist_host);

/* Choose X (D19): the smallest x in [0,8] whose 2^x-1 normal
 * exponent codes, placed at the top of the populated range (bins
 * e_max-2^x+2 .. e_max), hold at least (1 - flush_budget) of the non-zero
 * finite values (bins 1..254).  hist_host: 256 host counters. */
exmy_status exmy_choose_x(const uint64_t *hist_host, double flush_budget, int *x_out);

/* -------------------------------------------------------------- device ops */

/* Exponent histogram (A1): hist[b] += number of elements whose
 * 8-bit biased exponent field is b.  Bin 0 = zeros and input subnormals,
 * bin 255 = NaN/Inf (D18).  `hist`: device uint64[256], ACCUMULATED into
 * (zero it first for a fresh histogram).  Reads n elements once. */
exmy_status exmy_exponent_histogram(const void *in, int dtype, int64_t n,
                                    uint64_t *hist, void *stream);

/* Per-tensor metadata from a device histogram (A2): *meta =
 * top populated bin in [0,254] (0 if none).  One tiny launch; graph-safe. */
exmy_status exmy_emax_from_histogram(const uint64_t *hist, uint8_t *meta, void *stream);

/* Per-tensor metadata straight from the data (A2 without A1): *meta = the
 * largest 8-bit biased exponent field of a finite element, clamped to 254
 * (0 if none) -- the same byte exmy_emax_from_histogram gives -- as one
 * read-only max reduction (CTAs combine with a byte compare-and-swap on the
 * 32-bit word holding *meta; the other three bytes are preserved).  Needs a
 * 16-byte aligned `in` (else EXMY_E_ALIGN: use the histogram path).  Use it
 * when X is already chosen and only the bias is data-derived. */
exmy_status exmy_max_exponent(const void *in, int dtype, int64_t n, uint8_t *meta, void *stream);

/* Emulation / quantize (A3): out[i] = the eXmY grid value nearest
 * to in[i] (RTNE, saturating, subnormals, signed zero), converted RTNE to
 * the same container dtype (D21); NaN/Inf bit patterns pass through
 * unchanged.  in/out: n elements of `dtype`; out may alias in. */
exmy_status exmy_quantize(const void *in, void *out, int dtype, int64_t n,
                          int x, int y, const uint8_t *meta, void *stream);

/* Encode = type conversion (A4) + power-of-2 bit packing
 * (A5), fused: codes never touch HBM.
 *   in: (rows, cols) row-major fp32/bf16; packed: n*k/8 bytes (layout above).
 *   NaN/Inf (D9): code 0 in the packed stream; (index, fp32 bits) of the
 *   first sp_capacity of them in ascending index order in sp_index[] /
 *   sp_bits[] (device); sp_count[0] (device uint64) is SET to the total
 *   number of specials, even when it exceeds capacity (the entries past the
 *   capacity are not written; check after the stream syncs).  The
 *   histogram's bin 255 is that count.  The list is built after the encode
 *   kernel by ordered stream compaction (no sort): with sp_capacity > 0,
 *   sp_count must point to EXMY_SPECIALS_WORDS uint64 of device workspace
 *   (word 0 = the count, then 1024 per-range counts and a fix-up flag:
 *   the fast per-tensor kernels leave tiles holding NaN/Inf to a fix-up pass
 *   that encodes them on the vector path with code 0 in their lanes); with
 *   sp_capacity == 0 one word is enough.  Without NaN/Inf (word 0 == 0) the two compaction
 *   launches return at once.  sp_index/sp_bits may be NULL iff
 *   sp_capacity == 0; sp_count may be NULL only if the input is known to
 *   hold no NaN/Inf.  The same convention holds for every *_encode* call
 *   below except the grouped ones (per-entry lists of one count word). */
#define EXMY_SPECIALS_WORDS 1026
int exmy_specials_words(void);   /* == EXMY_SPECIALS_WORDS */
exmy_status exmy_encode(const void *in, int dtype, int64_t rows, int64_t cols, int axis,
                        int x, int y, const uint8_t *meta, uint8_t *packed,
                        int64_t *sp_index, uint32_t *sp_bits, uint64_t *sp_count,
                        int64_t sp_capacity, void *stream);

/* Decode = unpack (A6) + dequantize (A7), fused: out[i] = value of code i
 * rounded RTNE to out_dtype (D21); then min(*sp_count, sp_capacity) specials
 * are written back from their fp32 bits (bf16 out: the top 16 bits, quiet
 * bit forced if a NaN payload would vanish, D9).  sp_* may all be NULL/0
 * when the tensor holds no specials.  Decode of a row shard: pass the
 * shard's own segment bytes (see the layout note) and its row count. */
exmy_status exmy_decode(const uint8_t *packed, int64_t rows, int64_t cols, int axis,
                        int x, int y, const uint8_t *meta,
                        const int64_t *sp_index, const uint32_t *sp_bits,
                        const uint64_t *sp_count, int64_t sp_capacity,
                        void *out, int out_dtype, void *stream);

/* Test/diagnostic knobs (process-global, not thread-safe; default 0).
 * exmy_debug_force_generic(1) routes every element through the integer
 * generic encode/decode paths instead of the fast paths, so both can be
 * checked against the oracle; exmy_debug_hist_mode selects the histogram
 * counter-update variant (0: lane-private read-modify-write, 1: lane-private
 * shared-memory atomics, 2: the same atomics with both bf16 elements'
 * counter offsets from one shift+mask, 3: lane-pair 16-bit counters,
 * 4 (default): one 32-bit counter table per CTA with a column per lane,
 * shared by all its warps -- conflict-free, constant increment).
 * exmy_debug_hist_blocks(b) caps the histogram grid at b CTAs (0: auto) so
 * tests reach the counter-overflow flushes with small inputs.  Pass -1 to
 * query.  Return the previous value. */
int exmy_debug_force_generic(int on);
int exmy_debug_hist_mode(int mode);
/* ROWS encode kernel choice: 1 = TMA-staged persistent kernel (bulk copies
 * into a shared-memory ring), 0 = register-pipelined tiles; -1 queries.
 * Returns the previous value. */
int exmy_debug_enc_tma(int on);
/* exmy_encode_rowwise for rows of 9 KB .. 72 KB: 1 = the thread-block-cluster
 * kernel (row-group slabs in distributed shared memory, one HBM read), 0 =
 * the two-pass / two-launch paths (the default: measured faster, DESIGN.md
 * section 12); -1 queries.  Returns the previous value. */
int exmy_debug_rowwise_cluster(int on);
int exmy_debug_hist_blocks(int blocks);

/* Roofline probe, not part of the codec: reads in_bytes
 * (a multiple of 16 KB, 16-byte aligned) and writes out_bytes (a multiple of
 * 16; each 16 KB input chunk's CTA writes its share) with the codec kernels' access shape and no
 * arithmetic, so read 2 B / write 0.875 B per element times the HBM limit of
 * an e3m3 bf16 encode's traffic mix.  Errors: E_SHAPE, E_ARG, E_ALIGN. */
exmy_status exmy_debug_probe(const void *in, int64_t in_bytes, void *out, int64_t out_bytes, void *stream);

/* ------------------------------------------------------- block metadata */
/* Blocks ("a tensor, a row, a column, a sub row or even a 2D
 * tile"; per-row metadata is the paper's quality recipe): the
 * (rows, cols) row-major tensor is tiled by block_rows x block_cols blocks,
 * block_rows | rows and block_cols | cols (else EXMY_E_SHAPE).  Block (i, j)
 * owns metadata byte meta[i * (cols / block_cols) + j] (device memory).
 *   tensor: (rows, cols)   row: (1, cols)   column: (rows, 1)
 *   sub-row of length L: (1, L)   2-D tile: (r, c)
 * Every element is coded exactly as the per-tensor calls would code it with
 * its block's e_max.  The fast kernels need block_cols % 4 == 0 (ROWS
 * encode), % 8 (COLS, and ROWS decode to bf16) and block_rows == 1 or
 * % 8 == 0; other shapes take a scalar kernel with identical results. */
typedef enum { EXMY_SCHEME_MAX_BEFORE = 0, EXMY_SCHEME_MAX_AFTER = 1 } exmy_scheme;

/* Per-block metadata.  MAX_BEFORE: the largest 8-bit
 * biased exponent field of a finite element of the block (the maximum
 * exponent before rounding).  MAX_AFTER: the biased exponent of the block's
 * largest magnitude after rounding it RTNE to y mantissa bits in its own
 * binade (so 3.9 with y=1 gives 129, "it always rounds up to 4.0").  NaN/Inf
 * are ignored; a block with no finite non-zero element gets 0; results are
 * clamped to 254.  Kernels: one warp per block, or for sub-row blocks of
 * <= 32 16-byte vectors (1 x 32, per-row blocks of narrow rows) a segmented
 * reduction over contiguous 16 KB chunks; whole-tensor metadata is
 * exmy_max_exponent / exmy_exponent_histogram. */
exmy_status exmy_block_max_exponent(const void *in, int dtype, int64_t rows, int64_t cols,
                                    int64_t block_rows, int64_t block_cols, int y, int scheme,
                                    uint8_t *meta, void *stream);

/* exmy_quantize / exmy_encode / exmy_decode with block metadata; arguments
 * as the per-tensor calls plus the block shape. */
exmy_status exmy_quantize_blocked(const void *in, void *out, int dtype, int64_t rows, int64_t cols,
                                  int64_t block_rows, int64_t block_cols, int x, int y,
                                  const uint8_t *meta, void *stream);
exmy_status exmy_encode_blocked(const void *in, int dtype, int64_t rows, int64_t cols, int axis,
                                int64_t block_rows, int64_t block_cols, int x, int y,
                                const uint8_t *meta, uint8_t *packed, int64_t *sp_index,
                                uint32_t *sp_bits, uint64_t *sp_count, int64_t sp_capacity,
                                void *stream);
exmy_status exmy_decode_blocked(const uint8_t *packed, int64_t rows, int64_t cols, int axis,
                                int64_t block_rows, int64_t block_cols, int x, int y,
                                const uint8_t *meta, const int64_t *sp_index,
                                const uint32_t *sp_bits, const uint64_t *sp_count,
                                int64_t sp_capacity, void *out, int out_dtype, void *stream);

/* Per-row metadata and encode in one call (the paper's per-row recipe,
 * P:622-627): meta[r] (device, rows bytes) := the row's
 * maximum exponent under `scheme`, then the tensor is encoded with block
 * (1, cols) -- bit-identical to exmy_block_max_exponent + exmy_encode_blocked.
 * ROWS with aligned rows of at most 9216 bytes runs one fused kernel: a
 * CTA stages its row group (8 rows) in shared memory with bulk
 * asynchronous copies (cp.async.bulk on an mbarrier) and computes the 8
 * maxima and the codes from there, so HBM is read once; rows up to 16 KB
 * run a fused kernel that re-reads the rows from L2 (evict_last /
 * evict_first policies); longer rows and COLS take two launches (row maxima,
 * then the blocked encode -- COLS rows of 64..512 columns through the
 * narrow-row kernel).  Measured in DESIGN.md §8b / §12.6. */
exmy_status exmy_encode_rowwise(const void *in, int dtype, int64_t rows, int64_t cols, int axis,
                                int x, int y, int scheme, uint8_t *meta, uint8_t *packed,
                                int64_t *sp_index, uint32_t *sp_bits, uint64_t *sp_count,
                                int64_t sp_capacity, void *stream);

/* Row gather-decode (embedding lookup, "decoding
 * ... during serving ... is performance critical").  Needs the COLS layout,
 * where row r is the contiguous byte range off_j + [r*cols*w_j/8,
 * (r+1)*cols*w_j/8) of every segment.  out[i, :] = decode(row row_index[i])
 * (n_index x cols, fp32/bf16, 16-byte aligned).  meta: the per-tensor byte
 * (meta_per_row = 0) or one byte per row (meta_per_row = 1, block 1 x cols).
 * Row indices must lie in [0, rows) (not checked on the device).  NaN/Inf
 * recorded out of band are NOT restored (decode the tensor for those). */
exmy_status exmy_decode_rows(const uint8_t *packed, int64_t rows, int64_t cols, int x, int y,
                             const uint8_t *meta, int meta_per_row, const int64_t *row_index,
                             int64_t n_index, void *out, int out_dtype, void *stream);

/* ------------------------------------------------ float scaling (reading D23)
 * Fig. 2's third scheme, "float scaling with maximum exponent of 127"
 * ("an additional bfloat16 or float32 scaling factor").
 * Each block_rows x block_cols block carries one fp32 metadata value, its
 * largest finite magnitude amax (0 if it has none); codes live on the
 * e_max = 127 grid, whose top is G (2 - 2^-y for x >= 1).  With amax =
 * A1 * 2^p, A1 in [1,2):
 *   encode  u = RN32(v * RN32(G/A1) * 2^-p), code = the e_max-127 code of u
 *           (the fp32 scaling factor RN32(G/A1))
 *   decode  out = RN32(g * amax / G), g the code's exact value at e_max 127
 *           (exact product and quotient rounded once, fp32 subnormals
 *           included; a zero result keeps the code's sign); bf16 = RN16(out)
 *           (reading D24).  Kernels: FMUL + FFMA with a two-term amax/G for
 *           results >= 2^-100, integer evaluation below that and for x = 8.
 * so each block's maximum decodes to exactly amax ("captures the largest
 * value in the block accurately").  Layout, specials and error codes
 * as exmy_encode_blocked / exmy_decode_blocked; scale is device memory,
 * (rows/block_rows) * (cols/block_cols) floats in block-row-major order. */

/* scale[b] := max |finite v| over block b (fp32).  One warp per block, or
 * for sub-row blocks of <= 32 16-byte vectors a segmented reduction (a
 * thread per vector, the block's lanes combined by shuffles). */
exmy_status exmy_block_float_scale(const void *in, int dtype, int64_t rows, int64_t cols,
                                   int64_t block_rows, int64_t block_cols, float *scale,
                                   void *stream);

/* Emulation: out = decode(encode(v)) in v's dtype, NaN/Inf passed through.
 * in/out 16-byte aligned and rows*cols a multiple of 8 (bf16) / 4 (fp32),
 * else E_ALIGN. */
exmy_status exmy_quantize_fs(const void *in, void *out, int dtype, int64_t rows, int64_t cols,
                             int64_t block_rows, int64_t block_cols, int x, int y,
                             const float *scale, void *stream);
exmy_status exmy_encode_fs(const void *in, int dtype, int64_t rows, int64_t cols, int axis,
                           int64_t block_rows, int64_t block_cols, int x, int y,
                           const float *scale, uint8_t *packed, int64_t *sp_index,
                           uint32_t *sp_bits, uint64_t *sp_count, int64_t sp_capacity,
                           void *stream);
exmy_status exmy_decode_fs(const uint8_t *packed, int64_t rows, int64_t cols, int axis,
                           int64_t block_rows, int64_t block_cols, int x, int y,
                           const float *scale, const int64_t *sp_index, const uint32_t *sp_bits,
                           const uint64_t *sp_count, int64_t sp_capacity, void *out,
                           int out_dtype, void *stream);

/* ----------------------------------- fused encode + all-gather (push)
 * SURVEY 8(f) row 2 ("encode before ... network
 * communication"; P:343-344 shards reconstruct independently).  The caller
 * (one rank) encodes its row shard: rows [row0, row0+rows) of a
 * (total_rows, cols) tensor, ROWS layout, under the GLOBAL metadata byte
 * `meta`, and the kernel writes the shard's packed bytes straight into each
 * of the `ndst` destination buffers (a host array of device pointers, each
 * total_rows*cols*k/8 bytes: normally every rank's gathered buffer, peers'
 * mapped over NVLink through CUDA IPC / symmetric memory) at the shard's
 * global offsets.  Once every rank has run (and the group has synchronised)
 * every buffer holds exactly exmy_encode of the whole tensor: the
 * all-gather happens in the encode's own stores.  rows, row0, total_rows
 * multiples of 8, cols % 4 == 0, 1 <= ndst <= 8; destination segments
 * aligned as for exmy_encode's vector path, else E_ALIGN.  Specials: the
 * shard's NaN/Inf with GLOBAL element indices, sorted. */
exmy_status exmy_encode_push(const void *in, int dtype, int64_t rows, int64_t cols, int64_t row0,
                             int64_t total_rows, int x, int y, const uint8_t *meta,
                             uint8_t *const *dst, int ndst, int64_t *sp_index, uint32_t *sp_bits,
                             uint64_t *sp_count, int64_t sp_capacity, void *stream);

/* NVLS multicast form of exmy_encode_push (P:298,
 * P:536): identical arguments except one destination, `mc_dst`, a multicast
 * address of the gathered packed buffer (e.g. torch symmetric memory's
 * multicast_ptr) bound on every GPU of the node.  Each 4 / 8 / 16-byte
 * segment store is one multimem.st, replicated to every bound GPU by the
 * NVSwitch, instead of one store per peer.  Same bytes as exmy_encode_push
 * into every bound buffer; the caller synchronises (stream + barrier) before
 * peers read.  E_ALIGN as exmy_encode_push. */
exmy_status exmy_encode_push_multicast(const void *in, int dtype, int64_t rows, int64_t cols,
                                       int64_t row0, int64_t total_rows, int x, int y, const uint8_t *meta,
                                       uint8_t *mc_dst, int64_t *sp_index, uint32_t *sp_bits,
                                       uint64_t *sp_count, int64_t sp_capacity, void *stream);

/* Pull decode, the mirror of exmy_encode_push ("decode
 * reads peers' packed shards over NVLink"): decodes the whole
 * (nsrc * shard_rows, cols) tensor whose row shard s is the independent
 * packed tensor (ROWS layout, shard_rows x cols) at srcs[s] -- on a node,
 * every rank's packed shard mapped into this process -- so the all-gather of
 * packed bytes happens in the decode's loads.  Same per-tensor metadata for
 * every shard (the global e_max); 1 <= nsrc <= 8, shard_rows % 8 == 0;
 * out (fp32 / bf16) 16-byte aligned with cols a multiple of 4 / 8, shard
 * segments aligned as exmy_decode's vector path, else E_ALIGN.  Out-of-band
 * NaN/Inf are not restored (as exmy_decode with no specials). */
exmy_status exmy_decode_pull(const uint8_t *const *srcs, int nsrc, int64_t shard_rows, int64_t cols,
                             int x, int y, const uint8_t *meta, void *out, int out_dtype, void *stream);

/* ------------------------------------------ grouped launch (tensor table)
 * a model is many tensors (Llama-3 8B: 291, P:600-606
 * "the weights of Llama"), each compressed under its own per-tensor
 * metadata.  These calls run the per-tensor max exponent,
 * encode (ROWS) and decode over a whole table in a constant number of
 * launches, bit-identical to calling exmy_max_exponent / exmy_encode /
 * exmy_decode on each entry.
 *
 * Usage: fill exmy_group_entry[n] (host), call exmy_group_plan into a host
 * buffer of exmy_group_plan_bytes(n) bytes, copy those bytes once to device
 * memory (16-byte aligned), then pass both copies to the group calls (the
 * host copy sizes the launch, the device copy is what the kernels read).  A
 * plan stays valid while its buffers do and can be captured in a CUDA
 * graph.  All entries share one input dtype, one format (x, y) and one
 * output dtype. */
typedef struct exmy_group_entry {
    const void *in;           /* encode / max: rows*cols elements (dtype), 16-byte aligned; may be NULL for decode-only plans */
    void *out;                /* decode: rows*cols elements (out_dtype), 16-byte aligned; may be NULL for encode-only plans */
    uint8_t *packed;          /* rows*cols*k/8 bytes, ROWS layout (exmy_encode's), 16-byte aligned */
    uint8_t *meta;            /* device, one byte: the tensor's max biased exponent (written by exmy_group_max_exponent) */
    int64_t *sp_index;        /* specials as in exmy_encode / exmy_decode (per entry); all may be NULL / 0 */
    uint32_t *sp_bits;
    uint64_t *sp_count;
    int64_t sp_capacity;
    int64_t rows, cols;       /* rows % 8 == 0, cols % 4 == 0 (ROWS layout, 8x4-element tiles) */
} exmy_group_entry;

/* Size of the plan for n entries (n >= 1). */
size_t exmy_group_plan_bytes(int n);

/* Validate the table and write the plan into `plan` (host, plan_bytes >=
 * exmy_group_plan_bytes(n)).  dtype: input dtype; out_dtype: decode output.
 * Errors: E_DTYPE, E_FORMAT, E_SHAPE (rows%8, cols%4, n < 1), E_ALIGN
 * (an entry pointer not 16-byte aligned), E_ARG (NULL packed/meta, plan too
 * small), E_CAPACITY (negative capacity).  Entries with rows*cols == 0 are
 * allowed and skipped. */
exmy_status exmy_group_plan(const exmy_group_entry *entries, int n, int dtype, int x, int y,
                            int out_dtype, void *plan, size_t plan_bytes);

/* Same table, per-row metadata ("quantized the weights with the
 * maximum exponent of each row"): entry i's `meta` points to rows bytes
 * (8-byte aligned), byte r = row r's max biased exponent; the group calls
 * then run per row, bit-identical to exmy_block_max_exponent (1 x cols,
 * scheme 0) / exmy_encode_blocked / exmy_decode_blocked (ROWS) per entry.
 * Extra requirement: cols % 8 == 0 (E_SHAPE); meta not 8-byte aligned:
 * E_ALIGN.  exmy_group_max_exponent on such a plan is one launch. */
exmy_status exmy_group_plan_rows(const exmy_group_entry *entries, int n, int dtype, int x, int y,
                                 int out_dtype, void *plan, size_t plan_bytes);

/* meta of every entry := its max biased exponent over finite elements
 * (== exmy_max_exponent / the top histogram bin; 0 for all-zero tensors).
 * Two launches (clear, reduce).  Needs every entry's `in`. */
exmy_status exmy_group_max_exponent(const void *plan_host, const void *plan_device, void *stream);

/* Encode every entry (ROWS) under its meta byte; per-entry specials as in
 * exmy_encode (counts cleared, list sorted by index).  Three launches. */
exmy_status exmy_group_encode(const void *plan_host, const void *plan_device, void *stream);

/* Per-row plans only (else E_ARG): every row's byte (max before rounding)
 * AND the encode in one call, == exmy_group_max_exponent + exmy_group_encode
 * on the same plan.  Entries whose rows are <= 9216 bytes (bf16 <= 4608
 * columns, fp32 <= 2304) and a multiple of 16 bytes are read from HBM once:
 * each row group is staged in shared memory by bulk asynchronous copies,
 * its 8 maxima and its codes computed from there (like exmy_encode_rowwise);
 * the other entries take the two passes.  Two to five launches. */
exmy_status exmy_group_encode_rowwise(const void *plan_host, const void *plan_device, void *stream);

/* Decode every entry into its `out` (+ out-of-band specials).  Two launches. */
exmy_status exmy_group_decode(const void *plan_host, const void *plan_device, void *stream);

/* ------------------------------------------------ checkpoint container
 * "encoding and decoding tensors and checkpoints"
 * (P:17-18); file layout after S:369-378 (little-endian):
 *   "EXMY" | version u8 = 2 | entry_count u32, then per tensor
 *   name_len u16 | name | rank u8 | dims u32 x rank | x u8 | y u8 | scheme u8
 *   (0 max-before, 1 max-after, 2 float-scale) | block_kind u8 (0 tensor,
 *   1 row, 2 col, 3 sub-row + L u32, 4 tile + r u32, c u32) | flags u8 (bit0
 *   scale, bit1 specials, bit2 COLS packing, bit3 bf16 source) | (offset u64,
 *   length u64) of metadata, each packed segment (descending width), scale
 *   array, specials | crc32 u32 (IEEE) of the tensor's payload bytes;
 *   payloads follow the manifest, one tensor's sections contiguous.
 * Specials are stored as count (u64 index, u32 fp32 pattern) records
 * (version 2; version-1 files stored the indices, then the patterns, and
 * are still read).  Host code (pread / pwrite); every buffer here is HOST
 * memory. */
typedef struct exmy_ckpt_tensor {
    const char *name;              /* unique, <= 65535 bytes */
    int rank;                      /* 0..8 */
    int64_t dims[8];               /* each < 2^32; prod(dims) % 8 == 0 */
    int x, y, scheme, block_kind;
    int64_t block_p0, block_p1;    /* sub-row L / tile (r, c) */
    int axis;                      /* EXMY_AXIS_ROWS / COLS */
    int src_dtype;                 /* EXMY_F32 / EXMY_BF16 */
    const void *meta;              /* metadata bytes (u8 e_max per block) */
    int64_t meta_bytes;
    const void *packed;            /* the n*k/8 packed bytes, segments in order */
    int64_t packed_bytes;
    const void *scale;             /* float-scale metadata (fp32 per block) or NULL */
    int64_t scale_bytes;
    const int64_t *sp_index;       /* specials (sorted) */
    const uint32_t *sp_bits;
    int64_t specials_count;
} exmy_ckpt_tensor;

typedef struct exmy_ckpt exmy_ckpt;   /* opaque reader */

/* Write n tensors; returns the file size in bytes, or -status (E_ARG,
 * E_SHAPE: packed_bytes != prod(dims)*k/8, E_IO).  n = 0 writes a valid
 * empty container. */
int64_t exmy_ckpt_write(const char *path, const exmy_ckpt_tensor *tensors, int n);

/* Open: reads the header and manifest only (E_IO, E_CONTAINER for bad
 * magic / version / truncated manifest / sections outside the file or
 * overlapping / segment lengths != prod(dims)*w/8 / metadata or scale
 * lengths that do not match the block grid / allocation failure). */
exmy_status exmy_ckpt_open(const char *path, exmy_ckpt **out);
int exmy_ckpt_count(const exmy_ckpt *h);
/* Tensor i's manifest entry: sizes filled, data pointers NULL; `name` stays
 * valid until exmy_ckpt_close. */
exmy_status exmy_ckpt_info(const exmy_ckpt *h, int i, exmy_ckpt_tensor *info);
/* index of the tensor called `name`, -1 if none */
int exmy_ckpt_find(const exmy_ckpt *h, const char *name);
/* Lazy read of tensor i: each non-NULL destination (host) receives exactly
 * that section (sizes from exmy_ckpt_info); no other tensor's bytes are
 * touched.  No CRC check (see exmy_ckpt_verify); a specials index outside
 * [0, prod(dims)) returns E_CONTAINER. */
exmy_status exmy_ckpt_read(exmy_ckpt *h, int i, void *meta, void *packed, void *scale,
                           int64_t *sp_index, uint32_t *sp_bits);
/* Recompute tensor i's CRC32 over its payload: EXMY_OK or E_CHECKSUM. */
exmy_status exmy_ckpt_verify(exmy_ckpt *h, int i);
/* payload bytes read through this handle so far (instrumentation) */
int64_t exmy_ckpt_bytes_read(const exmy_ckpt *h);
void exmy_ckpt_close(exmy_ckpt *h);

/* Embedding bag over a COLS-packed table ("decode fused
 * into a ... embedding-bag prologue"; config 5; reading D25).  out[b, :] =
 * the fp32 pool of rows indices[offsets[b] .. offsets[b+1]) -- each row
 * decoded exactly as exmy_decode does, accumulated in fp32 in index order
 * (acc + v, or fma(weights[i], v, acc) when weights != NULL); mode 0 sum,
 * 1 mean (divide by the bag size); empty bags give +0.  Decoded rows never
 * reach HBM.  indices / offsets (nbags + 1 entries) / weights are device
 * arrays; meta is one byte (meta_per_row = 0) or one per row; out is
 * (nbags, cols) fp32, 16-byte aligned; packed 8-byte aligned.  Row indices
 * must lie in [0, rows) (not checked).  Out-of-band NaN/Inf are not
 * restored (as exmy_decode_rows). */
exmy_status exmy_embedding_bag(const uint8_t *packed, int64_t rows, int64_t cols, int x, int y,
                               const uint8_t *meta, int meta_per_row, const int64_t *indices,
                               const int64_t *offsets, int64_t nbags, const float *weights,
                               int mode, float *out, void *stream);

/* Decode fused into a matrix-vector product ("decode
 * fused into the consumer"; serving decode is "performance critical",
 * P:296-298; reading D26).  out[i, n] = sum_c act[i, c] * W[n, c] for the
 * ROWS-packed weight matrix W (rows x cols, k = 1+x+y <= 8) and m fp32
 * activation rows act (m x cols, row-major, 16-byte aligned); out is fp32
 * (m x rows, row-major).  The decoded W never reaches HBM: each pass over
 * <= 8 activation rows reads the packed bytes once.  meta: one device byte
 * (per tensor) or `rows` bytes (meta_per_row = 1, the (1, cols) blocks of
 * exmy_block_max_exponent / exmy_encode_rowwise).  Sums are fp32 in a fixed
 * order (see exmy_gemv.cuh): not bit-identical to another summation order;
 * the tests bound the error by the fp32 dot-product bound.  NaN/Inf weights
 * from the encode's specials list (sp_index / sp_bits / sp_count /
 * sp_capacity as written by exmy_encode; capacity 0: none) are applied
 * afterwards.  Requires rows % 8 == 0, cols % 4 == 0, packed 16-byte
 * aligned.  EXMY_E_FORMAT for k = 9. */
/* exmy_gemv kernel choice: 1 (default) = packed bytes staged in shared
 * memory by bulk asynchronous copies when cols % 16 == 0, 0 = the
 * register-pipelined kernel for every shape; -1 queries.  Returns the
 * previous value. */
int exmy_debug_gemv_bulk(int on);
exmy_status exmy_gemv(const uint8_t *packed, int64_t rows, int64_t cols, int x, int y,
                      const uint8_t *meta, int meta_per_row, const int64_t *sp_index,
                      const uint32_t *sp_bits, const unsigned long long *sp_count, int64_t sp_capacity,
                      const float *act, int64_t m, float *out, void *stream);

/* ------------------------------------------------ host-buffer conveniences */

/* End-to-end encode of a HOST tensor (pinned memory recommended): H2D copy
 * into `dev_in` (caller-owned device scratch of n*esize bytes), histogram ->
 * e_max -> encode into `dev_packed` (device, n*k/8 bytes), D2H copy of the
 * packed bytes into `host_packed` and of the metadata byte into
 * `host_meta`.  `dev_hist` (uint64[256]) and `dev_meta` (uint8) are device
 * scratch; specials as in exmy_encode (device arrays).  Asynchronous on
 * `stream`: host buffers are valid after the stream syncs. */
exmy_status exmy_encode_host(const void *host_in, int dtype, int64_t rows, int64_t cols,
                             int axis, int x, int y,
                             void *dev_in, uint64_t *dev_hist, uint8_t *dev_meta,
                             uint8_t *dev_packed, int64_t *sp_index, uint32_t *sp_bits,
                             uint64_t *sp_count, int64_t sp_capacity,
                             uint8_t *host_packed, uint8_t *host_meta, void *stream);

/* End-to-end decode of HOST packed bytes: H2D copy into `dev_packed`, decode
 * into `dev_out`, D2H copy into `host_out`.  meta is a device byte. */
exmy_status exmy_decode_host(const uint8_t *host_packed, int64_t rows, int64_t cols, int axis,
                             int x, int y, const uint8_t *meta,
                             const int64_t *sp_index, const uint32_t *sp_bits,
                             const uint64_t *sp_count, int64_t sp_capacity,
                             uint8_t *dev_packed, void *dev_out, int out_dtype,
                             void *host_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* EXMY_H */
