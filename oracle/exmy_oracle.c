/*
 * exmy_oracle.c -- plain, slow, scalar CPU oracle for the eXmY tensor codec.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may link, load or
 * call this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code, header,
 * table or constant with paper_2405_13938_b200/csrc (the CUDA path).
 *
 * Every function follows the plain definition in the paper (P:n = line n of
 * PAPER.md, S:n = line n of SPEC.md) or, where the paper is silent, the
 * reading numbered Dn in DESIGN.md "Readings".  No blocking, no bit tricks:
 *
 *   quantize  = the grid point nearest to the exact input value, ties to the
 *               code whose LSB is 0 (y = 0: to the even fp32 exponent),
 *               saturating at the largest magnitude (
 *               D5-D8).  Implemented as: enumerate all
 *               2^(k-1) magnitude codes, compute their exact values in fp64,
 *               sort them (qsort, a library primitive), binary-search the two
 *               neighbours of |v| and compare |v| with their exact midpoint.
 *   code value = (-1)^s (2^y+m) 2^(e-bias-y) for e>=1, (-1)^s m 2^(1-bias-y)
 *               for e=0 or x=0 (Table 1, subnormals P:172-175; D3),
 *               with bias = 2^x + 126 - e_max (metadata = maximum biased
 *               exponent; D1).
 *   pack      = power-of-2 decomposition of k, widest segment takes the most
 *               significant code bits, element i of a group at bits
 *               [w*i, w*i+w) of a little-endian 8w-bit container
 *               (Fig. 3; D12-D16).
 *
 * Exactness of the fp64 arithmetic used here: every fp32 value and every grid
 * value of a format with x<=8, y<=23, e_max in [0,254] is a normal fp64
 * number (smallest grid quantum 2^(1-382-23) > 2^-1022), the sum of two
 * adjacent grid values has at most y+3 significant bits, and /2 is exact; so
 * every comparison below is exact.  Values are built with ldexp from
 * integers, never by reinterpreting host floats, so host FTZ/DAZ modes cannot
 * matter.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#include "exmy_oracle.h"

/* ---------------------------------------------------------------- formats */

int oracle_format_valid(int x, int y, int e_max)
{
    if (x < 0 || x > 8 || y < 0 || y > 23) return 0;
    if (1 + x + y > ORACLE_MAX_K) return 0;
    if (e_max < 0 || e_max > 254) return 0;           /* D4 */
    return 1;
}

/* bias from metadata, D1: the top exponent code 2^x-1 sits at fp32 biased
 * exponent e_max, i.e. (2^x - 1) - bias + 127 = e_max. */
int oracle_bias(int x, int e_max) { return (1 << x) + 126 - e_max; }

/* Exact value of a magnitude code (sign bit excluded), Table 1 + P:172-175. */
double oracle_code_magnitude(uint32_t mag, int x, int y, int e_max)
{
    int bias = oracle_bias(x, e_max);
    uint32_t e = (x == 0) ? 0u : (mag >> y);
    uint32_t m = mag & ((1u << y) - 1u);
    if (e == 0)                                   /* subnormal / x=0 (D3) */
        return ldexp((double)m, 1 - bias - y);
    return ldexp((double)((1u << y) + m), (int)e - bias - y);
}

double oracle_code_value(uint32_t code, int x, int y, int e_max)
{
    int k = 1 + x + y;
    uint32_t s = (code >> (k - 1)) & 1u;
    double a = oracle_code_magnitude(code & ((1u << (k - 1)) - 1u), x, y, e_max);
    return s ? -a : a;   /* -0.0 for the negative zero code (D10) */
}

/* ------------------------------------------------------------- the grid */

typedef struct { double v; uint32_t mag; } grid_pt;

static int cmp_grid(const void *a, const void *b)
{
    double va = ((const grid_pt *)a)->v, vb = ((const grid_pt *)b)->v;
    return (va > vb) - (va < vb);
}

typedef struct { grid_pt *pts; uint32_t n; int x, y, e_max; } grid;

static int grid_build(grid *g, int x, int y, int e_max)
{
    g->n = 1u << (x + y);
    g->x = x; g->y = y; g->e_max = e_max;
    g->pts = (grid_pt *)malloc(sizeof(grid_pt) * g->n);
    if (!g->pts) return -1;
    for (uint32_t c = 0; c < g->n; ++c) {
        g->pts[c].v = oracle_code_magnitude(c, x, y, e_max);
        g->pts[c].mag = c;
    }
    qsort(g->pts, g->n, sizeof(grid_pt), cmp_grid);
    return 0;
}

static void grid_free(grid *g) { free(g->pts); g->pts = NULL; }

/* exact real value of an fp32 bit pattern (finite only) */
static double f32_value(uint32_t u)
{
    uint32_t E = (u >> 23) & 0xFFu, f = u & 0x7FFFFFu;
    double a = (E == 0) ? ldexp((double)f, -149)
                        : ldexp((double)(f | 0x800000u), (int)E - 150);
    return (u >> 31) ? -a : a;
}

/* nearest magnitude code to |v| (v finite), D5-D8 */
static uint32_t grid_nearest(const grid *g, double a)
{
    /* i = number of grid points with value <= a  (a >= 0 and grid[0] = 0) */
    uint32_t lo = 0, hi = g->n;
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (g->pts[mid].v <= a) lo = mid + 1; else hi = mid;
    }
    uint32_t i = lo;                 /* >= 1 */
    const grid_pt *below = &g->pts[i - 1];
    if (below->v == a) return below->mag;
    if (i == g->n) return below->mag;             /* above max: saturate (D7) */
    const grid_pt *above = &g->pts[i];
    double midpoint = (below->v + above->v) / 2.0;   /* exact, see header */
    if (a < midpoint) return below->mag;
    if (a > midpoint) return above->mag;
    /* tie (D6): for y >= 1 the code whose LSB -- the mantissa LSB -- is 0
     * (round-to-nearest-even).  For y = 0 there is no mantissa bit: the
     * paper's Eigen RTNE extended to zero mantissa bits keeps the
     * fp32 pattern whose last kept bit, the exponent LSB, is 0, i.e. the
     * neighbour whose fp32 biased exponent is even (the same rule as D22's
     * "after rounding" exponent).  Zero (exponent field 0) wins the tie with
     * the smallest non-zero value (D8). */
    if (g->y == 0) {
        if (below->v == 0.0) return below->mag;
        int e;
        (void)frexp(below->v, &e);                       /* below = 2^(e-1) */
        return ((e - 1 + 127) & 1) ? above->mag : below->mag;
    }
    return (below->mag & 1u) ? above->mag : below->mag;
}

/* ------------------------------------------- exact value -> fp32 / bf16 */

/* RTNE of an exact fp64 value to a binary format with p significand bits
 * (incl. the implicit bit) and 8 exponent bits, bias 127 (fp32: p=24, bf16:
 * p=8).  Returns the bit pattern in the low 1+8+(p-1) bits.  Plain
 * round-to-nearest-even on the quantum 2^(max(E,-126) - (p-1)). */
static uint32_t round_to_ieee8(double v, int p)
{
    uint32_t sign = signbit(v) ? 1u : 0u;
    double a = fabs(v);
    uint32_t sbit = sign << (p - 1 + 8);
    if (a == 0.0) return sbit;
    int e;
    (void)frexp(a, &e);               /* a = f * 2^e, f in [0.5,1) => E = e-1 */
    int E = e - 1;
    if (E < -126) E = -126;
    int qe = E - (p - 1);             /* exponent of the output quantum */
    double s = ldexp(a, -qe);         /* exact scaling: s < 2^p */
    double fl = floor(s);
    double frac = s - fl;             /* exact */
    uint64_t r = (uint64_t)fl;
    if (frac > 0.5 || (frac == 0.5 && (r & 1u))) r += 1;
    if (r == 0) return sbit;
    if (r == (1ull << p)) { r >>= 1; qe += 1; }   /* carry into next binade */
    uint32_t bits;
    if (r < (1ull << (p - 1))) {
        bits = (uint32_t)r;           /* subnormal output (qe == -126-(p-1)) */
    } else {
        int ef = qe + (p - 1) + 127;
        if (ef >= 255) bits = 0xFFu << (p - 1);   /* overflow -> Inf (never hit for k<=9) */
        else bits = ((uint32_t)ef << (p - 1)) | (uint32_t)(r - (1ull << (p - 1)));
    }
    return sbit | bits;
}

uint32_t oracle_round_f32(double v) { return round_to_ieee8(v, 24); }
uint16_t oracle_round_bf16(double v) { return (uint16_t)round_to_ieee8(v, 8); }

/* ------------------------------------------------------ element codecs */

static int is_special(uint32_t u) { return ((u >> 23) & 0xFFu) == 0xFFu; }

/* k-bit code of the finite fp32 pattern u: sign bit always from u (D10). */
static uint32_t encode_finite(const grid *g, uint32_t u)
{
    int k = 1 + g->x + g->y;
    uint32_t s = u >> 31;
    double a = fabs(f32_value(u));
    return (s << (k - 1)) | grid_nearest(g, a);
}

/* per-element codes without packing (specials -> code 0, flagged) */
int oracle_encode_codes(const void *in, int dtype, int64_t n, int x, int y, int e_max,
                        uint16_t *codes, uint8_t *special)
{
    if (!oracle_format_valid(x, y, e_max)) return -1;
    grid g;
    if (grid_build(&g, x, y, e_max)) return -1;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t u = (dtype == ORACLE_BF16) ? ((uint32_t)((const uint16_t *)in)[i] << 16)
                                            : ((const uint32_t *)in)[i];
        special[i] = (uint8_t)is_special(u);
        codes[i] = special[i] ? 0 : (uint16_t)encode_finite(&g, u);
    }
    grid_free(&g);
    return 0;
}

int oracle_encode_element(uint32_t u, int x, int y, int e_max, uint32_t *code)
{
    if (!oracle_format_valid(x, y, e_max)) return -1;
    if (is_special(u)) { *code = 0; return 1; }
    grid g;
    if (grid_build(&g, x, y, e_max)) return -1;
    *code = encode_finite(&g, u);
    grid_free(&g);
    return 0;
}

/* ------------------------------------------------------------ histogram */

/* histogram of the 8-bit biased exponent field; bin 255 holds
 * NaN/Inf (D18), bin 0 holds zeros and input subnormals (D11). */
void oracle_histogram(const void *in, int dtype, int64_t n, uint64_t hist[256])
{
    for (int64_t i = 0; i < n; ++i) {
        uint32_t u = (dtype == ORACLE_BF16) ? ((uint32_t)((const uint16_t *)in)[i] << 16)
                                            : ((const uint32_t *)in)[i];
        hist[(u >> 23) & 0xFFu] += 1;
    }
}

/* metadata = maximum biased exponent before rounding. */
int oracle_emax(const uint64_t hist[256])
{
    for (int b = 254; b >= 0; --b)
        if (hist[b]) return b;
    return 0;
}

/* P:473-478 (D19): the smallest x whose 2^x-1 normal exponent codes, placed
 * at the top of the populated range, cover at least (1-budget) of the
 * non-zero finite values. */
int oracle_choose_x(const uint64_t hist[256], double budget)
{
    int e_max = oracle_emax(hist);
    uint64_t total = 0;
    for (int b = 1; b <= 254; ++b) total += hist[b];
    for (int x = 0; x <= 8; ++x) {
        uint64_t covered = 0;
        for (int b = e_max - (1 << x) + 2; b <= e_max; ++b)
            if (b >= 1) covered += hist[b];
        if ((double)covered >= (1.0 - budget) * (double)total) return x;
    }
    return 8;
}

/* ------------------------------------------------------------- quantize */

static uint32_t load_u32(const void *in, int dtype, int64_t i)
{
    return (dtype == ORACLE_BF16) ? ((uint32_t)((const uint16_t *)in)[i] << 16)
                                  : ((const uint32_t *)in)[i];
}

static void store_value(void *out, int dtype, int64_t i, double v)
{
    if (dtype == ORACLE_BF16) ((uint16_t *)out)[i] = oracle_round_bf16(v);
    else ((uint32_t *)out)[i] = oracle_round_f32(v);
}

/* Emulation: fp -> nearest grid value -> same container dtype,
 * NaN/Inf passed through bit-exactly (D9, D21). */
int oracle_quantize(const void *in, void *out, int dtype, int64_t n, int x, int y, int e_max)
{
    if (!oracle_format_valid(x, y, e_max)) return -1;
    grid g;
    if (grid_build(&g, x, y, e_max)) return -1;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t u = load_u32(in, dtype, i);
        if (is_special(u)) {
            if (dtype == ORACLE_BF16) ((uint16_t *)out)[i] = ((const uint16_t *)in)[i];
            else ((uint32_t *)out)[i] = u;
            continue;
        }
        uint32_t code = encode_finite(&g, u);
        store_value(out, dtype, i, oracle_code_value(code, x, y, e_max));
    }
    grid_free(&g);
    return 0;
}

/* --------------------------------------------------------- bit packing */

int oracle_segments(int k, int widths[4], int64_t n, int64_t offsets[4])
{
    int ns = 0;
    int64_t off = 0;
    for (int w = 8; w >= 1; w >>= 1) {
        if (k & w) {
            widths[ns] = w;
            if (offsets) offsets[ns] = off;
            off += n * w / 8;
            ++ns;
        }
    }
    return ns;
}

/* element index (row-major) of lane i of container idx */
static int64_t lane_element(int64_t idx, int i, int64_t rows, int64_t cols, int axis)
{
    (void)rows;
    if (axis == ORACLE_ROWS) {          /* container (g,c): elements (8g+i, c) */
        int64_t g = idx / cols, c = idx % cols;
        return (8 * g + i) * cols + c;
    } else {                            /* container (r,g): elements (r, 8g+i) */
        int64_t gpr = cols / 8;
        int64_t r = idx / gpr, g = idx % gpr;
        return r * cols + 8 * g + i;
    }
}

int oracle_shape_ok(int64_t rows, int64_t cols, int axis)
{
    if (rows < 0 || cols < 0) return 0;
    if (axis == ORACLE_ROWS) return rows % 8 == 0;
    if (axis == ORACLE_COLS) return cols % 8 == 0;
    return 0;
}

/* P:311-353, Fig. 3; D12-D16.  codes are uint16 k-bit codes, row-major. */
int oracle_pack(const uint16_t *codes, int64_t rows, int64_t cols, int axis, int k, uint8_t *packed)
{
    if (k < 1 || k > ORACLE_MAX_PACK_K || !oracle_shape_ok(rows, cols, axis)) return -1;
    int64_t n = rows * cols;
    int widths[4]; int64_t offs[4];
    int ns = oracle_segments(k, widths, n, offs);
    int hi = k;
    for (int j = 0; j < ns; ++j) {
        int w = widths[j], lo = hi - w;
        uint32_t fmask = (1u << w) - 1u;
        uint8_t *seg = packed + offs[j];
        if (w == 8) {                   /* D15: byte passthrough, element order */
            for (int64_t e = 0; e < n; ++e) seg[e] = (uint8_t)((codes[e] >> lo) & 0xFFu);
        } else {
            int64_t ncont = n / 8;
            for (int64_t idx = 0; idx < ncont; ++idx) {
                uint32_t cont = 0;
                for (int i = 0; i < 8; ++i) {
                    uint32_t field = ((uint32_t)codes[lane_element(idx, i, rows, cols, axis)] >> lo) & fmask;
                    cont |= field << (w * i);
                }
                for (int b = 0; b < w; ++b)          /* little-endian container */
                    seg[idx * w + b] = (uint8_t)(cont >> (8 * b));
            }
        }
        hi = lo;
    }
    return 0;
}

int oracle_unpack(const uint8_t *packed, int64_t rows, int64_t cols, int axis, int k, uint16_t *codes)
{
    if (k < 1 || k > ORACLE_MAX_PACK_K || !oracle_shape_ok(rows, cols, axis)) return -1;
    int64_t n = rows * cols;
    int widths[4]; int64_t offs[4];
    int ns = oracle_segments(k, widths, n, offs);
    for (int64_t e = 0; e < n; ++e) codes[e] = 0;
    int hi = k;
    for (int j = 0; j < ns; ++j) {
        int w = widths[j], lo = hi - w;
        uint32_t fmask = (1u << w) - 1u;
        const uint8_t *seg = packed + offs[j];
        if (w == 8) {
            for (int64_t e = 0; e < n; ++e) codes[e] |= (uint16_t)((uint32_t)seg[e] << lo);
        } else {
            int64_t ncont = n / 8;
            for (int64_t idx = 0; idx < ncont; ++idx) {
                uint32_t cont = 0;
                for (int b = 0; b < w; ++b) cont |= (uint32_t)seg[idx * w + b] << (8 * b);
                for (int i = 0; i < 8; ++i) {
                    uint32_t field = (cont >> (w * i)) & fmask;
                    codes[lane_element(idx, i, rows, cols, axis)] |= (uint16_t)(field << lo);
                }
            }
        }
        hi = lo;
    }
    return 0;
}

/* --------------------------------------------------------- encode/decode */

/* Type conversion then bit packing.  NaN/Inf are kept out of
 * band (D9): code 0 in the packed stream plus (index, fp32 bits)
 * in ascending index order.  Returns the number of specials (all of them,
 * even beyond capacity), or -1 on invalid arguments. */
int64_t oracle_encode(const void *in, int dtype, int64_t rows, int64_t cols, int axis,
                      int x, int y, int e_max, uint8_t *packed,
                      int64_t *sp_index, uint32_t *sp_bits, int64_t sp_capacity)
{
    if (!oracle_format_valid(x, y, e_max) || !oracle_shape_ok(rows, cols, axis)) return -1;
    if (1 + x + y > ORACLE_MAX_PACK_K) return -1;
    int64_t n = rows * cols;
    uint16_t *codes = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(n ? n : 1));
    if (!codes) return -1;
    grid g;
    if (grid_build(&g, x, y, e_max)) { free(codes); return -1; }
    int64_t ns = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t u = load_u32(in, dtype, i);
        if (is_special(u)) {
            codes[i] = 0;
            if (ns < sp_capacity) { sp_index[ns] = i; sp_bits[ns] = u; }
            ++ns;
        } else {
            codes[i] = (uint16_t)encode_finite(&g, u);
        }
    }
    grid_free(&g);
    oracle_pack(codes, rows, cols, axis, 1 + x + y, packed);
    free(codes);
    return ns;
}

/* Unpack then code -> exact value -> RTNE to out dtype (D21); specials are
 * written back from their original fp32 bits (bf16 out: top 16 bits, quiet
 * bit forced if a NaN payload would vanish, D9). */
int oracle_decode(const uint8_t *packed, int64_t rows, int64_t cols, int axis,
                  int x, int y, int e_max,
                  const int64_t *sp_index, const uint32_t *sp_bits, int64_t sp_count,
                  void *out, int out_dtype)
{
    if (!oracle_format_valid(x, y, e_max) || !oracle_shape_ok(rows, cols, axis)) return -1;
    if (1 + x + y > ORACLE_MAX_PACK_K) return -1;
    int64_t n = rows * cols;
    uint16_t *codes = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(n ? n : 1));
    if (!codes) return -1;
    oracle_unpack(packed, rows, cols, axis, 1 + x + y, codes);
    for (int64_t i = 0; i < n; ++i)
        store_value(out, out_dtype, i, oracle_code_value(codes[i], x, y, e_max));
    free(codes);
    for (int64_t j = 0; j < sp_count; ++j) {
        int64_t i = sp_index[j];
        uint32_t u = sp_bits[j];
        if (out_dtype == ORACLE_BF16) {
            uint16_t b = (uint16_t)(u >> 16);
            if ((u & 0x7FFFFFu) != 0 && (b & 0x7Fu) == 0) b |= 0x40u;   /* keep it a NaN */
            ((uint16_t *)out)[i] = b;
        } else {
            ((uint32_t *)out)[i] = u;
        }
    }
    return 0;
}

/* ====================================================== block metadata */
/* Blocks ("a tensor, a row, a column, a sub row or even a 2D
 * tile") are block_rows x block_cols tiles of the row-major (rows, cols)
 * tensor, block_rows | rows and block_cols | cols.  Block (i, j) owns
 * metadata byte meta[i * (cols / block_cols) + j]. */
int oracle_block_shape_ok(int64_t rows, int64_t cols, int64_t br, int64_t bc)
{
    if (rows < 0 || cols < 0 || br < 1 || bc < 1) return 0;
    if (rows % br || cols % bc) return 0;
    return 1;
}

static int64_t block_of(int64_t e, int64_t cols, int64_t br, int64_t bc)
{
    int64_t r = e / cols, c = e % cols;
    return (r / br) * (cols / bc) + c / bc;
}

/* biased exponent (fp32 convention) of |v| rounded to nearest with y mantissa
 * bits in its own binade, exponent range unbounded; <= 0 reported as 0
 * (P:225-226).  Ties go to the representation whose last kept bit is 0
 * (RTNE "extended ... to arbitrary number of mantissa bits"): the
 * mantissa LSB for y >= 1, the exponent LSB for y = 0 (reading D22). */
static int exponent_after_rounding(uint32_t u, int y)
{
    double a = fabs(f32_value(u));
    if (a == 0.0) return 0;
    int e;
    (void)frexp(a, &e);               /* a in [2^(e-1), 2^e) */
    int E = e - 1;
    double s = ldexp(a, y - E);       /* in [2^y, 2^(y+1)), exact */
    double fl = floor(s), frac = s - fl;
    double r = fl;
    int lsb_odd = (y >= 1) ? (fmod(fl, 2.0) != 0.0) : (((E + 127) & 1) != 0);
    if (frac > 0.5 || (frac == 0.5 && lsb_odd)) r += 1.0;
    if (r >= ldexp(1.0, y + 1)) E += 1;   /* carry into the next binade */
    int be = E + 127;
    return be < 0 ? 0 : be;
}

/* Per-block metadata.  scheme 0 = maximum exponent before rounding (the
 * largest 8-bit biased exponent field of a finite element);
 * scheme 1 = after rounding to y mantissa bits.
 * NaN/Inf are ignored; a block without finite elements gets 0; results are
 * clamped to [0,254] (D4). */
int oracle_block_max_exponent(const void *in, int dtype, int64_t rows, int64_t cols,
                              int64_t br, int64_t bc, int y, int scheme, uint8_t *meta)
{
    if (!oracle_block_shape_ok(rows, cols, br, bc) || y < 0 || y > 23 || (scheme != 0 && scheme != 1)) return -1;
    int64_t nb = (rows / br) * (cols / bc);
    for (int64_t b = 0; b < nb; ++b) meta[b] = 0;
    for (int64_t e = 0; e < rows * cols; ++e) {
        uint32_t u = load_u32(in, dtype, e);
        if (is_special(u)) continue;
        int be = scheme == 0 ? (int)((u >> 23) & 0xFFu) : exponent_after_rounding(u, y);
        if (be > 254) be = 254;
        int64_t b = block_of(e, cols, br, bc);
        if (be > meta[b]) meta[b] = (uint8_t)be;
    }
    return 0;
}

/* grids for every metadata value, built on first use */
typedef struct { grid g[255]; int built[255]; int x, y; } grid_cache;

static const grid *cache_get(grid_cache *gc, int e_max)
{
    if (!gc->built[e_max]) {
        if (grid_build(&gc->g[e_max], gc->x, gc->y, e_max)) return NULL;
        gc->built[e_max] = 1;
    }
    return &gc->g[e_max];
}

static void cache_free(grid_cache *gc)
{
    for (int i = 0; i < 255; ++i)
        if (gc->built[i]) grid_free(&gc->g[i]);
}

static int meta_at(const uint8_t *meta, int64_t e, int64_t cols, int64_t br, int64_t bc)
{
    int m = meta[block_of(e, cols, br, bc)];
    return m > 254 ? 254 : m;
}

/* Emulation with block metadata: element e is quantized on the grid of its
 * block's e_max. */
int oracle_quantize_blocked(const void *in, void *out, int dtype, int64_t rows, int64_t cols,
                            int64_t br, int64_t bc, int x, int y, const uint8_t *meta)
{
    if (!oracle_format_valid(x, y, 0) || !oracle_block_shape_ok(rows, cols, br, bc)) return -1;
    grid_cache *gc = (grid_cache *)calloc(1, sizeof(grid_cache));
    if (!gc) return -1;
    gc->x = x; gc->y = y;
    for (int64_t e = 0; e < rows * cols; ++e) {
        uint32_t u = load_u32(in, dtype, e);
        if (is_special(u)) {
            if (dtype == ORACLE_BF16) ((uint16_t *)out)[e] = ((const uint16_t *)in)[e];
            else ((uint32_t *)out)[e] = u;
            continue;
        }
        int em = meta_at(meta, e, cols, br, bc);
        const grid *g = cache_get(gc, em);
        uint32_t code = encode_finite(g, u);
        store_value(out, dtype, e, oracle_code_value(code, x, y, em));
    }
    cache_free(gc);
    free(gc);
    return 0;
}

int64_t oracle_encode_blocked(const void *in, int dtype, int64_t rows, int64_t cols, int axis,
                              int64_t br, int64_t bc, int x, int y, const uint8_t *meta, uint8_t *packed,
                              int64_t *sp_index, uint32_t *sp_bits, int64_t sp_capacity)
{
    if (!oracle_format_valid(x, y, 0) || !oracle_shape_ok(rows, cols, axis) ||
        !oracle_block_shape_ok(rows, cols, br, bc) || 1 + x + y > ORACLE_MAX_PACK_K) return -1;
    int64_t n = rows * cols;
    uint16_t *codes = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(n ? n : 1));
    grid_cache *gc = (grid_cache *)calloc(1, sizeof(grid_cache));
    if (!codes || !gc) { free(codes); free(gc); return -1; }
    gc->x = x; gc->y = y;
    int64_t ns = 0;
    for (int64_t e = 0; e < n; ++e) {
        uint32_t u = load_u32(in, dtype, e);
        if (is_special(u)) {
            codes[e] = 0;
            if (ns < sp_capacity) { sp_index[ns] = e; sp_bits[ns] = u; }
            ++ns;
        } else {
            codes[e] = (uint16_t)encode_finite(cache_get(gc, meta_at(meta, e, cols, br, bc)), u);
        }
    }
    cache_free(gc);
    free(gc);
    oracle_pack(codes, rows, cols, axis, 1 + x + y, packed);
    free(codes);
    return ns;
}

int oracle_decode_blocked(const uint8_t *packed, int64_t rows, int64_t cols, int axis,
                          int64_t br, int64_t bc, int x, int y, const uint8_t *meta,
                          const int64_t *sp_index, const uint32_t *sp_bits, int64_t sp_count,
                          void *out, int out_dtype)
{
    if (!oracle_format_valid(x, y, 0) || !oracle_shape_ok(rows, cols, axis) ||
        !oracle_block_shape_ok(rows, cols, br, bc) || 1 + x + y > ORACLE_MAX_PACK_K) return -1;
    int64_t n = rows * cols;
    uint16_t *codes = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(n ? n : 1));
    if (!codes) return -1;
    oracle_unpack(packed, rows, cols, axis, 1 + x + y, codes);
    for (int64_t e = 0; e < n; ++e)
        store_value(out, out_dtype, e, oracle_code_value(codes[e], x, y, meta_at(meta, e, cols, br, bc)));
    free(codes);
    for (int64_t j = 0; j < sp_count; ++j) {
        int64_t i = sp_index[j];
        uint32_t u = sp_bits[j];
        if (out_dtype == ORACLE_BF16) {
            uint16_t b = (uint16_t)(u >> 16);
            if ((u & 0x7FFFFFu) != 0 && (b & 0x7Fu) == 0) b |= 0x40u;
            ((uint16_t *)out)[i] = b;
        } else {
            ((uint32_t *)out)[i] = u;
        }
    }
    return 0;
}

/* ======================================================= float scaling */
/* The third Fig. 2 scheme, "float scaling with maximum exponent of 127"
 * ("an additional bfloat16 or float32 scaling factor").
 * Reading D23: every block stores one fp32 metadata value, its
 * largest finite magnitude amax, and uses e_max = 127, whose grid top is
 * G = the largest magnitude code's value at e_max 127.  The block is mapped
 * onto that grid by the fp32 factor RN32(G/amax) and mapped back by amax/G,
 * so its maximum lands on G and comes back as amax ("captures the largest
 * value in the block accurately").  With amax = A1 * 2^p, A1 in [1, 2):
 *   encode  r  = RN32(G / A1)                 (the fp32 scaling factor)
 *           u  = RN32(v * r * 2^-p)           (exact product, rounded once)
 *           code = the e_max-127 code of u    (as oracle_encode)
 *   decode  out = RN32(g * amax / G)          (g = the code's exact value at
 *           e_max 127; the exact product and quotient, rounded once, fp32
 *           subnormals included; a zero result keeps the code's sign)
 *           bf16 output = RN16 of that fp32 value  (reading D24)
 * amax = 0 (no finite non-zero element): u = v * 0, codes are signed zeros,
 * and they decode to signed zeros. */

double oracle_fs_grid_top(int x, int y)
{
    return oracle_code_magnitude((1u << (x + y)) - 1u, x, y, 127);
}

/* amax = A1 * 2^p, A1 in [1, 2) (subnormal amax normalised) */
static void fs_split(uint32_t amax_bits, double *A1, int *p)
{
    double a = f32_value(amax_bits & 0x7FFFFFFFu);
    int e;
    double f = frexp(a, &e);          /* a = f * 2^e, f in [0.5, 1) */
    *A1 = 2.0 * f;                    /* exact */
    *p = e - 1;
}

/* The fp32 value nearest to the exact quotient num / den of two positive
 * doubles (ties to the even pattern, fp32 subnormals included), where den has
 * at most 26 significant bits.  No division result is trusted: starting from
 * a guess, the answer is the fp32 t with
 *     den * (t - ulp/2)  <=  num  <=  den * (t + ulp/2),
 * checked with exact products -- every midpoint between neighbouring fp32
 * values has at most 25 significant bits, so den * midpoint is an exact
 * double (<= 51 bits) and each comparison below is exact. */
static uint32_t rn32_quotient(double num, double den)
{
    uint32_t t = oracle_round_f32(num / den);         /* a guess: within one step */
    for (;;) {
        double vt = f32_value(t);
        if (t < 0x7F7FFFFFu) {                        /* compare with the midpoint above */
            double mid = (vt + f32_value(t + 1u)) / 2.0;
            double dm = den * mid;
            if (num > dm || (num == dm && (t & 1u))) { t += 1u; continue; }
        }
        if (t > 0u) {                                 /* and with the midpoint below */
            double mid = (vt + f32_value(t - 1u)) / 2.0;
            double dm = den * mid;
            if (num < dm || (num == dm && (t & 1u))) { t -= 1u; continue; }
        }
        return t;
    }
}

/* fp32 bits of the per-block float-scale metadata: the largest finite |v| */
int oracle_block_float_scale(const void *in, int dtype, int64_t rows, int64_t cols,
                             int64_t br, int64_t bc, uint32_t *amax)
{
    if (!oracle_block_shape_ok(rows, cols, br, bc)) return -1;
    int64_t nb = (rows / br) * (cols / bc);
    for (int64_t b = 0; b < nb; ++b) amax[b] = 0;
    for (int64_t e = 0; e < rows * cols; ++e) {
        uint32_t u = load_u32(in, dtype, e);
        if (is_special(u)) continue;
        int64_t b = block_of(e, cols, br, bc);
        if (fabs(f32_value(u)) > f32_value(amax[b])) amax[b] = u & 0x7FFFFFFFu;
    }
    return 0;
}

/* the fp32 encode factor RN32(G / A1) of a block (amax != 0) */
uint32_t oracle_fs_factor(uint32_t amax, int x, int y)
{
    double A1;
    int p;
    fs_split(amax, &A1, &p);
    return rn32_quotient(oracle_fs_grid_top(x, y), A1);   /* A1: <= 24 significant bits */
}

/* scaled fp32 value u of the finite element v (bits) under block max amax */
uint32_t oracle_fs_scale_in(uint32_t v, uint32_t amax, int x, int y)
{
    if ((amax & 0x7FFFFFFFu) == 0) return v & 0x80000000u;      /* v * 0 */
    double A1;
    int p;
    fs_split(amax, &A1, &p);
    uint32_t r = oracle_fs_factor(amax, x, y);
    double prod = f32_value(v) * f32_value(r);                  /* exact: 24 x 24 bits */
    return oracle_round_f32(ldexp(prod, -p));                   /* exact scaling, one rounding */
}

/* decoded fp32 bits of code under block max amax (reading D23):
 * RN32(g * amax / G), g the exact value of the code at e_max 127 */
uint32_t oracle_fs_scale_out(uint32_t code, uint32_t amax, int x, int y)
{
    int k = 1 + x + y;
    uint32_t sign = ((code >> (k - 1)) & 1u) << 31;
    double g = fabs(oracle_code_value(code, x, y, 127));   /* exact, a normal fp64 */
    double a = f32_value(amax & 0x7FFFFFFFu);
    if (g == 0.0 || a == 0.0) return sign;                 /* signed zero */
    /* g * a is exact (<= 24 + 24 significant bits); G has <= 24 */
    return rn32_quotient(g * a, oracle_fs_grid_top(x, y)) | sign;
}

static uint32_t fs_encode_code(const grid *g127, uint32_t u_in, uint32_t amax)
{
    return encode_finite(g127, oracle_fs_scale_in(u_in, amax, g127->x, g127->y));
}

static void fs_store(void *out, int dtype, int64_t i, uint32_t f32bits)
{
    if (dtype == ORACLE_BF16) ((uint16_t *)out)[i] = oracle_round_bf16(f32_value(f32bits));
    else ((uint32_t *)out)[i] = f32bits;
}

int oracle_quantize_fs(const void *in, void *out, int dtype, int64_t rows, int64_t cols,
                       int64_t br, int64_t bc, int x, int y, const uint32_t *amax)
{
    if (!oracle_format_valid(x, y, 127) || !oracle_block_shape_ok(rows, cols, br, bc)) return -1;
    grid g;
    if (grid_build(&g, x, y, 127)) return -1;
    for (int64_t e = 0; e < rows * cols; ++e) {
        uint32_t u = load_u32(in, dtype, e);
        if (is_special(u)) {
            if (dtype == ORACLE_BF16) ((uint16_t *)out)[e] = ((const uint16_t *)in)[e];
            else ((uint32_t *)out)[e] = u;
            continue;
        }
        uint32_t a = amax[block_of(e, cols, br, bc)];
        fs_store(out, dtype, e, oracle_fs_scale_out(fs_encode_code(&g, u, a), a, x, y));
    }
    grid_free(&g);
    return 0;
}

int64_t oracle_encode_fs(const void *in, int dtype, int64_t rows, int64_t cols, int axis,
                         int64_t br, int64_t bc, int x, int y, const uint32_t *amax, uint8_t *packed,
                         int64_t *sp_index, uint32_t *sp_bits, int64_t sp_capacity)
{
    if (!oracle_format_valid(x, y, 127) || !oracle_shape_ok(rows, cols, axis) ||
        !oracle_block_shape_ok(rows, cols, br, bc) || 1 + x + y > ORACLE_MAX_PACK_K) return -1;
    int64_t n = rows * cols;
    uint16_t *codes = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(n ? n : 1));
    grid g;
    if (!codes || grid_build(&g, x, y, 127)) { free(codes); return -1; }
    int64_t ns = 0;
    for (int64_t e = 0; e < n; ++e) {
        uint32_t u = load_u32(in, dtype, e);
        if (is_special(u)) {
            codes[e] = 0;
            if (ns < sp_capacity) { sp_index[ns] = e; sp_bits[ns] = u; }
            ++ns;
        } else {
            codes[e] = (uint16_t)fs_encode_code(&g, u, amax[block_of(e, cols, br, bc)]);
        }
    }
    grid_free(&g);
    oracle_pack(codes, rows, cols, axis, 1 + x + y, packed);
    free(codes);
    return ns;
}

int oracle_decode_fs(const uint8_t *packed, int64_t rows, int64_t cols, int axis,
                     int64_t br, int64_t bc, int x, int y, const uint32_t *amax,
                     const int64_t *sp_index, const uint32_t *sp_bits, int64_t sp_count,
                     void *out, int out_dtype)
{
    if (!oracle_format_valid(x, y, 127) || !oracle_shape_ok(rows, cols, axis) ||
        !oracle_block_shape_ok(rows, cols, br, bc) || 1 + x + y > ORACLE_MAX_PACK_K) return -1;
    int64_t n = rows * cols;
    uint16_t *codes = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(n ? n : 1));
    if (!codes) return -1;
    oracle_unpack(packed, rows, cols, axis, 1 + x + y, codes);
    for (int64_t e = 0; e < n; ++e)
        fs_store(out, out_dtype, e, oracle_fs_scale_out(codes[e], amax[block_of(e, cols, br, bc)], x, y));
    free(codes);
    for (int64_t j = 0; j < sp_count; ++j) {
        int64_t i = sp_index[j];
        uint32_t u = sp_bits[j];
        if (out_dtype == ORACLE_BF16) {
            uint16_t b = (uint16_t)(u >> 16);
            if ((u & 0x7FFFFFu) != 0 && (b & 0x7Fu) == 0) b |= 0x40u;
            ((uint16_t *)out)[i] = b;
        } else {
            ((uint32_t *)out)[i] = u;
        }
    }
    return 0;
}

/* ================================================= embedding bag (decode + pool) */
/* SURVEY 8(f) row 3, "decode fused into a GEMM/embedding-bag prologue" (config 5,
 * P:293-298 serving decode is performance critical).  Reading D25: bag b pools
 * the rows indices[offsets[b] .. offsets[b+1]) of a COLS-packed (rows, cols)
 * table: each row decoded to fp32 exactly as oracle_decode does (NaN/Inf kept
 * out of band are NOT restored, as exmy_decode_rows), then accumulated in fp32
 * in index order, acc = RN32(acc + v), or acc = RN32(w v + acc) (one fused
 * rounding) with per-sample weights; mode 1 (mean) divides by the bag size
 * (RN32); an empty bag gives +0. */

/* code of element (r, c) of a COLS-packed table: container g = r*(cols/8) + c/8,
 * lane c%8, segment bits as oracle_pack lays them out */
static uint32_t cols_code_at(const uint8_t *packed, int64_t rows, int64_t cols, int k, int64_t r, int64_t c)
{
    int widths[4];
    int64_t offs[4];
    int ns = oracle_segments(k, widths, rows * cols, offs);
    int64_t g = r * (cols / 8) + c / 8;
    int lane = (int)(c % 8);
    uint32_t code = 0;
    int hi = k;
    for (int s = 0; s < ns; ++s) {
        int w = widths[s], lo = hi - w;
        const uint8_t *seg = packed + offs[s];
        uint32_t field;
        if (w == 8) {
            field = seg[r * cols + c];
        } else {
            uint32_t cont = 0;
            for (int b = 0; b < w; ++b) cont |= (uint32_t)seg[g * w + b] << (8 * b);
            field = (cont >> (w * lane)) & ((1u << w) - 1u);
        }
        code |= field << lo;
        hi = lo;
    }
    return code;
}

int oracle_embedding_bag(const uint8_t *packed, int64_t rows, int64_t cols, int x, int y,
                         const uint8_t *meta, int meta_per_row, const int64_t *indices,
                         const int64_t *offsets, int64_t nbags, const float *weights, int mode,
                         float *out)
{
    if (!oracle_format_valid(x, y, 0) || cols % 8 || (mode != 0 && mode != 1)) return -1;
    int k = 1 + x + y;
    for (int64_t b = 0; b < nbags; ++b) {
        int64_t i0 = offsets[b], i1 = offsets[b + 1];
        for (int64_t c = 0; c < cols; ++c) {
            volatile float acc = 0.0f;
            for (int64_t i = i0; i < i1; ++i) {
                int64_t r = indices[i];
                int e = meta[meta_per_row ? r : 0];
                if (e > 254) e = 254;
                uint32_t vb = oracle_round_f32(oracle_code_value(cols_code_at(packed, rows, cols, k, r, c), x, y, e));
                float v;
                memcpy(&v, &vb, 4);
                if (weights) acc = fmaf(weights[i], v, acc);   /* one rounding of w v + acc */
                else acc = acc + v;
            }
            if (mode == 1 && i1 > i0) acc = acc / (float)(i1 - i0);
            out[b * cols + c] = acc;
        }
    }
    return 0;
}
