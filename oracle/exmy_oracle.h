/* exmy_oracle.h -- TEST INFRASTRUCTURE ONLY (see exmy_oracle.c).
 * The oracle's own declarations; deliberately independent of include/exmy.h. */
#ifndef EXMY_ORACLE_H
#define EXMY_ORACLE_H
#include <stdint.h>

#define ORACLE_F32 0
#define ORACLE_BF16 1
#define ORACLE_ROWS 0
#define ORACLE_COLS 1
#define ORACLE_MAX_K 16       /* element codecs (k=16 serves the fp16/bf16 pins) */
#define ORACLE_MAX_PACK_K 15  /* power-of-2 decomposition into {8,4,2,1} */

#ifdef __cplusplus
extern "C" {
#endif
int oracle_format_valid(int x, int y, int e_max);
int oracle_bias(int x, int e_max);
double oracle_code_magnitude(uint32_t mag, int x, int y, int e_max);
double oracle_code_value(uint32_t code, int x, int y, int e_max);
uint32_t oracle_round_f32(double v);
uint16_t oracle_round_bf16(double v);
int oracle_encode_codes(const void *in, int dtype, int64_t n, int x, int y, int e_max,
                        uint16_t *codes, uint8_t *special);
int oracle_encode_element(uint32_t u, int x, int y, int e_max, uint32_t *code);
void oracle_histogram(const void *in, int dtype, int64_t n, uint64_t hist[256]);
int oracle_emax(const uint64_t hist[256]);
int oracle_choose_x(const uint64_t hist[256], double budget);
int oracle_quantize(const void *in, void *out, int dtype, int64_t n, int x, int y, int e_max);
int oracle_segments(int k, int widths[4], int64_t n, int64_t offsets[4]);
int oracle_shape_ok(int64_t rows, int64_t cols, int axis);
int oracle_pack(const uint16_t *codes, int64_t rows, int64_t cols, int axis, int k, uint8_t *packed);
int oracle_unpack(const uint8_t *packed, int64_t rows, int64_t cols, int axis, int k, uint16_t *codes);
int64_t oracle_encode(const void *in, int dtype, int64_t rows, int64_t cols, int axis,
                      int x, int y, int e_max, uint8_t *packed,
                      int64_t *sp_index, uint32_t *sp_bits, int64_t sp_capacity);
int oracle_decode(const uint8_t *packed, int64_t rows, int64_t cols, int axis,
                  int x, int y, int e_max,
                  const int64_t *sp_index, const uint32_t *sp_bits, int64_t sp_count,
                  void *out, int out_dtype);
int oracle_block_shape_ok(int64_t rows, int64_t cols, int64_t br, int64_t bc);
int oracle_block_max_exponent(const void *in, int dtype, int64_t rows, int64_t cols,
                              int64_t br, int64_t bc, int y, int scheme, uint8_t *meta);
int oracle_quantize_blocked(const void *in, void *out, int dtype, int64_t rows, int64_t cols,
                            int64_t br, int64_t bc, int x, int y, const uint8_t *meta);
int64_t oracle_encode_blocked(const void *in, int dtype, int64_t rows, int64_t cols, int axis,
                              int64_t br, int64_t bc, int x, int y, const uint8_t *meta, uint8_t *packed,
                              int64_t *sp_index, uint32_t *sp_bits, int64_t sp_capacity);
int oracle_decode_blocked(const uint8_t *packed, int64_t rows, int64_t cols, int axis,
                          int64_t br, int64_t bc, int x, int y, const uint8_t *meta,
                          const int64_t *sp_index, const uint32_t *sp_bits, int64_t sp_count,
                          void *out, int out_dtype);
/* float scaling (reading D23) */
double oracle_fs_grid_top(int x, int y);
int oracle_block_float_scale(const void *in, int dtype, int64_t rows, int64_t cols,
                             int64_t br, int64_t bc, uint32_t *amax);
uint32_t oracle_fs_factor(uint32_t amax, int x, int y);
uint32_t oracle_fs_scale_in(uint32_t v, uint32_t amax, int x, int y);
uint32_t oracle_fs_scale_out(uint32_t code, uint32_t amax, int x, int y);
int oracle_quantize_fs(const void *in, void *out, int dtype, int64_t rows, int64_t cols,
                       int64_t br, int64_t bc, int x, int y, const uint32_t *amax);
int64_t oracle_encode_fs(const void *in, int dtype, int64_t rows, int64_t cols, int axis,
                         int64_t br, int64_t bc, int x, int y, const uint32_t *amax, uint8_t *packed,
                         int64_t *sp_index, uint32_t *sp_bits, int64_t sp_capacity);
int oracle_decode_fs(const uint8_t *packed, int64_t rows, int64_t cols, int axis,
                     int64_t br, int64_t bc, int x, int y, const uint32_t *amax,
                     const int64_t *sp_index, const uint32_t *sp_bits, int64_t sp_count,
                     void *out, int out_dtype);

/* embedding bag over a COLS-packed table (reading D25) */
int oracle_embedding_bag(const uint8_t *packed, int64_t rows, int64_t cols, int x, int y,
                         const uint8_t *meta, int meta_per_row, const int64_t *indices,
                         const int64_t *offsets, int64_t nbags, const float *weights, int mode,
                         float *out);

#ifdef __cplusplus
}
#endif
#endif
