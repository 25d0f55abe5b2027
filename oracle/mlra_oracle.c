/*
 * mlra_oracle.c — CPU restatement of the ModuLoRA hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it. The product path (libmlra.so) never links or calls it.
 *
 * Parity status: PINNED. tests/test_oracle_golden.py checks every function
 * here bit-for-bit against fixtures produced by the reference itself
 * (oracle/_ref/libmlra_ref.so, built from /root/reference/proj/src by
 * oracle/Makefile; generator: tests/golden/make_golden.py), and against the
 * known-answer tests of /root/reference/proj/tests.
 *
 * All arithmetic is IEEE f64 in the reference's own evaluation order, so the
 * results are bit-identical to the reference (compile with -ffp-contract=off,
 * no fast-math; see oracle/Makefile).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Rng — rng.hpp:15-57. mt19937_64 + the reference's hand-written mappings. */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_rng;

ORC_EXPORT void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  }
  r->idx = 312;
}

static void orc_rng_twist(orc_rng* r) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  for (int i = 0; i < 312; ++i) {
    uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % 312] & lower);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
  }
  r->idx = 0;
}

/* std::mt19937_64::operator() */
ORC_EXPORT uint64_t orc_rng_next_u64(orc_rng* r) {
  if (r->idx >= 312) orc_rng_twist(r);
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* rng.hpp:24-26 */
ORC_EXPORT double orc_rng_uniform(orc_rng* r) {
  return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:30-35 (cosine branch only, no cached spare) */
ORC_EXPORT double orc_rng_gaussian(orc_rng* r) {
  const double u1 = 1.0 - orc_rng_uniform(r);
  const double u2 = orc_rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* rng.hpp:42-44 */
ORC_EXPORT uint64_t orc_rng_uniform_index(orc_rng* r, uint64_t n) {
  return orc_rng_next_u64(r) % n;
}

/* rng.hpp:52-57 (splitmix64 finalizer) */
ORC_EXPORT uint64_t orc_mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* DenseMatrix::gaussian — matrix.cpp:62-67: row-major fill, mean + std*g. */
ORC_EXPORT void orc_gaussian_fill(uint64_t seed, double* out, uint64_t n,
                                  double mean, double stddev) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = mean + stddev * orc_rng_gaussian(&r);
}

/* ------------------------------------------------------------------------ */
/* Bitpack — bitpack.cpp:25-112. LSB-first stream over the whole matrix.     */
/* ------------------------------------------------------------------------ */
ORC_EXPORT int orc_supported_bits(int bits) {
  return bits == 2 || bits == 3 || bits == 4 || bits == 8;
}

/* bitpack.cpp:64-66 */
ORC_EXPORT uint64_t orc_packed_word_count(uint64_t count, int bits) {
  return (count * (uint64_t)bits + 31) / 32;
}

/* bitpack.cpp:25-35 */
ORC_EXPORT uint32_t orc_read_code(const uint32_t* words, int bits,
                                  uint64_t index) {
  const uint64_t bit = index * (uint64_t)bits;
  const uint64_t word = bit / 32, off = bit % 32;
  const uint32_t mask = (1u << bits) - 1u;
  uint64_t v = words[word] >> off;
  if (off + (uint64_t)bits > 32) v |= (uint64_t)words[word + 1] << (32 - off);
  return (uint32_t)v & mask;
}

/* bitpack.cpp:68-91. Returns 0, or -1 (ConfigError) / -2 (RangeError at
 * *bad_index). `words` must hold orc_packed_word_count(count, bits) words. */
ORC_EXPORT int orc_pack(const uint32_t* codes, uint64_t count, int bits,
                        uint32_t* words, uint64_t* bad_index) {
  if (!orc_supported_bits(bits)) return -1;
  const uint32_t limit = 1u << bits;
  memset(words, 0, orc_packed_word_count(count, bits) * sizeof(uint32_t));
  for (uint64_t i = 0; i < count; ++i) {
    const uint32_t c = codes[i];
    if (c >= limit) {
      if (bad_index) *bad_index = i;
      return -2;
    }
    const uint64_t bit = i * (uint64_t)bits;
    const uint64_t word = bit / 32, off = bit % 32;
    words[word] |= c << off;
    if (off + (uint64_t)bits > 32) words[word + 1] |= c >> (32 - off);
  }
  return 0;
}

/* bitpack.cpp:37-60. 0 ok, -1 ConfigError, -3 FormatError{BadField}. */
ORC_EXPORT int orc_validate_packed(const uint32_t* words, uint64_t word_count,
                                   uint64_t count, int bits) {
  if (!orc_supported_bits(bits)) return -1;
  if (word_count != orc_packed_word_count(count, bits)) return -3;
  const uint64_t used = count * (uint64_t)bits;
  if (word_count) {
    const uint64_t tail = word_count * 32 - used;
    if (tail > 0 && tail < 32 && (words[word_count - 1] >> (32 - tail)) != 0)
      return -3;
  }
  return 0;
}

/* bitpack.cpp:93-98 */
ORC_EXPORT int orc_unpack(const uint32_t* words, uint64_t word_count,
                          uint64_t count, int bits, uint32_t* out) {
  int st = orc_validate_packed(words, word_count, count, bits);
  if (st) return st;
  for (uint64_t i = 0; i < count; ++i) out[i] = orc_read_code(words, bits, i);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Quantize — quantize.cpp:24-44 (grid), 163-184 (RTN), 117-155 (dequant).  */
/* ------------------------------------------------------------------------ */

/* quantize.cpp:24-36 */
static void orc_compute_grid(const double* vals, uint64_t n, int bits,
                             float* scale, float* zero) {
  double lo = vals[0], hi = vals[0];
  for (uint64_t i = 0; i < n; ++i) {
    lo = vals[i] < lo ? vals[i] : lo; /* std::min(lo, v) */
    hi = hi < vals[i] ? vals[i] : hi; /* std::max(hi, v) */
  }
  const double levels = (double)((1 << bits) - 1);
  *zero = (float)lo;
  *scale = (hi > lo) ? (float)((hi - lo) / levels) : 1.0f;
  if (!(*scale > 0.0f)) *scale = 1.0f;
}

/* quantize.cpp:38-44 */
static uint32_t orc_code_on_grid(double w, float scale, float zero, int bits) {
  const double levels = (double)((1 << bits) - 1);
  double c = round((w - (double)zero) / (double)scale);
  if (c < 0.0) c = 0.0;
  if (levels < c) c = levels;
  return (uint32_t)c;
}

/* quantize.cpp:163-184. group == 0 selects per-row grids (quantize.cpp:78-80).
 * Returns 0 / -1 ConfigError / -4 DimensionError. */
ORC_EXPORT int orc_quantize_rtn(const double* w, uint64_t rows, uint64_t cols,
                                int bits, uint64_t group, uint32_t* words,
                                float* scales, float* zeros) {
  if (group == 0) group = cols;
  if (rows == 0 || cols == 0) return -4;
  if (!orc_supported_bits(bits)) return -1;
  if (cols % group != 0) return -1;
  const uint64_t ng = cols / group;
  uint32_t* codes = (uint32_t*)malloc(rows * cols * sizeof(uint32_t));
  for (uint64_t i = 0; i < rows; ++i) {
    for (uint64_t g = 0; g < ng; ++g) {
      float s, z;
      orc_compute_grid(w + i * cols + g * group, group, bits, &s, &z);
      scales[i * ng + g] = s;
      zeros[i * ng + g] = z;
      for (uint64_t j = g * group; j < (g + 1) * group; ++j)
        codes[i * cols + j] = orc_code_on_grid(w[i * cols + j], s, z, bits);
    }
  }
  orc_pack(codes, rows * cols, bits, words, NULL);
  free(codes);
  return 0;
}

/* quantize.cpp:82-115 (QuantizedMatrix::validate). 0 ok; -1 ConfigError;
 * -3 FormatError; -5 NumericError. */
ORC_EXPORT int orc_validate_qmatrix(uint64_t rows, uint64_t cols, int bits,
                                    int packed_bits, uint64_t group,
                                    uint64_t code_count, uint64_t n_scales,
                                    uint64_t n_zeros, const float* scales) {
  if (!orc_supported_bits(bits)) return -1;
  if (packed_bits != bits) return -1;
  if (rows == 0 || cols == 0 || group == 0 || cols % group != 0) return -1;
  if (code_count != rows * cols) return -3;
  const uint64_t ng = rows * (cols / group);
  if (n_scales != ng || n_zeros != ng) return -3;
  for (uint64_t i = 0; i < n_scales; ++i)
    if (!(scales[i] > 0.0f)) return -5;
  return 0;
}

/* quantize.cpp:123-137: W[i,j] = double(s)*c + double(z), one f64 rounding. */
ORC_EXPORT void orc_dequantize(const uint32_t* words, uint64_t rows,
                               uint64_t cols, int bits, uint64_t group,
                               const float* scales, const float* zeros,
                               double* out) {
  const uint64_t ng = cols / group;
  for (uint64_t i = 0; i < rows; ++i) {
    for (uint64_t j = 0; j < cols; ++j) {
      const uint64_t gidx = i * ng + j / group;
      const uint32_t c = orc_read_code(words, bits, i * cols + j);
      out[i * cols + j] = (double)scales[gidx] * (double)c + (double)zeros[gidx];
    }
  }
}

/* quantize.cpp:139-155 */
ORC_EXPORT void orc_dequantize_row(const uint32_t* words, uint64_t cols,
                                   int bits, uint64_t group,
                                   const float* scales, const float* zeros,
                                   uint64_t row, double* out) {
  const uint64_t ng = cols / group;
  for (uint64_t j = 0; j < cols; ++j) {
    const uint64_t gidx = row * ng + j / group;
    const uint32_t c = orc_read_code(words, bits, row * cols + j);
    out[j] = (double)scales[gidx] * (double)c + (double)zeros[gidx];
  }
}

/* The device's "materialize" contract: the f32 / bf16 images of
 * the f64 dequantized value. fp32 = RN(f64); bf16 = RN_even(fp32). */
ORC_EXPORT void orc_dequantize_f32(const uint32_t* words, uint64_t rows,
                                   uint64_t cols, int bits, uint64_t group,
                                   const float* scales, const float* zeros,
                                   float* out) {
  const uint64_t ng = cols / group;
  for (uint64_t i = 0; i < rows; ++i) {
    for (uint64_t j = 0; j < cols; ++j) {
      const uint64_t gidx = i * ng + j / group;
      const uint32_t c = orc_read_code(words, bits, i * cols + j);
      const double v = (double)scales[gidx] * (double)c + (double)zeros[gidx];
      out[i * cols + j] = (float)v;
    }
  }
}

/* The built-in non-affine plugin "cb2" (include/mlra.h mlra_cb2_create) —
 * the device form of the black-box Quantizer hook (quantize.hpp:91-106). The
 * reference hosts such plugins but ships none, so this
 * decode law is pinned by the known-answer test in tests/test_cb2.py
 * (hand-computed values) rather than by reference output. One u16 code per 8
 * consecutive row entries: bits 0-7 index codebook[256][8], bit 8+j negates
 * entry j; per-(row, group) f32 scale:
 *   out[i, 8u+j] = RN_f32(s[i, (8u+j)/g] * (+-cb[idx][j]))   (one IEEE multiply) */
ORC_EXPORT void orc_cb2_dequant_f32(const uint16_t* codes, uint64_t rows, uint64_t cols,
                                    uint64_t group, const float* codebook,
                                    const float* scales, float* out) {
  const uint64_t ng = cols / group, cpr = cols / 8;
  for (uint64_t i = 0; i < rows; ++i) {
    for (uint64_t u = 0; u < cpr; ++u) {
      const uint16_t code = codes[i * cpr + u];
      const float* e = codebook + (uint64_t)(code & 0xFFu) * 8;
      for (uint64_t j = 0; j < 8; ++j) {
        const float s = scales[i * ng + (8 * u + j) / group];
        float m = e[j];
        if ((code >> (8 + j)) & 1u) m = -m;
        out[i * cols + 8 * u + j] = s * m;
      }
    }
  }
}

/* The built-in plugin "e8p" (include/mlra.h mlra_e8p_create): QuIP#'s E8P
 * lattice codebook. Parity status: the reference ships no such plugin
 * (SPEC.md:8, :251), so this restatement of the decode law is pinned by the
 * hand-derived known answers and the lattice-membership checks of
 * tests/test_e8p.py, not by reference output.
 *
 * Abs table: (i) every vector of {1/2, 3/2, 5/2}^8 with squared norm <= 10 in
 * lexicographic order of 2|a| (227), then (ii) the 29 norm-12 patterns of
 * {1/2, 3/2}^8 listed below (QuIP#'s E8P12 construction: 256 patterns). A code
 * (one u16 per 8 row entries): bits 0-7 pattern index, bits 8-14 negate entries
 * 0-6, entry 7 negated iff (number of negations among 0-6 + the pattern's
 * coordinate sum) is odd, bit 15 = +1/4 shift (else -1/4). Then
 *   out[i, 8u+j] = RN_f32(s[i, (8u+j)/g] * (sign_j * a_j + shift)). */
static const uint8_t ORC_E8P_NORM12[29][8] = {
    {3, 1, 1, 1, 3, 3, 3, 3}, {1, 3, 1, 1, 3, 3, 3, 3}, {1, 1, 3, 1, 3, 3, 3, 3},
    {1, 1, 1, 3, 3, 3, 3, 3}, {3, 3, 3, 1, 3, 3, 1, 1}, {3, 3, 3, 1, 3, 1, 3, 1},
    {3, 3, 3, 1, 1, 3, 3, 1}, {3, 3, 3, 1, 3, 1, 1, 3}, {3, 3, 3, 1, 1, 3, 1, 3},
    {3, 3, 3, 1, 1, 1, 3, 3}, {3, 3, 1, 3, 3, 3, 1, 1}, {3, 3, 1, 3, 3, 1, 3, 1},
    {3, 3, 1, 3, 1, 3, 3, 1}, {3, 3, 1, 3, 3, 1, 1, 3}, {3, 3, 1, 3, 1, 3, 1, 3},
    {3, 3, 1, 3, 1, 1, 3, 3}, {3, 1, 3, 3, 3, 3, 1, 1}, {3, 1, 3, 3, 3, 1, 3, 1},
    {3, 1, 3, 3, 1, 3, 3, 1}, {3, 1, 3, 3, 3, 1, 1, 3}, {3, 1, 3, 3, 1, 3, 1, 3},
    {1, 3, 3, 3, 1, 1, 3, 3}, {1, 3, 3, 3, 3, 3, 1, 1}, {1, 3, 3, 3, 3, 1, 3, 1},
    {1, 3, 3, 3, 1, 3, 3, 1}, {1, 3, 3, 3, 3, 1, 1, 3}, {1, 3, 3, 3, 1, 3, 1, 3},
    {1, 1, 3, 3, 1, 3, 3, 3}, {3, 3, 1, 1, 3, 3, 3, 1}};

/* 2|a| of the 256 patterns, row-major (the oracle's own enumeration). */
ORC_EXPORT void orc_e8p_abs_table(int32_t* twice_abs) {
  int n = 0;
  for (int d0 = 1; d0 <= 5; d0 += 2)
  for (int d1 = 1; d1 <= 5; d1 += 2)
  for (int d2 = 1; d2 <= 5; d2 += 2)
  for (int d3 = 1; d3 <= 5; d3 += 2)
  for (int d4 = 1; d4 <= 5; d4 += 2)
  for (int d5 = 1; d5 <= 5; d5 += 2)
  for (int d6 = 1; d6 <= 5; d6 += 2)
  for (int d7 = 1; d7 <= 5; d7 += 2) {
    const int d[8] = {d0, d1, d2, d3, d4, d5, d6, d7};
    int norm4 = 0;
    for (int j = 0; j < 8; ++j) norm4 += d[j] * d[j];
    if (norm4 > 40) continue;
    for (int j = 0; j < 8; ++j) twice_abs[n * 8 + j] = d[j];
    ++n;
  }
  for (int i = 0; i < 29; ++i, ++n)
    for (int j = 0; j < 8; ++j) twice_abs[n * 8 + j] = ORC_E8P_NORM12[i][j];
}

ORC_EXPORT void orc_e8p_dequant_f32(const uint16_t* codes, uint64_t rows, uint64_t cols,
                                    uint64_t group, const float* scales, float* out) {
  int32_t t[256 * 8];
  orc_e8p_abs_table(t);
  const uint64_t ng = cols / group, cpr = cols / 8;
  for (uint64_t i = 0; i < rows; ++i) {
    for (uint64_t u = 0; u < cpr; ++u) {
      const uint32_t code = codes[i * cpr + u];
      const int32_t* a2 = t + (code & 0xFFu) * 8;
      int sum2 = 0, flips = 0;
      for (int j = 0; j < 8; ++j) sum2 += a2[j];
      for (int j = 0; j < 7; ++j) flips += (code >> (8 + j)) & 1u;
      const int neg7 = ((flips + sum2 / 2) & 1);  /* even total flips + coordinate sum */
      for (int j = 0; j < 8; ++j) {
        const int neg = j < 7 ? (int)((code >> (8 + j)) & 1u) : neg7;
        /* value in quarters: sign * 2|a| * 2 +- 1, exact */
        const int q4 = (neg ? -2 * a2[j] : 2 * a2[j]) + ((code >> 15) ? 1 : -1);
        const float v = (float)q4 * 0.25f;
        const float s = scales[i * ng + (8 * u + (uint64_t)j) / group];
        out[i * cols + 8 * u + j] = s * v;
      }
    }
  }
}

/* The built-in "lut" plugin (include/mlra.h mlra_lut_create; e.g. QLoRA's NF4):
 * codes in the reference's bitstream (bitpack.cpp:25-35), a per-matrix table of
 * 2^bits f32 levels and a per-(row, group) f32 scale:
 *   out[i, j] = RN_f32(s[i, j/g] * lut[c[i, j]])   (one IEEE multiply) */
ORC_EXPORT void orc_lut_dequant_f32(const uint32_t* words, uint64_t rows, uint64_t cols,
                                    int bits, uint64_t group, const float* lut,
                                    const float* scales, float* out) {
  const uint64_t ng = cols / group;
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t j = 0; j < cols; ++j) {
      const uint32_t c = orc_read_code(words, bits, i * cols + j);
      out[i * cols + j] = scales[i * ng + j / group] * lut[c];
    }
}

ORC_EXPORT uint16_t orc_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) /* NaN */
    return (uint16_t)((u >> 16) | 0x0040u);
  const uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb;
  return (uint16_t)(u >> 16);
}

ORC_EXPORT float orc_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* ------------------------------------------------------------------------ */
/* Dense f64 arithmetic — matrix.cpp:81-129 (fixed i-k-j order).             */
/* ------------------------------------------------------------------------ */

/* matrix.cpp:81-97: out[m×n] = a[m×k]·b[k×n], out zero-initialised. */
ORC_EXPORT void orc_matmul(const double* a, const double* b, uint64_t m,
                           uint64_t k, uint64_t n, double* out) {
  memset(out, 0, m * n * sizeof(double));
  for (uint64_t i = 0; i < m; ++i) {
    for (uint64_t p = 0; p < k; ++p) {
      const double aip = a[i * k + p];
      for (uint64_t j = 0; j < n; ++j) out[i * n + j] += aip * b[p * n + j];
    }
  }
}

/* matrix.cpp:99-107 */
static void orc_transpose(const double* a, uint64_t r, uint64_t c, double* out) {
  for (uint64_t i = 0; i < r; ++i)
    for (uint64_t j = 0; j < c; ++j) out[j * r + i] = a[i * c + j];
}

/* ------------------------------------------------------------------------ */
/* Low-precision linear — lowprec_linear.cpp:150-247 (WeightMaterialize).    */
/* ------------------------------------------------------------------------ */

/* lowprec_linear.cpp:158-171: out[s,i] = Σ_j x[s,j]·W[i,j], in-order sum.
 * `w` is the f64 dequantized matrix [d_out × d_in]. */
ORC_EXPORT void orc_lp_forward_dense(const double* w, uint64_t d_out,
                                     uint64_t d_in, const double* x,
                                     uint64_t m, double* out) {
  for (uint64_t s = 0; s < m; ++s) {
    for (uint64_t i = 0; i < d_out; ++i) {
      double acc = 0.0;
      const double* wrow = w + i * d_in;
      for (uint64_t j = 0; j < d_in; ++j) acc += x[s * d_in + j] * wrow[j];
      out[s * d_out + i] = acc;
    }
  }
}

/* lowprec_linear.cpp:207-221: grad_in[s,j] += g[s,i]·W[i,j], i outer. */
ORC_EXPORT void orc_lp_backward_dense(const double* w, uint64_t d_out,
                                      uint64_t d_in, const double* g,
                                      uint64_t m, double* grad_in) {
  memset(grad_in, 0, m * d_in * sizeof(double));
  for (uint64_t s = 0; s < m; ++s) {
    for (uint64_t i = 0; i < d_out; ++i) {
      const double gv = g[s * d_out + i];
      const double* wrow = w + i * d_in;
      for (uint64_t j = 0; j < d_in; ++j) grad_in[s * d_in + j] += gv * wrow[j];
    }
  }
}

/* ------------------------------------------------------------------------ */
/* ModuLoRA layer — lora.cpp:52-72 forward, tape replay for backward          */
/* (autodiff.cpp:101-139, 145-193, 315-327). A: [d_out×r], B: [d_in×r].       */
/* ------------------------------------------------------------------------ */

/* y = ((base + scaling·((x·B)·Aᵀ)) + bias), each step rounded as the tape
 * does: matmul (i-k-j), scale, add (a += b), bias_add. xb_out: [m×r]. */
ORC_EXPORT void orc_layer_forward_dense(const double* w, uint64_t d_out,
                                        uint64_t d_in, const double* a,
                                        const double* b, uint64_t r,
                                        double scaling, const double* bias,
                                        const double* x, uint64_t m, double* y,
                                        double* xb_out) {
  double* base = (double*)malloc(m * d_out * sizeof(double));
  double* xb = xb_out ? xb_out : (double*)malloc(m * r * sizeof(double));
  double* at = (double*)malloc(r * d_out * sizeof(double));
  double* ab = (double*)malloc(m * d_out * sizeof(double));
  orc_lp_forward_dense(w, d_out, d_in, x, m, base);      /* lora.cpp:65-66 */
  orc_matmul(x, b, m, d_in, r, xb);                       /* lora.cpp:68 */
  orc_transpose(a, d_out, r, at);                         /* lora.cpp:69 */
  orc_matmul(xb, at, m, r, d_out, ab);
  for (uint64_t i = 0; i < m * d_out; ++i) {
    const double low = ab[i] * scaling;                   /* lora.cpp:70 */
    const double sum = base[i] + low;                     /* add */
    y[i] = sum + (bias ? bias[i % d_out] : 0.0);          /* bias_add */
  }
  free(base);
  if (!xb_out) free(xb);
  free(at);
  free(ab);
}

/* Reverse replay of the 7 records of layer_forward for upstream grad g:
 *   bias_add → dbias = Σ_rows g (autodiff.cpp:183-191)
 *   add → g to both sides; scalar_mul → dab = scale(g, c)
 *   matmul(xb, Aᵀ) → d(xb) = dab·A ; d(Aᵀ) = xbᵀ·dab ; transpose → dA
 *   matmul(x, B) → dx = d(xb)·Bᵀ ; dB = xᵀ·d(xb)
 *   lp_linear → dx += g·W
 * dx may be NULL (x not requiring grad skips both dx contributions,
 * autodiff.cpp:136 / :150). dbias may be NULL (frozen bias). */
ORC_EXPORT void orc_layer_backward_dense(const double* w, uint64_t d_out,
                                         uint64_t d_in, const double* a,
                                         const double* b, uint64_t r,
                                         double scaling, const double* x,
                                         const double* xb, const double* g,
                                         uint64_t m, double* dx, double* da,
                                         double* db, double* dbias) {
  if (dbias) {
    memset(dbias, 0, d_out * sizeof(double));
    for (uint64_t i = 0; i < m; ++i)
      for (uint64_t j = 0; j < d_out; ++j) dbias[j] += g[i * d_out + j];
  }
  double* dab = (double*)malloc(m * d_out * sizeof(double));
  for (uint64_t i = 0; i < m * d_out; ++i) dab[i] = g[i] * scaling;
  /* d(xb) = dab · transpose(Aᵀ) = dab · A  ([m×d_out]·[d_out×r]) */
  double* dxb = (double*)malloc(m * r * sizeof(double));
  orc_matmul(dab, a, m, d_out, r, dxb);
  /* d(Aᵀ) = transpose(xb) · dab  ([r×m]·[m×d_out]) then dA = its transpose */
  double* xbt = (double*)malloc(r * m * sizeof(double));
  orc_transpose(xb, m, r, xbt);
  double* dat = (double*)malloc(r * d_out * sizeof(double));
  orc_matmul(xbt, dab, r, m, d_out, dat);
  orc_transpose(dat, r, d_out, da);
  /* matmul(x, B): dB = transpose(x) · d(xb) */
  double* xt = (double*)malloc(d_in * m * sizeof(double));
  orc_transpose(x, m, d_in, xt);
  orc_matmul(xt, dxb, d_in, m, r, db);
  if (dx) {
    double* bt = (double*)malloc(r * d_in * sizeof(double));
    orc_transpose(b, d_in, r, bt);
    orc_matmul(dxb, bt, m, r, d_in, dx); /* first accumulation: 0 + v = v */
    double* gx = (double*)malloc(m * d_in * sizeof(double));
    orc_lp_backward_dense(w, d_out, d_in, g, m, gx);
    for (uint64_t i = 0; i < m * d_in; ++i) dx[i] += gx[i];
    free(bt);
    free(gx);
  }
  free(dab);
  free(dxb);
  free(xbt);
  free(dat);
  free(xt);
}

/* ------------------------------------------------------------------------ */
/* AdamW::step — train.cpp:81-134 (one parameter; the caller loops over the  */
/* parameter list in order and stops at the first non-finite gradient, which */
/* the reference reports with NumericError, train.cpp:113-117).              */
/* ------------------------------------------------------------------------ */
/* Returns 0, or 6 (NumericError) without touching p/m/v when g holds a
 * non-finite value. */
ORC_EXPORT int orc_adamw_step(double beta1, double beta2, double eps, double weight_decay,
                              uint64_t step_index, double lr, uint64_t n, double* p,
                              double* m, double* v, const double* g) {
  for (uint64_t j = 0; j < n; ++j)
    if (!isfinite(g[j])) return 6;                           /* :113-117 */
  const double t = (double)step_index + 1.0;                 /* :99 */
  const double bc1 = 1.0 - pow(beta1, t);                    /* :100 */
  const double bc2 = 1.0 - pow(beta2, t);                    /* :101 */
  for (uint64_t j = 0; j < n; ++j) {                         /* :122-129 */
    m[j] = beta1 * m[j] + (1.0 - beta1) * g[j];
    v[j] = beta2 * v[j] + (1.0 - beta2) * g[j] * g[j];
    const double mhat = m[j] / bc1;
    const double vhat = v[j] / bc2;
    p[j] = p[j] * (1.0 - lr * weight_decay) - lr * mhat / (sqrt(vhat) + eps);
  }
  return 0;
}
