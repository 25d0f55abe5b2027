// common.cuh — device-resident frozen weight layout and the exact dequant unit.
//
// Device layout of a QuantizedMatrix (quantize.hpp:29-48):
//   * codes: the reference's LSB-first bitstream (bitpack.cpp:25-35), but laid
//     out ROW-PADDED: rows_pad x cols_pad codes, each row starting on a word
//     (rows_pad, cols_pad = multiples of 256). When rows and cols are already
//     multiples of 256 this IS the reference's whole-matrix stream, uploaded
//     verbatim (every BASELINE shape); otherwise a relayout kernel builds it.
//     Pad codes are 0.
//   * grid: float2 {s', z} per (row, group), rows_pad x ng_pad. s' = +s when the
//     group is "fma-certified" (fmaf(s,c,z) == (float)(double(s)*c+double(z))
//     for every code c), else -s (validate() guarantees s > 0, so the sign bit
//     is free). Pad groups are {1, 0}, so pad entries dequantize to exactly 0.
//
// Dequant contract: the f32 value of an entry is
// RN_f32(double(s)*c + double(z)) — bit-identical to (float) of the
// reference's f64 dequantize (quantize.cpp:123-137). Certified groups compute
// it with one fp32 FMA (exact: the f64 sum is exact there, so both roundings
// coincide); uncertified groups take the f64 path. bf16 = RN(f32).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace mlra {

struct QWeightDev {
  int64_t rows, cols;          // logical d_out (N), d_in (K)
  int64_t rows_pad, cols_pad;  // multiples of 256
  int bits;
  int64_t group;               // group size along cols (divides cols)
  int64_t ng_pad;              // grid row stride in groups: ceil(cols_pad/group) rounded to even
  int64_t row_words;           // 32-bit words per padded row = cols_pad*bits/32
  const uint32_t* words;       // rows_pad * row_words (+ 4 words slack)
  const float2* grid;          // rows_pad * ng_pad
  const float* lut = nullptr;  // lut plugin: 16 f32 levels (grid = {s, 0}); null = affine
};

// Device state of the built-in "cb2" codebook plugin (codebook.cu).
struct Cb2Dev {
  int64_t rows, cols, group, ng;  // ng = cols / group
  const uint16_t* codes;          // [rows x cols/8]
  // Device codebook layout (host-converted at upload; shared-memory gathers are
  // random, so the layout sets the bank-conflict cost):
  //  bf16 != 0: every magnitude is exactly a bf16 -> uint4[256], entry i = 8 bf16
  //             (one 16-B gather per code; products stay exact in f32);
  //  bf16 == 0: float4[2][256]: entries 0-3 of code i at [0][i], 4-7 at [1][i]
  //             (each gather's 16-B slot spans all 8 bank groups).
  const void* codebook;           // 16-B aligned
  int bf16;
  const float* scales;            // [rows x ng]
  // e8p != 0: the E8P lattice codebook (mlra_e8p_create): codebook = uint4[256]
  // of bf16 (|a| + 1/4) rows, uint4[256] of (|a| - 1/4) rows, then uint32[8]
  // "odd" bits (the abs pattern's coordinate sum is odd); see e8p_decode_signs.
  int e8p;
};

// E8P code -> (negate mask, use-(|a|+1/4) mask) of its 8 entries. Code bits:
// 0-7 abs-pattern index, 8-14 signs of entries 0-6, 15 the shift (+1/4 when
// set, -1/4 otherwise); entry 7's sign makes the count of negated entries
// congruent to the pattern's coordinate sum mod 2, so sign(a)·|a| lies in E8's
// half-integer coset (D8 + 1/2) before the shift. Entry j's value is
// sign_j · (|a_j| + sign_j·shift): the magnitude is |a_j| + 1/4 exactly when
// (negated_j XOR shift bit) is set.
__host__ __device__ __forceinline__ void e8p_decode_signs(uint32_t code, uint32_t odd,
                                                          uint32_t* neg, uint32_t* plus) {
  const uint32_t sb = (code >> 8) & 0x7Fu;
  uint32_t par = sb;
  par ^= par >> 4;
  par ^= par >> 2;
  par ^= par >> 1;
  const uint32_t n = sb | ((((par & 1u) ^ odd) & 1u) << 7);
  *neg = n;
  *plus = n ^ ((code >> 15) ? 0xFFu : 0u);
}

// Bits of the 8 consecutive codes of unit `u` (codes 8u..8u+7) of a
// word-aligned row, at the LSB of the result (bitpack.cpp:25-35 restated for
// 8 codes at a time).
template <int BITS>
__device__ __forceinline__ uint64_t load_unit(const uint32_t* __restrict__ rw, int64_t u) {
  if constexpr (BITS == 4) {
    return __ldg(rw + u);
  } else if constexpr (BITS == 8) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(rw) + u);
    return static_cast<uint64_t>(v.x) | (static_cast<uint64_t>(v.y) << 32);
  } else if constexpr (BITS == 2) {
    const uint32_t w = __ldg(rw + (u >> 1));
    return (w >> ((u & 1) * 16)) & 0xFFFFu;
  } else {  // 3 bits: 24-bit unit at bit 24u, may straddle two words
    const int64_t bit = u * 24;
    const int64_t w0 = bit >> 5;
    const uint32_t off = static_cast<uint32_t>(bit & 31);
    uint64_t v = __ldg(rw + w0) >> off;
    if (off > 8) v |= static_cast<uint64_t>(__ldg(rw + w0 + 1)) << (32 - off);
    return v & 0xFFFFFFu;
  }
}

__device__ __forceinline__ float code_to_f32(uint32_t c) {
  // exact int -> float for c < 2^23 without the I2F pipe
  return __int_as_float(0x4B000000u | c) - 8388608.0f;
}

// One dequantized entry, exact per the contract above. sg = signed scale.
__device__ __forceinline__ float deq_entry(uint32_t c, float sg, float z) {
  if (sg > 0.0f) return __fmaf_rn(sg, code_to_f32(c), z);
  return __double2float_rn(__fma_rn(static_cast<double>(-sg), static_cast<double>(c),
                                    static_cast<double>(z)));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// 8 codes sharing one grid entry -> 8 f32 values.
template <int BITS>
__device__ __forceinline__ void deq8_f32(uint64_t v, float2 g, float (&f)[8]) {
  constexpr uint32_t mask = (1u << BITS) - 1u;
  if (g.x > 0.0f) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      f[i] = __fmaf_rn(g.x, code_to_f32(static_cast<uint32_t>(v >> (BITS * i)) & mask), g.y);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      f[i] = deq_entry(static_cast<uint32_t>(v >> (BITS * i)) & mask, g.x, g.y);
  }
}

template <int BITS>
__device__ __forceinline__ uint4 deq8_bf16(uint64_t v, float2 g) {
  float f[8];
  deq8_f32<BITS>(v, g, f);
  uint4 o;
  o.x = pack_bf16x2(f[0], f[1]);
  o.y = pack_bf16x2(f[2], f[3]);
  o.z = pack_bf16x2(f[4], f[5]);
  o.w = pack_bf16x2(f[6], f[7]);
  return o;
}

// Packed-f32x2 ops (sm_100 FADD2 / FFMA2): same IEEE rounding per lane as the
// scalar forms, so results stay bit-identical to deq8_f32.
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint32_t f2_to_bf16x2(uint64_t p) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;"
      : "=r"(d)
      : "f"(__uint_as_float(static_cast<uint32_t>(p >> 32))),
        "f"(__uint_as_float(static_cast<uint32_t>(p))));
  return d;
}

// Magic-float words (0x4B000000 | c) of the 8 codes of a unit, in order.
template <int BITS>
__device__ __forceinline__ void unit_magic(uint32_t v, uint32_t (&m)[8]) {
  if constexpr (BITS == 4) {
    // nibbles 2j / 2j+1 live in byte j of lo / hi; PRMT drops each byte under
    // the 0x4B exponent byte in one instruction
    const uint32_t lo = v & 0x0F0F0F0Fu, hi = (v >> 4) & 0x0F0F0F0Fu;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      m[2 * j] = __byte_perm(lo, 0x4B000000u, 0x7540u | j);
      m[2 * j + 1] = __byte_perm(hi, 0x4B000000u, 0x7540u | j);
    }
  } else if constexpr (BITS == 2) {
    // spread the 2-bit fields into nibbles (x: codes 0,2,4,6; y: codes 1,3,5,7),
    // then the 4-bit byte-permute path: lo byte j = nibble 2j, hi byte j = nibble 2j+1
    const uint32_t w = (v & 0x3333u) | (((v >> 2) & 0x3333u) << 16);
    const uint32_t lo = w & 0x0F0F0F0Fu, hi = (w >> 4) & 0x0F0F0F0Fu;
    // lo bytes = codes (0, 4, 1, 5), hi bytes = codes (2, 6, 3, 7)
    m[0] = __byte_perm(lo, 0x4B000000u, 0x7540u);
    m[1] = __byte_perm(lo, 0x4B000000u, 0x7542u);
    m[2] = __byte_perm(hi, 0x4B000000u, 0x7540u);
    m[3] = __byte_perm(hi, 0x4B000000u, 0x7542u);
    m[4] = __byte_perm(lo, 0x4B000000u, 0x7541u);
    m[5] = __byte_perm(lo, 0x4B000000u, 0x7543u);
    m[6] = __byte_perm(hi, 0x4B000000u, 0x7541u);
    m[7] = __byte_perm(hi, 0x4B000000u, 0x7543u);
  } else {
    constexpr uint32_t mask = (1u << BITS) - 1u;
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = ((v >> (BITS * i)) & mask) | 0x4B000000u;
  }
}

// Fast unit: 8 codes (BITS <= 4, packed in v) sharing grid g -> 8 bf16.
// deq8_bf16_cert assumes a certified group (caller checked g.x > 0).
// Certified groups: FADD2 (exact code -> float) + FFMA2 (one rounding) +
// cvt.rn.bf16x2; uncertified groups take the exact f64 path.
template <int BITS>
__device__ __forceinline__ uint4 deq8_bf16_cert(uint32_t v, float2 g) {
  uint32_t m[8];
  unit_magic<BITS>(v, m);
  const uint64_t neg = 0xCB000000CB000000ull;  // (-2^23, -2^23)
  const uint64_t s2 = (static_cast<uint64_t>(__float_as_uint(g.x)) << 32) | __float_as_uint(g.x);
  const uint64_t z2 = (static_cast<uint64_t>(__float_as_uint(g.y)) << 32) | __float_as_uint(g.y);
  uint32_t o[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint64_t pr = (static_cast<uint64_t>(m[2 * j + 1]) << 32) | m[2 * j];
    o[j] = f2_to_bf16x2(f2_fma(f2_add(pr, neg), s2, z2));
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}
template <int BITS>
__device__ __forceinline__ uint4 deq8_bf16_fast(uint32_t v, float2 g) {
  if (!(g.x > 0.0f)) return deq8_bf16<BITS>(v, g);
  return deq8_bf16_cert<BITS>(v, g);
}

// General unit: groups may change inside the 8 codes (group % 8 != 0; only the
// small ragged reference-test shapes hit this).
template <int BITS>
__device__ __forceinline__ void deq8_f32_general(uint64_t v, const float2* __restrict__ grow,
                                                 int64_t k0, int64_t group, float (&f)[8]) {
  constexpr uint32_t mask = (1u << BITS) - 1u;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 g = __ldg(grow + (k0 + i) / group);
    f[i] = deq_entry(static_cast<uint32_t>(v >> (BITS * i)) & mask, g.x, g.y);
  }
}

template <int BITS>
__device__ __forceinline__ uint4 deq8_bf16_general(uint64_t v, const float2* __restrict__ grow,
                                                   int64_t k0, int64_t group) {
  float f[8];
  deq8_f32_general<BITS>(v, grow, k0, group, f);
  uint4 o;
  o.x = pack_bf16x2(f[0], f[1]);
  o.y = pack_bf16x2(f[2], f[3]);
  o.z = pack_bf16x2(f[4], f[5]);
  o.w = pack_bf16x2(f[6], f[7]);
  return o;
}

}  // namespace mlra
