// qgemm_dev.cuh — device helpers shared by the 1-CTA (qgemm.cu) and CTA-pair
// (qgemm2.cu) fused dequant GEMMs.
#pragma once
#include <stdint.h>

#include "common.cuh"
#include "ptx.cuh"
#include "qgemm.h"

namespace mlra {
namespace qg {

constexpr int BM = 128;
constexpr int BK = 64;
#ifndef MLRA_PROD_NS
#define MLRA_PROD_NS 128  // backoff of the TMA producers' empty/qempty waits
#endif
#ifndef MLRA_EPI_NS
#define MLRA_EPI_NS 64  // backoff of the epilogue's tfull wait
#endif
#ifndef MLRA_STAGES
#define MLRA_STAGES 4
#endif
constexpr int STAGES = MLRA_STAGES;
constexpr int PROD_NS = MLRA_PROD_NS;
constexpr int EPI_NS = MLRA_EPI_NS;
constexpr int MAX_QS = 4;
constexpr int W_TILE = BM * BK * 2;  // 16 KB
constexpr int T_TILE = 256 * BK * 2;  // 32 KB: the pair kernel's stage (2 x 128 tokens), the 1-CTA kernel's at 256 tokens
constexpr int EPI_WARP0 = 4;
constexpr int DQ_WARP0 = 8;
constexpr int NUM_DQ_WARPS = 8;
constexpr int NUM_DQ_THREADS = NUM_DQ_WARPS * 32;
constexpr int NUM_THREADS = (DQ_WARP0 + NUM_DQ_WARPS) * 32;
constexpr int UNITS_PER_GROUP_THREAD = (BM * BK / 8) / (NUM_DQ_THREADS / 2);  // 8
constexpr int SMEM_LIMIT = 232448;
constexpr int SMEM_FIXED = 1024 + STAGES * (W_TILE + T_TILE) + 512;
// 1-CTA kernel with 128-token tiles: half-size activation stages, so a deeper
// ring (6 stages) fits — at small m its k-block rate is bound by the latency of
// one stage's round trip (dequant/TMA -> MMA -> commit -> refill), not by MMA.
#ifndef MLRA_STAGES128
#define MLRA_STAGES128 6
#endif
__host__ __device__ constexpr int qgemm1_stages(int tbn) { return tbn == 128 ? MLRA_STAGES128 : STAGES; }
__host__ __device__ constexpr int qgemm1_smem_fixed(int tbn) {
  return 1024 + qgemm1_stages(tbn) * (W_TILE + tbn * BK * 2) + 512;
}

// Unit u (0..1023) of a stage -> byte offset of its 16-byte chunk inside the
// SW128 operand tile, plus its position in the packed tile.
//  K-major (forward): tile = 128 rows x 64 k; unit = (r = u/8, k8 = u%8);
//     canonical K-major SW128: row r at r*128, chunk k8 at (k8 ^ r%8)*16.
//  MN-major (dX):     tile = 64 reduction rows (n) x 128 output cols (k);
//     unit = (n = u/16, k8 = u%16); 64-column chunk c = k8/8 at c*8192,
//     row n at n*128, 16-byte column group (k8%8 ^ n%8).
template <bool MN>
__device__ __forceinline__ uint32_t unit_soff(int u) {
  if constexpr (!MN) {
    const int r = u >> 3, k8 = u & 7;
    return r * 128 + ((k8 ^ (r & 7)) << 4);
  } else {
    const int n = u >> 4, k8 = u & 15;
    return (k8 >> 3) * 8192 + n * 128 + (((k8 & 7) ^ (n & 7)) << 4);
  }
}

// Packed unit j (8 codes) of a Q-ring row (16*BITS bytes = 128 codes) at
// shared address `row`.
template <int BITS>
__device__ __forceinline__ uint32_t q_unit(uint32_t row, int j) {
  if constexpr (BITS == 4) {
    return lds32(row + j * 4);
  } else if constexpr (BITS == 2) {
    return lds16(row + j * 2);
  } else {
    const int off = j * 3;
    const uint32_t a = row + (off & ~3);
    return __funnelshift_r(lds32(a), lds32(a + 4), (off & 3) * 8) & 0xFFFFFFu;
  }
}

// Group index of the first code of 128-code block `blk` along the code rows.
// group >= 128: blk / (group/128) via the host's round-up reciprocal (exact for
// blk < 2^32 / divisor; 0 encodes divisor 1) instead of a runtime-divisor
// divide on every stage's critical path.
__device__ __forceinline__ int pair_group(int blk, const GemmArgs& p) {
  if (p.q_group_shift >= 0) return blk << (7 - p.q_group_shift);
  return p.q_group_magic == 0u ? blk : static_cast<int>(__umulhi(static_cast<uint32_t>(blk),
                                                                p.q_group_magic));
}

// One thread's share of a dequant stage: UPT units of 8 codes (rows rbase +
// i*ROW_STEP of the Q stage) -> bf16 into the SW128 W tile. All code and grid
// loads issue first; a single warp vote on the per-group certificates then
// selects the branch-free FADD2/FFMA2 path for all units, so the units overlap
// instead of serialising behind a per-unit branch.
template <int BITS, int UPT, int ROW_STEP>
__device__ __forceinline__ void dequant_units(uint32_t qc, uint32_t qg, uint32_t st,
                                              const uint32_t (&soff)[UPT], int unit, int gsub,
                                              int rbase, int gbox) {
  constexpr int QROW = 16 * BITS;
  uint32_t v[UPT];
  float2 g[UPT];
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const int row = rbase + i * ROW_STEP;
    v[i] = q_unit<BITS>(qc + row * QROW, unit);
    g[i] = lds_f2(qg + row * gbox + gsub * 8);
  }
  bool ok = true;
#pragma unroll
  for (int i = 0; i < UPT; ++i) ok = ok && (g[i].x > 0.0f);
  if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
    for (int i = 0; i < UPT; ++i) sts128(st + soff[i], deq8_bf16_cert<BITS>(v[i], g[i]));
  } else {
#pragma unroll
    for (int i = 0; i < UPT; ++i) sts128(st + soff[i], deq8_bf16_fast<BITS>(v[i], g[i]));
  }
}

// The cb2 codebook plugin's tile decode (codebook.cu, fused path): BITS tag
// kCb2Bits selects it; its packed stream has the 2-bit geometry (one u16 code
// per 8 weights), so the Q ring is loaded exactly as for BITS = 2 and only the
// decode differs. `cbs` = shared address of the bf16-exact codebook, uint4[256].
constexpr int kCb2Bits = 18;
// The lut plugin (a per-matrix table of 2^b f32 levels, e.g. NF4): BITS tag
// kLutTag + b; its codes are the plain b-bit stream, so only the decode differs.
constexpr int kLutTag = 32;
// The e8p plugin (E8P lattice codebook): the cb2 stream geometry, decode by
// e8p_decode_signs over (|a| +- 1/4) tables (qgemm.h kE8pSmemBytes).
constexpr int kE8pBits = 19;
template <int BITS>
constexpr bool is_lut() { return BITS > kLutTag; }
template <int BITS>
constexpr int q_geom_bits() {
  return (BITS == kCb2Bits || BITS == kE8pBits) ? 2 : (BITS > kLutTag ? BITS - kLutTag : BITS);
}

__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}

template <int UPT, int ROW_STEP>
__device__ __forceinline__ void dequant_units_cb2(uint32_t qc, uint32_t qg, uint32_t st,
                                                  const uint32_t (&soff)[UPT], int unit, int gsub,
                                                  int rbase, int gbox, uint32_t cbs) {
  constexpr int QROW = 32;  // 128 weights x 2 bits
  uint32_t v[UPT];
  float sc[UPT];
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const int row = rbase + i * ROW_STEP;
    v[i] = lds16(qc + row * QROW + unit * 2);
    sc[i] = lds_f2(qg + row * gbox + gsub * 8).x;
  }
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const uint4 q = lds128(cbs + ((v[i] & 0xFFu) << 4));
    const float s = fabsf(sc[i]);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    uint32_t o[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const float a = __fmul_rn(s, __uint_as_float(w[p] << 16));
      const float b = __fmul_rn(s, __uint_as_float(w[p] & 0xFFFF0000u));
      o[p] = pack_bf16x2(a, b) ^ ((((v[i] >> (8 + 2 * p)) & 3u) * 0x40008000u) & 0x80008000u);
    }
    sts128(st + soff[i], make_uint4(o[0], o[1], o[2], o[3]));
  }
}

// The e8p plugin's tile decode. Entry j of a code is sign_j·(|a_j| + sign_j·t)
// = sign_j·|a_j| + t (t = +-1/4 from bit 15, sign_j^2 = 1), exact in fp32, so
// w_j = RN_f32(s · (sign_j·|a_j| + t)) — bit for bit the law of
// k_cb2_materialize's e8p path (sign_j·RN(s·(|a_j| +- 1/4)); RN is odd-symmetric).
// ONE shared-memory gather per code, as in the cb2 decode: `tab` holds the 256
// bf16 |a| rows (built by the kernel prologue from the (|a| +- 1/4) tables)
// with the pattern's odd-sum bit in the (otherwise zero) sign bit of entry 0;
// the negate byte (e8p_decode_signs) and its sign-bit masks are ALU work.
template <int UPT, int ROW_STEP>
__device__ __forceinline__ void dequant_units_e8p(uint32_t qc, uint32_t qg, uint32_t st,
                                                  const uint32_t (&soff)[UPT], int unit, int gsub,
                                                  int rbase, int gbox, uint32_t tab) {
  constexpr int QROW = 32;  // 128 weights x 2 bits
  uint32_t v[UPT];
  float sc[UPT];
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const int row = rbase + i * ROW_STEP;
    v[i] = lds16(qc + row * QROW + unit * 2);
    sc[i] = lds_f2(qg + row * gbox + gsub * 8).x;
  }
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const uint4 A = lds128(tab + ((v[i] & 0xFFu) << 4));
    const uint32_t sb = (v[i] >> 8) & 0x7Fu;
    const uint32_t n = sb | (((__popc(sb) ^ (A.x >> 15)) & 1u) << 7);  // negate byte
    const uint32_t w[4] = {A.x & 0xFFFF7FFFu, A.y, A.z, A.w};
    const float t = (v[i] >> 15) ? 0.25f : -0.25f;
    const float s = fabsf(sc[i]);
    uint32_t o[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const uint32_t ws = w[p] ^ ((((n >> (2 * p)) & 3u) * 0x40008000u) & 0x80008000u);
      o[p] = pack_bf16x2(__fmul_rn(s, __uint_as_float(ws << 16) + t),
                         __fmul_rn(s, __uint_as_float(ws & 0xFFFF0000u) + t));
    }
    sts128(st + soff[i], make_uint4(o[0], o[1], o[2], o[3]));
  }
}

// The lut plugin's tile decode: w = RN_f32(s · lut[c]) -> bf16, the same
// law as k_materialize_lut (materialize.cu), so fused == materialized bit for
// bit. `lut` = shared address of the 16-float table: 16 consecutive words sit
// in 16 distinct banks, so the per-code gathers never conflict.
template <int B, int UPT, int ROW_STEP>
__device__ __forceinline__ void dequant_units_lut(uint32_t qc, uint32_t qg, uint32_t st,
                                                  const uint32_t (&soff)[UPT], int unit, int gsub,
                                                  int rbase, int gbox, uint32_t lut) {
  constexpr int QROW = 16 * B;
  constexpr uint32_t mask = (1u << B) - 1u;
  uint32_t v[UPT];
  float sc[UPT];
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const int row = rbase + i * ROW_STEP;
    v[i] = q_unit<B>(qc + row * QROW, unit);
    sc[i] = lds_f2(qg + row * gbox + gsub * 8).x;
  }
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    uint32_t o[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const float a = __fmul_rn(sc[i], __uint_as_float(lds32(lut + (((v[i] >> (B * 2 * p)) & mask) << 2))));
      const float b =
          __fmul_rn(sc[i], __uint_as_float(lds32(lut + (((v[i] >> (B * (2 * p + 1))) & mask) << 2))));
      o[p] = pack_bf16x2(a, b);
    }
    sts128(st + soff[i], make_uint4(o[0], o[1], o[2], o[3]));
  }
}

struct TileIter {
  int m_tiles;
  int n_tiles;
  __device__ __forceinline__ void coords(int tile, int& m, int& n) const {
    m = tile % m_tiles;
    n = tile / m_tiles;
  }
};

}  // namespace qg
}  // namespace mlra
