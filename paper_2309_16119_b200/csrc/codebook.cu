// codebook.cu — the built-in non-affine plugins "cb2" and "e8p" (include/mlra.h,
// mlra_cb2_create): a QuIP#-style 2-bit vector codebook behind the device
// dequant hook (the GPU form of Quantizer::matvec, quantize.hpp:98-105).
//
// Format: one u16 code per 8 consecutive row entries — bits 0-7 index a
// 256 x 8 f32 magnitude codebook, bit 8+j negates entry j — and one f32 scale
// per (row, group) along cols. Ŵ[i, 8u+j] = RN_f32(s · ±cb[idx][j]) (one IEEE
// multiply, so bit-exact against oracle/mlra_oracle.c orc_cb2_dequant), then
// RN to bf16 for the GEMM operand.
//
// "e8p" (mlra_e8p_create) is QuIP#'s E8P lattice codebook in the same u16-per-8
// format: the 16 bits select one of 2^16 points of E8 + 1/4 (common.cuh
// e8p_decode_signs); Ŵ = RN_f32(s · value), value exact in bf16.
//
// k_cb2_materialize is HBM-bound: 0.25 B of code + 4/g B of scale read and
// 2 (bf16) or 4 (f32) B written per entry. The codebook lives in shared memory
// in a bank-conflict-aware layout (Cb2Dev); every warp store covers a
// contiguous 512 B.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace mlra {

namespace {

constexpr int kCbThreads = 256;
constexpr int kCbPerThread = 4;

// Magnitudes of a code's 8 entries from the shared codebook.
template <bool CB16>
__device__ __forceinline__ void cb2_mags(uint32_t code, const uint4* cbh, const float4* cb0,
                                         const float4* cb1, float (&m)[8]) {
  const uint32_t i = code & 0xFFu;
  if constexpr (CB16) {
    const uint4 q = cbh[i];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      m[2 * p] = __uint_as_float(w[p] << 16);
      m[2 * p + 1] = __uint_as_float(w[p] & 0xFFFF0000u);
    }
  } else {
    const float4 a = cb0[i], b = cb1[i];
    m[0] = a.x, m[1] = a.y, m[2] = a.z, m[3] = a.w;
    m[4] = b.x, m[5] = b.y, m[6] = b.z, m[7] = b.w;
  }
}

// E8P: the 8 magnitudes |a_j| + t·(1 - 2·neg_j) of a code (t = +-1/4 from bit
// 15; exact) and its negate byte (common.cuh e8p_decode_signs), from ONE
// shared-memory gather: `tab` = the 256 bf16 |a| rows with the pattern's
// odd-sum bit in the (zero) sign bit of entry 0 (staged by k_cb2_materialize).
__device__ __forceinline__ uint32_t e8p_mags(uint32_t code, const uint4* tab, float (&m)[8]) {
  const uint4 A = tab[code & 0xFFu];
  const uint32_t sb = (code >> 8) & 0x7Fu;
  const uint32_t n = sb | (((__popc(sb) ^ (A.x >> 15)) & 1u) << 7);
  const float t = (code >> 15) ? 0.25f : -0.25f;
  const uint32_t w[4] = {A.x & 0xFFFF7FFFu, A.y, A.z, A.w};
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    m[2 * p] = __uint_as_float(w[p] << 16) + (((n >> (2 * p)) & 1u) ? -t : t);
    m[2 * p + 1] = __uint_as_float(w[p] & 0xFFFF0000u) + (((n >> (2 * p + 1)) & 1u) ? -t : t);
  }
  return n;
}

// E8P bf16 output straight from the signed |a| row: w_j = RN_f32(s·(sign_j·|a_j| + t))
// (the fused GEMM decode's law, qgemm_dev.cuh dequant_units_e8p; identical bits
// to sign_j·RN(s·(|a_j| +- 1/4)) since RN is odd-symmetric) — no per-entry
// magnitude select, one sign-mask XOR per pair.
__device__ __forceinline__ uint4 e8p_bf16(uint32_t code, const uint4* tab, float s) {
  const uint4 A = tab[code & 0xFFu];
  const uint32_t sb = (code >> 8) & 0x7Fu;
  const uint32_t n = sb | (((__popc(sb) ^ (A.x >> 15)) & 1u) << 7);
  const float t = (code >> 15) ? 0.25f : -0.25f;
  const uint32_t w[4] = {A.x & 0xFFFF7FFFu, A.y, A.z, A.w};
  uint32_t o[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const uint32_t ws = w[p] ^ ((((n >> (2 * p)) & 3u) * 0x40008000u) & 0x80008000u);
    o[p] = pack_bf16x2(__fmul_rn(s, __uint_as_float(ws << 16) + t),
                       __fmul_rn(s, __uint_as_float(ws & 0xFFFF0000u) + t));
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// One code -> 8 bf16 outputs. Products RN_f32(s·mag) (scalar IEEE
// multiplies); the sign is applied after rounding (RN commutes with negation):
// the mask of entries (2p, 2p+1) is ((code >> (8+2p)) & 3) * 0x40008000 &
// 0x80008000 — bit 15 and bit 31 of the packed pair — 3 ops per pair.
template <bool VEC>
__device__ __forceinline__ void cb2_emit(void* __restrict__ out, int64_t o, uint32_t sg, float s,
                                         const float (&m)[8]) {
  // sg: negate bit per entry (cb2: code >> 8; e8p: e8p_decode_signs)
  float f[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) f[e] = __fmul_rn(s, m[e]);
  uint4 v;
  v.x = pack_bf16x2(f[0], f[1]) ^ ((((sg) & 3u) * 0x40008000u) & 0x80008000u);
  v.y = pack_bf16x2(f[2], f[3]) ^ ((((sg >> 2) & 3u) * 0x40008000u) & 0x80008000u);
  v.z = pack_bf16x2(f[4], f[5]) ^ ((((sg >> 4) & 3u) * 0x40008000u) & 0x80008000u);
  v.w = pack_bf16x2(f[6], f[7]) ^ ((((sg >> 6) & 3u) * 0x40008000u) & 0x80008000u);
  if constexpr (VEC) {
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + o) = v;
  } else {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 8; ++e)
      reinterpret_cast<uint16_t*>(out)[o + e] = static_cast<uint16_t>(w[e >> 1] >> (16 * (e & 1)));
  }
}

// f32 output, half a code per thread: entries 4h..4h+3 of the code, one
// 16-B store — adjacent lanes write adjacent 16 B, so each warp store covers
// a contiguous 512 B (a whole code per lane would leave 32-B gaps per store).
template <bool VEC, bool CB16, bool E8P>
__device__ __forceinline__ void cb2_emit_half(float* __restrict__ out, int64_t o, uint32_t code,
                                              float s, int h, const uint4* cbh, const float4* cb0,
                                              const float4* cb1, const uint32_t* odd) {
  const uint32_t i = code & 0xFFu;
  float m[4];
  uint32_t sg = code >> (8 + 4 * h);
  if constexpr (E8P) {
    float m8[8];
    sg = e8p_mags(code, cbh, m8) >> (4 * h);
#pragma unroll
    for (int e = 0; e < 4; ++e) m[e] = m8[4 * h + e];
  } else if constexpr (CB16) {
    const uint4 q = cbh[i];
    const uint32_t a = h ? q.z : q.x, b = h ? q.w : q.y;
    m[0] = __uint_as_float(a << 16), m[1] = __uint_as_float(a & 0xFFFF0000u);
    m[2] = __uint_as_float(b << 16), m[3] = __uint_as_float(b & 0xFFFF0000u);
  } else {
    const float4 v = h ? cb1[i] : cb0[i];
    m[0] = v.x, m[1] = v.y, m[2] = v.z, m[3] = v.w;
  }
  float f[4];
#pragma unroll
  for (int e = 0; e < 4; ++e)
    f[e] = __uint_as_float(__float_as_uint(__fmul_rn(s, m[e])) ^ (((sg >> e) & 1u) << 31));
  if constexpr (VEC) {
    *reinterpret_cast<float4*>(out + o) = make_float4(f[0], f[1], f[2], f[3]);
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) out[o + e] = f[e];
  }
}

// Work items = (row, pass of kCbThreads * kCbPerThread codes) strided over a
// resident-size grid (the 8 KB codebook is staged into shared memory once per
// CTA); the (row, pass) of a thread's next item advances incrementally (no
// per-item division). Software-pipelined: the codes and scales of the next item
// are loaded before the current item is decoded (ncu: the one-pass-at-a-time
// form was long-scoreboard bound at 32% of DRAM bandwidth). Within a pass a
// thread owns kCbPerThread codes strided by the block size, so each warp store
// covers a contiguous 512 B (bf16).
template <bool F32, bool VEC, bool CB16, bool E8P>
__global__ void __launch_bounds__(kCbThreads) k_cb2_materialize(
    const Cb2Dev c, int64_t row0, int64_t nrows, int64_t col0, int64_t ncols,
    void* __restrict__ out, int64_t ld, int gshift) {
  // cb2: 256 (bf16 rows) or 512 (f32 halves) float4; e8p: the 256 |a| rows (e8p_mags)
  constexpr int NCB = CB16 ? 256 : 512;
  __shared__ float4 cbs[NCB];
  const uint4* cbh = reinterpret_cast<const uint4*>(cbs);
  const float4* cb0 = cbs;
  const float4* cb1 = cbs + 256;
  const uint32_t* odd = nullptr;
  if constexpr (E8P) {  // |a| = (|a| + 1/4) - 1/4 (bf16-exact), odd bit -> sign bit of entry 0
    const uint4* src = reinterpret_cast<const uint4*>(c.codebook);
    const uint32_t* oddw = reinterpret_cast<const uint32_t*>(src + 512);
    for (int i = threadIdx.x; i < 256; i += kCbThreads) {
      const uint4 pr = __ldg(src + i);
      const uint32_t pw[4] = {pr.x, pr.y, pr.z, pr.w};
      uint32_t aw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        aw[q] = pack_bf16x2(__uint_as_float(pw[q] << 16) - 0.25f,
                            __uint_as_float(pw[q] & 0xFFFF0000u) - 0.25f);
      aw[0] |= ((__ldg(oddw + (i >> 5)) >> (i & 31)) & 1u) << 15;
      reinterpret_cast<uint4*>(cbs)[i] = make_uint4(aw[0], aw[1], aw[2], aw[3]);
    }
  } else {
    for (int i = threadIdx.x; i < NCB; i += kCbThreads)
      cbs[i] = __ldg(reinterpret_cast<const float4*>(c.codebook) + i);
  }
  constexpr int SH = F32 ? 1 : 0;  // work unit: a code (bf16) or half a code (f32)
  const int ncodes = static_cast<int>(ncols >> 3);
  const int nunits = ncodes << SH;
  const int ucol0 = static_cast<int>(col0 >> 3);
  const int64_t cpr = c.cols >> 3;  // codes per full row
  const int gdiv = static_cast<int>(c.group);
  constexpr int CH = kCbThreads * kCbPerThread;
  const int ipr = (nunits + CH - 1) / CH;  // passes per row
  const int drow = static_cast<int>(gridDim.x) / ipr, dpass = static_cast<int>(gridDim.x) % ipr;
  int64_t rr = static_cast<int64_t>(blockIdx.x) / ipr;
  int pass = static_cast<int>(blockIdx.x) % ipr;
  uint32_t code[kCbPerThread];
  float scl[kCbPerThread];
  auto fetch = [&](int64_t r, int ps) {
    const int base = ps * CH + static_cast<int>(threadIdx.x);
    const uint16_t* crow = c.codes + (row0 + r) * cpr + ucol0;
    const float* srow = c.scales + (row0 + r) * c.ng;
#pragma unroll
    for (int j = 0; j < kCbPerThread; ++j) {
      const int it = base + j * kCbThreads;
      const int ci = it >> SH;
      const int k = (ucol0 + ci) << 3;
      code[j] = it < nunits ? __ldg(crow + ci) : 0u;
      scl[j] = it < nunits ? __ldg(srow + (gshift >= 0 ? (k >> gshift) : k / gdiv)) : 0.0f;
    }
  };
  if (rr < nrows) fetch(rr, pass);
  __syncthreads();
  while (rr < nrows) {
    uint32_t cur[kCbPerThread];
    float cs[kCbPerThread];
#pragma unroll
    for (int j = 0; j < kCbPerThread; ++j) {
      cur[j] = code[j];
      cs[j] = scl[j];
    }
    const int64_t r_cur = rr;
    const int p_cur = pass;
    pass += dpass;
    rr += drow;
    if (pass >= ipr) {
      pass -= ipr;
      ++rr;
    }
    if (rr < nrows) fetch(rr, pass);  // next item in flight
    const int base = p_cur * CH + static_cast<int>(threadIdx.x);
    void* orow = F32 ? static_cast<void*>(reinterpret_cast<float*>(out) + r_cur * ld)
                     : static_cast<void*>(reinterpret_cast<__nv_bfloat16*>(out) + r_cur * ld);
#pragma unroll
    for (int j = 0; j < kCbPerThread; ++j) {
      const int it = base + j * kCbThreads;
      if (it >= nunits) break;
      if constexpr (F32) {
        cb2_emit_half<VEC, CB16, E8P>(static_cast<float*>(orow), static_cast<int64_t>(it) << 2,
                                      cur[j], cs[j], it & 1, cbh, cb0, cb1, odd);
      } else {
        if constexpr (E8P) {
          const uint4 v = e8p_bf16(cur[j], cbh, cs[j]);
          const int64_t o = static_cast<int64_t>(it) << 3;
          if constexpr (VEC) {
            *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(orow) + o) = v;
          } else {
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 8; ++e)
              reinterpret_cast<uint16_t*>(orow)[o + e] = static_cast<uint16_t>(w[e >> 1] >> (16 * (e & 1)));
          }
        } else {
          float m[8];
          cb2_mags<CB16>(cur[j], cbh, cb0, cb1, m);
          cb2_emit<VEC>(orow, static_cast<int64_t>(it) << 3, cur[j] >> 8, cs[j], m);
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_cb2_materialize(const Cb2Dev& c, int64_t row0, int64_t nrows, int64_t col0,
                                   int64_t ncols, void* out, int64_t ld, bool f32,
                                   cudaStream_t st) {
  if (nrows <= 0 || ncols <= 0) return cudaSuccess;
  const bool vec = (ld % 8 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  int gshift = -1;
  for (int s = 3; s < 31; ++s)
    if ((int64_t{1} << s) == c.group) gshift = s;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;  // one resident wave
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cb2_materialize<false, true, false, false>,
                                                    kCbThreads, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int64_t cap = static_cast<int64_t>(sms) * per_sm;
  const int64_t nunits = (ncols >> 3) << (f32 ? 1 : 0);
  const int64_t items = nrows * ((nunits + kCbThreads * kCbPerThread - 1) / (kCbThreads * kCbPerThread));
  const dim3 grid(static_cast<unsigned>(items < cap ? items : cap));
  note_launch();
#define MLRA_CB2_LAUNCH(F, V, H, E)                                                          \
  k_cb2_materialize<F, V, H, E><<<grid, kCbThreads, 0, st>>>(c, row0, nrows, col0, ncols, out, \
                                                             ld, gshift)
  if (c.e8p) {
    if (f32) {
      if (vec) MLRA_CB2_LAUNCH(true, true, true, true); else MLRA_CB2_LAUNCH(true, false, true, true);
    } else {
      if (vec) MLRA_CB2_LAUNCH(false, true, true, true); else MLRA_CB2_LAUNCH(false, false, true, true);
    }
  } else if (c.bf16) {
    if (f32) {
      if (vec) MLRA_CB2_LAUNCH(true, true, true, false); else MLRA_CB2_LAUNCH(true, false, true, false);
    } else {
      if (vec) MLRA_CB2_LAUNCH(false, true, true, false); else MLRA_CB2_LAUNCH(false, false, true, false);
    }
  } else {
    if (f32) {
      if (vec) MLRA_CB2_LAUNCH(true, true, false, false); else MLRA_CB2_LAUNCH(true, false, false, false);
    } else {
      if (vec) MLRA_CB2_LAUNCH(false, true, false, false); else MLRA_CB2_LAUNCH(false, false, false, false);
    }
  }
#undef MLRA_CB2_LAUNCH
  return cudaGetLastError();
}

}  // namespace mlra
