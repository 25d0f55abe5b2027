// rht.cu — the randomized Hadamard transform of activations (QuIP#'s
// incoherence processing, "orthogonal matrices multiplication in the forward
// and backward passes"), for layers whose weights were
// quantized in a rotated basis W~ = U W V^T with U = H_b·diag(s_u),
// V = H_b·diag(s_v) block-diagonal (b-wide orthonormal Walsh-Hadamard blocks
// times random signs; b | d, b a power of two, so every LLaMA width works —
// e.g. 6656 = 13 x 512, 17920 = 35 x 512):
//   forward  y = U^T (W~ (V x)),      backward dx = V^T (W~^T (U dy)).
// One kernel per application, HBM-bound (2 B read + 2 or 4 B written per
// element): one warp per b-wide block of one row, b/32 contiguous elements per
// lane (coalesced 16-B-multiple loads), log2(b/32) butterfly stages in
// registers and 5 across lanes (shfl.xor), fp32 arithmetic, the 1/sqrt(b)
// normalisation folded into the last stage.
//   mode 0 (apply):   out = H_b · diag(s) · in / sqrt(b)      (V x, U dy)
//   mode 1 (inverse): out = diag(s) · H_b · in / sqrt(b)      (V^T d~x, U^T y~)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include "../../include/mlra.h"
#include "kernels.h"

namespace mlra {

namespace {

template <int E, bool OUT_F32>
__global__ void __launch_bounds__(256) k_rht(const __nv_bfloat16* __restrict__ in, int64_t rows,
                                            int64_t cols, int64_t ld_in,
                                            const float* __restrict__ signs, int inverse,
                                            void* __restrict__ out, int64_t ld_out) {
  constexpr int B = 32 * E;
  const int lane = threadIdx.x & 31;
  const int64_t seg = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nseg = rows * (cols / B);
  if (seg >= nseg) return;
  const int64_t r = seg / (cols / B), c0 = (seg - r * (cols / B)) * B + lane * E;
  float v[E];
  const __nv_bfloat16* src = in + r * ld_in + c0;
#pragma unroll
  for (int e = 0; e < E; e += 2) {
    const __nv_bfloat162 p = *reinterpret_cast<const __nv_bfloat162*>(src + e);
    v[e] = __bfloat162float(p.x);
    v[e + 1] = __bfloat162float(p.y);
  }
  if (!inverse) {
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] *= __ldg(signs + c0 + e);
  }
#pragma unroll
  for (int h = 1; h < E; h <<= 1) {  // in-register stages
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if ((e & h) == 0) {
        const float a = v[e], b = v[e + h];
        v[e] = a + b;
        v[e + h] = a - b;
      }
    }
  }
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {  // cross-lane stages (element stride m·E)
    const bool hi = lane & m;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float o = __shfl_xor_sync(0xffffffffu, v[e], m);
      v[e] = hi ? o - v[e] : v[e] + o;
    }
  }
  const float norm = rsqrtf(static_cast<float>(B));
#pragma unroll
  for (int e = 0; e < E; ++e) {
    v[e] *= norm;
    if (inverse) v[e] *= __ldg(signs + c0 + e);
  }
  if constexpr (OUT_F32) {
    float* dst = reinterpret_cast<float*>(out) + r * ld_out + c0;
#pragma unroll
    for (int e = 0; e < E; e += 2) *reinterpret_cast<float2*>(dst + e) = make_float2(v[e], v[e + 1]);
  } else {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(out) + r * ld_out + c0;
#pragma unroll
    for (int e = 0; e < E; e += 2)
      *reinterpret_cast<__nv_bfloat162*>(dst + e) = __floats2bfloat162_rn(v[e], v[e + 1]);
  }
}

// Tensor-core form for b = 16·A (A in {16, 32, 64}: b = 256, 512, 1024). A
// block x (b elements) is the A x 16 matrix M[a][c] = x[16a + c]; with Sylvester
// ordering H_b = H_A (x) H_16, so H_b·x = vec(H_A · M · H_16) (H symmetric).
// One warp per block, two bf16 mma.sync m16n8k16 stages, fp32 accumulation:
//  1. M1^T = H_16 · M^T: the x values are exact bf16 operands (B fragments
//     loaded straight from global, sign flips applied to the bf16 bits);
//  2. Y = H_A · M1: step 1's fp32 accumulator fragments are exactly step 2's
//     B fragments (row/col of the m16n8 C layout = k/n of the B layout of the
//     transpose), split into three bf16 parts (hi + mid + lo = the full 24-bit
//     fp32 value), so the product of the +-1 entries stays fp32-exact.
// H entries are (-1)^popc(i & j). Output fragments hold 2 consecutive
// elements per lane. Same law as the butterfly kernel up to fp32 summation
// order; no shuffles (the butterfly kernel's 5 cross-lane stages made it
// shuffle-bound at ~1 TB/s).
__device__ __forceinline__ uint32_t h_pair(int i, int j) {  // bf16x2 {H[i][j], H[i][j+1]}
  const uint32_t lo = (__popc(i & j) & 1) ? 0xBF80u : 0x3F80u;
  const uint32_t hi = (__popc(i & (j + 1)) & 1) ? 0xBF80u : 0x3F80u;
  return lo | (hi << 16);
}

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t sign_mask2(const float* s) {  // flip bf16 sign bits where s < 0
  const float2 v = __ldg(reinterpret_cast<const float2*>(s));
  return (v.x < 0.0f ? 0x8000u : 0u) | (v.y < 0.0f ? 0x80000000u : 0u);
}

// three-way bf16 split of two fp32 values: parts[p] = bf16x2 of part p
__device__ __forceinline__ void split3(float x, float y, uint32_t (&parts)[3]) {
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
    parts[p] = *reinterpret_cast<const uint32_t*>(&h);
    x -= __bfloat162float(h.x);
    y -= __bfloat162float(h.y);
  }
}

constexpr int kRhtRing = 4;  // blocks in flight per warp (cp.async ring)

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// RING: every warp keeps kRhtRing blocks in flight through a shared-memory ring
// filled by cp.async (16-B aligned rows; the register-prefetch form had one
// block of prefetch per warp and was latency-bound: ncu 27 % DRAM, 30 % tensor)
template <int A, bool OUT_F32, bool RING>
__global__ void __launch_bounds__(256, A <= 32 ? 3 : 1) k_rht_tc(const __nv_bfloat16* __restrict__ in, int64_t rows,
                                               int64_t cols, int64_t ld_in,
                                               const float* __restrict__ signs, int inverse,
                                               void* __restrict__ out, int64_t ld_out) {
  constexpr int B = 16 * A, NT1 = A / 8, MT = A / 16;
  constexpr int SLOT = B * 2;              // bytes of one block
  constexpr int CPL = SLOT / (16 * 32);    // 16-B copies per lane per block
  extern __shared__ __align__(16) unsigned char rht_ring[];
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t nblk = cols / B, total = rows * nblk;
  const int64_t warp0 = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  // H_16 A fragments (step 1), loop invariant
  const uint32_t h0 = h_pair(g, 2 * tq), h1 = h_pair(g + 8, 2 * tq), h2 = h_pair(g, 2 * tq + 8),
                 h3 = h_pair(g + 8, 2 * tq + 8);
  const float norm = rsqrtf(static_cast<float>(B));
  const uint32_t wring = static_cast<uint32_t>(__cvta_generic_to_shared(rht_ring)) +
                         static_cast<uint32_t>(threadIdx.x >> 5) * (kRhtRing * SLOT);
  auto issue = [&](int64_t b, int slot) {  // block b -> ring slot (one commit group)
    if (b < total) {
      const int64_t r = b / nblk, c0 = (b - r * nblk) * B;
      const unsigned char* src = reinterpret_cast<const unsigned char*>(in + r * ld_in + c0);
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        cp_async16(wring + slot * SLOT + (lane + 32 * c) * 16, src + (lane + 32 * c) * 16);
    }
    cp_async_commit();
  };
  uint32_t nb0[NT1], nb1[NT1];
  auto load = [&](int64_t b) {
    const int64_t r = b / nblk, c0 = (b - r * nblk) * B;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(in + r * ld_in + c0);
#pragma unroll
    for (int j = 0; j < NT1; ++j) {
      const int e = 16 * (8 * j + g) + 2 * tq;  // element of b0 (b1: e + 8)
      nb0[j] = __ldg(src + e / 2);
      nb1[j] = __ldg(src + e / 2 + 4);
    }
  };
  if constexpr (RING) {
#pragma unroll
    for (int d = 0; d < kRhtRing - 1; ++d) issue(warp0 + d * nwarps, d);
  } else {
    if (warp0 < total) load(warp0);
  }
  int it = 0;
  for (int64_t blk = warp0; blk < total; blk += nwarps, ++it) {
    const int64_t r = blk / nblk, c0 = (blk - r * nblk) * B;
    uint32_t cb0[NT1], cb1[NT1];
    if constexpr (RING) {
      issue(blk + (kRhtRing - 1) * nwarps, (it + kRhtRing - 1) % kRhtRing);
      cp_async_wait<kRhtRing - 1>();  // this block's group has landed (own copies)
      __syncwarp();                    // ... and every lane's
      const uint32_t sl = wring + (it % kRhtRing) * SLOT;
#pragma unroll
      for (int j = 0; j < NT1; ++j) {
        const int e = 16 * (8 * j + g) + 2 * tq;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cb0[j]) : "r"(sl + e * 2));
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cb1[j]) : "r"(sl + e * 2 + 16));
      }
      __syncwarp();  // the slot is refilled by the next iteration's issue
    } else {
#pragma unroll
      for (int j = 0; j < NT1; ++j) {
        cb0[j] = nb0[j];
        cb1[j] = nb1[j];
      }
      if (blk + nwarps < total) load(blk + nwarps);
    }
    // step 1: C1[j] = (H_16 · M^T) restricted to a in [8j, 8j + 8)
    float c1[NT1][4];
#pragma unroll
    for (int j = 0; j < NT1; ++j) {
      const int e = 16 * (8 * j + g) + 2 * tq;
      uint32_t b0 = cb0[j], b1 = cb1[j];
      if (!inverse) {
        b0 ^= sign_mask2(signs + c0 + e);
        b1 ^= sign_mask2(signs + c0 + e + 8);
      }
      c1[j][0] = c1[j][1] = c1[j][2] = c1[j][3] = 0.0f;
      mma16816(c1[j], h0, h1, h2, h3, b0, b1);
    }
    // step 2: Y = H_A · M1, B fragments from C1 (three bf16 parts each)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int kt = 0; kt < MT; ++kt) {
          const uint32_t a0 = h_pair(16 * mt + g, 16 * kt + 2 * tq),
                         a1 = h_pair(16 * mt + g + 8, 16 * kt + 2 * tq),
                         a2 = h_pair(16 * mt + g, 16 * kt + 2 * tq + 8),
                         a3 = h_pair(16 * mt + g + 8, 16 * kt + 2 * tq + 8);
          uint32_t p0[3], p1[3];
          split3(c1[2 * kt][2 * nt], c1[2 * kt][2 * nt + 1], p0);
          split3(c1[2 * kt + 1][2 * nt], c1[2 * kt + 1][2 * nt + 1], p1);
#pragma unroll
          for (int p = 0; p < 3; ++p) mma16816(acc, a0, a1, a2, a3, p0[p], p1[p]);
        }
        // acc: Y[16mt + g][8nt + 2tq .. +1] and Y[16mt + g + 8][...] -> elements i, i + 128
        const int i0 = 16 * (16 * mt + g) + 8 * nt + 2 * tq;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = i0 + 128 * h;
          float y0 = acc[2 * h] * norm, y1 = acc[2 * h + 1] * norm;
          if (inverse) {
            const float2 s = __ldg(reinterpret_cast<const float2*>(signs + c0 + i));
            y0 *= s.x;
            y1 *= s.y;
          }
          if constexpr (OUT_F32) {
            *reinterpret_cast<float2*>(reinterpret_cast<float*>(out) + r * ld_out + c0 + i) =
                make_float2(y0, y1);
          } else {
            *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(out) + r * ld_out +
                                               c0 + i) = __floats2bfloat162_rn(y0, y1);
          }
        }
      }
    }
  }
  if constexpr (RING) cp_async_wait<0>();
}

template <int A>
cudaError_t rht_tc(const void* in, int64_t rows, int64_t cols, int64_t ld_in, const float* signs,
                   int inverse, void* out, int64_t ld_out, bool f32, cudaStream_t st) {
  const int64_t total = rows * (cols / (16 * A));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_sm = A <= 32 ? 3 : 1;
  int64_t blocks = (total + 7) / 8;
  if (blocks > per_sm * static_cast<int64_t>(sms)) blocks = per_sm * static_cast<int64_t>(sms);
  const bool ring = ld_in % 8 == 0 && reinterpret_cast<uintptr_t>(in) % 16 == 0 &&
                    getenv("MLRA_RHT_NORING") == nullptr;
  const int smem = ring ? 8 * kRhtRing * 16 * A * 2 : 0;
  note_launch();
  const auto* x = static_cast<const __nv_bfloat16*>(in);
  const dim3 grid(static_cast<unsigned>(blocks));
#define MLRA_RHT_LAUNCH(F, R)                                                                  \
  do {                                                                                         \
    if (R) {                                                                                   \
      static bool attr = false;                                                                \
      if (!attr) {                                                                             \
        cudaFuncSetAttribute(k_rht_tc<A, F, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                             smem);                                                            \
        attr = true;                                                                           \
      }                                                                                        \
    }                                                                                          \
    k_rht_tc<A, F, R><<<grid, 256, smem, st>>>(x, rows, cols, ld_in, signs, inverse, out, ld_out); \
  } while (0)
  if (f32) {
    if (ring) MLRA_RHT_LAUNCH(true, true); else MLRA_RHT_LAUNCH(true, false);
  } else {
    if (ring) MLRA_RHT_LAUNCH(false, true); else MLRA_RHT_LAUNCH(false, false);
  }
#undef MLRA_RHT_LAUNCH
  return cudaGetLastError();
}

template <int E>
cudaError_t rht_e(const void* in, int64_t rows, int64_t cols, int64_t ld_in, const float* signs,
                  int inverse, void* out, int64_t ld_out, bool f32, cudaStream_t st) {
  const int64_t segs = rows * (cols / (32 * E));
  const int64_t blocks = (segs + 7) / 8;
  if (blocks > 0x7FFFFFFF) return cudaErrorInvalidValue;
  note_launch();
  if (f32)
    k_rht<E, true><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(in), rows, cols, ld_in, signs, inverse, out, ld_out);
  else
    k_rht<E, false><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(in), rows, cols, ld_in, signs, inverse, out, ld_out);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_rht(const void* in, int64_t rows, int64_t cols, int64_t ld_in,
                       const float* signs, int inverse, int block, void* out, int64_t ld_out,
                       bool f32, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  // tensor-core form for b >= 256 (MLRA_RHT_BUTTERFLY=1: the butterfly kernel, A/B)
  static const bool use_tc = getenv("MLRA_RHT_BUTTERFLY") == nullptr;
  switch (block) {
    case 64: return rht_e<2>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st);
    case 128: return rht_e<4>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st);
    case 256: return use_tc ? rht_tc<16>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st)
                            : rht_e<8>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st);
    case 512: return use_tc ? rht_tc<32>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st)
                            : rht_e<16>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st);
    case 1024: return use_tc ? rht_tc<64>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st)
                             : rht_e<32>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mlra
