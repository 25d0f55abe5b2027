// codebook.cu — the built-in non-affine plugin "cb2" (include/mlra.h,
// mlra_cb2_create): a QuIP#-style 2-bit vector codebook behind the device
// dequant hook (the GPU form of Quantizer::matvec, quantize.hpp:98-105).
//
// Format: one u16 code per 8 consecutive row entries — bits 0-7 index a
// 256 x 8 f32 magnitude codebook, bit 8+j negates entry j — and one f32 scale
// per (row, group) along cols. Ŵ[i, 8u+j] = RN_f32(s · ±cb[idx][j]) (one IEEE
// multiply, so bit-exact against oracle/mlra_oracle.c orc_cb2_dequant), then
// RN to bf16 for the GEMM operand.
//
// k_cb2_materialize is HBM-bound: 0.25 B of code + 4/g B of scale read and
// 2 (bf16) or 4 (f32) B written per entry. The 8 KB codebook lives in shared
// memory (one float4 pair per code lookup); each thread owns 4 codes strided
// by the block size so a warp's 16-B stores cover a contiguous 512 B (bf16).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace mlra {

namespace {

constexpr int kCbThreads = 256;
constexpr int kCbPerThread = 4;

template <bool F32, bool VEC>
__global__ void __launch_bounds__(kCbThreads) k_cb2_materialize(
    const Cb2Dev c, int64_t row0, int64_t nrows, int64_t col0, int64_t ncols,
    void* __restrict__ out, int64_t ld, int gshift) {
  __shared__ float4 cb[256 * 2];
  for (int i = threadIdx.x; i < 512; i += kCbThreads)
    cb[i] = __ldg(reinterpret_cast<const float4*>(c.codebook) + i);
  __syncthreads();
  const int ncodes = static_cast<int>(ncols >> 3);
  const int ucol0 = static_cast<int>(col0 >> 3);
  const int64_t cpr = c.cols >> 3;  // codes per full row
  for (int64_t rr = blockIdx.y; rr < nrows; rr += gridDim.y) {
    const int64_t r = row0 + rr;
    const uint16_t* crow = c.codes + r * cpr;
    const float* srow = c.scales + r * c.ng;
    const int base = blockIdx.x * (kCbThreads * kCbPerThread) + threadIdx.x;
#pragma unroll
    for (int j = 0; j < kCbPerThread; ++j) {
      const int it = base + j * kCbThreads;
      if (it >= ncodes) break;
      const int u = ucol0 + it;  // code index within the row
      const uint32_t code = __ldg(crow + u);
      const int k = u << 3;      // first column of the code
      const float s = __ldg(srow + (gshift >= 0 ? (k >> gshift) : k / static_cast<int>(c.group)));
      const float4 m0 = cb[(code & 0xFFu) * 2], m1 = cb[(code & 0xFFu) * 2 + 1];
      const float mag[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
      float f[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t neg = (code >> (8 + e)) & 1u;
        f[e] = __uint_as_float(__float_as_uint(__fmul_rn(s, mag[e])) ^ (neg << 31));
      }
      const int64_t o = rr * ld + (static_cast<int64_t>(it) << 3);
      if constexpr (VEC) {
        if constexpr (F32) {
          float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + o);
          p[0] = make_float4(f[0], f[1], f[2], f[3]);
          p[1] = make_float4(f[4], f[5], f[6], f[7]);
        } else {
          uint4 v;
          v.x = pack_bf16x2(f[0], f[1]);
          v.y = pack_bf16x2(f[2], f[3]);
          v.z = pack_bf16x2(f[4], f[5]);
          v.w = pack_bf16x2(f[6], f[7]);
          *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + o) = v;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if constexpr (F32)
            reinterpret_cast<float*>(out)[o + e] = f[e];
          else
            reinterpret_cast<__nv_bfloat16*>(out)[o + e] = __float2bfloat16_rn(f[e]);
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
  const int64_t ncodes = ncols >> 3;
  const unsigned gx =
      static_cast<unsigned>((ncodes + kCbThreads * kCbPerThread - 1) / (kCbThreads * kCbPerThread));
  const unsigned gy = static_cast<unsigned>(nrows < 65535 ? nrows : 65535);
  const dim3 grid(gx, gy);
  note_launch();
  if (f32) {
    if (vec)
      k_cb2_materialize<true, true><<<grid, kCbThreads, 0, st>>>(c, row0, nrows, col0, ncols, out,
                                                                 ld, gshift);
    else
      k_cb2_materialize<true, false><<<grid, kCbThreads, 0, st>>>(c, row0, nrows, col0, ncols,
                                                                  out, ld, gshift);
  } else {
    if (vec)
      k_cb2_materialize<false, true><<<grid, kCbThreads, 0, st>>>(c, row0, nrows, col0, ncols,
                                                                  out, ld, gshift);
    else
      k_cb2_materialize<false, false><<<grid, kCbThreads, 0, st>>>(c, row0, nrows, col0, ncols,
                                                                   out, ld, gshift);
  }
  return cudaGetLastError();
}

}  // namespace mlra
