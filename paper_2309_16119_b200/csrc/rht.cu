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
  switch (block) {
    case 64: return rht_e<2>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st);
    case 128: return rht_e<4>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st);
    case 256: return rht_e<8>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st);
    case 512: return rht_e<16>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st);
    case 1024: return rht_e<32>(in, rows, cols, ld_in, signs, inverse, out, ld_out, f32, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mlra
