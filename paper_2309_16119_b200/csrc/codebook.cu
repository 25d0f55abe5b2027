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
__device__ __forceinline__ void cb2_store(void* __restrict__ out, int64_t o, const float (&f)[8]) {
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

// Work items = (row, pass of kCbThreads * kCbPerThread codes) strided over a
// resident-size grid (the 8 KB codebook is staged into shared memory once per
// CTA). Software-pipelined: the codes and scales of the next item are loaded
// before the current item is decoded, so a load latency is exposed once per
// CTA, not once per pass (ncu: the one-pass-at-a-time form was long-scoreboard
// bound at 32% of DRAM bandwidth). Within a pass a thread owns kCbPerThread
// codes strided by the block size, so each warp store covers a contiguous
// 512 B (bf16).
template <bool F32, bool VEC>
__global__ void __launch_bounds__(kCbThreads) k_cb2_materialize(
    const Cb2Dev c, int64_t row0, int64_t nrows, int64_t col0, int64_t ncols,
    void* __restrict__ out, int64_t ld, int gshift) {
  __shared__ float4 cb[256 * 2];
  for (int i = threadIdx.x; i < 512; i += kCbThreads)
    cb[i] = __ldg(reinterpret_cast<const float4*>(c.codebook) + i);
  const int ncodes = static_cast<int>(ncols >> 3);
  const int ucol0 = static_cast<int>(col0 >> 3);
  const int64_t cpr = c.cols >> 3;  // codes per full row
  const int gdiv = static_cast<int>(c.group);
  constexpr int CH = kCbThreads * kCbPerThread;
  const int ipr = (ncodes + CH - 1) / CH;  // passes per row
  const int64_t items = nrows * ipr;
  uint32_t code[kCbPerThread];
  float scl[kCbPerThread];
  auto fetch = [&](int64_t item) {
    const int64_t rr = item / ipr;
    const int base = static_cast<int>(item - rr * ipr) * CH + threadIdx.x;
    const uint16_t* crow = c.codes + (row0 + rr) * cpr + ucol0;
    const float* srow = c.scales + (row0 + rr) * c.ng;
#pragma unroll
    for (int j = 0; j < kCbPerThread; ++j) {
      const int it = base + j * kCbThreads;
      const int k = (ucol0 + it) << 3;
      code[j] = it < ncodes ? __ldg(crow + it) : 0u;
      scl[j] = it < ncodes ? __ldg(srow + (gshift >= 0 ? (k >> gshift) : k / gdiv)) : 0.0f;
    }
  };
  int64_t item = blockIdx.x;
  if (item < items) fetch(item);
  __syncthreads();
  for (; item < items; item += gridDim.x) {
    uint32_t cur[kCbPerThread];
    float cs[kCbPerThread];
#pragma unroll
    for (int j = 0; j < kCbPerThread; ++j) {
      cur[j] = code[j];
      cs[j] = scl[j];
    }
    if (item + gridDim.x < items) fetch(item + gridDim.x);  // next item in flight
    const int64_t rr = item / ipr;
    const int base = static_cast<int>(item - rr * ipr) * CH + threadIdx.x;
#pragma unroll
    for (int j = 0; j < kCbPerThread; ++j) {
      const int it = base + j * kCbThreads;
      if (it >= ncodes) break;
      const float4 m0 = cb[(cur[j] & 0xFFu) * 2], m1 = cb[(cur[j] & 0xFFu) * 2 + 1];
      const float mag[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
      float f[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t neg = (cur[j] >> (8 + e)) & 1u;
        f[e] = __uint_as_float(__float_as_uint(__fmul_rn(cs[j], mag[e])) ^ (neg << 31));
      }
      cb2_store<F32, VEC>(out, rr * ld + (static_cast<int64_t>(it) << 3), f);
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
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cb2_materialize<true, true>,
                                                    kCbThreads, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int64_t cap = static_cast<int64_t>(sms) * per_sm;
  const int64_t ncodes = ncols >> 3;
  const int64_t items = nrows * ((ncodes + kCbThreads * kCbPerThread - 1) / (kCbThreads * kCbPerThread));
  const dim3 grid(static_cast<unsigned>(items < cap ? items : cap));
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
