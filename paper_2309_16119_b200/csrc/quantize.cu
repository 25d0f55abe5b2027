// quantize.cu — RtnQuantizer::quantize on the device (quantize.hpp:108-113,
// quantize.cpp:24-44 + 163-184): the built-in Quantizer plugin's quantize()
// side, producing the reference's QuantizedMatrix layout bit-for-bit.
//
//  * k_rtn_grid: one warp per (row, group): exact f64 min / max over the
//    group, then zero = (float)lo, scale = (float)((hi - lo) / (2^b - 1))
//    (1 when hi == lo or the rounded scale is not positive) — compute_grid.
//  * k_rtn_pack: one thread per output u32 word of the LSB-first bitstream over
//    the whole row-major matrix (bitpack.cpp:68-91): every code whose bits
//    intersect the word is recomputed as clamp(round((w - z) / s), 0, 2^b - 1)
//    in f64 (code_on_grid; CUDA round() is round-half-away like std::round) and
//    OR-ed in, so straddling codes need no cross-thread exchange.
// f32 weights are widened exactly, i.e. the result equals the reference's
// quantize_rtn((double)w).
#include <cuda_runtime.h>

#include "kernels.h"

namespace mlra {

namespace {

template <typename T>
__device__ __forceinline__ double ld_w(const T* w, int64_t i) {
  return static_cast<double>(__ldg(w + i));
}

template <typename T>
__global__ void k_rtn_grid(const T* __restrict__ w, int64_t rows, int64_t cols, int64_t group,
                           int bits, float* __restrict__ scales, float* __restrict__ zeros) {
  const int64_t ng = cols / group;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int64_t gi = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       gi < rows * ng; gi += warps) {
    const int64_t r = gi / ng, g = gi - r * ng;
    const T* p = w + r * cols + g * group;
    // The reference scans in index order keeping the FIRST of equal extremes
    // (std::min / std::max keep their first argument on ties), which decides
    // the sign of a zero extreme: carry the index and break ties by it.
    double lo = ld_w(p, lane < group ? lane : 0), hi = lo;
    int64_t li = lane < group ? lane : 0, hix = li;
#pragma unroll 4
    for (int64_t j = lane; j < group; j += 32) {
      const double v = ld_w(p, j);
      if (v < lo) lo = v, li = j;
      if (hi < v) hi = v, hix = j;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double l2 = __shfl_xor_sync(0xffffffffu, lo, o);
      const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
      const int64_t li2 = __shfl_xor_sync(0xffffffffu, li, o);
      const int64_t hi2 = __shfl_xor_sync(0xffffffffu, hix, o);
      if (l2 < lo || (!(lo < l2) && li2 < li)) lo = l2, li = li2;
      if (hi < h2 || (!(h2 < hi) && hi2 < hix)) hi = h2, hix = hi2;
    }
    if (lane == 0) {
      const double levels = static_cast<double>((1 << bits) - 1);
      float s = hi > lo ? __double2float_rn(__ddiv_rn(__dsub_rn(hi, lo), levels)) : 1.0f;
      if (!(s > 0.0f)) s = 1.0f;
      scales[gi] = s;
      zeros[gi] = __double2float_rn(lo);
    }
  }
}

template <typename T>
__global__ void k_rtn_pack(const T* __restrict__ w, int64_t rows, int64_t cols, int64_t group,
                           int bits, const float* __restrict__ scales,
                           const float* __restrict__ zeros, uint64_t nwords,
                           uint32_t* __restrict__ words) {
  const uint64_t count = static_cast<uint64_t>(rows) * static_cast<uint64_t>(cols);
  const int64_t ng = cols / group;
  const double levels = static_cast<double>((1 << bits) - 1);
  for (uint64_t wi = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; wi < nwords;
       wi += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t b0 = wi * 32;
    const uint64_t c_first = b0 / bits;
    uint64_t c_last = (b0 + 31) / bits;
    if (c_last >= count) c_last = count - 1;
    // (row, col, group) of the first code once; the rest advance incrementally
    // (64-bit divides per code dominated this kernel)
    int64_t r = static_cast<int64_t>(c_first / cols), j = static_cast<int64_t>(c_first % cols);
    int64_t gcol = j / group, jg = j - gcol * group;
    uint32_t out = 0;
    for (uint64_t c = c_first; c <= c_last; ++c) {
      const int64_t gi = r * ng + gcol;
      const double z = static_cast<double>(__ldg(zeros + gi));
      const double s = static_cast<double>(__ldg(scales + gi));
      double q = round(__ddiv_rn(__dsub_rn(ld_w(w, static_cast<int64_t>(c)), z), s));
      q = q < 0.0 ? 0.0 : (q > levels ? levels : q);  // std::clamp
      const uint32_t code = static_cast<uint32_t>(q);
      const int64_t sh = static_cast<int64_t>(c * bits) - static_cast<int64_t>(b0);
      out |= sh >= 0 ? code << sh : code >> (-sh);
      if (++jg == group) {
        jg = 0;
        ++gcol;
      }
      if (++j == cols) {
        j = 0;
        jg = 0;
        gcol = 0;
        ++r;
      }
    }
    words[wi] = out;
  }
}

int grid_blocks(int64_t work, int per_block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t b = (work + per_block - 1) / per_block;
  if (b > 16LL * sms) b = 16LL * sms;
  return static_cast<int>(b < 1 ? 1 : b);
}

template <typename T>
cudaError_t rtn_t(const T* w, int64_t rows, int64_t cols, int64_t group, int bits,
                  uint32_t* words, uint64_t nwords, float* scales, float* zeros, cudaStream_t st) {
  note_launch();
  k_rtn_grid<T><<<grid_blocks(rows * (cols / group), 8), 256, 0, st>>>(w, rows, cols, group, bits,
                                                                       scales, zeros);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  note_launch();
  k_rtn_pack<T><<<grid_blocks(static_cast<int64_t>(nwords), 256), 256, 0, st>>>(
      w, rows, cols, group, bits, scales, zeros, nwords, words);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_rtn_grid(const double* w, int64_t rows, int64_t cols, int64_t group, int bits,
                            float* scales, float* zeros, cudaStream_t st) {
  note_launch();
  k_rtn_grid<double><<<grid_blocks(rows * (cols / group), 8), 256, 0, st>>>(w, rows, cols, group,
                                                                            bits, scales, zeros);
  return cudaGetLastError();
}

cudaError_t launch_quantize_rtn(const void* w, bool f64, int64_t rows, int64_t cols, int64_t group,
                                int bits, uint32_t* words, uint64_t nwords, float* scales,
                                float* zeros, cudaStream_t st) {
  if (f64)
    return rtn_t(static_cast<const double*>(w), rows, cols, group, bits, words, nwords, scales,
                 zeros, st);
  return rtn_t(static_cast<const float*>(w), rows, cols, group, bits, words, nwords, scales, zeros,
               st);
}

}  // namespace mlra
