// materialize.cu — K1 (the plugin's materialize()) and the upload-time kernels.
//
//  * k_relayout: reference whole-matrix bitstream (bitpack.cpp:25-35) ->
//    row-padded device layout (common.cuh). Only for shapes whose rows are
//    not already word-aligned multiples of 256.
//  * k_grid: f32 scales/zeros (quantize.hpp:36-37) -> signed float2 grid with
//    the per-group fma certificate (common.cuh).
//  * k_materialize: Ŵ = RN(double(s)·c + double(z)) (quantize.cpp:123-137,
//    139-155) into f32 or bf16, bit-exact with (float)dequantize().
//    HBM-bound: reads b/8 + 8/g bytes and writes 2 or 4 bytes per entry.
//  * k_materialize_lut: the lut plugin's Ŵ = RN_f32(s · lut[c]).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace mlra {

namespace {

__device__ __forceinline__ uint32_t read_code_ref(const uint32_t* __restrict__ w, int bits,
                                                  uint64_t index) {
  // bitpack.cpp:25-35
  const uint64_t bit = index * static_cast<uint64_t>(bits);
  const uint64_t word = bit >> 5, off = bit & 31;
  uint64_t v = w[word] >> off;
  if (off + bits > 32) v |= static_cast<uint64_t>(w[word + 1]) << (32 - off);
  return static_cast<uint32_t>(v) & ((1u << bits) - 1u);
}

__global__ void k_relayout(const uint32_t* __restrict__ src, int64_t rows, int64_t cols, int bits,
                           int64_t row_words, int64_t rows_pad, uint32_t* __restrict__ dst) {
  const int64_t total = rows_pad * row_words;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / row_words, w = i % row_words;
    uint32_t out = 0;
    if (r < rows) {
      // codes whose bits intersect [32w, 32w+32) of this padded row
      const int64_t b0 = w * 32;
      const int64_t c_first = b0 / bits, c_last = (b0 + 31) / bits;
      for (int64_t c = c_first; c <= c_last; ++c) {
        if (c >= cols) break;
        const uint32_t code = read_code_ref(src, bits, static_cast<uint64_t>(r * cols + c));
        const int64_t sh = c * bits - b0;  // may be negative for the straddling first code
        if (sh >= 0)
          out |= code << sh;
        else
          out |= code >> (-sh);
      }
    }
    dst[i] = out;
  }
}

__global__ void k_grid(const float* __restrict__ scales, const float* __restrict__ zeros,
                       int64_t rows, int64_t ng, int64_t rows_pad, int64_t ng_pad, int bits,
                       float2* __restrict__ grid, int* __restrict__ n_uncertified) {
  const int64_t total = rows_pad * ng_pad;
  int local = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / ng_pad, g = i % ng_pad;
    float s = 1.0f, z = 0.0f;
    if (r < rows && g < ng) {
      s = scales[r * ng + g];
      z = zeros[r * ng + g];
    }
    bool cert = true;
    const uint32_t levels = 1u << bits;
    for (uint32_t c = 0; c < levels; ++c) {
      const float fast = __fmaf_rn(s, code_to_f32(c), z);
      const float exact = __double2float_rn(
          __fma_rn(static_cast<double>(s), static_cast<double>(c), static_cast<double>(z)));
      if (__float_as_uint(fast) != __float_as_uint(exact)) {
        cert = false;
        break;
      }
    }
    if (!cert) ++local;
    grid[i] = make_float2(cert ? s : -s, z);
  }
  if (local) atomicAdd(n_uncertified, local);
}

// One thread per 8-entry unit of the (logical) matrix.
// Tile form: columns [col0, col0 + ncols) of rows [row0, row0 + nrows), col0 % 8 == 0.
template <int BITS, bool F32, bool VEC>
__global__ void __launch_bounds__(256) k_materialize(const QWeightDev q, int64_t row0,
                                                     int64_t nrows, int64_t col0, int64_t ncols,
                                                     void* __restrict__ out, int64_t ld) {
  const int64_t upr = (ncols + 7) / 8;  // units per tile row
  const int64_t total = nrows * upr;
  const int64_t col_end = ncols;  // valid extent of a tile row
  const bool fast_group = (q.group % 8) == 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t rr = i / upr, u = i % upr;
    const int64_t r = row0 + rr;
    const int64_t ua = col0 / 8 + u;  // unit index within the row
    const uint64_t v = load_unit<BITS>(q.words + r * q.row_words, ua);
    const float2* grow = q.grid + r * q.ng_pad;
    float f[8];
    if (fast_group)
      deq8_f32<BITS>(v, __ldg(grow + (ua * 8) / q.group), f);
    else
      deq8_f32_general<BITS>(v, grow, ua * 8, q.group, f);
    const int64_t k0 = u * 8;
    if constexpr (VEC) {  // cols % 8 == 0 and ld % 8 == 0: aligned vector stores
      if constexpr (F32) {
        float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + rr * ld + k0);
        o[0] = make_float4(f[0], f[1], f[2], f[3]);
        o[1] = make_float4(f[4], f[5], f[6], f[7]);
      } else {
        uint4 o;
        o.x = pack_bf16x2(f[0], f[1]);
        o.y = pack_bf16x2(f[2], f[3]);
        o.z = pack_bf16x2(f[4], f[5]);
        o.w = pack_bf16x2(f[6], f[7]);
        *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + rr * ld + k0) = o;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (k0 + j < col_end) {
          if constexpr (F32)
            reinterpret_cast<float*>(out)[rr * ld + k0 + j] = f[j];
          else
            reinterpret_cast<__nv_bfloat16*>(out)[rr * ld + k0 + j] = __float2bfloat16_rn(f[j]);
        }
      }
    }
  }
}

// Bandwidth path (2-D grid, one row per blockIdx.y, no 64-bit divides): each
// thread owns 4 items strided by 32 so every warp store covers a contiguous
// 512 B. Items are 8-code units (bf16 out, one 16-B store) or 4-code quads
// (f32 out, one 16-B store). Requires group % 8 == 0 (one grid entry per item).
template <int BITS>
__device__ __forceinline__ uint32_t quad_bits(const uint32_t* __restrict__ rw, int64_t qd) {
  const int64_t bit = qd * 4 * BITS;
  const int64_t w0 = bit >> 5;
  const uint32_t off = static_cast<uint32_t>(bit & 31);
  const uint32_t lo = __ldg(rw + w0);
  const uint32_t hi = off + 4 * BITS > 32 ? __ldg(rw + w0 + 1) : 0u;
  constexpr uint32_t qmask = 4 * BITS >= 32 ? 0xFFFFFFFFu : ((1u << (4 * BITS)) - 1u);
  return __funnelshift_r(lo, hi, off) & qmask;
}

// Uncertified groups (rare: the per-group fp32-FMA exactness check failed at
// upload) take the exact f64 path out of line, so the hot loop keeps few registers.
template <int BITS>
__device__ __noinline__ uint4 deq8_bf16_slow(uint32_t v, float2 g) {
  return deq8_bf16<BITS>(v, g);
}

template <int BITS, bool F32, int GSHIFT>
__global__ void __launch_bounds__(128) k_materialize_fast(const QWeightDev q, int64_t row0,
                                                          void* __restrict__ out, int64_t ld,
                                                          int64_t items, int gshift) {
  constexpr int CODES = F32 ? 4 : 8;
  constexpr int IPT = 4;  // items per thread, strided by 32: every warp store covers 512 B
  const int64_t r = row0 + blockIdx.y;
  const uint32_t* rw = q.words + r * q.row_words;
  const float2* grow = q.grid + r * q.ng_pad;
  const int base = static_cast<int>(blockIdx.x) * 512 + (threadIdx.x >> 5) * 128 + (threadIdx.x & 31);
  const int n = static_cast<int>(items);
  const int gs = GSHIFT >= 0 ? GSHIFT : gshift;
  // every item's code bits and grid entry are requested before any is decoded
  // (the loop with an early exit issued them one at a time: long-scoreboard bound)
  uint64_t v[IPT];
  float2 g[IPT];
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int it = base + 32 * j;
    if (it < n) {
      const int k0 = it * CODES;
      g[j] = __ldg(grow + (gs >= 0 ? (k0 >> gs) : k0 / static_cast<int>(q.group)));
      if constexpr (F32)
        v[j] = quad_bits<BITS>(rw, it);
      else
        v[j] = load_unit<BITS>(rw, it);
    }
  }
  if constexpr (F32) {
    float* orow = reinterpret_cast<float*>(out) + static_cast<int64_t>(blockIdx.y) * ld;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const int it = base + 32 * j;
      if (it >= n) break;
      constexpr uint32_t mask = (1u << BITS) - 1u;
      const uint32_t vv = static_cast<uint32_t>(v[j]);
      float f[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) f[i] = deq_entry((vv >> (BITS * i)) & mask, g[j].x, g[j].y);
      *reinterpret_cast<float4*>(orow + it * CODES) = make_float4(f[0], f[1], f[2], f[3]);
    }
  } else {
    __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(out) + static_cast<int64_t>(blockIdx.y) * ld;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const int it = base + 32 * j;
      if (it >= n) break;
      uint4 o;
      if constexpr (BITS <= 4)
        o = g[j].x > 0.0f ? deq8_bf16_cert<BITS>(static_cast<uint32_t>(v[j]), g[j])
                          : deq8_bf16_slow<BITS>(static_cast<uint32_t>(v[j]), g[j]);
      else
        o = deq8_bf16<BITS>(v[j], g[j]);
      *reinterpret_cast<uint4*>(orow + it * CODES) = o;
    }
  }
}

// The lut plugin's materialize (mlra_lut_create): Ŵ[i, j] = RN_f32(s · lut[c]),
// s = the {s, 0} grid entry of (i, j/g). group % 8 == 0 (checked at upload), so
// every 8-code unit shares one scale. Block rows over blockIdx.y, 128 units per
// block along x (contiguous 16-B stores per warp); the table sits in 16
// conflict-free shared words.
template <int BITS, bool F32, bool VEC>
__global__ void __launch_bounds__(128) k_materialize_lut(const QWeightDev q, int64_t row0,
                                                         int64_t nrows, int64_t u0, int64_t units,
                                                         void* __restrict__ out, int64_t ld,
                                                         int gshift) {
  constexpr int UPT = 4;  // units per thread, strided by the block: 4 loads in flight
  __shared__ float lut[16];
  if (threadIdx.x < 16) lut[threadIdx.x] = __ldg(q.lut + threadIdx.x);
  __syncthreads();
  constexpr uint32_t mask = (1u << BITS) - 1u;
  for (int64_t rr = blockIdx.y; rr < nrows; rr += gridDim.y) {
    const int64_t r = row0 + rr;
    const uint32_t* rw = q.words + r * q.row_words;
    const float2* grow = q.grid + r * q.ng_pad;
    for (int64_t it0 = static_cast<int64_t>(blockIdx.x) * (128 * UPT) + threadIdx.x; it0 < units;
         it0 += static_cast<int64_t>(gridDim.x) * (128 * UPT)) {
      uint32_t v[UPT];
      float s[UPT];
#pragma unroll
      for (int j = 0; j < UPT; ++j) {
        const int64_t it = it0 + j * 128;
        if (it < units) {
          const int64_t ua = u0 + it;
          v[j] = static_cast<uint32_t>(load_unit<BITS>(rw, ua));
          const int64_t k = ua * 8;
          s[j] = __ldg(grow + (gshift >= 0 ? (k >> gshift) : k / q.group)).x;
        }
      }
#pragma unroll
      for (int j = 0; j < UPT; ++j) {
        const int64_t it = it0 + j * 128;
        if (it >= units) break;
        float f[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = __fmul_rn(s[j], lut[(v[j] >> (BITS * i)) & mask]);
        const int64_t o = rr * ld + it * 8;
        if constexpr (F32) {
          float* op = reinterpret_cast<float*>(out) + o;
          if constexpr (VEC) {
            reinterpret_cast<float4*>(op)[0] = make_float4(f[0], f[1], f[2], f[3]);
            reinterpret_cast<float4*>(op)[1] = make_float4(f[4], f[5], f[6], f[7]);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) op[i] = f[i];
          }
        } else {
          const uint4 w = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                                     pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
          __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(out) + o;
          if constexpr (VEC) {
            *reinterpret_cast<uint4*>(op) = w;
          } else {
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              op[2 * i] = __ushort_as_bfloat16(static_cast<unsigned short>(ws[i] & 0xFFFFu));
              op[2 * i + 1] = __ushort_as_bfloat16(static_cast<unsigned short>(ws[i] >> 16));
            }
          }
        }
      }
    }
  }
}

int grid_for(int64_t work, int per_block);

template <int BITS>
cudaError_t materialize_lut_bits(const QWeightDev& q, int64_t row0, int64_t nrows, int64_t col0,
                                 int64_t ncols, void* out, int64_t ld, bool f32,
                                 cudaStream_t st) {
  const int64_t units = ncols / 8;
  const bool vec = ld % (f32 ? 4 : 8) == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
  int gshift = -1;
  for (int sft = 3; sft < 31; ++sft)
    if ((int64_t{1} << sft) == q.group) gshift = sft;
  const int64_t bx = (units + 511) / 512;
  int64_t by = static_cast<int64_t>(grid_for(nrows * bx, 1)) / bx;
  if (by < 1) by = 1;
  if (by > nrows) by = nrows;
  if (by > 65535) by = 65535;
  const dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(by));
  note_launch();
  if (f32) {
    if (vec)
      k_materialize_lut<BITS, true, true><<<grid, 128, 0, st>>>(q, row0, nrows, col0 / 8, units,
                                                                 out, ld, gshift);
    else
      k_materialize_lut<BITS, true, false><<<grid, 128, 0, st>>>(q, row0, nrows, col0 / 8, units,
                                                                  out, ld, gshift);
  } else {
    if (vec)
      k_materialize_lut<BITS, false, true><<<grid, 128, 0, st>>>(q, row0, nrows, col0 / 8, units,
                                                                  out, ld, gshift);
    else
      k_materialize_lut<BITS, false, false><<<grid, 128, 0, st>>>(q, row0, nrows, col0 / 8,
                                                                   units, out, ld, gshift);
  }
  return cudaGetLastError();
}

cudaError_t materialize_lut(const QWeightDev& q, int64_t row0, int64_t nrows, int64_t col0,
                            int64_t ncols, void* out, int64_t ld, bool f32, cudaStream_t st) {
  if (col0 % 8 != 0 || ncols % 8 != 0) return cudaErrorInvalidValue;
  switch (q.bits) {
    case 2: return materialize_lut_bits<2>(q, row0, nrows, col0, ncols, out, ld, f32, st);
    case 3: return materialize_lut_bits<3>(q, row0, nrows, col0, ncols, out, ld, f32, st);
    case 4: return materialize_lut_bits<4>(q, row0, nrows, col0, ncols, out, ld, f32, st);
    default: return cudaErrorInvalidValue;
  }
}

int grid_for(int64_t work, int per_block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (work + per_block - 1) / per_block;
  const int64_t cap = static_cast<int64_t>(sms) * 16;
  if (blocks > cap) blocks = cap;
  return static_cast<int>(blocks < 1 ? 1 : blocks);
}

template <int BITS>
cudaError_t materialize_tile_bits(const QWeightDev& q, int64_t row0, int64_t nrows, int64_t col0,
                                  int64_t ncols, void* out, int64_t ld, bool f32, bool vec,
                                  cudaStream_t st) {
  const int64_t units = nrows * ((ncols + 7) / 8);
  const int blocks = grid_for(units, 256);
  note_launch();
  if (f32) {
    if (vec)
      k_materialize<BITS, true, true><<<blocks, 256, 0, st>>>(q, row0, nrows, col0, ncols, out, ld);
    else
      k_materialize<BITS, true, false><<<blocks, 256, 0, st>>>(q, row0, nrows, col0, ncols, out, ld);
  } else {
    if (vec)
      k_materialize<BITS, false, true><<<blocks, 256, 0, st>>>(q, row0, nrows, col0, ncols, out, ld);
    else
      k_materialize<BITS, false, false><<<blocks, 256, 0, st>>>(q, row0, nrows, col0, ncols, out,
                                                                ld);
  }
  return cudaGetLastError();
}

template <int BITS>
cudaError_t materialize_bits(const QWeightDev& q, int64_t row0, int64_t nrows, void* out,
                             int64_t ld, bool f32, cudaStream_t st) {
  const bool vec = (q.cols % 8 == 0) && (ld % 8 == 0) &&
                   (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  if (vec && q.group % 8 == 0 && nrows <= 65535) {
    const int64_t items = f32 ? q.cols / 4 : q.cols / 8;
    int gshift = -1;
    for (int sft = 3; sft < 31; ++sft)
      if ((int64_t{1} << sft) == q.group) gshift = sft;
    dim3 grid(static_cast<unsigned>((items + 511) / 512), static_cast<unsigned>(nrows));
    note_launch();
    // the LLaMA group (128) gets a compile-time shift
    if (f32) {
      if (gshift == 7)
        k_materialize_fast<BITS, true, 7><<<grid, 128, 0, st>>>(q, row0, out, ld, items, gshift);
      else
        k_materialize_fast<BITS, true, -1><<<grid, 128, 0, st>>>(q, row0, out, ld, items, gshift);
    } else {
      if (gshift == 7)
        k_materialize_fast<BITS, false, 7><<<grid, 128, 0, st>>>(q, row0, out, ld, items, gshift);
      else
        k_materialize_fast<BITS, false, -1><<<grid, 128, 0, st>>>(q, row0, out, ld, items, gshift);
    }
    return cudaGetLastError();
  }
  return materialize_tile_bits<BITS>(q, row0, nrows, 0, q.cols, out, ld, f32, vec, st);
}

}  // namespace

cudaError_t launch_relayout(const uint32_t* src, int64_t rows, int64_t cols, int bits,
                            int64_t row_words, int64_t rows_pad, uint32_t* dst,
                            cudaStream_t st) {
  note_launch();
  k_relayout<<<grid_for(rows_pad * row_words, 256), 256, 0, st>>>(src, rows, cols, bits,
                                                                  row_words, rows_pad, dst);
  return cudaGetLastError();
}

cudaError_t launch_grid(const float* scales, const float* zeros, int64_t rows, int64_t ng,
                        int64_t rows_pad, int64_t ng_pad, int bits, float2* grid,
                        int* n_uncertified, cudaStream_t st) {
  note_launch();
  k_grid<<<grid_for(rows_pad * ng_pad, 256), 256, 0, st>>>(scales, zeros, rows, ng, rows_pad,
                                                           ng_pad, bits, grid, n_uncertified);
  return cudaGetLastError();
}

cudaError_t launch_materialize(const QWeightDev& q, int64_t row0, int64_t nrows, void* out,
                               int64_t ld, bool f32, cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  if (q.lut) return materialize_lut(q, row0, nrows, 0, q.cols, out, ld, f32, st);
  switch (q.bits) {
    case 2: return materialize_bits<2>(q, row0, nrows, out, ld, f32, st);
    case 3: return materialize_bits<3>(q, row0, nrows, out, ld, f32, st);
    case 4: return materialize_bits<4>(q, row0, nrows, out, ld, f32, st);
    case 8: return materialize_bits<8>(q, row0, nrows, out, ld, f32, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_materialize_tile(const QWeightDev& q, int64_t row0, int64_t nrows, int64_t col0,
                                    int64_t ncols, void* out, int64_t ld, bool f32,
                                    cudaStream_t st) {
  if (nrows <= 0 || ncols <= 0) return cudaSuccess;
  if (q.lut) return materialize_lut(q, row0, nrows, col0, ncols, out, ld, f32, st);
  if (col0 == 0 && ncols == q.cols) return launch_materialize(q, row0, nrows, out, ld, f32, st);
  const bool vec = (ncols % 8 == 0) && (ld % 8 == 0) &&
                   (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  switch (q.bits) {
    case 2: return materialize_tile_bits<2>(q, row0, nrows, col0, ncols, out, ld, f32, vec, st);
    case 3: return materialize_tile_bits<3>(q, row0, nrows, col0, ncols, out, ld, f32, vec, st);
    case 4: return materialize_tile_bits<4>(q, row0, nrows, col0, ncols, out, ld, f32, vec, st);
    case 8: return materialize_tile_bits<8>(q, row0, nrows, col0, ncols, out, ld, f32, vec, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mlra
