// lora_thin.cu — K4/K5/K6: the skinny rank-r adapter products.
//
//  k_rowdot (K4, K5a): out[t, j] = Σ_k act[t,k]·W[k,j]   (m x r, reduction over d)
//     XB  = X·B   — matmul(t, x, B)           lora.cpp:68
//     dYA = dY·A  — d(xb) = dab·A              autodiff.cpp:150-152 on lora.cpp:69
//     Also emits bf16(s·out) into the zero-padded LoRA operand of the
//     tensor-core GEMM's extra K block (qgemm.cu).
//     Warp per TT tokens; lanes stride d in 8-element vectors; W chunks staged
//     in padded (bank-conflict-free) shared memory; warp-shuffle reduction.
//  k_coldot (K5b, K6): out[n, j] += s·Σ_t act[t,n]·V[t,j]  (d x r, reduction over tokens)
//     dA = s·dYᵀ·XB   — d(Aᵀ) = xbᵀ·dab, transposed   autodiff.cpp:153-155, :315-320
//     dB = s·Xᵀ·dYA   — dB = xᵀ·d(xb)                   autodiff.cpp:153-155
//     dbias = Σ_t dY  — bias_add backward                autodiff.cpp:183-191
//     Thread per 2 columns (coalesced bf16x2 rows), V rows broadcast from
//     shared memory, token range split across CTAs, fp32 atomics at the end.
// All accumulation is fp32.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace mlra {

namespace {

template <int RC, int TT>
__global__ void __launch_bounds__(256)
    k_rowdot(const __nv_bfloat16* __restrict__ act, int64_t lda, int64_t m, int64_t kd,
             const float* __restrict__ W, int64_t ldw, int rc, float scale,
             float* __restrict__ out, int64_t ldo, __nv_bfloat16* __restrict__ pad,
             int64_t ldp) {
  extern __shared__ float wsm[];  // [32 lanes][8*RC + 4]
  constexpr int LS = 8 * RC + 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t_base = (static_cast<int64_t>(blockIdx.x) * 8 + warp) * TT;
  float acc[TT][RC];
#pragma unroll
  for (int tt = 0; tt < TT; ++tt)
#pragma unroll
    for (int j = 0; j < RC; ++j) acc[tt][j] = 0.0f;

  for (int64_t k0 = 0; k0 < kd; k0 += 256) {
    __syncthreads();
    for (int i = threadIdx.x; i < 256 * RC; i += 256) {
      const int kl = i / RC, j = i % RC;
      const int64_t k = k0 + kl;
      const float v = (k < kd && j < rc) ? W[k * ldw + j] : 0.0f;
      wsm[(kl >> 3) * LS + (kl & 7) * RC + j] = v;
    }
    __syncthreads();
    float a[TT][8];
    const int64_t kq = k0 + lane * 8;
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) {
      const int64_t t = t_base + tt;
      if (t < m && kq + 8 <= kd) {
        const uint4 u = *reinterpret_cast<const uint4*>(act + t * lda + kq);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          a[tt][2 * e] = f.x;
          a[tt][2 * e + 1] = f.y;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          a[tt][e] = (t < m && kq + e < kd) ? __bfloat162float(act[t * lda + kq + e]) : 0.0f;
      }
    }
    const float* wl = wsm + lane * LS;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
      for (int j = 0; j < RC; j += 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(wl + kk * RC + j);
#pragma unroll
        for (int tt = 0; tt < TT; ++tt) {
          acc[tt][j] = __fmaf_rn(a[tt][kk], w4.x, acc[tt][j]);
          acc[tt][j + 1] = __fmaf_rn(a[tt][kk], w4.y, acc[tt][j + 1]);
          acc[tt][j + 2] = __fmaf_rn(a[tt][kk], w4.z, acc[tt][j + 2]);
          acc[tt][j + 3] = __fmaf_rn(a[tt][kk], w4.w, acc[tt][j + 3]);
        }
      }
    }
  }
#pragma unroll
  for (int tt = 0; tt < TT; ++tt) {
#pragma unroll
    for (int j = 0; j < RC; ++j) {
      float v = acc[tt][j];
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      acc[tt][j] = v;
    }
    const int64_t t = t_base + tt;
    if (t < m) {
#pragma unroll
      for (int j = 0; j < RC; ++j) {
        if ((j & 31) == lane && j < rc) {
          out[t * ldo + j] = acc[tt][j];
          if (pad) pad[t * ldp + j] = __float2bfloat16_rn(scale * acc[tt][j]);
        }
      }
    }
  }
}

template <int RC>
__global__ void __launch_bounds__(128)
    k_coldot(const __nv_bfloat16* __restrict__ act, int64_t lda, int64_t m, int64_t nd,
             const float* __restrict__ V, int64_t ldv, int rc, float scale, int64_t t_per_block,
             float* __restrict__ out, int64_t ldo, float* __restrict__ colsum) {
  __shared__ __align__(16) float vsm[64 * RC];
  const int64_t n0 = (static_cast<int64_t>(blockIdx.x) * 128 + threadIdx.x) * 2;
  const int64_t tb = static_cast<int64_t>(blockIdx.y) * t_per_block;
  const int64_t te = (tb + t_per_block < m) ? tb + t_per_block : m;
  float acc0[RC], acc1[RC];
#pragma unroll
  for (int j = 0; j < RC; ++j) acc0[j] = acc1[j] = 0.0f;
  float cs0 = 0.0f, cs1 = 0.0f;
  const bool pair = n0 + 1 < nd;
  for (int64_t t0 = tb; t0 < te; t0 += 64) {
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * RC; i += 128) {
      const int tl = i / RC, j = i % RC;
      const int64_t t = t0 + tl;
      vsm[i] = (t < te && j < rc) ? V[t * ldv + j] : 0.0f;
    }
    __syncthreads();
    const int nt = static_cast<int>((te - t0) < 64 ? (te - t0) : 64);
    if (n0 < nd) {
#pragma unroll 4
      for (int tl = 0; tl < nt; ++tl) {
        const int64_t t = t0 + tl;
        float a0, a1 = 0.0f;
        if (pair) {
          const float2 f =
              __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(act + t * lda + n0));
          a0 = f.x;
          a1 = f.y;
        } else {
          a0 = __bfloat162float(act[t * lda + n0]);
        }
        cs0 += a0;
        cs1 += a1;
        const float* vr = vsm + tl * RC;
#pragma unroll
        for (int j = 0; j < RC; j += 4) {
          const float4 v = *reinterpret_cast<const float4*>(vr + j);
          acc0[j] = __fmaf_rn(a0, v.x, acc0[j]);
          acc0[j + 1] = __fmaf_rn(a0, v.y, acc0[j + 1]);
          acc0[j + 2] = __fmaf_rn(a0, v.z, acc0[j + 2]);
          acc0[j + 3] = __fmaf_rn(a0, v.w, acc0[j + 3]);
          acc1[j] = __fmaf_rn(a1, v.x, acc1[j]);
          acc1[j + 1] = __fmaf_rn(a1, v.y, acc1[j + 1]);
          acc1[j + 2] = __fmaf_rn(a1, v.z, acc1[j + 2]);
          acc1[j + 3] = __fmaf_rn(a1, v.w, acc1[j + 3]);
        }
      }
    }
  }
  if (n0 < nd) {
#pragma unroll
    for (int j = 0; j < RC; ++j)
      if (j < rc) atomicAdd(out + n0 * ldo + j, scale * acc0[j]);
    if (colsum) atomicAdd(colsum + n0, cs0);
    if (pair) {
#pragma unroll
      for (int j = 0; j < RC; ++j)
        if (j < rc) atomicAdd(out + (n0 + 1) * ldo + j, scale * acc1[j]);
      if (colsum) atomicAdd(colsum + n0 + 1, cs1);
    }
  }
}

__global__ void k_pad_bf16(const float* __restrict__ src, int64_t rows, int64_t cols,
                           int64_t lds, __nv_bfloat16* __restrict__ dst, int64_t rows_pad,
                           int64_t ldd) {
  const int64_t total = rows_pad * ldd;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / ldd, c = i % ldd;
    dst[i] = __float2bfloat16_rn((r < rows && c < cols) ? src[r * lds + c] : 0.0f);
  }
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <int RC>
cudaError_t rowdot_rc(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                      const float* W, int64_t ldw, int rc, float scale, float* out, int64_t ldo,
                      __nv_bfloat16* pad, int64_t ldp, cudaStream_t st) {
  constexpr int TT = 64 / RC;
  const size_t smem = 32 * (8 * RC + 4) * sizeof(float);
  auto kern = k_rowdot<RC, TT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t blocks = (m + 8 * TT - 1) / (8 * TT);
  note_launch();
  kern<<<static_cast<unsigned>(blocks), 256, smem, st>>>(act, lda, m, kd, W, ldw, rc, scale,
                                                         out, ldo, pad, ldp);
  return cudaGetLastError();
}

template <int RC>
cudaError_t coldot_rc(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t nd,
                      const float* V, int64_t ldv, int rc, float scale, float* out, int64_t ldo,
                      float* colsum, cudaStream_t st) {
  const int64_t bx = (nd + 255) / 256;
  int64_t splits = (4 * sm_count() + bx - 1) / bx;
  const int64_t max_splits = (m + 63) / 64;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  int64_t tpb = (m + splits - 1) / splits;
  tpb = (tpb + 63) / 64 * 64;
  splits = (m + tpb - 1) / tpb;
  dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(splits));
  note_launch();
  k_coldot<RC><<<grid, 128, 0, st>>>(act, lda, m, nd, V, ldv, rc, scale, tpb, out, ldo, colsum);
  return cudaGetLastError();
}

}  // namespace

// rank up to 256 in chunks of at most 64 columns
cudaError_t launch_rowdot(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                          const float* W, int64_t r, float scale, float* out,
                          __nv_bfloat16* pad, int64_t ldp, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  for (int64_t j0 = 0; j0 < r; j0 += 64) {
    const int rc = static_cast<int>(r - j0 < 64 ? r - j0 : 64);
    __nv_bfloat16* p = pad ? pad + j0 : nullptr;
    cudaError_t e;
    if (rc <= 8)
      e = rowdot_rc<8>(act, lda, m, kd, W + j0, r, rc, scale, out + j0, r, p, ldp, st);
    else if (rc <= 16)
      e = rowdot_rc<16>(act, lda, m, kd, W + j0, r, rc, scale, out + j0, r, p, ldp, st);
    else if (rc <= 32)
      e = rowdot_rc<32>(act, lda, m, kd, W + j0, r, rc, scale, out + j0, r, p, ldp, st);
    else
      e = rowdot_rc<64>(act, lda, m, kd, W + j0, r, rc, scale, out + j0, r, p, ldp, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_coldot(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t nd,
                          const float* V, int64_t r, float scale, float* out, float* colsum,
                          cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  for (int64_t j0 = 0; j0 < r; j0 += 64) {
    const int rc = static_cast<int>(r - j0 < 64 ? r - j0 : 64);
    float* cs = j0 == 0 ? colsum : nullptr;
    cudaError_t e;
    if (rc <= 8)
      e = coldot_rc<8>(act, lda, m, nd, V + j0, r, rc, scale, out + j0, r, cs, st);
    else if (rc <= 16)
      e = coldot_rc<16>(act, lda, m, nd, V + j0, r, rc, scale, out + j0, r, cs, st);
    else if (rc <= 32)
      e = coldot_rc<32>(act, lda, m, nd, V + j0, r, rc, scale, out + j0, r, cs, st);
    else
      e = coldot_rc<64>(act, lda, m, nd, V + j0, r, rc, scale, out + j0, r, cs, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_pad_bf16(const float* src, int64_t rows, int64_t cols, int64_t lds,
                            __nv_bfloat16* dst, int64_t rows_pad, int64_t ldd, cudaStream_t st) {
  int64_t blocks = (rows_pad * ldd + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  note_launch();
  k_pad_bf16<<<static_cast<unsigned>(blocks), 256, 0, st>>>(src, rows, cols, lds, dst, rows_pad,
                                                            ldd);
  return cudaGetLastError();
}

}  // namespace mlra
