// thin_mma.cu — K4/K5/K6 on tensor cores: the skinny rank-r adapter products.
//
//  k_rowmma (K4, K5a): out[t, j] = Σ_k act[t,k]·W[k,j]   (m x r; reduction over d)
//     XB  = X·B   — matmul(t, x, B)               lora.cpp:68
//     dYA = dY·A  — d(xb) = dab·A                  autodiff.cpp:150-152 on lora.cpp:69
//  k_colmma (K5b, K6): out[n, j] += s·Σ_t act[t,n]·V[t,j]  (d x r; reduction over tokens)
//     dA = s·dYᵀ·XB   — d(Aᵀ) = xbᵀ·dab, transposed   autodiff.cpp:153-155, :315-320
//     dB = s·Xᵀ·dYA   — dB = xᵀ·d(xb)                  autodiff.cpp:153-155
//     dbias = Σ_t dY  — bias_add backward (a ones column of V)  autodiff.cpp:183-191
//
// These are HBM-bound (r flop/B): each CTA streams 64-row activation tiles
// through a cp.async double buffer and runs bf16 mma.sync m16n8k16 against the
// rank-r factor. The fp32 factor is split into bf16 hi + lo parts (two MMAs),
// so the product keeps ~16 mantissa bits (fp32-grade
// intermediates); activations are exact bf16. Split-K / split-token CTAs
// combine with fp32 atomics.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace mlra {

namespace {

constexpr int TILE = 64;      // rows (tokens or n) per CTA tile, and K chunk
constexpr int PADW = 72;      // padded smem row (bf16): conflict-free ldmatrix
constexpr int NS = 4;         // cp.async pipeline depth (chunks in flight per CTA)
constexpr int thin_smem_bytes(int nt) { return (NS * TILE * PADW + NS * 2 * 8 * nt * PADW) * 2; }

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Load a 64-row x 64-col bf16 tile (rows r0.., cols c0..) of a row-major
// matrix [rows x cols] (leading dim ld) into padded smem; zero-fill outside.
__device__ __forceinline__ void load_tile(uint32_t dst, const __nv_bfloat16* src, int64_t ld,
                                          int64_t rows, int64_t cols, int64_t r0, int64_t c0) {
  for (int i = threadIdx.x; i < TILE * 8; i += blockDim.x) {
    const int rr = i >> 3, cc = (i & 7) * 8;
    const int64_t r = r0 + rr, c = c0 + cc;
    int bytes = 0;
    const __nv_bfloat16* p = src;
    if (r < rows && c < cols) {
      const int64_t rem = cols - c;
      bytes = rem >= 8 ? 16 : static_cast<int>(rem) * 2;
      p = src + r * ld + c;
    }
    cp_async16(dst + (rr * PADW + cc) * 2, p, bytes);
  }
}

// Load factor rows [0, 8*NT) x cols [c0, c0+64) of a [8*NT x ld] bf16 matrix
// (hi and lo planes) into padded smem.
template <int NT>
__device__ __forceinline__ void load_factor(uint32_t dst, const __nv_bfloat16* hi,
                                            const __nv_bfloat16* lo, int64_t ld, int64_t c0) {
  constexpr int ROWS = 8 * NT;
  for (int i = threadIdx.x; i < 2 * ROWS * 8; i += blockDim.x) {
    const int plane = i / (ROWS * 8), j = i % (ROWS * 8);
    const int rr = j >> 3, cc = (j & 7) * 8;
    const __nv_bfloat16* p = (plane ? lo : hi) + rr * ld + c0 + cc;
    cp_async16(dst + ((plane * ROWS + rr) * PADW + cc) * 2, p, 16);
  }
}

// out[t, j] (+)= Σ_k act[t, k] · Wt[j, k]   (Wt = W transposed, hi/lo bf16, [8NT x kpad])
template <int NT>
__global__ void __launch_bounds__(128)
    k_rowmma(const __nv_bfloat16* __restrict__ act, int64_t lda, int64_t m, int64_t kd,
             const __nv_bfloat16* __restrict__ wt_hi, const __nv_bfloat16* __restrict__ wt_lo,
             int64_t ldw, int64_t k_per_split, float* __restrict__ out, int64_t ldo, int rc) {
  constexpr int ROWS = 8 * NT;
  extern __shared__ __align__(16) __nv_bfloat16 thin_smem[];
  __nv_bfloat16* const sa0 = thin_smem;                      // NS act tiles
  __nv_bfloat16* const sw0 = thin_smem + NS * TILE * PADW;   // NS factor tiles (hi+lo)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * TILE;
  const int64_t ks = static_cast<int64_t>(blockIdx.y) * k_per_split;
  const int64_t ke = ks + k_per_split < kd ? ks + k_per_split : kd;
  const int nch = static_cast<int>((ke - ks + TILE - 1) / TILE);
  float acc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.0f;
  for (int c = 0; c < NS - 1; ++c) {
    if (c < nch) {
      load_tile(su32(sa0 + c * TILE * PADW), act, lda, m, ke, t0, ks + c * TILE);
      load_factor<NT>(su32(sw0 + c * 2 * ROWS * PADW), wt_hi, wt_lo, ldw, ks + c * TILE);
    }
    cp_commit();
  }
  for (int c = 0; c < nch; ++c) {
    const int pf = c + NS - 1, b = c % NS;
    if (pf < nch) {
      load_tile(su32(sa0 + (pf % NS) * TILE * PADW), act, lda, m, ke, t0, ks + pf * TILE);
      load_factor<NT>(su32(sw0 + (pf % NS) * 2 * ROWS * PADW), wt_hi, wt_lo, ldw, ks + pf * TILE);
    }
    cp_commit();
    cp_wait<NS - 1>();
    __syncthreads();
    const uint32_t abase =
        su32(sa0 + b * TILE * PADW) + ((warp * 16 + (lane & 15)) * PADW + (lane >> 4) * 8) * 2;
    const __nv_bfloat16* wsm = sw0 + b * 2 * ROWS * PADW;
#pragma unroll
    for (int k16 = 0; k16 < 4; ++k16) {
      uint32_t a[4];
      ldsm_x4(abase + k16 * 32, a);
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const __nv_bfloat16* wh = wsm + (n * 8 + g) * PADW + k16 * 16 + 2 * tq;
        const __nv_bfloat16* wl = wh + ROWS * PADW;
        mma_bf16(acc[n], a, *reinterpret_cast<const uint32_t*>(wh),
                 *reinterpret_cast<const uint32_t*>(wh + 8));
        mma_bf16(acc[n], a, *reinterpret_cast<const uint32_t*>(wl),
                 *reinterpret_cast<const uint32_t*>(wl + 8));
      }
    }
    __syncthreads();
  }
  const int64_t ta = t0 + warp * 16 + g, tb = ta + 8;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int j = n * 8 + 2 * tq;
    if (ta < m) {
      if (j < rc) atomicAdd(out + ta * ldo + j, acc[n][0]);
      if (j + 1 < rc) atomicAdd(out + ta * ldo + j + 1, acc[n][1]);
    }
    if (tb < m) {
      if (j < rc) atomicAdd(out + tb * ldo + j, acc[n][2]);
      if (j + 1 < rc) atomicAdd(out + tb * ldo + j + 1, acc[n][3]);
    }
  }
}

// out[n, j] += scale · Σ_t act[t, n] · Vt[j, t]   (Vt = V transposed, hi/lo bf16, [8NT x ldv])
// Columns j >= rc of the product go to colsum (the ones column) when j == rc.
template <int NT>
__global__ void __launch_bounds__(128)
    k_colmma(const __nv_bfloat16* __restrict__ act, int64_t lda, int64_t m, int64_t nd,
             const __nv_bfloat16* __restrict__ vt_hi, const __nv_bfloat16* __restrict__ vt_lo,
             int64_t ldv, int64_t t_per_split, float scale, float* __restrict__ out, int64_t ldo,
             int rc, float* __restrict__ colsum) {
  constexpr int ROWS = 8 * NT;
  extern __shared__ __align__(16) __nv_bfloat16 thin_smem[];
  __nv_bfloat16* const sa0 = thin_smem;
  __nv_bfloat16* const sv0 = thin_smem + NS * TILE * PADW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * TILE;
  const int64_t ts = static_cast<int64_t>(blockIdx.y) * t_per_split;
  const int64_t te = ts + t_per_split < m ? ts + t_per_split : m;
  const int nch = static_cast<int>((te - ts + TILE - 1) / TILE);
  float acc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.0f;
  for (int c = 0; c < NS - 1; ++c) {
    if (c < nch) {
      load_tile(su32(sa0 + c * TILE * PADW), act, lda, te, nd, ts + c * TILE, n0);
      load_factor<NT>(su32(sv0 + c * 2 * ROWS * PADW), vt_hi, vt_lo, ldv, ts + c * TILE);
    }
    cp_commit();
  }
  for (int c = 0; c < nch; ++c) {
    const int pf = c + NS - 1, b = c % NS;
    if (pf < nch) {
      load_tile(su32(sa0 + (pf % NS) * TILE * PADW), act, lda, te, nd, ts + pf * TILE, n0);
      load_factor<NT>(su32(sv0 + (pf % NS) * 2 * ROWS * PADW), vt_hi, vt_lo, ldv, ts + pf * TILE);
    }
    cp_commit();
    cp_wait<NS - 1>();
    __syncthreads();
    // A fragment (M = n, K = t) from the [t][n] tile via transposed ldmatrix:
    // lane l addresses row t = (l & 7) + 8*(l >> 4), col n = warp*16 + 8*((l >> 3) & 1)
    const uint32_t abase = su32(sa0 + b * TILE * PADW) +
                           (((lane & 7) + ((lane >> 4) << 3)) * PADW + warp * 16 +
                            ((lane >> 3) & 1) * 8) * 2;
    const __nv_bfloat16* vsm = sv0 + b * 2 * ROWS * PADW;
#pragma unroll
    for (int k16 = 0; k16 < 4; ++k16) {
      uint32_t a[4];
      ldsm_x4_t(abase + k16 * 16 * PADW * 2, a);
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const __nv_bfloat16* vh = vsm + (n * 8 + g) * PADW + k16 * 16 + 2 * tq;
        const __nv_bfloat16* vl = vh + ROWS * PADW;
        mma_bf16(acc[n], a, *reinterpret_cast<const uint32_t*>(vh),
                 *reinterpret_cast<const uint32_t*>(vh + 8));
        mma_bf16(acc[n], a, *reinterpret_cast<const uint32_t*>(vl),
                 *reinterpret_cast<const uint32_t*>(vl + 8));
      }
    }
    __syncthreads();
  }
  const int64_t na = n0 + warp * 16 + g, nb = na + 8;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = n * 8 + 2 * tq + h;
      if (j < rc) {
        if (na < nd) atomicAdd(out + na * ldo + j, scale * acc[n][h]);
        if (nb < nd) atomicAdd(out + nb * ldo + j, scale * acc[n][2 + h]);
      } else if (j == rc && colsum != nullptr) {
        if (na < nd) atomicAdd(colsum + na, acc[n][h]);
        if (nb < nd) atomicAdd(colsum + nb, acc[n][2 + h]);
      }
    }
  }
}

// One launch for a layer pass's small conversion / zeroing jobs (PrepBatch):
// grid-stride over the concatenated index spaces of up to kMaxPrep tasks.
__global__ void k_prep(const PrepBatch b) {
  const int64_t total = b.offs[b.n];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int t = 0;
    while (i >= b.offs[t + 1]) ++t;
    const PrepTask& k = b.t[t];
    const int64_t j = i - b.offs[t];
    switch (k.kind) {
      case PrepTask::kZeroF32:
        reinterpret_cast<float*>(k.dst)[j] = 0.0f;
        break;
      case PrepTask::kZeroBf16:
        reinterpret_cast<__nv_bfloat16*>(k.dst)[j] = __float2bfloat16_rn(0.0f);
        break;
      case PrepTask::kSplitT: {  // hi/lo planes [rows_out x ldd] of src^T (cols = r)
        const int64_t row = j / k.ldd, col = j % k.ldd;
        float v = 0.0f;
        if (col < k.rows) {
          if (row < k.cols)
            v = k.src[col * k.lds + row];
          else if (row == k.cols && k.ones)
            v = 1.0f;
        }
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        reinterpret_cast<__nv_bfloat16*>(k.dst)[j] = h;
        reinterpret_cast<__nv_bfloat16*>(k.dst2)[j] = __float2bfloat16_rn(v - __bfloat162float(h));
        break;
      }
      case PrepTask::kPadBf16: {  // dst [rows_out x ldd] = bf16(scale * src) zero-padded
        const int64_t row = j / k.ldd, col = j % k.ldd;
        const float v = (row < k.rows && col < k.cols) ? k.scale * k.src[row * k.lds + col] : 0.0f;
        reinterpret_cast<__nv_bfloat16*>(k.dst)[j] = __float2bfloat16_rn(v);
        break;
      }
    }
  }
}

int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

int blocks_for(int64_t work) {
  int64_t b = (work + 255) / 256;
  if (b > 16 * sms()) b = 16 * sms();
  return static_cast<int>(b < 1 ? 1 : b);
}

template <int NT>
cudaError_t rowmma_nt(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                      const __nv_bfloat16* hi, const __nv_bfloat16* lo, int64_t ldw, float* out,
                      int64_t ldo, int64_t r, cudaStream_t st) {
  const int64_t tb = (m + TILE - 1) / TILE;
  const int64_t kchunks = (kd + TILE - 1) / TILE;
  int64_t splits = (4 * sms() + tb - 1) / tb;
  if (splits > kchunks) splits = kchunks;
  if (splits < 1) splits = 1;
  const int64_t kps = (kchunks + splits - 1) / splits * TILE;
  splits = (kd + kps - 1) / kps;
  dim3 grid(static_cast<unsigned>(tb), static_cast<unsigned>(splits));
  const int smem = thin_smem_bytes(NT);
  cudaError_t e = cudaFuncSetAttribute(k_rowmma<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch();
  k_rowmma<NT><<<grid, 128, smem, st>>>(act, lda, m, kd, hi, lo, ldw, kps, out, ldo,
                                        static_cast<int>(r));
  return cudaGetLastError();
}

template <int NT>
cudaError_t colmma_nt(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t nd,
                      const __nv_bfloat16* hi, const __nv_bfloat16* lo, int64_t ldv, float scale,
                      float* out, int64_t ldo, int64_t r, float* colsum, cudaStream_t st) {
  const int64_t nb = (nd + TILE - 1) / TILE;
  const int64_t tchunks = (m + TILE - 1) / TILE;
  int64_t splits = (4 * sms() + nb - 1) / nb;
  if (splits > tchunks) splits = tchunks;
  if (splits < 1) splits = 1;
  const int64_t tps = (tchunks + splits - 1) / splits * TILE;
  splits = (m + tps - 1) / tps;
  dim3 grid(static_cast<unsigned>(nb), static_cast<unsigned>(splits));
  const int smem = thin_smem_bytes(NT);
  cudaError_t e = cudaFuncSetAttribute(k_colmma<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch();
  k_colmma<NT><<<grid, 128, smem, st>>>(act, lda, m, nd, hi, lo, ldv, tps, scale, out, ldo,
                                        static_cast<int>(r), colsum);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_prep(const PrepBatch& b, cudaStream_t st) {
  if (b.n == 0 || b.offs[b.n] == 0) return cudaSuccess;
  note_launch();
  k_prep<<<blocks_for(b.offs[b.n]), 256, 0, st>>>(b);
  return cudaGetLastError();
}

int thin_rows(int64_t r, bool ones) { return static_cast<int>((r + (ones ? 1 : 0) + 7) / 8 * 8); }

#define MLRA_NT_DISPATCH(NTV, CALL)            \
  switch (NTV) {                               \
    case 1: return CALL(1);                    \
    case 2: return CALL(2);                    \
    case 3: return CALL(3);                    \
    case 4: return CALL(4);                    \
    case 5: return CALL(5);                    \
    case 6: return CALL(6);                    \
    case 7: return CALL(7);                    \
    case 8: return CALL(8);                    \
    case 9: return CALL(9);                    \
    default: return cudaErrorInvalidValue;     \
  }

cudaError_t launch_rowmma(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                          const __nv_bfloat16* wt_hi, const __nv_bfloat16* wt_lo, int64_t ldw,
                          float* out, int64_t ldo, int64_t r, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
#define CALL_ROW(N) rowmma_nt<N>(act, lda, m, kd, wt_hi, wt_lo, ldw, out, ldo, r, st)
  MLRA_NT_DISPATCH(thin_rows(r, false) / 8, CALL_ROW)
#undef CALL_ROW
}

cudaError_t launch_colmma(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t nd,
                          const __nv_bfloat16* vt_hi, const __nv_bfloat16* vt_lo, int64_t ldv,
                          float scale, float* out, int64_t ldo, int64_t r, float* colsum,
                          cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
#define CALL_COL(N) colmma_nt<N>(act, lda, m, nd, vt_hi, vt_lo, ldv, scale, out, ldo, r, colsum, st)
  MLRA_NT_DISPATCH(thin_rows(r, colsum != nullptr) / 8, CALL_COL)
#undef CALL_COL
}

}  // namespace mlra
