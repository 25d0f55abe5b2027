// optq.cu — OptqQuantizer::quantize on the device (
// quantize.hpp:62-77, 115-125; quantize.cpp:186-255; linalg.cpp:13-71),
// bit-identical to the reference.
//
// Every f64 value the reference computes is the end of a fixed, in-order chain
// of IEEE operations (mul then add/sub: the reference is built without FMA
// contraction). Each kernel below evaluates the same chains in the same order
// with explicitly rounded intrinsics (__dmul_rn / __dadd_rn / __dsub_rn /
// __ddiv_rn, never contracted) and takes its parallelism from the independent
// chains only:
//  * k_hessian: H = XᵀX (matrix.cpp:81-97), one chain over the samples per
//    entry, smem-tiled;
//  * k_damp: mean of diag(H), H_ii += damping·mean (quantize.cpp:198-204);
//  * k_chol_step: cholesky_lower (linalg.cpp:13-34) right-looking — step k
//    finalizes column k and applies its term to every trailing entry, which is
//    exactly the reference's k-ascending subtraction order per entry;
//  * k_spd_solve: spd_inverse's per-column forward / back solves (linalg.cpp:
//    36-58), one thread per column (the back solve's k-ascending order forbids
//    a right-looking schedule), then k_symmetrize (:59-66);
//  * the column sweep (quantize.cpp:231-252) is row-parallel: for each row the
//    residual entry r(i,k) receives e_j·U(j,k) for j ascending. k_sweep keeps
//    that order per entry but defers the far-column terms: a CTA owns 32 rows,
//    walks 32-column blocks, first applies all earlier columns' terms to the
//    block as an in-order tiled product (E·U, compute-bound), then sweeps the
//    block column by column.
#include <cuda_runtime.h>

#include "kernels.h"

namespace mlra {

namespace {

__device__ __forceinline__ double msub(double s, double a, double b) {
  return __dsub_rn(s, __dmul_rn(a, b));
}

// H[n x n] = Xᵀ X, X [m x n] row-major: H(i,j) = ((0 + x0i·x0j) + x1i·x1j) + ...
constexpr int HT = 32;
__global__ void __launch_bounds__(256) k_hessian(const double* __restrict__ x, int64_t m, int64_t n,
                                                 double* __restrict__ h) {
  __shared__ double sa[HT][HT + 1], sb[HT][HT + 1];  // [sample][col]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * HT, j0 = static_cast<int64_t>(blockIdx.x) * HT;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t p0 = 0; p0 < m; p0 += HT) {
    for (int r = ty; r < HT; r += 8) {
      const int64_t p = p0 + r;
      sa[r][tx] = (p < m && i0 + tx < n) ? x[p * n + i0 + tx] : 0.0;
      sb[r][tx] = (p < m && j0 + tx < n) ? x[p * n + j0 + tx] : 0.0;
    }
    __syncthreads();
    const int pn = m - p0 < HT ? static_cast<int>(m - p0) : HT;
    for (int pp = 0; pp < pn; ++pp) {
      const double b = sb[pp][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(sa[pp][ty * 4 + q], b));
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = i0 + ty * 4 + q, j = j0 + tx;
    if (i < n && j < n) h[i * n + j] = acc[q];
  }
}

__global__ void k_damp(double* __restrict__ h, int64_t n, double damping) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mean = 0.0;
  for (int64_t i = 0; i < n; ++i) mean = __dadd_rn(mean, h[i * n + i]);
  mean = __ddiv_rn(mean, static_cast<double>(n));
  const double add = __dmul_rn(damping, mean);
  for (int64_t i = 0; i < n; ++i) h[i * n + i] = __dadd_rn(h[i * n + i], add);
}

// Step k of the right-looking Cholesky on S (lower part, in place): column k of
// S is final (every term j < k applied). L(:, k) = S(:, k) / sqrt(S(k, k));
// S(i, j) -= L(i, k)·L(j, k) for k < j <= i. bad: first pivot with S(k,k) <= 0.
__global__ void __launch_bounds__(256) k_chol_step(double* __restrict__ s, double* __restrict__ l,
                                                   int64_t n, int64_t k, int* __restrict__ bad) {
  const double d = s[k * n + k];
  const double lkk = sqrt(d);
  const int64_t t = n - k - 1;  // trailing extent
  if (blockIdx.y == 0 && blockIdx.x == 0) {  // finalize column k (block (0,0) also updates below)
    for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x)
      l[i * n + k] = i == k ? lkk : __ddiv_rn(s[i * n + k], lkk);
    if (threadIdx.x == 0 && !(d > 0.0)) atomicMin(bad, static_cast<int>(k));
  }
  // 32 x 32 tiles of the trailing lower triangle, 4 entries per thread
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  if (bj > bi || t <= 0) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j = k + 1 + bj * 32 + tx;
  if (j >= n) return;
  const double ljk = __ddiv_rn(s[j * n + k], lkk);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = k + 1 + bi * 32 + ty * 4 + q;
    if (i < n && i >= j) {
      const double lik = __ddiv_rn(s[i * n + k], lkk);
      s[i * n + j] = msub(s[i * n + j], lik, ljk);
    }
  }
}

// spd_inverse per column `col` (one thread each): L y = e_col, then Lᵀ x = y,
// both with the reference's k-ascending chains. y / x live column-interleaved
// (entry i of column col at [i * n + col]) so a warp's accesses coalesce.
__global__ void k_spd_solve(const double* __restrict__ l, int64_t n, double* __restrict__ y,
                            double* __restrict__ inv) {
  const int64_t col = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (col >= n) return;
  for (int64_t i = 0; i < n; ++i) {
    double s = i == col ? 1.0 : 0.0;
    const double* li = l + i * n;
#pragma unroll 4
    for (int64_t k = 0; k < i; ++k) s = msub(s, __ldg(li + k), y[k * n + col]);
    y[i * n + col] = __ddiv_rn(s, __ldg(li + i));
  }
  for (int64_t ii = n; ii-- > 0;) {
    double s = y[ii * n + col];
#pragma unroll 4
    for (int64_t k = ii + 1; k < n; ++k) s = msub(s, __ldg(l + k * n + ii), inv[k * n + col]);
    inv[ii * n + col] = __ddiv_rn(s, __ldg(l + ii * n + ii));
  }
}

__global__ void k_symmetrize(double* __restrict__ a, int64_t n) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t / n, j = t % n;
    if (j > i) {
      const double v = __dmul_rn(0.5, __dadd_rn(a[i * n + j], a[j * n + i]));
      a[i * n + j] = v;
      a[j * n + i] = v;
    }
  }
}

// U = Lᵀ (upper), the strictly-lower part zero (transpose of a lower L).
__global__ void k_transpose_lower(const double* __restrict__ l, int64_t n, double* __restrict__ u) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = t / n, j = t % n;
    u[t] = j >= i ? l[j * n + i] : 0.0;
  }
}

// code_on_grid (quantize.cpp:38-44) on the f32 grid of the entry's group.
__device__ __forceinline__ uint32_t code_on(double w, float s, float z, double levels) {
  double c = round(__ddiv_rn(__dsub_rn(w, static_cast<double>(z)), static_cast<double>(s)));
  c = c < 0.0 ? 0.0 : (c > levels ? levels : c);
  return static_cast<uint32_t>(c);
}

// The column sweep. CTA = 32 rows; block = 32 columns; 256 threads, thread
// (tx, ty) owns rows ty*4..ty*4+3 of column tx of the block.
constexpr int SR = 32, SB = 32;
__global__ void __launch_bounds__(256) k_sweep(const double* __restrict__ w, const double* __restrict__ u,
                                               int64_t rows, int64_t cols, int64_t group, int bits,
                                               const float* __restrict__ scales,
                                               const float* __restrict__ zeros,
                                               double* __restrict__ e_all, uint32_t* __restrict__ codes) {
  __shared__ double se[SR][SB + 1];  // e of (row, column) for the staged column chunk
  __shared__ double su[SB][SB + 1];  // U rows of the staged chunk x the block's columns
  __shared__ double st[SR][SB + 1];  // the block's residual tile
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * SR;
  const int64_t ng = cols / group;
  const double levels = static_cast<double>((1 << bits) - 1);
  for (int64_t c0 = 0; c0 < cols; c0 += SB) {
    const int64_t k = c0 + tx;
    double t[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = r0 + ty * 4 + q;
      t[q] = (i < rows && k < cols) ? w[i * cols + k] : 0.0;
    }
    // deferred terms of every earlier column, j ascending
    for (int64_t j0 = 0; j0 < c0; j0 += SB) {
      for (int rr = ty; rr < SR; rr += 8) {
        const int64_t i = r0 + rr;
        se[rr][tx] = i < rows ? e_all[i * cols + j0 + tx] : 0.0;
        su[rr][tx] = k < cols ? u[(j0 + rr) * cols + k] : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int jj = 0; jj < SB; ++jj) {
        const double uj = su[jj][tx];
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] = msub(t[q], se[ty * 4 + q][jj], uj);
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) st[ty * 4 + q][tx] = t[q];
    // U rows of this block's own columns
    for (int rr = ty; rr < SB; rr += 8)
      su[rr][tx] = (c0 + rr < cols && k < cols) ? u[(c0 + rr) * cols + k] : 0.0;
    __syncthreads();
    const int nb = cols - c0 < SB ? static_cast<int>(cols - c0) : SB;
    for (int jj = 0; jj < nb; ++jj) {
      const int64_t j = c0 + jj;
      if (threadIdx.x < SR) {  // one thread per row quantizes column j
        const int64_t i = r0 + threadIdx.x;
        double e = 0.0;
        if (i < rows) {
          const double rij = st[threadIdx.x][jj];
          const float s = scales[i * ng + j / group], z = zeros[i * ng + j / group];
          const uint32_t c = code_on(rij, s, z, levels);
          codes[i * cols + j] = c;
          const double what = __dadd_rn(__dmul_rn(static_cast<double>(s), static_cast<double>(c)),
                                        static_cast<double>(z));
          e = __ddiv_rn(__dsub_rn(rij, what), su[jj][jj]);
          e_all[i * cols + j] = e;
        }
        se[threadIdx.x][jj] = e;
      }
      __syncthreads();
      if (tx > jj) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st[ty * 4 + q][tx] = msub(st[ty * 4 + q][tx], se[ty * 4 + q][jj], su[jj][tx]);
      }
      __syncthreads();
    }
  }
}

// codes [rows x cols] -> the reference's whole-matrix LSB-first bitstream
__global__ void k_pack_codes(const uint32_t* __restrict__ codes, uint64_t count, int bits,
                             uint64_t nwords, uint32_t* __restrict__ words) {
  for (uint64_t wi = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; wi < nwords;
       wi += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t b0 = wi * 32;
    uint64_t c_last = (b0 + 31) / bits;
    if (c_last >= count) c_last = count - 1;
    uint32_t out = 0;
    for (uint64_t c = b0 / bits; c <= c_last; ++c) {
      const int64_t sh = static_cast<int64_t>(c * bits) - static_cast<int64_t>(b0);
      const uint32_t v = codes[c];
      out |= sh >= 0 ? v << sh : v >> (-sh);
    }
    words[wi] = out;
  }
}

int blocks_for(int64_t work, int per_block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t b = (work + per_block - 1) / per_block;
  if (b > 16LL * sms) b = 16LL * sms;
  return static_cast<int>(b < 1 ? 1 : b);
}

// cholesky_lower of a (n x n, consumed as scratch) into l; bad = first failing pivot or n
cudaError_t cholesky(double* a, double* l, int64_t n, int* bad, cudaStream_t st) {
  for (int64_t k = 0; k < n; ++k) {
    const int64_t t = n - k - 1;
    const unsigned nb = static_cast<unsigned>(t > 0 ? (t + 31) / 32 : 1);
    note_launch();
    k_chol_step<<<dim3(nb, nb), 256, 0, st>>>(a, l, n, k, bad);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_optq_workspace(const double* calib, int64_t m, int64_t n, double damping,
                                  double* hessian, double* upper, double* scratch, int* bad,
                                  cudaStream_t st) {
  // scratch: 2 n^2 doubles
  double* a = scratch;
  double* b = scratch + n * n;
  const unsigned nt = static_cast<unsigned>((n + HT - 1) / HT);
  note_launch();
  k_hessian<<<dim3(nt, nt), 256, 0, st>>>(calib, m, n, hessian);
  note_launch();
  k_damp<<<1, 32, 0, st>>>(hessian, n, damping);
  cudaError_t e = cudaMemcpyAsync(a, hessian, n * n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b, 0, n * n * sizeof(double), st)) != cudaSuccess) return e;
  if ((e = cholesky(a, b, n, bad, st)) != cudaSuccess) return e;  // b = L
  // inverse through the column solves: y scratch in `a`, result in `upper` (temp)
  note_launch();
  k_spd_solve<<<static_cast<unsigned>((n + 63) / 64), 64, 0, st>>>(b, n, a, upper);
  note_launch();
  k_symmetrize<<<blocks_for(n * n, 256), 256, 0, st>>>(upper, n);
  // second factorization (of the inverse; its pivots cannot fail once the first succeeded
  // in exact arithmetic — a failure is still reported through `bad` as n + pivot)
  if ((e = cudaMemsetAsync(b, 0, n * n * sizeof(double), st)) != cudaSuccess) return e;
  if ((e = cholesky(upper, b, n, bad + 1, st)) != cudaSuccess) return e;
  note_launch();
  k_transpose_lower<<<blocks_for(n * n, 256), 256, 0, st>>>(b, n, upper);
  return cudaGetLastError();
}

cudaError_t launch_optq_sweep(const double* w, const double* upper, int64_t rows, int64_t cols,
                              int64_t group, int bits, const float* scales, const float* zeros,
                              double* e_scratch, uint32_t* codes, uint32_t* words, uint64_t nwords,
                              cudaStream_t st) {
  note_launch();
  k_sweep<<<static_cast<unsigned>((rows + SR - 1) / SR), 256, 0, st>>>(
      w, upper, rows, cols, group, bits, scales, zeros, e_scratch, codes);
  note_launch();
  k_pack_codes<<<blocks_for(static_cast<int64_t>(nwords), 256), 256, 0, st>>>(
      codes, static_cast<uint64_t>(rows * cols), bits, nwords, words);
  return cudaGetLastError();
}

}  // namespace mlra
