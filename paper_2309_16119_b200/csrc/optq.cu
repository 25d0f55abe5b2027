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
//  * k_fwd_solve / k_back_solve: spd_inverse's per-column solves (linalg.cpp:
//    36-58), one thread per column (forward: 32 chains per thread through the
//    far terms; back: a serial chain per column — its k-ascending order
//    forbids a right-looking schedule — with operands loaded a batch ahead),
//    then k_symmetrize (:59-66);
//  * the column sweep (quantize.cpp:231-252) is row-parallel: for each row the
//    residual entry r(i,k) receives e_j·U(j,k) for j ascending. k_sweep keeps
//    that order per entry but defers the far-column terms: a CTA owns 32 rows,
//    walks 32-column blocks, first applies all earlier columns' terms to the
//    block as an in-order tiled product (E·U, compute-bound), then sweeps the
//    block column by column.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace mlra {

namespace {

__device__ __forceinline__ double msub(double s, double a, double b) {
  return __dsub_rn(s, __dmul_rn(a, b));
}

constexpr int CP = 32;  // panel width of the blocked factor / solve kernels

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
// S is final (every term j < k applied). L(:, k) = S(:, k) / sqrt(S(k, k)),
// stored transposed (lt row k = L column k, i.e. lt = Lᵀ, upper);
// S(i, j) -= L(i, k)·L(j, k) for k < j <= i. bad: first pivot with S(k,k) <= 0.
__global__ void __launch_bounds__(256) k_chol_step(double* __restrict__ s, double* __restrict__ lt,
                                                   int64_t n, int64_t k, int* __restrict__ bad) {
  const double d = s[k * n + k];
  const double lkk = sqrt(d);
  const int64_t t = n - k - 1;  // trailing extent
  if (blockIdx.y == 0 && blockIdx.x == 0) {  // finalize column k (block (0,0) also updates below)
    for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x)
      lt[k * n + i] = i == k ? lkk : __ddiv_rn(s[i * n + k], lkk);
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

// spd_inverse per column `col` (one thread each; y / x column-interleaved:
// entry i of column col at [i * n + col], so a warp's accesses coalesce).
// Forward solve L y = e_col: y[i] = (δ - Σ_{k<i} L(i,k)·y[k]) / L(i,i), k
// ascending. The far terms (k below the current 32-row block) come first in
// every chain, so a thread carries the 32 chains of a block at once (ILP 32)
// through the far terms, staged 32 x 32 from Lᵀ in shared memory, then
// finishes the block's triangle in order.
constexpr int FB = 32;
__global__ void __launch_bounds__(64) k_fwd_solve(const double* __restrict__ lt, int64_t n,
                                                  double* __restrict__ y) {
  __shared__ double sl[FB][FB + 1];  // sl[kk][q] = L(i0 + q, k0 + kk)
  const int64_t col = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (int64_t i0 = 0; i0 < n; i0 += FB) {
    double sv[FB];
#pragma unroll
    for (int q = 0; q < FB; ++q) sv[q] = (i0 + q == col) ? 1.0 : 0.0;
    for (int64_t k0 = 0; k0 < i0; k0 += FB) {
      __syncthreads();
      for (int t = threadIdx.x; t < FB * FB; t += blockDim.x) {
        const int kk = t / FB, q = t % FB;
        sl[kk][q] = i0 + q < n ? lt[(k0 + kk) * n + i0 + q] : 0.0;
      }
      __syncthreads();
      if (col < n) {
#pragma unroll 4
        for (int kk = 0; kk < FB; ++kk) {
          const double yk = y[(k0 + kk) * n + col];
#pragma unroll
          for (int q = 0; q < FB; ++q) sv[q] = msub(sv[q], sl[kk][q], yk);
        }
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < FB * FB; t += blockDim.x) {  // the block's own triangle
      const int kk = t / FB, q = t % FB;
      sl[kk][q] = (i0 + q < n && i0 + kk < n) ? lt[(i0 + kk) * n + i0 + q] : 0.0;
    }
    __syncthreads();
    if (col < n) {
#pragma unroll
      for (int q = 0; q < FB; ++q) {
        if (i0 + q >= n) break;
        double v = sv[q];
        for (int kk = 0; kk < q; ++kk) v = msub(v, sl[kk][q], y[(i0 + kk) * n + col]);
        y[(i0 + q) * n + col] = __ddiv_rn(v, sl[q][q]);
      }
    }
  }
}

// Blocked forward solves for all columns at once (Y = L⁻¹ column by column,
// Y[i][col] at [i * n + col]): the chain of y[i][col] is δ − Σ_{k<i} L(i,k)·y[k][col]
// with k ascending, then / L(i,i). Row panels of 32: the earlier panels'
// terms arrive through the trailing updates (k ascending per panel and
// inside it), the panel's own terms in k_fwd_panel. Entries with col > i stay
// exactly +0 (every term multiplies a +0 y), so those tiles are skipped.
__global__ void k_identity(double* __restrict__ y, int64_t n) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[t] = (t / n == t % n) ? 1.0 : 0.0;
}

__global__ void __launch_bounds__(256) k_fwd_panel(const double* __restrict__ lt, int64_t n,
                                                   int64_t p0, double* __restrict__ y) {
  __shared__ double dl[CP][CP + 1];  // dl[i][k] = L(p0 + i, p0 + k)
  const int pw = n - p0 < CP ? static_cast<int>(n - p0) : CP;
  for (int t = threadIdx.x; t < CP * CP; t += blockDim.x) {
    const int i = t / CP, k = t % CP;
    dl[i][k] = (i < pw && k <= i) ? lt[(p0 + k) * n + p0 + i] : 0.0;
  }
  __syncthreads();
  const int64_t col = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (col >= n || col >= p0 + pw) return;  // col beyond the panel: its rows here stay +0
  double yv[CP];
#pragma unroll
  for (int i = 0; i < CP; ++i) {
    if (i < pw) {
      double v = y[(p0 + i) * n + col];
#pragma unroll
      for (int k = 0; k < CP; ++k)
        if (k < i) v = msub(v, dl[i][k], yv[k]);
      yv[i] = __ddiv_rn(v, dl[i][i]);
      y[(p0 + i) * n + col] = yv[i];
    }
  }
}

__global__ void __launch_bounds__(256) k_fwd_trail(const double* __restrict__ lt, int64_t n,
                                                   int64_t p0, double* __restrict__ y) {
  __shared__ double li[CP][CP + 1], yp[CP][CP + 1];  // li[k][row], yp[k][col]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r0 = p0 + CP + static_cast<int64_t>(blockIdx.y) * 32;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32;
  if (c0 > r0 + 31) return;  // every column past every row of the tile: exact zeros
  for (int k = ty; k < CP; k += 8) {
    li[k][tx] = r0 + tx < n ? lt[(p0 + k) * n + r0 + tx] : 0.0;
    yp[k][tx] = c0 + tx < n ? y[(p0 + k) * n + c0 + tx] : 0.0;
  }
  __syncthreads();
  const int64_t col = c0 + tx;
  if (col >= n) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = ty * 4 + q;
    const int64_t i = r0 + r;
    if (i < n) {
      double v = y[i * n + col];
#pragma unroll
      for (int k = 0; k < CP; ++k) v = msub(v, li[k][r], yp[k][tx]);
      y[i * n + col] = v;
    }
  }
}

// Back solve Lᵀ x = y: x[ii] = (y[ii] - Σ_{k>ii} L(k,ii)·x[k]) / L(ii,ii), k
// ascending — a serial chain per column (chain ii starts with x[ii+1]). The
// operands stream in order (row ii of Lᵀ, the column's own x), so they are
// loaded a batch ahead of the dependent subtractions.
constexpr int BB = 8;
__global__ void __launch_bounds__(64) k_back_solve(const double* __restrict__ lt, int64_t n,
                                                   const double* __restrict__ y,
                                                   double* __restrict__ x) {
  const int64_t col = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (col >= n) return;
  for (int64_t ii = n; ii-- > 0;) {
    const double* lr = lt + ii * n;
    double s = y[ii * n + col];
    int64_t k = ii + 1;
    double la[BB], xa[BB];
    if (k + BB <= n) {
#pragma unroll
      for (int b = 0; b < BB; ++b) {
        la[b] = __ldg(lr + k + b);
        xa[b] = x[(k + b) * n + col];
      }
      for (; k + 2 * BB <= n; k += BB) {
        double lb[BB], xb[BB];
#pragma unroll
        for (int b = 0; b < BB; ++b) {  // next batch in flight
          lb[b] = __ldg(lr + k + BB + b);
          xb[b] = x[(k + BB + b) * n + col];
        }
#pragma unroll
        for (int b = 0; b < BB; ++b) s = msub(s, la[b], xa[b]);
#pragma unroll
        for (int b = 0; b < BB; ++b) {
          la[b] = lb[b];
          xa[b] = xb[b];
        }
      }
#pragma unroll
      for (int b = 0; b < BB; ++b) s = msub(s, la[b], xa[b]);
      k += BB;
    }
    for (; k < n; ++k) s = msub(s, __ldg(lr + k), x[k * n + col]);
    x[ii * n + col] = __ddiv_rn(s, __ldg(lr + ii));
  }
}

// The same back solve with the operand streams staged in shared memory: one
// warp per 32 columns; for each chain ii the rows x[k][col0..col0+31] (256 B)
// and Lᵀ[ii][k] of k in (ii, n) arrive in 64-row chunks by cp.async, double
// buffered, so the dependent subtractions read shared memory while the next
// chunk is in flight.
constexpr int XCH = 64;
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(
                   __cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int XNB = 4;  // chunk buffers: up to XNB - 1 chunks in flight ahead of the chain
__global__ void __launch_bounds__(32) k_back_solve_sm(const double* __restrict__ lt, int64_t n,
                                                      const double* __restrict__ y,
                                                      double* __restrict__ x) {
  extern __shared__ __align__(16) double bsm[];
  double (*sx)[XCH][32] = reinterpret_cast<double (*)[XCH][32]>(bsm);
  double (*sl)[XCH] = reinterpret_cast<double (*)[XCH]>(bsm + XNB * XCH * 32);
  const int lane = threadIdx.x;
  const int64_t col0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int64_t col = col0 + lane;
  const bool full = col0 + 32 <= n;  // whole 256-B rows (else per-lane scalar path)
  for (int64_t ii = n; ii-- > 0;) {
    const double* lr = lt + ii * n;
    double s = col < n ? y[ii * n + col] : 0.0;
    const int64_t k0 = ii + 1;
    const int nch = static_cast<int>((n - k0 + XCH - 1) / XCH);
    auto stage = [&](int c) {  // chunk c: rows [k0 + c·XCH, +XCH) ∩ [k0, n), buffer c % XNB
      const int buf = c % XNB;
      const int64_t kb = k0 + static_cast<int64_t>(c) * XCH;
      const int rows = n - kb < XCH ? static_cast<int>(n - kb) : XCH;
      if (full) {
        for (int t = lane; t < rows * 16; t += 32) {  // 16 x 16 B per row
          const int r = t >> 4, cc = t & 15;
          cp16(&sx[buf][r][2 * cc], x + (kb + r) * n + col0 + 2 * cc);
        }
      } else if (col < n) {
        for (int r = 0; r < rows; ++r) sx[buf][r][lane] = x[(kb + r) * n + col];
      }
      for (int r = lane; r < rows; r += 32) sl[buf][r] = __ldg(lr + kb + r);
    };
    for (int c = 0; c < XNB - 1; ++c) {  // prologue: one commit group per slot
      if (c < nch) stage(c);
      cp_commit();
    }
    for (int c = 0; c < nch; ++c) {
      if (c + XNB - 1 < nch) stage(c + XNB - 1);
      cp_commit();
      cp_wait<XNB - 1>();  // chunk c has landed
      __syncwarp();
      const int buf = c % XNB;
      const int64_t kb = k0 + static_cast<int64_t>(c) * XCH;
      const int rows = n - kb < XCH ? static_cast<int>(n - kb) : XCH;
      const double* slb = sl[buf];
      if (rows == XCH) {
#pragma unroll 16
        for (int r = 0; r < XCH; ++r) s = msub(s, slb[r], sx[buf][r][lane]);
      } else {
        for (int r = 0; r < rows; ++r) s = msub(s, slb[r], sx[buf][r][lane]);
      }
      __syncwarp();
    }
    cp_wait<0>();
    if (col < n) x[ii * n + col] = __ddiv_rn(s, __ldg(lr + ii));
    __threadfence_block();
    __syncwarp();
  }
}
constexpr int kBackSmem = XNB * XCH * 32 * 8 + XNB * XCH * 8;

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

// Blocked right-looking Cholesky, 32-column panels. The order of every chain
// is the reference's: entry (i, j) receives its terms k ascending — the terms
// of earlier panels from the trailing updates (in panel order, k ascending
// inside each), then the panel's own terms k in [p0, j) inside k_chol_panel.
// Panel p0: every CTA factors the 32 x 32 diagonal block into shared memory
// (column by column, as cholesky_lower does), then one thread per panel row
// i >= p0 + 32 finishes its 32 entries L(i, p0..p0+31) from registers.
__global__ void __launch_bounds__(256) k_chol_panel(const double* __restrict__ s,
                                                    double* __restrict__ lt, int64_t n, int64_t p0,
                                                    int* __restrict__ bad) {
  __shared__ double d[CP][CP + 1];  // d[i][j]: S then L of the diagonal block
  const int pw = n - p0 < CP ? static_cast<int>(n - p0) : CP;
  for (int t = threadIdx.x; t < CP * CP; t += blockDim.x) {
    const int i = t / CP, j = t % CP;
    d[i][j] = (i < pw && j <= i) ? s[(p0 + i) * n + p0 + j] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < pw; ++j) {
    if (threadIdx.x == 0) {
      double v = d[j][j];
      for (int k = 0; k < j; ++k) v = msub(v, d[j][k], d[j][k]);
      if (!(v > 0.0) && blockIdx.x == 0) atomicMin(bad, static_cast<int>(p0 + j));
      d[j][j] = sqrt(v);
    }
    __syncthreads();
    const int i = j + 1 + static_cast<int>(threadIdx.x);
    if (i < pw) {
      double v = d[i][j];
      for (int k = 0; k < j; ++k) v = msub(v, d[i][k], d[j][k]);
      d[i][j] = __ddiv_rn(v, d[j][j]);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0)  // the diagonal block's columns of Lᵀ
    for (int t = threadIdx.x; t < CP * CP; t += blockDim.x) {
      const int i = t / CP, j = t % CP;
      if (i < pw && j <= i) lt[(p0 + j) * n + p0 + i] = d[i][j];
    }
  const int64_t i = p0 + pw + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double lr[CP];
#pragma unroll
  for (int j = 0; j < CP; ++j) {
    if (j < pw) {
      double v = s[i * n + p0 + j];
#pragma unroll
      for (int k = 0; k < CP; ++k)
        if (k < j) v = msub(v, lr[k], d[j][k]);
      lr[j] = __ddiv_rn(v, d[j][j]);
      lt[(p0 + j) * n + i] = lr[j];
    }
  }
}

// Trailing update after panel p0: S(i, j) -= L(i, k)·L(j, k), k = p0 .. p0+31
// ascending, for p0 + 32 <= j <= i. 32 x 32 tiles of the lower triangle.
__global__ void __launch_bounds__(256) k_chol_trail(double* __restrict__ s,
                                                    const double* __restrict__ lt, int64_t n,
                                                    int64_t p0) {
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  if (bj > bi) return;
  __shared__ double li[CP][CP + 1], lj[CP][CP + 1];  // [k][row]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t q0 = p0 + CP, i0 = q0 + bi * 32, j0 = q0 + bj * 32;
  for (int k = ty; k < CP; k += 8) {
    li[k][tx] = i0 + tx < n ? lt[(p0 + k) * n + i0 + tx] : 0.0;
    lj[k][tx] = j0 + tx < n ? lt[(p0 + k) * n + j0 + tx] : 0.0;
  }
  __syncthreads();
  const int64_t j = j0 + tx;
  if (j >= n) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = ty * 4 + q;
    const int64_t i = i0 + r;
    if (i < n && i >= j) {
      double v = s[i * n + j];
#pragma unroll
      for (int k = 0; k < CP; ++k) v = msub(v, li[k][r], lj[k][tx]);
      s[i * n + j] = v;
    }
  }
}

// cholesky_lower of a (n x n, consumed as scratch) into lt = Lᵀ; bad = first failing pivot
cudaError_t cholesky(double* a, double* l, int64_t n, int* bad, cudaStream_t st) {
  if (getenv("MLRA_OPTQ_CHOL_STEP")) {  // dev A/B: one launch per column
    for (int64_t k = 0; k < n; ++k) {
      const int64_t t = n - k - 1;
      const unsigned nb = static_cast<unsigned>(t > 0 ? (t + 31) / 32 : 1);
      note_launch();
      k_chol_step<<<dim3(nb, nb), 256, 0, st>>>(a, l, n, k, bad);
    }
    return cudaGetLastError();
  }
  for (int64_t p0 = 0; p0 < n; p0 += CP) {
    const int64_t rest = n - p0 - CP;  // rows below the diagonal block
    const unsigned pb = static_cast<unsigned>(rest > 0 ? (rest + 255) / 256 : 1);
    note_launch();
    k_chol_panel<<<pb, 256, 0, st>>>(a, l, n, p0, bad);
    if (rest > 0) {
      const unsigned tb = static_cast<unsigned>((rest + 31) / 32);
      note_launch();
      k_chol_trail<<<dim3(tb, tb), 256, 0, st>>>(a, l, n, p0);
    }
  }
  return cudaGetLastError();
}

}  // namespace

// dev-only phase timer (MLRA_OPTQ_PROFILE=1): CUDA events on the stream, printed to stderr
struct PhaseTimer {
  bool on = getenv("MLRA_OPTQ_PROFILE") != nullptr;
  cudaStream_t st;
  cudaEvent_t ev[8];
  const char* name[8];
  int n = 0;
  explicit PhaseTimer(cudaStream_t s) : st(s) {}
  void mark(const char* nm) {
    if (!on || n == 8) return;
    cudaEventCreate(&ev[n]);
    cudaEventRecord(ev[n], st);
    name[n++] = nm;
  }
  ~PhaseTimer() {
    if (!on || n < 2) return;
    cudaEventSynchronize(ev[n - 1]);
    for (int i = 1; i < n; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      fprintf(stderr, "optq %-12s %9.3f ms\n", name[i], ms);
    }
    for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
  }
};

cudaError_t launch_optq_workspace(const double* calib, int64_t m, int64_t n, double damping,
                                  double* hessian, double* upper, double* scratch, int* bad,
                                  cudaStream_t st) {
  // scratch: 2 n^2 doubles
  double* a = scratch;
  double* b = scratch + n * n;
  PhaseTimer pt(st);
  pt.mark("start");
  const unsigned nt = static_cast<unsigned>((n + HT - 1) / HT);
  note_launch();
  k_hessian<<<dim3(nt, nt), 256, 0, st>>>(calib, m, n, hessian);
  note_launch();
  k_damp<<<1, 32, 0, st>>>(hessian, n, damping);
  pt.mark("hessian");
  cudaError_t e = cudaMemcpyAsync(a, hessian, n * n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(b, 0, n * n * sizeof(double), st)) != cudaSuccess) return e;
  if ((e = cholesky(a, b, n, bad, st)) != cudaSuccess) return e;  // b = Lᵀ
  pt.mark("cholesky1");
  // inverse through the column solves: y in `a`, x (the inverse) in `upper`
  const unsigned sb = static_cast<unsigned>((n + 63) / 64);
  if (getenv("MLRA_OPTQ_FWD_THREAD")) {  // dev A/B: one thread per column, 32 chains each
    note_launch();
    k_fwd_solve<<<sb, 64, 0, st>>>(b, n, a);
  } else {
    note_launch();
    k_identity<<<blocks_for(n * n, 256), 256, 0, st>>>(a, n);
    for (int64_t p0 = 0; p0 < n; p0 += CP) {
      note_launch();
      k_fwd_panel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(b, n, p0, a);
      const int64_t rest = n - p0 - CP;
      if (rest > 0) {
        note_launch();
        k_fwd_trail<<<dim3(static_cast<unsigned>((n + 31) / 32),
                           static_cast<unsigned>((rest + 31) / 32)),
                      256, 0, st>>>(b, n, p0, a);
      }
    }
  }
  pt.mark("fwd_solve");
  note_launch();
  if (getenv("MLRA_OPTQ_BACK_LDG"))
    k_back_solve<<<sb, 64, 0, st>>>(b, n, a, upper);
  else
  {
    cudaFuncSetAttribute(k_back_solve_sm, cudaFuncAttributeMaxDynamicSharedMemorySize, kBackSmem);
    k_back_solve_sm<<<static_cast<unsigned>((n + 31) / 32), 32, kBackSmem, st>>>(b, n, a, upper);
  }
  pt.mark("back_solve");
  note_launch();
  k_symmetrize<<<blocks_for(n * n, 256), 256, 0, st>>>(upper, n);
  // second factorization (of the inverse; reported through bad[1]); its Lᵀ is U
  if ((e = cudaMemsetAsync(b, 0, n * n * sizeof(double), st)) != cudaSuccess) return e;
  if ((e = cholesky(upper, b, n, bad + 1, st)) != cudaSuccess) return e;
  pt.mark("cholesky2");
  e = cudaMemcpyAsync(upper, b, n * n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  pt.mark("copy");
  if (e != cudaSuccess) return e;
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
