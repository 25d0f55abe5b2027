// optim.cu — AdamW over the adapter parameters on the device.
//
// Restates AdamW::step (train.cpp:81-134) in IEEE f64 with the reference's
// evaluation order, every operation an explicit round-to-nearest intrinsic
// (no FMA contraction), so the f64 master values and moments are bit-identical
// to the reference's given the same gradients:
//   m = β1·m + (1-β1)·g
//   v = β2·v + ((1-β2)·g)·g
//   p = p·(1 - lr·wd) - (lr·(m/bc1)) / (sqrt(v/bc2) + eps)
// with bc1 = 1 - β1^t, bc2 = 1 - β2^t, (1-β1), (1-β2), (1 - lr·wd) evaluated
// on the host exactly as the reference does.
//
// One launch updates a whole flat bucket of parameters (the data-parallel
// gradient bucket, dp.py): the update is elementwise and identical for every
// parameter. The reference's per-parameter "non-finite gradient" check
// (train.cpp:113-117: parameters before the bad one are updated, it and the
// rest are not) becomes a first pass that records the smallest offending
// parameter index, and an update pass that skips parameters at or after it.
//
// HBM-bound: 8+8+8 (p, m, v read) + 4 or 8 (g) + 8+8+8 written (+4 for the
// f32 working copy the GEMMs consume) bytes per element.
#include <cuda_runtime.h>

#include "kernels.h"

namespace mlra {

namespace {

__device__ __forceinline__ int seg_of(const AdamwSegs& sg, int nseg, int64_t i) {
  int lo = 0, hi = nseg;  // off[lo] <= i < off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (sg.off[mid] <= i)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

template <typename G>
__device__ __forceinline__ double load_g(const G* g, int64_t i) {
  return static_cast<double>(__ldg(g + i));
}

template <typename G>
__global__ void k_adamw_check(const G* __restrict__ grad, int64_t n, const __grid_constant__ AdamwSegs sg,
                              int nseg, int* __restrict__ first_bad) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double g = load_g(grad, i);
    if (!isfinite(g)) atomicMin(first_bad, seg_of(sg, nseg, i));
  }
}

template <typename G>
__global__ void k_adamw_update(const G* __restrict__ grad, int64_t n,
                               const __grid_constant__ AdamwSegs sg, int nseg,
                               const int* __restrict__ first_bad, double* __restrict__ p,
                               double* __restrict__ m, double* __restrict__ v,
                               float* __restrict__ p32, AdamwConsts c) {
  const int bad = first_bad ? *first_bad : nseg;
  const int64_t limit = bad >= nseg ? n : sg.off[bad];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < limit;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double g = load_g(grad, i);
    const double mi = __dadd_rn(__dmul_rn(c.beta1, m[i]), __dmul_rn(c.one_m_beta1, g));
    const double vi =
        __dadd_rn(__dmul_rn(c.beta2, v[i]), __dmul_rn(__dmul_rn(c.one_m_beta2, g), g));
    const double mhat = __ddiv_rn(mi, c.bc1);
    const double vhat = __ddiv_rn(vi, c.bc2);
    const double step = __ddiv_rn(__dmul_rn(c.lr, mhat), __dadd_rn(__dsqrt_rn(vhat), c.eps));
    const double pi = __dsub_rn(__dmul_rn(p[i], c.decay), step);
    m[i] = mi;
    v[i] = vi;
    p[i] = pi;
    if (p32) p32[i] = __double2float_rn(pi);
  }
}

}  // namespace

cudaError_t launch_adamw(const void* grad, bool grad_f64, int64_t n, const AdamwSegs& offs, int nseg,
                         int* first_bad, double* p, double* m, double* v, float* p32,
                         const AdamwConsts& c, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (n + 255) / 256;
  if (blocks > 8LL * sms) blocks = 8LL * sms;
  const int nb = static_cast<int>(blocks);
  if (first_bad) {
    // "none" = any value >= nseg: 0x7f7f7f7f by a memset (capturable, no host source)
    cudaError_t e = cudaMemsetAsync(first_bad, 0x7f, sizeof(int), st);
    if (e != cudaSuccess) return e;
    note_launch();
    if (grad_f64)
      k_adamw_check<<<nb, 256, 0, st>>>(static_cast<const double*>(grad), n, offs, nseg, first_bad);
    else
      k_adamw_check<<<nb, 256, 0, st>>>(static_cast<const float*>(grad), n, offs, nseg, first_bad);
  }
  note_launch();
  if (grad_f64)
    k_adamw_update<<<nb, 256, 0, st>>>(static_cast<const double*>(grad), n, offs, nseg, first_bad,
                                       p, m, v, p32, c);
  else
    k_adamw_update<<<nb, 256, 0, st>>>(static_cast<const float*>(grad), n, offs, nseg, first_bad,
                                       p, m, v, p32, c);
  return cudaGetLastError();
}

}  // namespace mlra
